timeout 600 python -m pytest tests -m gpu -x -q -k fused 2>&1 | tail -3
timeout -s KILL 300 python tools/fused_diag.py ab_libs/new3.so ab_libs/new3.so:FUSED=1 ab_libs/head.so 8
timeout -s KILL 300 python tools/fused_diag.py ab_libs/head.so ab_libs/new3.so:FUSED=1 ab_libs/new3.so 8
