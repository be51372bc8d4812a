timeout 600 python -m pytest tests -m gpu -x -q -k fused 2>&1 | tail -3
timeout -s KILL 400 python tools/fused_diag.py ab_libs/new4.so ab_libs/new4.so:FUSED=1 ab_libs/new3.so:FUSED=1 16
timeout -s KILL 400 python tools/fused_diag.py ab_libs/new3.so:FUSED=1 ab_libs/new4.so:FUSED=1 ab_libs/new4.so 16
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
