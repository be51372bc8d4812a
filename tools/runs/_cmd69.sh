timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout -s KILL 400 python tools/fused_diag.py ab_libs/head.so ab_libs/new5.so ab_libs/new5.so:FUSED=1 16
timeout -s KILL 400 python tools/fused_diag.py ab_libs/new5.so:FUSED=1 ab_libs/new5.so ab_libs/head.so 16
