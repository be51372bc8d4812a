timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout -s KILL 400 python tools/fused_diag.py ab_libs/nopdl.so ab_libs/pdl.so ab_libs/pdl.so:FUSED=1 16
timeout -s KILL 400 python tools/fused_diag.py ab_libs/pdl.so:FUSED=1 ab_libs/pdl.so ab_libs/nopdl.so 16
timeout -s KILL 600 python tools/ab.py ab_libs/nopdl.so ab_libs/pdl.so 10
