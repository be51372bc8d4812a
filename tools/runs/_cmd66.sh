timeout -s KILL 400 python tools/fused_diag.py ab_libs/new3.so ab_libs/new3.so:FUSED=1 20
timeout -s KILL 400 python tools/fused_diag.py ab_libs/new3.so:FUSED=1 ab_libs/new3.so 20
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
