timeout 600 python -m pytest tests -m gpu -q -k "fused or streaming_decoder" 2>&1 | tail -3
timeout -s KILL 400 python tools/fused_diag.py ab_libs/new5.so ab_libs/mask.so ab_libs/mask.so:FUSED=1 ab_libs/new5.so:FUSED=1 10
