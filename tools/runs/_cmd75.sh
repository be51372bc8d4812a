timeout 600 python -m pytest tests -m gpu -x -q -k "streaming_decoder" 2>&1 | tail -15
timeout -s KILL 600 python tools/model_bench.py --chunks 8 2>&1 | tail -3
timeout -s KILL 900 python tools/model_bench.py --chunks 32 2>&1 | tail -3
