timeout 600 python -m pytest tests -m gpu -q -k "fused" 2>&1 | tail -3
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -1
