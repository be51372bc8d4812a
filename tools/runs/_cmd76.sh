timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout -s KILL 300 python bench.py --steps 3 --warmup 3 2>/dev/null | tail -c 150
timeout -s KILL 900 python tools/model_bench.py --chunks 32 2>&1 | tail -1
