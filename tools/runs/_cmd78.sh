for i in 1 2 3; do timeout 900 python -m pytest tests -m gpu -q -p no:randomly 2>&1 | tail -1; done
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout -s KILL 600 python bench.py 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['parity']['pass'], d['next2_fused']['ms_per_step'], d['ms_per_step'])"
