set -x
python -c "from paper_2604_16395_b200 import build; build.build()"
timeout 600 python -m pytest tests -m gpu -x -q -k fused 2>&1 | tail -30
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python bench.py --steps 10 --warmup 3 2>&1 | tail -2 > gpurun_out/bench52.json
cat gpurun_out/bench52.json | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['roofline']['achieved'], d['e2e']['value'])"
