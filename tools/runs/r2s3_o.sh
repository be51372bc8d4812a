#!/bin/bash
# round 2, session 3: bench with the C3 budget-split field
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null
timeout -s KILL 900 python bench.py > gpurun_out/o_bench.json 2> gpurun_out/o_bench.err; echo rc=$?; tail -3 gpurun_out/o_bench.err
python3 -c "
import json
d=json.loads(open('gpurun_out/o_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['roofline']['frac']); print(json.dumps(d['c3']))"
