#!/bin/bash
# round 2, session 3: full validation of HEAD -- smoke, GPU suite, bench, launch list
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null
echo "== smoke"; timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/y_smoke.txt 2>&1; tail -1 gpurun_out/y_smoke.txt
echo "== gpu tests"; timeout -s KILL 2400 python -m pytest tests -m gpu -q --tb=short > gpurun_out/y_gputests.txt 2>&1; tail -3 gpurun_out/y_gputests.txt
echo "== bench"; timeout -s KILL 900 python bench.py > gpurun_out/y_bench.json 2> gpurun_out/y_bench.err; echo rc=$?
python3 -c "
import json
d=json.loads(open('gpurun_out/y_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['c5']['value'], d['c3']['value'], d['c3']['budget_8192']['value'], d['c2t']['value'], [k for k in d if k.endswith('_error')])"
echo "== launches"; timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/y_launches.csv python bench.py --steps 1 --warmup 3 --no-side > /dev/null 2>&1; echo rc=$?
