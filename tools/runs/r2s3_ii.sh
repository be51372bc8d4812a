#!/bin/bash
# round 2, session 3: final validation of HEAD -- smoke, full GPU suite, bench
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null
echo "== smoke"; timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ii_smoke.txt 2>&1; tail -1 gpurun_out/ii_smoke.txt
echo "== gpu tests"; timeout -s KILL 2400 python -m pytest tests -m gpu -q --tb=short > gpurun_out/ii_gputests.txt 2>&1; tail -3 gpurun_out/ii_gputests.txt
echo "== bench"; timeout -s KILL 900 python bench.py > gpurun_out/ii_bench.json 2> gpurun_out/ii_bench.err; echo rc=$?
python3 -c "
import json
d=json.loads(open('gpurun_out/ii_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['c5']['value'], d['c3']['value'], d['c2t']['value'], d['fp8_kv']['value'], [k for k in d if k.endswith('_error')], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
