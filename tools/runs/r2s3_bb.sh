#!/bin/bash
# round 2, session 3: bench with C3 budget 2048 and 8192
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null
timeout -s KILL 900 python bench.py > gpurun_out/bb_bench.json 2> gpurun_out/bb_bench.err; echo rc=$?
python3 -c "
import json
d=json.loads(open('gpurun_out/bb_bench.json').read().strip().splitlines()[-1])
c=d['c3']; print(d['value'], d['roofline']['frac'], c['value'], c['roofline']['frac'], [(k, c[k]['steps_per_round'], round(c[k]['value'],1), round(c[k]['roofline']['frac'],3)) for k in c if k.startswith('budget')], c['parity'], [k for k in d if k.endswith('_error')], d['fp8_kv']['value'])"
