#!/bin/bash
# round 2, session 3: final validation of HEAD -- smoke, GPU suite, bench, launch list, ncu of the last C2 launch
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null
echo "== smoke"; timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/cc_smoke.txt 2>&1; tail -1 gpurun_out/cc_smoke.txt
echo "== gpu tests"; timeout -s KILL 2400 python -m pytest tests -m gpu -q --tb=short > gpurun_out/cc_gputests.txt 2>&1; tail -3 gpurun_out/cc_gputests.txt
echo "== bench"; timeout -s KILL 900 python bench.py > gpurun_out/cc_bench.json 2> gpurun_out/cc_bench.err; echo rc=$?
python3 -c "
import json
d=json.loads(open('gpurun_out/cc_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['c5']['value'], d['c3']['value'], d['c2t']['value'], d['fp8_kv']['value'], [k for k in d if k.endswith('_error')], d['clocks'])"
echo "== launches"; timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/cc_launches.csv python bench.py --steps 1 --warmup 3 --no-side > /dev/null 2>&1; echo rc=$?
echo "== ncu attn"; timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc2 -s 31 -c 1 -o gpurun_out/cc_attn_full python bench.py --steps 1 --warmup 3 --no-side > /dev/null 2>&1; echo rc=$?
echo "== reference arm"; timeout -s KILL 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/cc_reference.json 2> gpurun_out/cc_reference.err; echo rc=$?
