#!/bin/bash
# round 2, session 3: C4 mix waits vs swap-in prefetch distance / eviction look-ahead
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null
for v in "C4_PREFETCH=0" "C4_PREFETCH=1" "C4_PREFETCH=2" "C4_AHEAD=3 C4_PREFETCH=1" "C4_COOLING=0"; do
  env $v timeout -s KILL 900 python tools/bench_workloads.py c4mix > gpurun_out/ee_$(echo $v | tr ' =' '__').json 2>/dev/null
  python3 - "$v" gpurun_out/ee_$(echo $v | tr ' =' '__').json <<'PY'
import json, sys
d = json.loads(open(sys.argv[2]).read().strip().splitlines()[-1])
co, ov = d['compute_only'], d['overlap']
print(sys.argv[1], 'compute_only', round(co['ms']), 'serial', round(d['serial']['ms']), 'overlap', round(ov['ms']), 'busy', round(ov['compute_busy_ms']), 'waits', ov.get('stream_waits'))
PY
done
