#!/bin/bash
# round 2, session 3: C4 mix, reserve 0 vs 0.05 alternated (3 runs each)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null
for k in 1 2 3; do for v in "C4_RESERVE=0" "C4_RESERVE=0.05"; do
  env $v timeout -s KILL 900 python tools/bench_workloads.py c4mix > gpurun_out/hh.json 2>/dev/null
  python3 - "$v" <<'PY'
import json, sys
d = json.loads(open('gpurun_out/hh.json').read().strip().splitlines()[-1])
co, ov = d['compute_only'], d['overlap']
print(sys.argv[1], 'compute_only', round(co['ms']), 'serial', round(d['serial']['ms']), 'overlap', round(ov['ms']), 'overlap_cost', round(d['overlap_cost']['ms']), 'out_GB', round(ov['swap_out_bytes']/1e9, 2))
PY
done; done
