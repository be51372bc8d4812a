#!/bin/bash
# round 2, session 3: C4 mix with a free-block reserve (fraction of the GPU pool)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null
for v in "C4_RESERVE=0" "C4_RESERVE=0.05" "C4_RESERVE=0.1" "C4_RESERVE=0.05 C4_PREFETCH=1" "C4_RESERVE=0"; do
  env $v timeout -s KILL 900 python tools/bench_workloads.py c4mix > gpurun_out/gg.json 2>/dev/null
  python3 - "$v" <<'PY'
import json, sys
d = json.loads(open('gpurun_out/gg.json').read().strip().splitlines()[-1])
co, ov = d['compute_only'], d['overlap']
print(sys.argv[1], 'compute_only', round(co['ms']), 'serial', round(d['serial']['ms']), 'overlap', round(ov['ms']), 'busy', round(ov['compute_busy_ms']), 'out_GB', round(ov['swap_out_bytes']/1e9, 2), 'in_GB', round(ov['swap_in_bytes']/1e9, 2), 'waits', ov.get('stream_waits'), 'parity', d.get('parity', {}).get('pass') if isinstance(d.get('parity'), dict) else d.get('parity'))
PY
done
