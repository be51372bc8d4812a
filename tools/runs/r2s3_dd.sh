#!/bin/bash
# round 2, session 3: C4 mix with the runtime's inserted cross-stream wait counts
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null
timeout -s KILL 900 python tools/bench_workloads.py c4mix > gpurun_out/dd_c4mix.json 2> gpurun_out/dd_err.txt; echo rc=$?
python3 - <<'PY'
import json
d = json.loads(open('gpurun_out/dd_c4mix.json').read().strip().splitlines()[-1])
for m in ('compute_only', 'serial', 'overlap', 'overlap_cost'):
    x = d[m]
    print(m, round(x['ms']), 'busy', round(x['compute_busy_ms']), 'gap', round(x['compute_gap_ms'], 1), 'waits', x.get('stream_waits'), 'steps', x['steps'])
PY
