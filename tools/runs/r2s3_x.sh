#!/bin/bash
# round 2, session 3: C4 mix -- compute slows under overlapped swaps; stream priority / staging off
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null
for v in "C4_PRIO=0" "C4_PRIO=1" "C4_PRIO=0 S2L_SWAP_STAGE=0" "C4_PRIO=1 S2L_SWAP_STAGE=0"; do
  env $v timeout -s KILL 900 python tools/bench_workloads.py c4mix > gpurun_out/x_c4mix_$(echo $v | tr ' =' '__').json 2> gpurun_out/x_err.txt; echo "$v rc=$?"
done
python3 - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/x_c4mix_*.json')):
    d = json.loads(open(f).read().strip().splitlines()[-1])
    co, se, ov = d['compute_only'], d['serial'], d['overlap']
    print(f.split('x_c4mix_')[1], 'compute_only', round(co['ms']), 'serial', round(se['ms']), 'overlap', round(ov['ms']),
          'busy', round(ov['compute_busy_ms']), 'copy_out_ms', round(ov['copy_out']['ms']), 'copy_in_ms', round(ov['copy_in']['ms']),
          'overlap_frac', d.get('overlap_fraction'))
PY
