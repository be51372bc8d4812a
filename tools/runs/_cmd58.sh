python -m paper_2604_16395_b200.build --force > /dev/null
for a in 2 3 0 2; do C4_AHEAD=$a timeout -s KILL 800 python tools/bench_workloads.py c4mix > gpurun_out/c4a$a.jsonl 2>/dev/null; python -c "
import json;d=json.loads(open('gpurun_out/c4a$a.jsonl').read().strip().splitlines()[-1]);print('ahead $a', {k:round(d[k]['ms']) for k in ('compute_only','serial','overlap')}, 'out GB', d['overlap']['swap_out_bytes']/1e9, 'overlap_frac', round(d['overlap_frac'],3), d['parity']['pass'])"; done
