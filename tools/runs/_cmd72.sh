for A in 3 4 6; do
  C4_AHEAD=$A timeout -s KILL 900 python tools/bench_workloads.py c4mix > gpurun_out/c4mix_a$A.json 2> gpurun_out/c4mix_a$A.err
  python -c "
import json; d=json.loads(open('gpurun_out/c4mix_a$A.json').read().strip().splitlines()[-1])
print('ahead $A', {m: round(d[m]['ms'],1) for m in ('compute_only','serial','overlap','overlap_cost')}, 'busy', round(d['overlap']['compute_busy_ms'],1), 'out', d['overlap']['swap_out_bytes']/1e9, 'in', d['overlap']['swap_in_bytes']/1e9, 'frac', round(d['overlap_frac'],3), 'parity', d['parity']['pass'])"
done
C4_AHEAD=2 C4_TIMELINE=1 timeout -s KILL 900 python tools/bench_workloads.py c4mix > gpurun_out/c4mix_tl.json 2> gpurun_out/c4mix_tl.err
tail -40 gpurun_out/c4mix_tl.err
