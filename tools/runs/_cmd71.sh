timeout 600 python -m pytest tests -m gpu -x -q -k "c4_pressure_driver or fused_append_then_swap" 2>&1 | tail -2
for P in 0 1 2; do
  C4_PREFETCH=$P timeout -s KILL 900 python tools/bench_workloads.py c4mix > gpurun_out/c4mix_p$P.json 2> gpurun_out/c4mix_p$P.err
  python -c "
import json; d=json.loads(open('gpurun_out/c4mix_p$P.json').read().strip().splitlines()[-1])
print('prefetch $P', {m: round(d[m]['ms'],1) for m in ('compute_only','serial','overlap','overlap_cost')}, 'busy', round(d['overlap']['compute_busy_ms'],1), 'pref', d['overlap'].get('prefetched_swap_ins'), 'frac', round(d['overlap_frac'],3), 'parity', d['parity']['pass'])"
done
