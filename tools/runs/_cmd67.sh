R=s3
mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null
echo "== smoke"; timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
echo "== bench"; timeout -s KILL 600 python bench.py > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err; tail -c 300 gpurun_out/bench_$R.json
echo "== launches"; timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_$R.csv python bench.py --steps 1 --warmup 3 --no-side > /dev/null 2>&1; echo rc=$?
cat > /tmp/fused_run.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
import bench
from paper_2604_16395_b200 import s2l
torch.cuda.set_device(0)
rids, toks, data = bench.make_stream_data(0)
S = bench.Stream(rids, toks, data, "cuda:0")
ctx, pool = bench.make_ctx(0)
for _ in range(2):
    bench.run_step_fused(ctx, S)
torch.cuda.synchronize()
PY
echo "== launches fused"; timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_fused_$R.csv python /tmp/fused_run.py > /dev/null 2>&1; echo rc=$?
echo "== ncu fused attn"; timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc2 -s 31 -c 1 -o gpurun_out/attn_fused_full_$R python /tmp/fused_run.py > /dev/null 2>&1; echo rc=$?
echo "== sanitizer fused"; timeout -s KILL 600 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "fused_append_prefill_aligned and 8-2-16-2 or unaligned_falls_back" > gpurun_out/memcheck_fused_$R.txt 2>&1; echo rc=$?; tail -3 gpurun_out/memcheck_fused_$R.txt
