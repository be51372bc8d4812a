R=s4
mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null
echo "== smoke"; timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
echo "== tests"; timeout -s KILL 900 python -m pytest tests -m gpu -q 2>&1 | tail -1
echo "== bench"; timeout -s KILL 600 python bench.py > gpurun_out/bench_$R.json 2> gpurun_out/bench_$R.err; tail -c 200 gpurun_out/bench_$R.json
echo "== reference"; timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/reference_$R.json 2>/dev/null; tail -c 300 gpurun_out/reference_$R.json
echo "== launches"; timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches_$R.csv python bench.py --steps 1 --warmup 3 --no-side > /dev/null 2>&1; echo rc=$?
echo "== ncu attn"; timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc2 -s 31 -c 1 -o gpurun_out/attn_full_$R python bench.py --steps 1 --warmup 3 --no-side > /dev/null 2>&1; echo rc=$?
echo "== workloads"; timeout -s KILL 900 python tools/bench_workloads.py c3 c5 > gpurun_out/workloads_$R.jsonl 2> gpurun_out/workloads_$R.err; tail -c 300 gpurun_out/workloads_$R.jsonl
echo "== sanitizer"; timeout -s KILL 600 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "c1_full_walk or tc_gqa_ragged or fused" > gpurun_out/memcheck_$R.txt 2>&1; echo rc=$?; tail -3 gpurun_out/memcheck_$R.txt
