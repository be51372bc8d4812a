#!/bin/bash
# round 2, session 2: bench with the C2t field, C4 swap grid refresh, 2-rank bench
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
( time timeout -s KILL 900 python bench.py > gpurun_out/s_bench.json 2> gpurun_out/s_bench.err ) 2> gpurun_out/s_bench_time.txt
timeout -s KILL 900 python tools/bench_workloads.py c4 > gpurun_out/s_c4grid.jsonl 2> gpurun_out/s_c4grid.err
timeout -s KILL 900 python bench.py --gpus 2 --steps 1 --warmup 3 --no-side > gpurun_out/s_bench2.json 2> gpurun_out/s_bench2.err; echo "bench2 rc=$?"
cat gpurun_out/s_bench_time.txt; tail -c 200 gpurun_out/s_bench2.json; tail -3 gpurun_out/s_bench.err
