#!/bin/bash
# round 2, session 2: driver-style runs: reference arm, bench N=1 (default flags), bench --gpus 2 under torchrun
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
( time timeout -s KILL 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/ag_ref.json 2> gpurun_out/ag_ref.err ) 2> gpurun_out/ag_ref_time.txt
( time timeout -s KILL 900 python bench.py > gpurun_out/ag_bench.json 2> gpurun_out/ag_bench.err ) 2> gpurun_out/ag_bench_time.txt
timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 > gpurun_out/ag_bench2.json 2> gpurun_out/ag_bench2.err; echo "torchrun rc=$?"
cat gpurun_out/ag_ref.json | tail -c 600; grep real gpurun_out/ag_ref_time.txt gpurun_out/ag_bench_time.txt; tail -c 300 gpurun_out/ag_bench2.json
