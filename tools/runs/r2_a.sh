#!/bin/bash
# round 2, first GPU pass: full GPU suite, default bench, 2-rank bench on one GPU
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r2a_smi.txt 2>&1
python -m paper_2604_16395_b200.build > gpurun_out/r2a_build.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2a_gputests.txt 2>&1
echo "pytest exit $?" >> gpurun_out/r2a_gputests.txt
timeout 600 python bench.py > gpurun_out/r2a_bench.json 2> gpurun_out/r2a_bench.err
echo "bench exit $?" >> gpurun_out/r2a_bench.err
timeout 600 python bench.py --gpus 2 --no-side > gpurun_out/r2a_bench2.json 2> gpurun_out/r2a_bench2.err
echo "bench2 exit $?" >> gpurun_out/r2a_bench2.err
