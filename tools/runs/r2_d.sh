#!/bin/bash
# round 2: bench of the stale-max kernel (default build)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
timeout 600 python bench.py > gpurun_out/r2d_bench.json 2> gpurun_out/r2d_bench.err; echo "rc $?" >> gpurun_out/r2d_bench.err
