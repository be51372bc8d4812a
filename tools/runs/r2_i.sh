#!/bin/bash
# round 2: TMA append -- GPU suite, bench, A/B of append paths
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2i_gputests.txt 2>&1; echo "exit $?" >> gpurun_out/r2i_gputests.txt
timeout -s KILL 600 python bench.py > gpurun_out/r2i_bench.json 2> gpurun_out/r2i_bench.err; echo "rc $?" >> gpurun_out/r2i_bench.err
S2L_APPEND_TMA=0 timeout -s KILL 600 python bench.py --no-side > gpurun_out/r2i_bench_noTMA.json 2> gpurun_out/r2i_bench_noTMA.err
