#!/bin/bash
# round 2, session 2: poly share 2/8 as the default: GPU suite + bench
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/v_gputests.txt 2>&1; echo "exit $?" >> gpurun_out/v_gputests.txt
timeout -s KILL 900 python bench.py > gpurun_out/v_bench.json 2> gpurun_out/v_bench.err
tail -2 gpurun_out/v_gputests.txt; tail -c 200 gpurun_out/v_bench.json
