#!/bin/bash
# round 2, session 2: re-validate HEAD (GPU suite, bench) and the FA4 same-window comparison
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/a_smi.txt
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/a_gputests.txt 2>&1; echo "exit $?" >> gpurun_out/a_gputests.txt
timeout -s KILL 600 python bench.py > gpurun_out/a_bench.json 2> gpurun_out/a_bench.err
timeout -s KILL 900 python tools/fa4_compare.py --out gpurun_out/a_fa4.json > gpurun_out/a_fa4.log 2>&1; echo "exit $?" >> gpurun_out/a_fa4.log
tail -2 gpurun_out/a_gputests.txt; tail -c 600 gpurun_out/a_bench.json; tail -5 gpurun_out/a_fa4.log
