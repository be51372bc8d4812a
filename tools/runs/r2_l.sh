#!/bin/bash
# round 2: staged swaps for scattered ids -- parity of swap tests, C4 microbench grid
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "swap or hazard or c4 or scheduler or c1" > gpurun_out/r2l_tests.txt 2>&1; echo "exit $?" >> gpurun_out/r2l_tests.txt
timeout -s KILL 900 python tools/bench_workloads.py c4 > gpurun_out/r2l_c4.jsonl 2> gpurun_out/r2l_c4.err; echo "exit $?" >> gpurun_out/r2l_c4.err
