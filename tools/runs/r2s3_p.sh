#!/bin/bash
# round 2, session 3: the budget-split update-round GPU test
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "budget_split or c3_small" --durations=3 > gpurun_out/p_tests.txt 2>&1; echo "exit $?" >> gpurun_out/p_tests.txt; tail -8 gpurun_out/p_tests.txt
