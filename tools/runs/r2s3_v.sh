#!/bin/bash
# round 2, session 3: wide-token-row append path test + the append / FP8 / fused tests
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fp8.py -m gpu -q -x -p no:cacheprovider -k "wide or c1 or gqa or fp8 or fused or c3_small" > gpurun_out/v_tests.txt 2>&1; echo "exit $?" >> gpurun_out/v_tests.txt; tail -4 gpurun_out/v_tests.txt
