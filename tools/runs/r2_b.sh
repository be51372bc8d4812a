#!/bin/bash
# round 2: A/B of the attention softmax designs (split-S round-1 design vs whole-S + stale-max
# pipelined softmax with 1-3 polynomial pairs of 8), then the fast parity subset on the default
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
bash tools/ab_build.sh split1 "-DS2L_SPLIT_S=1" stale_p1 "-DS2L_POLY_PAIRS=1" stale_p2 "-DS2L_POLY_PAIRS=2" stale_p3 "-DS2L_POLY_PAIRS=3" > gpurun_out/r2b_ab.txt 2>&1
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m "gpu and not slow" -x -q -p no:cacheprovider > gpurun_out/r2b_parity.txt 2>&1
echo "exit $?" >> gpurun_out/r2b_parity.txt
