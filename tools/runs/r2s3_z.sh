#!/bin/bash
# round 2, session 3: FP8-pool kernel, ring-first placement (F1) vs Q first (F0)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
S2L_LIB=abl/F1.so timeout -s KILL 900 python -m pytest tests/test_gpu_fp8.py -m gpu -q -x -p no:cacheprovider > gpurun_out/z_tests.txt 2>&1; echo "exit $?" >> gpurun_out/z_tests.txt; tail -2 gpurun_out/z_tests.txt
for k in 1 2 3; do
timeout -s KILL 900 python tools/ab.py abl/F0.so:KV=1 abl/F1.so:KV=1 8 >> gpurun_out/z_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/F1.so:KV=1 abl/F0.so:KV=1 8 >> gpurun_out/z_ab.txt 2>&1
done
grep -v Warn gpurun_out/z_ab.txt
