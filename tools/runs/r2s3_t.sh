#!/bin/bash
# round 2, session 3: MMA issue in one inline-PTX block per 8 S / 4 PV MMAs (MB) vs per-MMA elect (HEAD)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
S2L_LIB=abl/MB.so timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "tc_ or c2 or gqa or block or split or fused" > gpurun_out/t_tests.txt 2>&1; echo "exit $?" >> gpurun_out/t_tests.txt; tail -2 gpurun_out/t_tests.txt
for k in 1 2; do
timeout -s KILL 900 python tools/ab.py abl/HEAD.so abl/MB.so 10 >> gpurun_out/t_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/MB.so abl/HEAD.so 10 >> gpurun_out/t_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/HEAD.so abl/MB.so --c5 4 >> gpurun_out/t_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/MB.so abl/HEAD.so --c5 4 >> gpurun_out/t_ab.txt 2>&1
done
grep -v Warn gpurun_out/t_ab.txt
