#!/bin/bash
# round 2, session 3: mbarrier block first (B1) vs after the tiles (B0)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
S2L_LIB=abl/B1.so timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fp8.py -m gpu -q -x -p no:cacheprovider -k "tc_ or c2_full or split or fused_append_prefill_aligned or fp8_tensor" > gpurun_out/ff_tests.txt 2>&1; echo "exit $?" >> gpurun_out/ff_tests.txt; tail -2 gpurun_out/ff_tests.txt
for k in 1 2; do
timeout -s KILL 900 python tools/ab.py abl/B0.so abl/B1.so 10 >> gpurun_out/ff_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/B1.so abl/B0.so 10 >> gpurun_out/ff_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/B0.so abl/B1.so --c5 4 >> gpurun_out/ff_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/B1.so abl/B0.so --c5 4 >> gpurun_out/ff_ab.txt 2>&1
done
grep -v Warn gpurun_out/ff_ab.txt
