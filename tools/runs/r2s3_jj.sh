#!/bin/bash
# round 2, session 3: prologue -- barrier init / TMEM alloc before the unit decode (PR1) vs after (PR0)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
S2L_LIB=abl/PR1.so timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fp8.py -m gpu -q -x -p no:cacheprovider -k "c1 or tc_ or c2 or split or fused or fp8_tensor or c3_small" > gpurun_out/jj_tests.txt 2>&1; echo "exit $?" >> gpurun_out/jj_tests.txt; tail -2 gpurun_out/jj_tests.txt
timeout -s KILL 900 python tools/step_ab.py abl/PR0.so abl/PR1.so 4 > gpurun_out/jj_steps.txt 2>&1
grep -v Warn gpurun_out/jj_steps.txt | tail -2
for k in 1 2; do
timeout -s KILL 900 python tools/ab.py abl/PR0.so abl/PR1.so 10 >> gpurun_out/jj_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/PR1.so abl/PR0.so 10 >> gpurun_out/jj_ab.txt 2>&1
done
timeout -s KILL 900 python tools/ab.py abl/PR0.so abl/PR1.so --c5 4 >> gpurun_out/jj_ab.txt 2>&1
grep -v Warn gpurun_out/jj_ab.txt
