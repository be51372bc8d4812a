#!/bin/bash
# round 2, session 3: Q tiles between ring slots 2 and 3 (M1) vs ring first (Q0 = the validated build, M0 = same via slot_off)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
S2L_LIB=abl/M1.so timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "tc_ or c2_full or split or fused_append_prefill_aligned" > gpurun_out/mm_tests.txt 2>&1; echo "exit $?" >> gpurun_out/mm_tests.txt; tail -2 gpurun_out/mm_tests.txt
for k in 1 2; do
timeout -s KILL 900 python tools/ab.py abl/Q0.so abl/M0.so abl/M1.so 10 >> gpurun_out/mm_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/M1.so abl/M0.so abl/Q0.so 10 >> gpurun_out/mm_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/Q0.so abl/M0.so abl/M1.so --c5 4 >> gpurun_out/mm_ab.txt 2>&1
done
grep -v Warn gpurun_out/mm_ab.txt
