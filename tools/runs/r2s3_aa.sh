#!/bin/bash
# round 2, session 3: TMEM column map (T0 = S0 S1 O0 O1, T1 = S0 O0 S1 O1, T2 = O0 O1 S0 S1)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for t in T1 T2; do S2L_LIB=abl/$t.so timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "tc_ or c2_full or split or peaky" > gpurun_out/aa_tests_$t.txt 2>&1; echo "$t exit $?"; done
for k in 1 2; do
timeout -s KILL 900 python tools/ab.py abl/T0.so abl/T1.so abl/T2.so 8 >> gpurun_out/aa_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/T2.so abl/T1.so abl/T0.so 8 >> gpurun_out/aa_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/T0.so abl/T1.so abl/T2.so --c5 4 >> gpurun_out/aa_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/T2.so abl/T1.so abl/T0.so --c5 4 >> gpurun_out/aa_ab.txt 2>&1
done
grep -v Warn gpurun_out/aa_ab.txt
