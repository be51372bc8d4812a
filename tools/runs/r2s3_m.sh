#!/bin/bash
# round 2, session 3: degree-2 exp2 polynomial (P1: share 2/8, P2: share 3/8) vs degree 3 (P0)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for k in 1 2; do
timeout -s KILL 900 python tools/ab.py abl/P0.so abl/P1.so abl/P2.so 10 >> gpurun_out/m_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/P2.so abl/P1.so abl/P0.so 10 >> gpurun_out/m_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/P0.so abl/P1.so abl/P2.so --c5 4 >> gpurun_out/m_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/P2.so abl/P1.so abl/P0.so --c5 4 >> gpurun_out/m_ab.txt 2>&1
done
grep -v Warn gpurun_out/m_ab.txt
S2L_LIB=abl/P1.so timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -x -p no:cacheprovider -k "peaky or needle or c2_full or c5" > gpurun_out/m_tests.txt 2>&1; echo "exit $?" >> gpurun_out/m_tests.txt; tail -2 gpurun_out/m_tests.txt
