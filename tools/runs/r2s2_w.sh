#!/bin/bash
# round 2, session 2: lazy-rescale threshold 8 vs 12 (log2 units)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout -s KILL 900 python tools/ab.py abl/new.so abl/thr12.so 10 > gpurun_out/w_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/thr12.so abl/new.so 10 >> gpurun_out/w_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/new.so abl/thr12.so --c5 5 >> gpurun_out/w_ab.txt 2>&1
S2L_LIB=abl/thr12.so timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -k "peaky or needle or c2" > gpurun_out/w_tests.txt 2>&1; echo "exit $?" >> gpurun_out/w_tests.txt
grep -v Warn gpurun_out/w_ab.txt; tail -2 gpurun_out/w_tests.txt
