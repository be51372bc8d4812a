#!/bin/bash
# round 2, session 3: append kernel without register spills in the wide-row instantiations (AP) vs HEAD
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
S2L_LIB=abl/AP.so timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fp8.py -m gpu -q -x -p no:cacheprovider -k "c1 or gqa or block or c3_small or fp8 or swap or fused" > gpurun_out/u_tests.txt 2>&1; echo "exit $?" >> gpurun_out/u_tests.txt; tail -2 gpurun_out/u_tests.txt
for k in 1 2 3; do timeout -s KILL 600 python tools/append_bench.py abl/HEAD.so abl/AP.so >> gpurun_out/u_app.txt 2>&1; timeout -s KILL 600 python tools/append_bench.py abl/AP.so abl/HEAD.so >> gpurun_out/u_app.txt 2>&1; done
grep -v Warn gpurun_out/u_app.txt
