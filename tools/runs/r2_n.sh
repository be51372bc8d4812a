#!/bin/bash
# round 2: FP8 KV cache tests, full GPU suite, poly A/B on C2 and C5
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
timeout -s KILL 600 python -m pytest tests/test_gpu_fp8.py -x -q -p no:cacheprovider > gpurun_out/r2n_fp8.txt 2>&1; echo "exit $?" >> gpurun_out/r2n_fp8.txt
timeout -s KILL 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2n_gputests.txt 2>&1; echo "exit $?" >> gpurun_out/r2n_gputests.txt
bash tools/ab_build.sh p1 "-DS2L_POLY_PAIRS=1" p2 "-DS2L_POLY_PAIRS=2" p3 "-DS2L_POLY_PAIRS=3" > gpurun_out/r2n_ab_c2.txt 2>&1
timeout -s KILL 600 python tools/ab.py /tmp/s2l_ab/p1.so /tmp/s2l_ab/p2.so /tmp/s2l_ab/p3.so --c5 4 > gpurun_out/r2n_ab_c5.txt 2>&1
