#!/bin/bash
# round 2, session 2: persistent attention CTAs (S2L_PERSIST=1): GPU suite both ways, A/B, CTA trace
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
S2L_PERSIST=1 timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_fp8.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r_gputests_persist.txt 2>&1; echo "exit $?" >> gpurun_out/r_gputests_persist.txt
tail -2 gpurun_out/r_gputests_persist.txt
timeout -s KILL 900 python tools/ab.py abl/base.so abl/new.so abl/new.so:S2L_PERSIST=1 8 > gpurun_out/r_ab.txt 2>&1
timeout -s KILL 600 python tools/ab.py abl/base.so abl/new.so:S2L_PERSIST=1 --c5 4 >> gpurun_out/r_ab.txt 2>&1
grep -v Warn gpurun_out/r_ab.txt
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r_gputests.txt 2>&1; echo "exit $?" >> gpurun_out/r_gputests.txt
tail -2 gpurun_out/r_gputests.txt
