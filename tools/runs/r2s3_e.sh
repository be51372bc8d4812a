#!/bin/bash
# round 2, session 3: persistent kernel with the store/scheduler warp in named barriers (no polling)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
cp abl/D.so paper_2604_16395_b200/libs2l.so; touch paper_2604_16395_b200/libs2l.so
echo "== parity"
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider > gpurun_out/e_tests.txt 2>&1; echo "exit $?" >> gpurun_out/e_tests.txt
tail -3 gpurun_out/e_tests.txt
grep -q "exit 0" gpurun_out/e_tests.txt || exit 1
S="abl/D.so:S2L_PERSIST=0 abl/D.so:S2L_PERSIST=1"
timeout -s KILL 900 python tools/ab.py $S 10 > gpurun_out/e_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/D.so:S2L_PERSIST=1 abl/D.so:S2L_PERSIST=0 10 >> gpurun_out/e_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py $S --c5 4 >> gpurun_out/e_ab.txt 2>&1
grep -v Warn gpurun_out/e_ab.txt | tail -8
S2L_PERSIST=1 timeout -s KILL 600 ncu --set full --clock-control none -k regex:attn_tc2 -s 63 -c 1 -o gpurun_out/e_c5_p1 python tools/c5_stream_once.py > gpurun_out/e_c5_p1.log 2>&1; echo "ncu rc=$?"
