#!/bin/bash
# round 2, session 3: persistent attention kernel (attn_tc2p_kernel) -- parity, then A/B vs the one-unit grid
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out abl
python -m paper_2604_16395_b200.build --force > /dev/null
cp paper_2604_16395_b200/libs2l.so abl/cur.so
echo "== parity (persistent default)"
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider > gpurun_out/b_tests.txt 2>&1; echo "exit $?" >> gpurun_out/b_tests.txt
tail -15 gpurun_out/b_tests.txt
grep -q "exit 0" gpurun_out/b_tests.txt || exit 1
echo "== A/B"
timeout -s KILL 900 python tools/ab.py abl/cur.so:S2L_PERSIST=0 abl/cur.so:S2L_PERSIST=1 10 > gpurun_out/b_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/cur.so:S2L_PERSIST=1 abl/cur.so:S2L_PERSIST=0 10 >> gpurun_out/b_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/cur.so:S2L_PERSIST=0 abl/cur.so:S2L_PERSIST=1 --c5 5 >> gpurun_out/b_ab.txt 2>&1
grep -v Warn gpurun_out/b_ab.txt | tail -12
echo "== bench"
timeout -s KILL 600 python bench.py > gpurun_out/b_bench.json 2> gpurun_out/b_bench.err; tail -c 300 gpurun_out/b_bench.json
