#!/bin/bash
# round 2: fused (L2 prefetch) vs plain A/B; append rows-per-warp variants; C4 mode at full size
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -k "fused" > gpurun_out/r2p_fused_tests.txt 2>&1; echo "exit $?" >> gpurun_out/r2p_fused_tests.txt
cp paper_2604_16395_b200/libs2l.so /tmp/cur.so
timeout -s KILL 900 python tools/ab.py /tmp/cur.so paper_2604_16395_b200/libs2l.so:FUSED=1 16 > gpurun_out/r2p_ab_fused.txt 2>&1
mkdir -p /tmp/s2l_ab
for R in 2 8; do S2L_NVCC_FLAGS="-DS2L_APPEND_ROWS=$R" python -m paper_2604_16395_b200.build --force > /dev/null 2>&1; cp paper_2604_16395_b200/libs2l.so /tmp/s2l_ab/rows$R.so; done
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
timeout -s KILL 600 python tools/append_bench.py /tmp/cur.so /tmp/s2l_ab/rows2.so /tmp/s2l_ab/rows8.so /tmp/cur.so > gpurun_out/r2p_append_rows.txt 2>&1
timeout -s KILL 1500 python bench.py --workload c4 --steps 2 > gpurun_out/r2p_c4.json 2> gpurun_out/r2p_c4.err; echo "rc $?" >> gpurun_out/r2p_c4.err
