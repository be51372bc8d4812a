#!/bin/bash
# round 2: FP8 KV kernel on f16 operands (one conversion per two E4M3 values) vs the bf16-operand
# FP8 kernel (abso/head.so, built from the previous commit); FP8 parity tests; full bench line
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
timeout -s KILL 600 python -m pytest tests/test_gpu_fp8.py -q -p no:cacheprovider > gpurun_out/r2q_fp8_tests.txt 2>&1; echo "exit $?" >> gpurun_out/r2q_fp8_tests.txt
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2q_smoke.txt 2>&1
cp paper_2604_16395_b200/libs2l.so /tmp/cur.so
timeout -s KILL 900 python tools/ab.py abso/head.so:KV=1 /tmp/cur.so:KV=1 abso/head.so /tmp/cur.so 8 > gpurun_out/r2q_ab_fp8.txt 2>&1
timeout -s KILL 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2q_bench.json 2> gpurun_out/r2q_bench.err
