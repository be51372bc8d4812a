#!/bin/bash
# round 2: first run of the CTA-pair kernel: quick parity, then A/B pair vs tc2
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -m "gpu and not slow" -x -q -p no:cacheprovider -k "tc_ or c2 or gqa or block" > gpurun_out/r2e_parity.txt 2>&1; echo "exit $?" >> gpurun_out/r2e_parity.txt
cp paper_2604_16395_b200/libs2l.so /tmp/cur.so
timeout -s KILL 400 python tools/ab.py /tmp/cur.so:S2L_ATTN_PAIR=1 paper_2604_16395_b200/libs2l.so:S2L_ATTN_PAIR=0 6 > gpurun_out/r2e_ab.txt 2>&1; echo "exit $?" >> gpurun_out/r2e_ab.txt
