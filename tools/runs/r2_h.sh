#!/bin/bash
# round 2: pair kernel -- parity subset, A/B vs tc2, then the trace build timeline
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -m "gpu and not slow" -x -q -p no:cacheprovider -k "tc_ or c2 or gqa or block" > gpurun_out/r2h_parity.txt 2>&1; echo "exit $?" >> gpurun_out/r2h_parity.txt
cp paper_2604_16395_b200/libs2l.so /tmp/cur.so
timeout -s KILL 400 python tools/ab.py /tmp/cur.so:S2L_ATTN_PAIR=1 paper_2604_16395_b200/libs2l.so:S2L_ATTN_PAIR=0 6 > gpurun_out/r2h_ab.txt 2>&1; echo "exit $?" >> gpurun_out/r2h_ab.txt
S2L_NVCC_FLAGS=-DS2L_TRACE python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
timeout -s KILL 300 python tools/trace_pair.py > gpurun_out/r2h_trace.txt 2>&1; echo "exit $?" >> gpurun_out/r2h_trace.txt
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
