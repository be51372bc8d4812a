#!/bin/bash
# round 2: timeline trace of the CTA-pair kernel (S2L_TRACE build)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
S2L_NVCC_FLAGS=-DS2L_TRACE python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
timeout -s KILL 300 python tools/trace_pair.py > gpurun_out/r2g_trace.txt 2>&1; echo "exit $?" >> gpurun_out/r2g_trace.txt
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
