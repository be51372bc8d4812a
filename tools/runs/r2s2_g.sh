#!/bin/bash
# round 2, session 2: event trace of CTA 0 (steady-state chain) + poly-share A/B on the new epilogue
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
S2L_NVCC_FLAGS="-DS2L_TRACE" python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
timeout -s KILL 300 python tools/trace_run.py > gpurun_out/g_trace.txt 2>&1
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
timeout -s KILL 600 python tools/ab.py abl/new.so abl/poly2.so abl/poly0.so 6 > gpurun_out/g_ab.txt 2>&1
tail -3 gpurun_out/g_trace.txt; grep -v Warn gpurun_out/g_ab.txt
