#!/bin/bash
# round 2, session 2: two MMA issuer warps: GPU suite, A/B (C2, C5), event trace
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/h_gputests.txt 2>&1; echo "exit $?" >> gpurun_out/h_gputests.txt
timeout -s KILL 900 python tools/ab.py abl/one.so abl/two.so abl/two_poly2.so 8 > gpurun_out/h_ab.txt 2>&1
timeout -s KILL 600 python tools/ab.py abl/one.so abl/two.so abl/two_poly2.so --c5 4 >> gpurun_out/h_ab.txt 2>&1
S2L_NVCC_FLAGS="-DS2L_TRACE" python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
timeout -s KILL 300 python tools/trace_run.py > gpurun_out/h_trace.txt 2>&1
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
tail -3 gpurun_out/h_gputests.txt; grep -v Warn gpurun_out/h_ab.txt; tail -2 gpurun_out/h_trace.txt
