#!/bin/bash
# round 2, session 2: warp-level P arrivals: parity, A/B, event trace
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fp8.py tests/test_gpu_fullsize.py -m gpu -x -q > gpurun_out/m_gputests.txt 2>&1; echo "exit $?" >> gpurun_out/m_gputests.txt
timeout -s KILL 900 python tools/ab.py abl/base.so abl/warparr.so 8 > gpurun_out/m_ab.txt 2>&1
timeout -s KILL 600 python tools/ab.py abl/base.so abl/warparr.so --c5 4 >> gpurun_out/m_ab.txt 2>&1
S2L_NVCC_FLAGS="-DS2L_TRACE" python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
timeout -s KILL 300 python tools/trace_run.py > gpurun_out/m_trace.txt 2>&1
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
tail -2 gpurun_out/m_gputests.txt; grep -v Warn gpurun_out/m_ab.txt; tail -1 gpurun_out/m_trace.txt
