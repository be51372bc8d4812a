#!/bin/bash
# round 2, session 2: sum-check fast path (no tile max): GPU suite, A/B vs HEAD, CTA trace
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/d_gputests.txt 2>&1; echo "exit $?" >> gpurun_out/d_gputests.txt
timeout -s KILL 600 python tools/ab.py abl/base.so abl/new.so 8 > gpurun_out/d_ab.txt 2>&1
timeout -s KILL 600 python tools/ab.py abl/base.so abl/new.so --c5 4 >> gpurun_out/d_ab.txt 2>&1
S2L_NVCC_FLAGS="-DS2L_CTATRACE" python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
timeout -s KILL 600 python tools/cta_trace.py 0 4 31 > gpurun_out/d_cta.jsonl 2> gpurun_out/d_cta.err
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
tail -3 gpurun_out/d_gputests.txt; cat gpurun_out/d_ab.txt | grep -v Warn; cat gpurun_out/d_cta.jsonl; tail -3 gpurun_out/d_cta.err
