#!/bin/bash
# round 2, session 2: K0/V0 pre-issue + wait_group.read epilogue: GPU suite, A/B, CTA trace, bench
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -x -q > gpurun_out/i_gputests.txt 2>&1; echo "exit $?" >> gpurun_out/i_gputests.txt
timeout -s KILL 900 python tools/ab.py abl/base.so abl/new.so 8 > gpurun_out/i_ab.txt 2>&1
timeout -s KILL 600 python tools/ab.py abl/base.so abl/new.so --c5 4 >> gpurun_out/i_ab.txt 2>&1
S2L_NVCC_FLAGS="-DS2L_CTATRACE" python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
timeout -s KILL 600 python tools/cta_trace.py 0 4 31 > gpurun_out/i_cta.jsonl 2> gpurun_out/i_cta.err
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
timeout -s KILL 900 python bench.py > gpurun_out/i_bench.json 2> gpurun_out/i_bench.err
tail -3 gpurun_out/i_gputests.txt; grep -v Warn gpurun_out/i_ab.txt; cat gpurun_out/i_cta.jsonl | cut -c1-900; tail -c 300 gpurun_out/i_bench.json
