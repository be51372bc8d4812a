#!/bin/bash
# round 2, session 2: CTA-phase traces of C2 attention launches + sustained-clock probe
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
timeout -s KILL 300 python tools/clock_probe.py > gpurun_out/b_clock.json 2> gpurun_out/b_clock.err
S2L_NVCC_FLAGS="-DS2L_CTATRACE" python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
timeout -s KILL 600 python tools/cta_trace.py 0 4 16 31 > gpurun_out/b_cta.jsonl 2> gpurun_out/b_cta.err
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
cat gpurun_out/b_clock.json; cat gpurun_out/b_cta.jsonl; tail -3 gpurun_out/b_cta.err
