#!/bin/bash
# round 2, session 2: CTA-phase trace with decode / epilogue sub-phases
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
S2L_NVCC_FLAGS="-DS2L_CTATRACE" python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
timeout -s KILL 600 python tools/cta_trace.py 0 4 31 > gpurun_out/e_cta.jsonl 2> gpurun_out/e_cta.err
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
cat gpurun_out/e_cta.jsonl; tail -3 gpurun_out/e_cta.err
