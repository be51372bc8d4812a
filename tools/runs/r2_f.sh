#!/bin/bash
# round 2: ncu of the CTA-pair kernel on the last C2 chunk
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:attn_pair -s 31 -c 1 -o gpurun_out/pair_full_r2f python bench.py --steps 1 --warmup 3 --no-side > gpurun_out/r2f_ncu.log 2>&1; echo rc=$? >> gpurun_out/r2f_ncu.log
