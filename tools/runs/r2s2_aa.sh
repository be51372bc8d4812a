#!/bin/bash
# round 2, session 2: final evidence of the current kernels: FA4 comparisons (C2, C5), ncu
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
timeout -s KILL 900 python tools/fa4_compare.py --out gpurun_out/aa_fa4_c2.json > gpurun_out/aa_fa4_c2.log 2>&1
timeout -s KILL 1200 python tools/fa4_compare.py --c5 --reps 3 --out gpurun_out/aa_fa4_c5.json > gpurun_out/aa_fa4_c5.log 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/aa_launches.csv python bench.py --steps 1 --warmup 3 --no-side > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc2 -s 31 -c 1 -o gpurun_out/aa_attn_full python bench.py --steps 1 --warmup 3 --no-side > /dev/null 2>&1
tail -1 gpurun_out/aa_fa4_c2.log; tail -1 gpurun_out/aa_fa4_c5.log; ls gpurun_out/aa_*
