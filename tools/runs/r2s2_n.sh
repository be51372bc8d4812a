#!/bin/bash
# round 2, session 2: ncu evidence of the current kernels (launch list, attention + append full sets)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/n_launches.csv python bench.py --steps 1 --warmup 3 --no-side > /dev/null 2>&1; echo launches rc=$?
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc2 -s 31 -c 1 -o gpurun_out/n_attn_full python bench.py --steps 1 --warmup 3 --no-side > /dev/null 2>&1; echo attn rc=$?
timeout -s KILL 600 ncu --set full --clock-control none -k regex:append -s 31 -c 1 -o gpurun_out/n_append_full python bench.py --steps 1 --warmup 3 --no-side > /dev/null 2>&1; echo append rc=$?
ls -la gpurun_out/n_*
