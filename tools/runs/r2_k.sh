#!/bin/bash
# round 2: append kernel alone: register vs TMA (events), plus ncu kernel durations
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
L=paper_2604_16395_b200/libs2l.so
timeout -s KILL 300 python tools/append_bench.py $L:S2L_APPEND_TMA=0 $L:S2L_APPEND_TMA=1 $L:S2L_APPEND_TMA=0 $L:S2L_APPEND_TMA=1 > gpurun_out/r2k_append.txt 2>&1
S2L_APPEND_TMA=0 timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:append -c 40 --csv python tools/append_bench.py $L > gpurun_out/r2k_ncu_reg.csv 2>/dev/null
S2L_APPEND_TMA=1 timeout -s KILL 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:append -c 40 --csv python tools/append_bench.py $L > gpurun_out/r2k_ncu_tma.csv 2>/dev/null
