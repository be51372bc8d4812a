#!/bin/bash
# round 2, session 3: exp2 polynomial share after the layout change -- bf16 2/8 (Q0) vs 3/8 (Q3); FP8 1/8 (Q0) vs 2/8 (QF2)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for k in 1 2; do
timeout -s KILL 900 python tools/ab.py abl/Q0.so abl/Q3.so 10 >> gpurun_out/ll_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/Q3.so abl/Q0.so 10 >> gpurun_out/ll_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/Q0.so abl/Q3.so --c5 4 >> gpurun_out/ll_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/Q0.so:KV=1 abl/QF2.so:KV=1 8 >> gpurun_out/ll_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/QF2.so:KV=1 abl/Q0.so:KV=1 8 >> gpurun_out/ll_ab.txt 2>&1
done
grep -v Warn gpurun_out/ll_ab.txt
