#!/bin/bash
# round 2, session 3: longer A/B of the ring-first placement (J1) vs the current layout (J0)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for k in 1 2 3; do
timeout -s KILL 900 python tools/ab.py abl/J0.so abl/J1.so 12 >> gpurun_out/j_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/J1.so abl/J0.so 12 >> gpurun_out/j_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/J0.so abl/J1.so --c5 4 >> gpurun_out/j_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/J1.so abl/J0.so --c5 4 >> gpurun_out/j_ab.txt 2>&1
done
grep -v Warn gpurun_out/j_ab.txt
