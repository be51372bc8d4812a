#!/bin/bash
# round 2, session 3: why the persistent kernel is slower in the steady state --
# ring depth (one-unit kernel with 3 slots) vs polling warps 2-3 (suspend-hint waits)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
S="abl/A.so:S2L_PERSIST=0 abl/C.so:S2L_PERSIST=0 abl/A.so:S2L_PERSIST=1 abl/B.so:S2L_PERSIST=1"
timeout -s KILL 900 python tools/ab.py $S 8 > gpurun_out/c_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py $S --c5 4 >> gpurun_out/c_ab.txt 2>&1
grep -v Warn gpurun_out/c_ab.txt | tail -12
