#!/bin/bash
# round 2, session 3: persistent kernel with the MMA steady loop peeled (X3)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
S="abl/HEAD.so abl/X3.so abl/X3.so:S2L_PERSIST_GRID=-1"
timeout -s KILL 900 python tools/ab.py $S --c5 4 > gpurun_out/s_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py $S 8 >> gpurun_out/s_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/X3.so abl/HEAD.so 8 >> gpurun_out/s_ab.txt 2>&1
grep -v Warn gpurun_out/s_ab.txt | tail -8
