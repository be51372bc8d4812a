#!/bin/bash
# round 2, session 3: persistent kernel with a flat softmax loop (X1) vs nested (X0) vs the library (HEAD)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
S="abl/HEAD.so abl/X0.so abl/X1.so abl/X1.so:S2L_PERSIST_GRID=-1"
timeout -s KILL 900 python tools/ab.py $S --c5 4 > gpurun_out/q_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py $S 8 >> gpurun_out/q_ab.txt 2>&1
grep -v Warn gpurun_out/q_ab.txt | tail -8
