#!/bin/bash
# round 2, session 3: persistent kernel with fewer live registers across the softmax loop
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
S="abl/F.so:S2L_PERSIST=0 abl/F.so:S2L_PERSIST=1,S2L_PERSIST_GRID=-1 abl/F.so:S2L_PERSIST=1,S2L_PERSIST_GRID=0"
timeout -s KILL 900 python tools/ab.py $S --c5 4 > gpurun_out/g_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py $S 8 >> gpurun_out/g_ab.txt 2>&1
grep -v Warn gpurun_out/g_ab.txt | tail -6
