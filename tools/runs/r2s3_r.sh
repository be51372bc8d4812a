#!/bin/bash
# round 2, session 3: bisect -- persistent kernel, one unit per CTA, with the one-unit kernel's MMA loop (X2)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
S="abl/HEAD.so abl/X1.so:S2L_PERSIST_GRID=-1 abl/X2.so:S2L_PERSIST_GRID=-1"
timeout -s KILL 900 python tools/ab.py $S --c5 4 > gpurun_out/r_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py $S 8 >> gpurun_out/r_ab.txt 2>&1
grep -v Warn gpurun_out/r_ab.txt | tail -6
