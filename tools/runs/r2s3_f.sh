#!/bin/bash
# round 2, session 3: persistent kernel steady state -- one unit per CTA through the persistent code
# (S2L_PERSIST_GRID=-1), and ring depth 2
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
S="abl/D.so:S2L_PERSIST=0 abl/D.so:S2L_PERSIST=1,S2L_PERSIST_GRID=-1 abl/D.so:S2L_PERSIST=1,S2L_PERSIST_GRID=0 abl/E.so:S2L_PERSIST=1,S2L_PERSIST_GRID=0"
timeout -s KILL 900 python tools/ab.py $S --c5 4 > gpurun_out/f_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py $S 8 >> gpurun_out/f_ab.txt 2>&1
grep -v Warn gpurun_out/f_ab.txt | tail -8
