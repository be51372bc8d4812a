#!/bin/bash
# round 2, session 3: shared-memory placement experiments (one-unit kernel with the ring at 128 KB; persistent with the ring first)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
S="abl/F.so:S2L_PERSIST=0 abl/I.so:S2L_PERSIST=0 abl/G.so:S2L_PERSIST=0 abl/F.so:S2L_PERSIST=1 abl/H.so:S2L_PERSIST=1"
timeout -s KILL 900 python tools/ab.py $S --c5 4 > gpurun_out/h_ab.txt 2>&1
grep -v Warn gpurun_out/h_ab.txt | tail -6
