#!/bin/bash
# round 2, session 3: per-step C2 A/B, persistent (F.so, S2L_PERSIST=1) vs one-unit kernel
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout -s KILL 900 python tools/step_ab.py abl/F.so:S2L_PERSIST=0 abl/F.so:S2L_PERSIST=1 abl/J1.so:S2L_PERSIST=0 4 > gpurun_out/n_steps.txt 2>&1
grep -v Warn gpurun_out/n_steps.txt | tail -4
