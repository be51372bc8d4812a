#!/bin/bash
# round 2, session 3: one-unit kernel, shared-memory placement (Q first vs ring first)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout -s KILL 900 python tools/ab.py abl/J0.so abl/J1.so --c5 5 > gpurun_out/i_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/J0.so abl/J1.so 10 >> gpurun_out/i_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/J1.so abl/J0.so 10 >> gpurun_out/i_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/J1.so abl/J0.so --c5 5 >> gpurun_out/i_ab.txt 2>&1
grep -v Warn gpurun_out/i_ab.txt | tail -8
