#!/bin/bash
# round 2, session 2: poly share 2/8 vs 3/8 vs 4/8 (C2 both orders, C5)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout -s KILL 900 python tools/ab.py abl/poly2.so abl/poly3.so abl/poly4.so 10 > gpurun_out/u_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/poly4.so abl/poly3.so abl/poly2.so 10 >> gpurun_out/u_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/poly2.so abl/poly3.so abl/poly4.so --c5 5 >> gpurun_out/u_ab.txt 2>&1
grep -v Warn gpurun_out/u_ab.txt
