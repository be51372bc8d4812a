#!/bin/bash
# round 2, session 3: FlashAttention-4 same-window comparison with the final kernel (C2 and C5)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null
timeout -s KILL 1200 python tools/fa4_compare.py --reps 5 --out gpurun_out/nn_fa4_c2.json > gpurun_out/nn_fa4_c2.log 2>&1; echo "c2 rc=$?"; tail -c 600 gpurun_out/nn_fa4_c2.json
timeout -s KILL 1200 python tools/fa4_compare.py --reps 3 --c5 --out gpurun_out/nn_fa4_c5.json > gpurun_out/nn_fa4_c5.log 2>&1; echo "c5 rc=$?"; tail -c 600 gpurun_out/nn_fa4_c5.json
