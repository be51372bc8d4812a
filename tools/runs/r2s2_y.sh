#!/bin/bash
# round 2, session 2: fused (NEXT-2) vs plain per-kernel breakdown + launch list of the fused step
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout -s KILL 600 python tools/fused_diag.py abl/cur.so abl/cur.so:FUSED=1 6 > gpurun_out/y_fused.txt 2>&1
cat > /tmp/fused_step.py <<'PY'
import sys, os, torch
sys.path.insert(0, os.getcwd())
import bench
torch.cuda.set_device(0)
rids, toks, data = bench.make_stream_data(0)
S = bench.Stream(rids, toks, data, "cuda:0")
ctx, pool = bench.make_ctx(0)
for _ in range(3):
    bench.run_step_fused(ctx, S)
torch.cuda.synchronize()
PY
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/y_launches_fused.csv python /tmp/fused_step.py > /dev/null 2>&1
python tools/ncu_summary.py launches gpurun_out/y_launches_fused.csv > gpurun_out/y_launches_fused.txt
grep -v Warn gpurun_out/y_fused.txt | tail -12; cat gpurun_out/y_launches_fused.txt
