#!/bin/bash
# round 2, session 3: ncu of the persistent vs one-unit kernel (C5 last chunk, C2 last chunk)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
cp abl/B.so paper_2604_16395_b200/libs2l.so; touch paper_2604_16395_b200/libs2l.so
for P in 0 1; do
  S2L_PERSIST=$P timeout -s KILL 600 ncu --set full --clock-control none -k regex:attn_tc2 -s 63 -c 1 -o gpurun_out/d_c5_p$P python tools/c5_stream_once.py > gpurun_out/d_c5_p$P.log 2>&1; echo "c5 p$P rc=$?"
  S2L_PERSIST=$P timeout -s KILL 600 ncu --set full --clock-control none -k regex:attn_tc2 -s 31 -c 1 -o gpurun_out/d_c2_p$P python bench.py --steps 1 --warmup 3 --no-side > gpurun_out/d_c2_p$P.log 2>&1; echo "c2 p$P rc=$?"
done
ls -la gpurun_out/
