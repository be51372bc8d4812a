#!/bin/bash
# ncu --set full of the last C2 attention launch for a build variant: tools/ncu_variant.sh <name> "<nvcc flags>"
name=$1; flags=$2
S2L_NVCC_FLAGS="$flags" python -m paper_2604_16395_b200.build --force > /dev/null || exit 1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:${KREGEX:-attn_tc2} -s 31 -c 1 \
  -o gpurun_out/$name python bench.py --steps 1 --warmup 3 --no-side > gpurun_out/$name.log 2>&1
echo "$name rc=$?"
