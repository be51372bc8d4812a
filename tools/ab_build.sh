#!/bin/bash
# tools/ab_build.sh name "flags" [name "flags" ...] -> /tmp/s2l_ab/<name>.so, then runs tools/ab.py
mkdir -p /tmp/s2l_ab; libs=()
while [ $# -ge 2 ]; do
  S2L_NVCC_FLAGS="$2" python -m paper_2604_16395_b200.build --force > /dev/null || { echo "build $1 failed"; exit 1; }
  cp paper_2604_16395_b200/libs2l.so /tmp/s2l_ab/$1.so; libs+=(/tmp/s2l_ab/$1.so); shift 2
done
python -m paper_2604_16395_b200.build --force > /dev/null
timeout -s KILL 600 python tools/ab.py "${libs[@]}" 6
