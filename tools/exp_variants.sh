#!/bin/bash
# Timing experiments: rebuild with each flag set, run the C2 bench (value, kernel TFLOP/s).
for flags in "$@"; do
  S2L_NVCC_FLAGS="$flags" python -m paper_2604_16395_b200.build --force > /dev/null 2>/tmp/exp_build.txt || { echo "[$flags] BUILD FAILED"; tail -5 /tmp/exp_build.txt; continue; }
  out=$(timeout -s KILL 150 python bench.py --no-side 2>/tmp/exp_err.txt | tail -1)
  echo "[$flags] $(echo "$out" | python -c 'import json,sys
try:
  d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["roofline"]["achieved"],1), d["parity"]["max_normwise_err"])
except Exception as e: print("FAILED", e)')"
done
python -m paper_2604_16395_b200.build --force > /dev/null
