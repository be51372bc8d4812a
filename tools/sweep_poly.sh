#!/bin/bash
# Rebuilds libs2l with different poly-exp2 fractions and runs the C2 bench (no side rows).
for n in ${@:-0 2 3 4}; do
  S2L_NVCC_FLAGS="-DS2L_POLY_PAIRS=$n" python -m paper_2604_16395_b200.build --force > /dev/null
  out=$(timeout -s KILL 150 python bench.py --no-side 2>/tmp/sweep_err.txt | tail -1)
  echo "poly_pairs=$n $(echo "$out" | python -c 'import json,sys
try:
  d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["roofline"]["achieved"],1), d["parity"]["max_normwise_err"])
except Exception as e: print("FAILED", e)')"
done
python -m paper_2604_16395_b200.build --force > /dev/null
