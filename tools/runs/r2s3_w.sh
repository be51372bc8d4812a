#!/bin/bash
# round 2, session 3: bench with guarded side fields (N = 1) and the two-rank one-GPU bench test
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null
timeout -s KILL 900 python bench.py > gpurun_out/w_bench.json 2> gpurun_out/w_bench.err; echo rc=$?
python3 -c "
import json
d=json.loads(open('gpurun_out/w_bench.json').read().strip().splitlines()[-1])
print(d['value'], d['roofline']['frac'], sorted(k for k in d if k.endswith('_error')), len(d))"
timeout -s KILL 900 python -m pytest tests/test_gpu_multirank.py -m gpu -q -x -p no:cacheprovider > gpurun_out/w_mr.txt 2>&1; echo "exit $?"; tail -2 gpurun_out/w_mr.txt
