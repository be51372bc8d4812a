#!/bin/bash
# round 2, session 2: C2t GPU test, poly-share A/B with more rounds (C2 step/kernel, C5 kernel)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "c2t or gqa_ragged" > gpurun_out/t_tests.txt 2>&1; echo "exit $?" >> gpurun_out/t_tests.txt
timeout -s KILL 900 python tools/ab.py abl/new.so abl/poly2.so 12 > gpurun_out/t_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/new.so abl/poly2.so --c5 6 >> gpurun_out/t_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/poly2.so abl/new.so 12 >> gpurun_out/t_ab.txt 2>&1
tail -2 gpurun_out/t_tests.txt; grep -v Warn gpurun_out/t_ab.txt
