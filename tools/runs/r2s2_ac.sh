#!/bin/bash
# round 2, session 2: predicated item scan in the unit decode: A/B (both orders), C5, CTA trace, parity subset
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout -s KILL 900 python tools/ab.py abl/base.so abl/new.so 10 > gpurun_out/ac_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/new.so abl/base.so 10 >> gpurun_out/ac_ab.txt 2>&1
timeout -s KILL 900 python tools/ab.py abl/base.so abl/new.so --c5 4 >> gpurun_out/ac_ab.txt 2>&1
S2L_NVCC_FLAGS="-DS2L_CTATRACE" python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
timeout -s KILL 600 python tools/cta_trace.py 0 31 > gpurun_out/ac_cta.jsonl 2> gpurun_out/ac_cta.err
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "gqa or c2t or tail_wave or many_items or more_than" > gpurun_out/ac_tests.txt 2>&1; echo "exit $?" >> gpurun_out/ac_tests.txt
grep -v Warn gpurun_out/ac_ab.txt; cut -c1-400 gpurun_out/ac_cta.jsonl; tail -2 gpurun_out/ac_tests.txt
