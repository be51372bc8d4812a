#!/bin/bash
# round 2, session 2: full GPU suite + compute-sanitizer (memcheck, racecheck, synccheck, initcheck)
# on the tests that cover the new epilogue (TMA-store output, split merge paths) and staged swaps
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
timeout -s KILL 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/p_gputests.txt 2>&1; echo "exit $?" >> gpurun_out/p_gputests.txt
T="c1_full_walk or tc_gqa_ragged or tail_wave or fused or scattered or fp8_attention_c1"
for tool in memcheck racecheck synccheck initcheck; do
  timeout -s KILL 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fp8.py -q -p no:cacheprovider -k "$T" > gpurun_out/p_san_$tool.txt 2>&1; echo "rc=$?" >> gpurun_out/p_san_$tool.txt
done
tail -2 gpurun_out/p_gputests.txt; for tool in memcheck racecheck synccheck initcheck; do echo "== $tool"; tail -3 gpurun_out/p_san_$tool.txt; done
