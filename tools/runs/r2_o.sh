#!/bin/bash
# round 2: re-validation -- full GPU suite, bench (FP8 field), sanitizers on the fixed tests
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
timeout -s KILL 600 python bench.py > gpurun_out/r2o_bench.json 2> gpurun_out/r2o_bench.err; echo "rc $?" >> gpurun_out/r2o_bench.err
timeout -s KILL 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r2o_gputests.txt 2>&1; echo "exit $?" >> gpurun_out/r2o_gputests.txt
T="test_c1_full_walk or test_tc_gqa_ragged or test_fused_append_prefill_aligned or test_swap_scattered or test_fp8"
for tool in memcheck racecheck synccheck initcheck; do
  timeout -s KILL 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fp8.py -q -p no:cacheprovider -k "$T" > gpurun_out/r2o_san_$tool.txt 2>&1; echo "rc=$?" >> gpurun_out/r2o_san_$tool.txt
done
