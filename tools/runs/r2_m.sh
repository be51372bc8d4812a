#!/bin/bash
# round 2 evidence pass: full GPU suite (incl. slow / multi-rank), bench, sanitizers, ncu
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,temperature.gpu --format=csv > gpurun_out/r2m_smi.txt 2>&1
timeout -s KILL 600 python bench.py > gpurun_out/r2m_bench.json 2> gpurun_out/r2m_bench.err; echo "rc $?" >> gpurun_out/r2m_bench.err
timeout -s KILL 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rA > gpurun_out/r2m_gputests.txt 2>&1; echo "exit $?" >> gpurun_out/r2m_gputests.txt
timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2m_launches.csv python bench.py --steps 1 --warmup 3 --no-side > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc2 -s 31 -c 1 -o gpurun_out/r2m_attn_full python bench.py --steps 1 --warmup 3 --no-side > /dev/null 2>&1
timeout -s KILL 600 ncu --set full --clock-control none -k regex:append -s 31 -c 1 -o gpurun_out/r2m_append_full python bench.py --steps 1 --warmup 3 --no-side > /dev/null 2>&1
T="test_c1_full_walk or test_tc_gqa_ragged or test_fused_append_prefill_aligned or test_swap_scattered"
for tool in memcheck racecheck synccheck initcheck; do
  timeout -s KILL 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "$T" > gpurun_out/r2m_san_$tool.txt 2>&1; echo "rc=$?" >> gpurun_out/r2m_san_$tool.txt
done
