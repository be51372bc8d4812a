#!/bin/bash
# round 2, session 3: evidence for the current kernel (ring-first layout): launch list, ncu full of the
# last C2 attention launch, the append, the last C5 chunk; sanitizers; reference arm
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null
echo "== launches"; timeout -s KILL 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/l_launches.csv python bench.py --steps 1 --warmup 3 --no-side > /dev/null 2>&1; echo rc=$?
echo "== ncu attn"; timeout -s KILL 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc2 -s 31 -c 1 -o gpurun_out/l_attn_full python bench.py --steps 1 --warmup 3 --no-side > /dev/null 2>&1; echo rc=$?
echo "== ncu append"; timeout -s KILL 600 ncu --set full --clock-control none -k regex:append -s 31 -c 1 -o gpurun_out/l_append_full python bench.py --steps 1 --warmup 3 --no-side > /dev/null 2>&1; echo rc=$?
echo "== ncu c5"; timeout -s KILL 600 ncu --set full --clock-control none -k regex:attn_tc2 -s 63 -c 1 -o gpurun_out/l_c5_full python tools/c5_stream_once.py > /dev/null 2>&1; echo rc=$?
echo "== sanitizers"
for tool in memcheck racecheck synccheck initcheck; do
  timeout -s KILL 900 compute-sanitizer --tool $tool --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "c1_full_walk or tc_gqa_ragged or tail_wave or fused_append_prefill_aligned or swap_scattered_ids_staged" > gpurun_out/l_san_$tool.txt 2>&1; echo "$tool rc=$?"; tail -2 gpurun_out/l_san_$tool.txt
done
echo "== reference arm"; timeout -s KILL 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/l_reference.json 2> gpurun_out/l_reference.err; tail -c 300 gpurun_out/l_reference.json
