python -m paper_2604_16395_b200.build --force > /dev/null
timeout -s KILL 1500 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_gpu_parity.py -q -x -k "hazards or scheduler_on_device or c4_pressure or c1_full_walk or tc_gqa_ragged or errors_and_edges" > gpurun_out/memcheck_wide.txt 2>&1; echo rc=$?; tail -6 gpurun_out/memcheck_wide.txt
