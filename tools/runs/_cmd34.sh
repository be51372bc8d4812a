python -m paper_2604_16395_b200.build --force > /dev/null
timeout -s KILL 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
C4_TIMELINE=1 timeout -s KILL 900 python tools/bench_workloads.py c4mix > gpurun_out/c4mix.jsonl 2> gpurun_out/c4mix.err; cat gpurun_out/c4mix.jsonl; tail -30 gpurun_out/c4mix.err
timeout -s KILL 900 python tools/ttft_sim.py crawler --qps 4 --n 32 --gemm > gpurun_out/ttft_crawler_test.json 2> gpurun_out/ttft_crawler_test.err; tail -8 gpurun_out/ttft_crawler_test.err
