python -m paper_2604_16395_b200.build --force > /dev/null
timeout -s KILL 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout -s KILL 900 python tools/bench_workloads.py c4mix > gpurun_out/c4mix.jsonl 2> gpurun_out/c4mix.err; cat gpurun_out/c4mix.jsonl; tail -3 gpurun_out/c4mix.err
