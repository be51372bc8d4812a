python -m paper_2604_16395_b200.build --force > /dev/null
C4_TIMELINE=1 timeout -s KILL 900 python tools/bench_workloads.py c4mix > gpurun_out/c4mix.jsonl 2> gpurun_out/c4mix.err; tail -60 gpurun_out/c4mix.err
