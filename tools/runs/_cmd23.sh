set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m paper_2604_16395_b200.build --force > /dev/null
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout -s KILL 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout -s KILL 600 python bench.py > gpurun_out/bench_r01b.json 2> gpurun_out/bench_r01b.err; cat gpurun_out/bench_r01b.json; tail -3 gpurun_out/bench_r01b.err
