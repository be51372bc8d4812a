#!/bin/bash
# round 2, session 3: ring-first layout default -- smoke, full GPU suite (incl. the new full-size C5 test), bench
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null
echo "== smoke"; timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/k_smoke.txt 2>&1; tail -1 gpurun_out/k_smoke.txt
echo "== gpu tests"; timeout -s KILL 1800 python -m pytest tests -m gpu -q -x --tb=short --durations=8 > gpurun_out/k_gputests.txt 2>&1; tail -14 gpurun_out/k_gputests.txt
echo "== bench"; timeout -s KILL 600 python bench.py > gpurun_out/k_bench.json 2> gpurun_out/k_bench.err; tail -c 200 gpurun_out/k_bench.json
