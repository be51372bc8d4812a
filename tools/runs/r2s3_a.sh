#!/bin/bash
# round 2, session 3: fresh-container re-validation at HEAD (build, smoke, GPU suite, bench)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null
echo "== smoke"; timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
echo "== gpu tests"; timeout -s KILL 1500 python -m pytest tests -m gpu -q -x --tb=short > gpurun_out/a_gputests.txt 2>&1; tail -3 gpurun_out/a_gputests.txt
echo "== bench"; timeout -s KILL 600 python bench.py > gpurun_out/a_bench.json 2> gpurun_out/a_bench.err; tail -c 600 gpurun_out/a_bench.json
