#!/bin/bash
# round 2, session 2: final validation after the FP8 staging change: smoke, GPU suite, bench
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1; echo "build rc=$?"
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ak_smoke.txt 2>&1; echo "smoke rc=$?"
timeout -s KILL 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ak_gputests.txt 2>&1; echo "exit $?" >> gpurun_out/ak_gputests.txt
timeout -s KILL 900 python bench.py > gpurun_out/ak_bench.json 2> gpurun_out/ak_bench.err
tail -1 gpurun_out/ak_smoke.txt; tail -2 gpurun_out/ak_gputests.txt; tail -c 150 gpurun_out/ak_bench.json
