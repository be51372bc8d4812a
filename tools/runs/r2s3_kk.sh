#!/bin/bash
# round 2, session 3: flakiness check -- the GPU suite twice more + smoke
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null
for k in 1 2; do timeout -s KILL 2400 python -m pytest tests -m gpu -q --tb=short -p no:cacheprovider > gpurun_out/kk_gputests_$k.txt 2>&1; echo "run $k: $(tail -1 gpurun_out/kk_gputests_$k.txt)"; done
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
