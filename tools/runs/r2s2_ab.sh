#!/bin/bash
# round 2, session 2: driver-style checks: smoke(), full GPU suite (new staged-swap and C2t cases)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/ab_build.txt 2>&1; echo "build rc=$?"
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ab_smoke.txt 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/ab_smoke.txt
timeout -s KILL 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/ab_gputests.txt 2>&1; echo "exit $?" >> gpurun_out/ab_gputests.txt
tail -2 gpurun_out/ab_gputests.txt
