#!/bin/bash
# round 2: TMA append -- GPU suite, then A/B: plain (register append) / plain (TMA append) / fused
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
python -m paper_2604_16395_b200.build --force > /dev/null 2>&1
timeout -s KILL 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2j_gputests.txt 2>&1; echo "exit $?" >> gpurun_out/r2j_gputests.txt
cp paper_2604_16395_b200/libs2l.so /tmp/a.so; cp paper_2604_16395_b200/libs2l.so /tmp/b.so
timeout -s KILL 600 python tools/ab.py /tmp/a.so:S2L_APPEND_TMA=0 /tmp/b.so:S2L_APPEND_TMA=1 paper_2604_16395_b200/libs2l.so:FUSED=1 12 > gpurun_out/r2j_ab.txt 2>&1
