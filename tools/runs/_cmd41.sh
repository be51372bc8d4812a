S2L_NVCC_FLAGS="-DS2L_TRACE" python -m paper_2604_16395_b200.build --force > /dev/null
echo "== default trace"; timeout -s KILL 300 python tools/trace_run.py 2>&1 | tail -4
python -m paper_2604_16395_b200.build --force > /dev/null
