bash tools/ab_build.sh base "" stale "-DS2L_STALE=1"
S2L_NVCC_FLAGS="-DS2L_STALE=1" python -m paper_2604_16395_b200.build --force > /dev/null
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m "gpu" -x -q 2>&1 | tail -3
S2L_NVCC_FLAGS="-DS2L_STALE=1 -DS2L_TRACE" python -m paper_2604_16395_b200.build --force > /dev/null
echo "== stale trace"; timeout -s KILL 300 python tools/trace_run.py 2>&1 | tail -4
python -m paper_2604_16395_b200.build --force > /dev/null
