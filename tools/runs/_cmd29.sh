bash tools/ab_build.sh base "" pq "-DS2L_PQ=1" pq_p3 "-DS2L_PQ=1 -DS2L_POLY_PAIRS=3"
S2L_NVCC_FLAGS="-DS2L_PQ=1" python -m paper_2604_16395_b200.build --force > /dev/null
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -m "gpu" -x -q -k "tc_ or c2 or reduced or peaky or split" 2>&1 | tail -3
S2L_NVCC_FLAGS="-DS2L_PQ=1 -DS2L_TRACE" python -m paper_2604_16395_b200.build --force > /dev/null
echo "== pq trace"; timeout -s KILL 300 python tools/trace_run.py 2>&1 | tail -4
python -m paper_2604_16395_b200.build --force > /dev/null
