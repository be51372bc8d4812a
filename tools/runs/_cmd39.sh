bash tools/ab_build.sh base "" sm64 "-DS2L_SM64=1" sm64_p4 "-DS2L_SM64=1 -DS2L_POLY_PAIRS=4" sm64_p1 "-DS2L_SM64=1 -DS2L_POLY_PAIRS=1"
S2L_NVCC_FLAGS="-DS2L_SM64=1" python -m paper_2604_16395_b200.build --force > /dev/null
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -m "gpu" -x -q -k "tc_ or c2 or reduced or peaky or split or c5 or c3" 2>&1 | tail -3
python -m paper_2604_16395_b200.build --force > /dev/null
