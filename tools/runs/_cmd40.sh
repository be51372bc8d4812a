bash tools/ab_build.sh sm64_p1 "-DS2L_SM64=1 -DS2L_POLY_PAIRS=1" sm64_p0 "-DS2L_SM64=1 -DS2L_POLY_PAIRS=0" nosplit_sm64_p1 "-DS2L_SM64=1 -DS2L_POLY_PAIRS=1 -DS2L_SPLIT_S=0" base_p1 "-DS2L_POLY_PAIRS=1"
S2L_NVCC_FLAGS="-DS2L_SM64=1 -DS2L_POLY_PAIRS=1" python -m paper_2604_16395_b200.build --force > /dev/null
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m "gpu" -x -q 2>&1 | tail -3
python -m paper_2604_16395_b200.build --force > /dev/null
