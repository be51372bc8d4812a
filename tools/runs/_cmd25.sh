# A/B: truncation packing of P, poly share
bash tools/ab_build.sh base "" trunc "-DS2L_PACK_TRUNC=1" trunc_p3 "-DS2L_PACK_TRUNC=1 -DS2L_POLY_PAIRS=3" p3 "-DS2L_POLY_PAIRS=3" trunc_p1 "-DS2L_PACK_TRUNC=1 -DS2L_POLY_PAIRS=1"
S2L_NVCC_FLAGS="-DS2L_PACK_TRUNC=1" python -m paper_2604_16395_b200.build --force > /dev/null
timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -m "gpu" -x -q 2>&1 | tail -3
