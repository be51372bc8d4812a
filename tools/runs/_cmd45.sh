S2L_NVCC_FLAGS="-DS2L_HSPLIT=1" python -m paper_2604_16395_b200.build --force > /dev/null
timeout -s KILL 300 python -m pytest tests/test_gpu_parity.py -m "gpu" -x -q -k "tc_gqa_ragged" 2>&1 | tail -3
bash tools/ab_build.sh base "" hsplit "-DS2L_HSPLIT=1"
S2L_NVCC_FLAGS="-DS2L_HSPLIT=1" python -m paper_2604_16395_b200.build --force > /dev/null
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m "gpu" -x -q 2>&1 | tail -3
python -m paper_2604_16395_b200.build --force > /dev/null
