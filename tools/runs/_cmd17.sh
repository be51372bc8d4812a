bash tools/exp_variants.sh "-DS2L_EXP_MMA_ONLY -DS2L_EXP_NO_S -DS2L_EXP_NO_PV" "-DS2L_EXP_MMA_ONLY -DS2L_EXP_NO_S -DS2L_EXP_NO_PV -DS2L_EXP_HALF_LOAD" ""
timeout -s KILL 200 python -m pytest tests/test_gpu_parity.py -q -x -k "c1 or ragged or swap or c3" 2>&1 | tail -2
bash tools/ncu_variant.sh prof_noload_mma "-DS2L_EXP_MMA_ONLY -DS2L_EXP_NO_S -DS2L_EXP_NO_PV"
python -m paper_2604_16395_b200.build --force > /dev/null
timeout -s KILL 300 ncu --set full --clock-control none -k regex:append -s 31 -c 1 -o gpurun_out/append2 python bench.py --steps 1 --warmup 3 --no-side > /dev/null 2>&1; echo append rc=$?
