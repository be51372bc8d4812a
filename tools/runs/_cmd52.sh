bash tools/ab_build.sh base "" headmajor "-DS2L_HEAD_MAJOR=1"
S2L_NVCC_FLAGS="-DS2L_HEAD_MAJOR=1" python -m paper_2604_16395_b200.build --force > /dev/null
timeout -s KILL 900 python -m pytest tests/test_gpu_parity.py -m "gpu" -x -q -k "tc_ or c2 or split or c5 or c3 or reduced" 2>&1 | tail -2
timeout -s KILL 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:attn_tc2 -s 31 -c 1 python bench.py --steps 1 --warmup 3 --no-side 2>&1 | grep -E "dram__bytes|duration" | head -4
python -m paper_2604_16395_b200.build --force > /dev/null
timeout -s KILL 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:attn_tc2 -s 31 -c 1 python bench.py --steps 1 --warmup 3 --no-side 2>&1 | grep -E "dram__bytes|duration" | head -4
