S2L_NVCC_FLAGS="-DS2L_HSPLIT=1 -DS2L_TRACE" python -m paper_2604_16395_b200.build --force > /dev/null
timeout -s KILL 300 python tools/trace_run.py > /dev/null 2>&1
python -m paper_2604_16395_b200.build --force > /dev/null
