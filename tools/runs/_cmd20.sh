S2L_NVCC_FLAGS="-DS2L_TRACE" python -m paper_2604_16395_b200.build --force > /dev/null
S2L_ATTN_V5=1 timeout -s KILL 300 python tools/trace_run.py 2>&1 | tail -60
python -m paper_2604_16395_b200.build --force > /dev/null
