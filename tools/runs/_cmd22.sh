python -m paper_2604_16395_b200.build --force > /dev/null
cp paper_2604_16395_b200/libs2l.so /tmp/cur.so
timeout -s KILL 300 python tools/ab.py /tmp/cur.so /tmp/cur.so:S2L_ATTN_V5=1 6
S2L_ATTN_V5=1 timeout -s KILL 600 python -m pytest tests/test_gpu_parity.py -m "gpu and not slow" -x -q 2>&1 | tail -3
