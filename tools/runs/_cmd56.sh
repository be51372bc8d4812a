mkdir -p /tmp/s2l_ab
python -m paper_2604_16395_b200.build --force > /dev/null; cp paper_2604_16395_b200/libs2l.so /tmp/s2l_ab/split.so
S2L_NVCC_FLAGS="-DS2L_SPLIT_S=0" python -m paper_2604_16395_b200.build --force > /dev/null; cp paper_2604_16395_b200/libs2l.so /tmp/s2l_ab/nosplit.so
python -m paper_2604_16395_b200.build --force > /dev/null
timeout -s KILL 600 python tools/ab.py /tmp/s2l_ab/split.so /tmp/s2l_ab/nosplit.so 20
timeout -s KILL 600 python tools/ab.py /tmp/s2l_ab/nosplit.so /tmp/s2l_ab/split.so 20
