mkdir -p /tmp/s2l_ab
for r in 2 4 8; do S2L_NVCC_FLAGS="-DS2L_APPEND_ROWS=$r" python -m paper_2604_16395_b200.build --force > /dev/null; cp paper_2604_16395_b200/libs2l.so /tmp/s2l_ab/rows$r.so; done
python -m paper_2604_16395_b200.build --force > /dev/null
git_old=$(ls /tmp/s2l_ab)
timeout -s KILL 300 python tools/append_bench.py /tmp/s2l_ab/rows2.so /tmp/s2l_ab/rows4.so /tmp/s2l_ab/rows8.so
nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/micro/softmax_bench2.cu -o /tmp/sb2 && /tmp/sb2
