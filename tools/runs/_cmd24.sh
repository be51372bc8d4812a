nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/micro/pipe_bench.cu -o /tmp/pipe_bench && /tmp/pipe_bench
nvcc -O3 -gencode arch=compute_100a,code=sm_100a tools/micro/softmax_bench.cu -o /tmp/sb && /tmp/sb
