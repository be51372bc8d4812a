S2L_DIST_BACKEND=gloo S2L_BENCH_DEVICE=0 timeout -s KILL 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 2>gpurun_out/tr2.err | tail -1 | cut -c1-400
echo rc=$?
timeout -s KILL 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 2 --warmup 3 2>/dev/null | tail -1 | cut -c1-300
