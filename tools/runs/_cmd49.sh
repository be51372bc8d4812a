python -m paper_2604_16395_b200.build --force > /dev/null
echo "== gpu tests"; timeout -s KILL 900 python -m pytest tests -m gpu -q 2>&1 | tail -2
bash tools/round_evidence.sh r01d
echo "== reference arm"; timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref_r01d.json 2> gpurun_out/ref_r01d.err; tail -c 300 gpurun_out/ref_r01d.json
echo "== torchrun 2 ranks on one GPU (gloo)"; S2L_BENCH_DEVICE=0 S2L_DIST_BACKEND=gloo timeout -s KILL 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 2 --warmup 3 --no-side > gpurun_out/tr2_r01d.json 2> gpurun_out/tr2_r01d.err; tail -c 500 gpurun_out/tr2_r01d.json; tail -3 gpurun_out/tr2_r01d.err
timeout -s KILL 900 python tools/bench_workloads.py c4mix > gpurun_out/c4mix_r01d.jsonl 2> gpurun_out/c4mix_r01d.err; tail -c 300 gpurun_out/c4mix_r01d.jsonl
