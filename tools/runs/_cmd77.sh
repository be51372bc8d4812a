mkdir -p gpurun_out
timeout -s KILL 1500 python tools/ttft_sim.py crawler --qps 8 --n 96 --model > gpurun_out/ttft_model_crawler_qps_8_n_96.jsonl 2> gpurun_out/ttft_model.err; tail -5 gpurun_out/ttft_model.err
