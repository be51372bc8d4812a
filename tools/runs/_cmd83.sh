mkdir -p gpurun_out
timeout -s KILL 1500 python tools/ttft_sim.py anns --qps 4 --n 96 --model > gpurun_out/ttft_model_anns_qps_4_n_96.jsonl 2> gpurun_out/ttft_model_anns.err; tail -5 gpurun_out/ttft_model_anns.err
