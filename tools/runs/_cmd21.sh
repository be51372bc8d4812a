S2L_ATTN_V5=1 KREGEX=attn_tc5 bash tools/ncu_variant.sh v5prof ""
python tools/ncu_stalls.py gpurun_out/v5prof.ncu-rep 50 > gpurun_out/v5_stalls.txt 2>&1
ncu -i gpurun_out/v5prof.ncu-rep --page raw --csv > gpurun_out/v5prof_raw.csv 2>&1
python tools/ncu_summary.py gpurun_out/v5prof.ncu-rep > gpurun_out/v5prof_summary.txt 2>&1
