python -m paper_2604_16395_b200.build --force > /dev/null
for spec in "crawler --qps 8 --n 96" "crawler --qps 16 --n 96" "anns --qps 4 --n 96" "anns --qps 16 --n 96" "anns --qps 8 --n 96 --delay-scale 30 --gpu-blocks 3072"; do
  name=$(echo $spec | tr ' ' '_' | tr -d '-')
  timeout -s KILL 900 python tools/ttft_sim.py $spec --gemm > gpurun_out/ttft2_$name.json 2> gpurun_out/ttft2_$name.err
  echo "== $spec"; grep '^{' gpurun_out/ttft2_$name.err | cut -c1-160
done
