python -m paper_2604_16395_b200.build --force > /dev/null
echo "== gpu tests"; timeout -s KILL 900 python -m pytest tests -m gpu -q 2>&1 | tail -3
bash tools/round_evidence.sh r01c
echo "== reference arm"; timeout -s KILL 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref_r01c.json 2> gpurun_out/ref_r01c.err; tail -c 600 gpurun_out/ref_r01c.json
