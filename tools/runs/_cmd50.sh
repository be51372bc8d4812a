python -m paper_2604_16395_b200.build --force > /dev/null
timeout -s KILL 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout -s KILL 600 python tools/e2e_diag.py 2>&1 | head -8
timeout -s KILL 600 python bench.py > gpurun_out/bench_r01e.json 2> gpurun_out/bench_r01e.err; python -c "
import json;d=json.load(open('gpurun_out/bench_r01e.json'));print('value',d['value'],'kernel',d['roofline']['achieved'],'e2e',d['e2e']['value'],'append',d['append']['achieved'])"
