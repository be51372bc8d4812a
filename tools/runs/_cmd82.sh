timeout -s KILL 600 python bench.py 2>/dev/null | tail -1 > gpurun_out/bench_s5.json; python -c "
import json; d=json.loads(open('gpurun_out/bench_s5.json').read())
print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['parity'], d['next2_fused'])"
