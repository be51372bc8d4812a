python -m paper_2604_16395_b200.build --force > /dev/null
timeout -s KILL 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout -s KILL 600 python tools/e2e_diag.py 2>&1 | tail -20
timeout -s KILL 600 python bench.py > gpurun_out/bench_inl.json 2> gpurun_out/bench_inl.err; python -c "
import json;d=json.load(open('gpurun_out/bench_inl.json'));print('value',d['value'],'kernel',d['roofline']['achieved'],'e2e',d['e2e']['value'],'append',d['append']['achieved'])"
timeout -s KILL 900 python tools/bench_workloads.py c4mix > gpurun_out/c4mix.jsonl 2> gpurun_out/c4mix.err; python -c "
import json;d=json.loads(open('gpurun_out/c4mix.jsonl').read().strip().splitlines()[-1]);print({k:d[k]['ms'] for k in ('compute_only','serial','overlap')}, d['hidden_copy_frac'])"
