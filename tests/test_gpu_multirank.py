"""Multi-rank runs of bench.py on one GPU (the driver's N-GPU launch path, gloo because the
ranks share the device): `--gpus 2` spawns two ranks itself, each rank owns its shard (C2/C3:
its requests; C5: its KV heads; C4: its requests), output rows are gathered to rank 0 and
checked against the fp64 oracle."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bench(*args, env=None, timeout=1500):
    e = dict(os.environ, **(env or {}))
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, env=e, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert lines, r.stdout[-2000:] + r.stderr[-2000:]
    return json.loads(lines[-1])


def test_bench_two_ranks_c2_c3_c5_sharded():
    d = _bench("--gpus", "2", "--steps", "1", "--warmup", "3", "--no-side")
    assert d["n_gpus"] == 2 and d["placement"]["ranks"] == 2
    assert d["parity"]["pass"] and d["parity"]["ranks"] == 2          # rows of both ranks' requests
    assert d["c5"]["parity"]["pass"] and d["c5"]["sharding"] == "kv heads 8/2 per rank"
    assert d["c3"]["parity"]["pass"]
    assert d["e2e"]["value"] > 0 and d["cpu_baseline"]["value"] > 0


def test_bench_two_ranks_c4_request_sharded():
    d = _bench("--gpus", "2", "--workload", "c4", "--steps", "1", "--warmup", "3",
               env={"S2L_C4_REQUESTS": "48"})
    assert d["n_gpus"] == 2 and d["config"]["requests"] == 48
    assert d["value"] > 0 and d["swap"]["out_bytes"] > 0 and d["swap"]["in_bytes"] > 0
    assert d["host_link_concurrent_aggregate_gbs"]["h2d"] > 0
