"""Samples nvidia-smi SM clocks / power every 50 ms while the C2 stream runs back to back for
~4 s (the bench's own timed region is too short for more than a few samples)."""
import json, os, statistics, subprocess, sys, time
import torch
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

torch.cuda.set_device(0)
rids, toks, data = bench.make_stream_data(0)
S = bench.Stream(rids, toks, data, "cuda:0")
ctx, pool = bench.make_ctx(0)
bench.run_step(ctx, S); torch.cuda.synchronize()
f = open("/tmp/clk.csv", "w")
pr = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap",
                       "--format=csv,noheader,nounits", "-lms", "50"], stdout=f)
time.sleep(0.5)
t0 = time.time(); n = 0
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
while time.time() - t0 < 4.0:
    for _ in range(20):
        bench.run_step(ctx, S); n += 1
    torch.cuda.synchronize()
e.record(); torch.cuda.synchronize()
pr.terminate(); pr.wait(); f.close()
rows = [l.split(",") for l in open("/tmp/clk.csv") if l.strip()]
mhz = [float(r[0]) for r in rows]; pw = [float(r[1]) for r in rows]
busy = [(m, p) for m, p in zip(mhz, pw) if p > 300]
ms = s.elapsed_time(e) / n
print(json.dumps({"steps": n, "ms_per_step": ms, "tflops": bench.step_flops() / (ms * 1e-3) / 1e12,
                  "samples": len(rows), "busy_samples": len(busy),
                  "sm_mhz_median_busy": statistics.median([b[0] for b in busy]) if busy else None,
                  "power_w_median_busy": statistics.median([b[1] for b in busy]) if busy else None,
                  "power_cap_active_frac": sum(1 for r in rows if "Active" in r[2]) / max(1, len(rows))}))
