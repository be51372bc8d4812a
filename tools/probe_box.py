"""Probe the GPU box: host-link (PCIe) bandwidth with pinned memory, SM count, host cores/RAM.

Used once per round to record the swap roofline denominator.
Measures a single 1 GiB pinned cudaMemcpyAsync H2D, D2H and both directions at once,
best of 10, with CUDA events.
"""
import json, os, subprocess, time
import torch

def bw(fn, nbytes, reps=10):
    best = 0.0
    for _ in range(reps):
        s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize(); s.record(); fn(); e.record(); torch.cuda.synchronize()
        ms = s.elapsed_time(e)
        best = max(best, nbytes / (ms * 1e-3) / 1e9)
    return best

def main():
    out = {}
    p = torch.cuda.get_device_properties(0)
    out["gpu"] = p.name; out["sms"] = p.multi_processor_count; out["mem_gb"] = p.total_memory / 1e9
    out["nproc"] = os.cpu_count()
    with open("/proc/meminfo") as f:
        for line in f:
            if line.startswith(("MemTotal", "MemAvailable")):
                k, v = line.split(":"); out[k] = int(v.split()[0]) * 1024
    n = 1 << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    out["h2d_gbs"] = bw(lambda: d.copy_(h, non_blocking=True), n)
    out["d2h_gbs"] = bw(lambda: h.copy_(d, non_blocking=True), n)
    s1 = torch.cuda.Stream(); s2 = torch.cuda.Stream()
    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur); s2.wait_stream(cur)
        with torch.cuda.stream(s1): d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2): h2.copy_(d2, non_blocking=True)
        cur.wait_stream(s1); cur.wait_stream(s2)
    out["bidir_gbs_total"] = bw(both, 2 * n)
    # smaller transfer sizes (block-sized) for context
    for sz in (64 << 10, 512 << 10, 2 << 20, 16 << 20):
        cnt = min(256, n // sz)
        def many():
            for i in range(cnt):
                d[i * sz:(i + 1) * sz].copy_(h[i * sz:(i + 1) * sz], non_blocking=True)
        out[f"h2d_gbs_{sz>>10}KiB_x{cnt}"] = bw(many, sz * cnt, reps=5)
    try:
        out["nvidia_smi"] = subprocess.run(["nvidia-smi", "--query-gpu=name,clocks.sm,clocks.max.sm,pcie.link.gen.current,pcie.link.width.current", "--format=csv,noheader"], capture_output=True, text=True).stdout.strip()
        out["topo"] = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout.strip()[:2000]
        out["lscpu"] = subprocess.run(["lscpu"], capture_output=True, text=True).stdout.strip()[:1500]
    except Exception as ex:  # noqa
        out["smi_err"] = str(ex)
    print(json.dumps(out, indent=1))
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/probe_box.json", "w") as f:
        json.dump(out, f, indent=1)

if __name__ == "__main__":
    main()
