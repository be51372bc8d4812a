"""Scattered-swap staging threshold sweep: bench.swap_cell (random 64 KiB GPU ids, L = 1) for a few
block counts with S2L_STAGE_MIN_RUNS = 2 / 4 / 16 (the library reads it at context creation)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402

torch.cuda.set_device(0)
link = bench.measure_link(torch.device("cuda:0"))
mode = sys.argv[1] if len(sys.argv) > 1 else "runs"
cells = ([(thr, "262144", 1, B) for thr in ("16", "4", "2") for B in (4, 8, 16, 32, 64)] if mode == "runs" else
         [("4", rb, L, B) for rb in ("262144", "4194304", "67108864") for L in (8, 32) for B in (8, 64, 512)])
for thr, rb, L, B in cells:
        os.environ["S2L_STAGE_MIN_RUNS"] = thr
        os.environ["S2L_STAGE_RUN_BYTES"] = rb
        c = bench.swap_cell(0, L, B, True)
        print(json.dumps({"min_runs": int(thr), "run_bytes": int(rb), "L": L, "blocks": B, "runs": c["gpu_id_runs"],
                          "out_frac": round(c["out_gbs"] / link["d2h"], 3), "in_frac": round(c["in_gbs"] / link["h2d"], 3),
                          "out_frac_call": round(c["out_gbs_call"] / link["d2h"], 3),
                          "in_frac_call": round(c["in_gbs_call"] / link["h2d"], 3)}), flush=True)
