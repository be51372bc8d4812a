"""Synthetic streaming traces shaped like the paper's retriever traces (inputs only: arrival
times, chunk counts, token ids; no method arithmetic).  The paper's traces are external
(P:L482); the marginals below follow Table 2, Fig. 6 (inter-chunk arrival,
P:L300) and Fig. 7 (chunks per query):

  crawler (append mode): total tokens ~ LogNormal(ln 5800, 0.976) (median 5.8K, P95 ~28.9K),
      U{6..10} chunks of near-equal size, inter-chunk gaps ~ LogNormal(ln 0.7007 s, 1.4)
      (median 700.7 ms, tens of ms to > 30 s);
  ANNS (update mode): total ~ LogNormal(ln 10000, 0.688) (median 10K, P95 ~31K), 1 + a
      geometric number of refinements (p = 0.45, capped at 8 chunks; most queries 1-3),
      gaps ~ LogNormal(ln 0.0367 s, 1.2) (median 36.7 ms); every chunk after the first is the
      whole refined input with its LCP uniform in [ceil(0.2 T), floor(0.8 T)] (reading Z14).
Query arrivals are Poisson at `qps`.  `delay_scale` stretches the gaps (Table 3 runs at 10x /
30x delays to induce memory pressure).  Totals are truncated to [lo, hi].

Each trace is a time-sorted list of chunk events (t, rid, n_chunks, tokens, new_input, mode).
"""
from __future__ import annotations

import math

import numpy as np

from . import workloads as W


def _ln(rng, median, sigma):
    return math.exp(math.log(median) + sigma * rng.standard_normal())


def crawler_trace(seed: int, n_queries: int, qps: float, lo: int = 256, hi: int = 32768,
                  delay_scale: float = 1.0):
    rng = np.random.default_rng(seed)
    t, ev = 0.0, []
    for rid in range(n_queries):
        t += rng.exponential(1.0 / qps)
        T = int(min(hi, max(lo, round(_ln(rng, 5800, 0.976)))))
        n = int(rng.integers(6, 11))
        toks = W.request_tokens(seed, rid, T)
        bounds = [T * i // n for i in range(n + 1)]
        tc = t
        for i in range(n):
            tc += delay_scale * _ln(rng, 0.7007, 1.4)
            ev.append((tc, rid, n, toks[bounds[i]:bounds[i + 1]], None, "append"))
    ev.sort(key=lambda e: (e[0], e[1]))
    return ev


def anns_trace(seed: int, n_queries: int, qps: float, lo: int = 512, hi: int = 32768,
               delay_scale: float = 1.0):
    rng = np.random.default_rng(seed)
    t, ev = 0.0, []
    for rid in range(n_queries):
        t += rng.exponential(1.0 / qps)
        T = int(min(hi, max(lo, round(_ln(rng, 10000, 0.688)))))
        n = int(min(8, 1 + rng.geometric(0.45) - 1))
        cur = W.request_tokens(seed, rid, T)
        tc = t + delay_scale * _ln(rng, 0.0367, 1.2)
        ev.append((tc, rid, n, None, cur, "update"))
        for i in range(1, n):
            p = int(rng.integers(-(-2 * T // 10), (8 * T) // 10 + 1))
            cur = W.updated_tokens(seed, rid, cur, p, T, i)
            tc += delay_scale * _ln(rng, 0.0367, 1.2)
            ev.append((tc, rid, n, None, cur, "update"))
    ev.sort(key=lambda e: (e[0], e[1]))
    return ev
