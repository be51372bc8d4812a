"""Recompute-vs-swap preemption cost model on B200 (host side).

The paper (§2.2, §4.3):
  * recomputation discards a victim's KV blocks and later re-prefills its ℓ tokens:
    C_recomp(ℓ) = recomputation_latency(ℓ)   (measured over 1K-128K tokens and
    fitted piecewise-linear "to account for memory bandwidth saturation");
  * swapping moves ⌈ℓ/k⌉ blocks out and later back in:
    C_swap(ℓ) = swap_latency(⌈ℓ/k⌉)           (⌈ℓ/k⌉·M_block / BW_PCIe, symmetric);
  * "Selecting between the two strategies requires comparing C_recomp(r) versus 2·C_swap(r)"
    (P:L79); the cheaper one is chosen, ties -> recompute.
The B200 profiles are measured with this library (tools/profile_costmodel.py): the recompute
curve is append + chunked-prefill attention of the KV-cache geometry (attention only — the
paper's C_prefill also contains the model GEMMs, which are out of scope here), times the number
of layers; the swap curve is s2l_swap_out + s2l_swap_in of C blocks.  Profiles are stored as
JSON.
"""
from __future__ import annotations

import bisect
import json
import math
from dataclasses import dataclass, field


@dataclass
class PiecewiseLinear:
    """y(x) through measured points (x sorted ascending): linear interpolation inside
    ("fit a piecewise-linear model"), the last segment's slope above the last sample,
    and below the first sample the line through the origin to it (a zero-length
    recompute or swap costs nothing; the paper profiles 1K-128K tokens only)."""
    xs: list
    ys: list

    def __post_init__(self):
        if len(self.xs) != len(self.ys) or len(self.xs) < 2:
            raise ValueError("need >= 2 points")
        pts = sorted(zip(self.xs, self.ys))
        self.xs = [float(x) for x, _ in pts]
        self.ys = [float(y) for _, y in pts]
        if len(set(self.xs)) != len(self.xs):
            raise ValueError("duplicate x")

    def __call__(self, x: float) -> float:
        xs, ys = self.xs, self.ys
        if x < xs[0] and xs[0] > 0:
            return ys[0] * max(x, 0.0) / xs[0]
        i = bisect.bisect_right(xs, x) - 1
        i = min(max(i, 0), len(xs) - 2)
        x0, x1, y0, y1 = xs[i], xs[i + 1], ys[i], ys[i + 1]
        return y0 + (y1 - y0) * (x - x0) / (x1 - x0)

    def to_json(self):
        return {"x": self.xs, "y": self.ys}

    @classmethod
    def from_json(cls, d):
        return cls(list(d["x"]), list(d["y"]))


@dataclass
class CostModel:
    block_size: int
    recompute_s: PiecewiseLinear            # tokens -> seconds
    swap_s: PiecewiseLinear                 # blocks -> seconds (one direction)
    meta: dict = field(default_factory=dict)

    def recompute_latency(self, tokens: int) -> float:
        """C_recomp(ℓ)."""
        return 0.0 if tokens <= 0 else max(0.0, self.recompute_s(tokens))

    def swap_latency(self, blocks: int) -> float:
        """C_swap for `blocks` blocks, one direction."""
        return 0.0 if blocks <= 0 else max(0.0, self.swap_s(blocks))

    def choose_eviction(self, computed_tokens: int) -> str:
        """'recompute' if C_recomp(ℓ) <= 2·C_swap(⌈ℓ/k⌉) else 'swap' (ties -> recompute)."""
        blocks = -(-computed_tokens // self.block_size)
        return "recompute" if self.recompute_latency(computed_tokens) <= 2.0 * self.swap_latency(blocks) else "swap"

    def crossover_tokens(self, lo: int | None = None, hi: int | None = None) -> int | None:
        """Smallest ℓ in [lo, hi] (default: the profiled token range) at which swapping becomes
        cheaper, by bisection on the sign of C_recomp(ℓ) - 2·C_swap(ℓ) (assumes one crossing
        in the range; None if recompute wins throughout)."""
        lo = int(self.recompute_s.xs[0]) if lo is None else lo
        hi = int(self.recompute_s.xs[-1]) if hi is None else hi
        f = lambda t: self.recompute_latency(t) - 2.0 * self.swap_latency(-(-t // self.block_size))
        if f(hi) <= 0:
            return None
        if f(lo) > 0:
            return lo
        while hi - lo > 1:
            mid = (lo + hi) // 2
            if f(mid) > 0:
                hi = mid
            else:
                lo = mid
        return hi

    def to_json(self):
        return {"block_size": self.block_size, "recompute_s": self.recompute_s.to_json(),
                "swap_s": self.swap_s.to_json(), "meta": self.meta}

    @classmethod
    def from_json(cls, d):
        return cls(d["block_size"], PiecewiseLinear.from_json(d["recompute_s"]),
                   PiecewiseLinear.from_json(d["swap_s"]), d.get("meta", {}))

    def save(self, path):
        with open(path, "w") as f:
            json.dump(self.to_json(), f, indent=1)

    @classmethod
    def load(cls, path):
        with open(path) as f:
            return cls.from_json(json.load(f))


def analytic(block_size: int, m_block_bytes: int, bw_bytes_per_s: float, c_prefill_s_per_token: float,
             max_tokens: int = 1 << 17) -> CostModel:
    """The paper's closed forms as a model: C_recomp = ℓ·C_prefill and
    C_swap = ⌈ℓ/k⌉·M_block / BW_PCIe, sampled at the ends (both are linear)."""
    rec = PiecewiseLinear([0, max_tokens], [0.0, max_tokens * c_prefill_s_per_token])
    nb = -(-max_tokens // block_size)
    swp = PiecewiseLinear([0, nb], [0.0, nb * m_block_bytes / bw_bytes_per_s])
    return CostModel(block_size, rec, swp, {"kind": "analytic"})
