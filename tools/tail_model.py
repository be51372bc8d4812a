"""Launch-tail model of the attention grid (host-side estimate, no GPU).

Units are dispatched in the kernel's longest-first order to the first free SM (the hardware's
in-order block dispatch = list scheduling); a unit costs FIX + STEP x (its KV tiles) cycles
(FIX ~12K cycles per CTA and STEP ~2820 per KV step from the CTA-phase trace, profiles/r02s2),
a split piece FIX + MERGE + STEP x tiles / s.  Prints makespan / ideal for the library's split
rule (s2l_host.cpp: split the last partial wave's units when it is at most half full) and for
the best rule found by exhaustive search over (tail units, split factor), on the C2 chunks and
on the C3 update round in token-budget steps of <= 8192 tokens.

    python tools/tail_model.py
"""
import heapq
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from synth import workloads as W  # noqa: E402

P, FIX, STEP, MERGE = 148, 12000, 2820, 7000


def units_of(items, G=4, hkv=8):
    """Per-unit KV-tile counts of one attention call: items [(q_pos, n_q)], pairs of 128-row tiles."""
    us, toks = [], 128 // G
    for q_pos, nq in items:
        pairs = -(-(-(-nq * G // 128)) // 2)
        for pr in range(pairs):
            tok_last = min((pr * 2 + 2) * toks, nq) - 1
            us += [(q_pos + tok_last) // 128 + 1] * hkv
    return sorted(us, reverse=True)


def makespan(us, first_split, s):
    cost = [FIX + STEP * t for t in us[:first_split]]
    for t in us[first_split:]:
        ss = min(s, t)
        cost += [FIX + MERGE + STEP * (t / ss)] * ss
    h = [0.0] * P
    for c in cost:
        heapq.heappush(h, heapq.heappop(h) + c)
    return max(h), sum(FIX + STEP * t for t in us) / P


def library_rule(us):
    U = len(us)
    rem = U % P
    if rem and rem * 2 <= P:
        s = min(P // rem, 8, min(us[U - rem:]))
        if s > 1:
            return makespan(us, U - rem, s)
    return makespan(us, U, 1)


def best_rule(us):
    best = makespan(us, len(us), 1)
    for k in range(4, min(len(us), 3 * P) + 1, 4):
        for s in (2, 3, 4, 6, 8):
            m = makespan(us, len(us) - k, s)
            if m[0] < best[0]:
                best = m
    return best


def main():
    for j in (0, 4, 8, 16, 31):
        us = units_of([(512 * j, 512)] * 8)
        a, b = library_rule(us), best_rule(us)
        print(f"C2 chunk {j:2d}: {len(us)} units, makespan / ideal: library rule {a[0] / a[1]:.4f}, best {b[0] / b[1]:.4f}")
    R, T = 32, 8192
    ps = W.c3_lcp_draws(W.seed_of(3), R, T)
    n = [T - int(p) for p in ps]
    steps, cur, fill = [], [], 0
    for r in range(R):
        done = 0
        while done < n[r]:
            take = min(n[r] - done, 8192 - fill)
            cur.append((int(ps[r]) + done, take))
            done += take
            fill += take
            if fill == 8192:
                steps.append(cur)
                cur, fill = [], 0
    if cur:
        steps.append(cur)
    a = b = ideal = 0.0
    for s in steps:
        us = units_of(s)
        x, y = library_rule(us), best_rule(us)
        a, b, ideal = a + x[0], b + y[0], ideal + x[1]
    print(f"C3 budget steps ({len(steps)}): makespan / ideal: library rule {a / ideal:.4f}, best {b / ideal:.4f}")


if __name__ == "__main__":
    main()
