"""STREAM2LLM hot-path ORACLE — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously-correct CPU implementation of what the streaming-prefill hot
path computes, written from the paper (arXiv 2604.16395, /root/reference/PAPER.md,
cited as P:Lnnn).  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may import it.  It shares no code with the CUDA
path (`paper_2604_16395_b200/`) and never imports it; the only shared module is the
seeded input generator `synth/`, which holds none of the method's arithmetic.

Modules
  lcp        — longest common prefix           pinned
  geometry   — M_KV, M_block, ceil(l/k)          pinned
  kvcache    — request/block state machine: allocate+append, LCP
               invalidation, swap-out/in, recompute preemption
                                   pinned
  attention  — causal GQA softmax attention over the contiguous
               per-request K/V, fp64             pinned
  fp8        — E4M3 codec of the optional FP8 KV cache (b = 1 instead
               of the paper's 2), from the format's
               definition                                               pinned

Every function states the passage it follows.  Parity pins live in tests/ (-m "not gpu").
"""
