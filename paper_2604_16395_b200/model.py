"""NEXT-4: the library's per-layer streaming API inside a decoder forward pass.

A Llama-3-style decoder stack (RMSNorm, fused QKV projection, rotary embedding, grouped-query
attention, output projection, SwiGLU MLP) prefilled chunk by chunk as context streams in
("chunked prefill ... the KV cache of earlier chunks is reused").  Per chunk:

  * s2l_append_chunk in reserve mode (k = v = NULL) allocates the chunk's blocks once;
  * per layer, the projections produce Q/K/V of the chunk's rows and ONE s2l_prefill_append
    launch writes that layer's K/V into the paged pool and computes the chunked-prefill
    attention over the cached prefix + the chunk (the hot path, libs2l);
  * the dense layers around it are plain library GEMMs (torch / cuBLAS) and elementwise ops.

Weights are random (seeded): the paper's experiments need trained models and datasets, which are
out of scope; this module exists to exercise and time the per-layer API
inside a real forward pass.  There is no CPU path: the attention is only ever computed by libs2l.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch

from . import s2l


@dataclass(frozen=True)
class Shape:
    layers: int
    hidden: int
    h_q: int
    h_kv: int
    d: int
    inter: int
    rope_theta: float = 500000.0
    eps: float = 1e-5


LLAMA3_8B = Shape(layers=32, hidden=4096, h_q=32, h_kv=8, d=128, inter=14336)


def _rms_norm(x: torch.Tensor, w: torch.Tensor, eps: float) -> torch.Tensor:
    xf = x.float()
    return (xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + eps) * w.float()).to(x.dtype)


def _rope(x: torch.Tensor, pos: torch.Tensor, theta: float) -> torch.Tensor:
    """Rotary embedding (half-split layout) of x [rows][heads][d] at absolute positions pos [rows]."""
    d = x.shape[-1]
    inv = theta ** (-torch.arange(0, d, 2, device=x.device, dtype=torch.float32) / d)
    ang = pos.to(torch.float32)[:, None] * inv[None, :]
    cos, sin = ang.cos()[:, None, :], ang.sin()[:, None, :]
    x1, x2 = x[..., : d // 2].float(), x[..., d // 2:].float()
    return torch.cat([x1 * cos - x2 * sin, x1 * sin + x2 * cos], dim=-1).to(x.dtype)


class StreamingDecoder:
    """Random-weight decoder whose attention runs through one libs2l context.

    ctx must be created for (shape.layers, h_q, h_kv, d, block size).  Each layer's K/V exist
    only after that layer's projection, so the per-layer call is the only way to store them:
    s2l_prefill_append is one launch when every q_pos is block-aligned, else a one-layer append
    launch followed by the attention launch."""

    def __init__(self, shape: Shape, ctx: "s2l.Context", vocab: int = 32768, seed: int = 0,
                 device: str = "cuda", scale: float = 0.02):
        self.s, self.ctx = shape, ctx
        g = torch.Generator(device=device).manual_seed(seed)
        bf = torch.bfloat16

        def w(*dims, std=scale):
            return (torch.randn(*dims, generator=g, device=device) * std).to(bf)

        qkv = (shape.h_q + 2 * shape.h_kv) * shape.d
        self.emb = w(vocab, shape.hidden, std=1.0)
        self.wqkv = [w(shape.hidden, qkv) for _ in range(shape.layers)]
        self.wo = [w(shape.h_q * shape.d, shape.hidden) for _ in range(shape.layers)]
        self.wgu = [w(shape.hidden, 2 * shape.inter) for _ in range(shape.layers)]
        self.wd = [w(shape.inter, shape.hidden) for _ in range(shape.layers)]
        self.n1 = [torch.ones(shape.hidden, device=device, dtype=bf) for _ in range(shape.layers)]
        self.n2 = [torch.ones(shape.hidden, device=device, dtype=bf) for _ in range(shape.layers)]

    def chunk(self, items, tokens: torch.Tensor, trace: list | None = None) -> torch.Tensor:
        """Prefills one chunk per item.  items: [(rid, q_pos, n, row)] (rows packed in item
        order, q_pos = the request's cached length); tokens: int64 [rows] on the device.
        Returns the last layer's hidden states [rows][hidden].  trace (optional) receives
        (layer, q, k, v, o) of every layer for checking."""
        s, ctx = self.s, self.ctx
        rows = int(tokens.shape[0])
        ctx.append_chunk([(r, None, n, row) for r, _, n, row in items], None, None, kv_rows=rows)
        pos = torch.cat([torch.arange(p, p + n, device=tokens.device) for _, p, n, _ in items])
        x = self.emb[tokens]
        o = torch.empty(rows, s.h_q, s.d, device=x.device, dtype=x.dtype)
        nq, nk = s.h_q * s.d, s.h_kv * s.d
        for layer in range(s.layers):
            h = _rms_norm(x, self.n1[layer], s.eps)
            qkv = h @ self.wqkv[layer]
            q = _rope(qkv[:, :nq].view(rows, s.h_q, s.d), pos, s.rope_theta)
            k = _rope(qkv[:, nq:nq + nk].view(rows, s.h_kv, s.d), pos, s.rope_theta)
            v = qkv[:, nq + nk:].contiguous().view(rows, s.h_kv, s.d)   # dense rows for the ABI
            ctx.prefill_append(layer, list(items), q, k, v, o)
            if trace is not None:
                trace.append((layer, q, k, v, o.clone()))
            x = x + o.view(rows, nq) @ self.wo[layer]
            h = _rms_norm(x, self.n2[layer], s.eps)
            gu = h @ self.wgu[layer]
            x = x + (torch.nn.functional.silu(gu[:, :s.inter]) * gu[:, s.inter:]) @ self.wd[layer]
        return x

    def flops_per_chunk(self, items) -> float:
        """Dense-layer GEMM FLOPs + causal attention FLOPs of one chunk() call."""
        s = self.s
        rows = sum(n for _, _, n, _ in items)
        per_tok = 2 * (s.hidden * (s.h_q + 2 * s.h_kv) * s.d + s.h_q * s.d * s.hidden
                       + s.hidden * 2 * s.inter + s.inter * s.hidden)
        attn = sum(4.0 * s.d * s.h_q * (n * p + n * (n + 1) / 2) for _, p, n, _ in items)
        return s.layers * (per_tok * rows + attn)
