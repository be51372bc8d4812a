"""FP8 E4M3 storage format of the optional FP8 KV cache -- TEST INFRASTRUCTURE
ONLY (see oracle/__init__.py).  The paper stores KV in 2-byte FP16 ("b: bytes per value,
typically 2 bytes for FP16", §2.1); an FP8 cache halves b.  This module writes the
format out from its definition (OCP 8-bit floating point, E4M3 "FN" variant):

    bit 7 sign, bits 6-3 exponent e (bias 7), bits 2-0 mantissa m;
    e = 0:       value = (-1)^s * 2^-6 * m/8             (subnormals, smallest 2^-9)
    1 <= e <= 15: value = (-1)^s * 2^(e-7) * (1 + m/8)    except e = 15, m = 7: NaN
    (no infinities; largest finite 0x7E = 448).

Encoding (what the library's K/V store does, reading Z20 in DESIGN.md): round to nearest
representable value, ties to the code with an even mantissa (round-to-nearest-even), values
beyond +-448 saturate to +-448 (the `satfinite` conversion); the codec is a table over all 256
codes, searched by value (nearest neighbour) -- no bit tricks.
"""
from __future__ import annotations

import numpy as np


def decode_table() -> np.ndarray:
    """float64 value of every code 0..255 (NaN for 0x7F / 0xFF)."""
    out = np.empty(256, dtype=np.float64)
    for c in range(256):
        s, e, m = (c >> 7) & 1, (c >> 3) & 15, c & 7
        if e == 15 and m == 7:
            v = np.nan
        elif e == 0:
            v = 2.0 ** -6 * (m / 8.0)
        else:
            v = 2.0 ** (e - 7) * (1.0 + m / 8.0)
        out[c] = -v if s else v
    return out


_TABLE = decode_table()
_FINITE = np.array([c for c in range(256) if not np.isnan(_TABLE[c])], dtype=np.int64)
MAX_FINITE = 448.0


def decode(codes: np.ndarray) -> np.ndarray:
    return _TABLE[np.asarray(codes, dtype=np.uint8).astype(np.int64)]


def encode(x: np.ndarray) -> np.ndarray:
    """Nearest finite E4M3 code (ties -> even mantissa; +-0 keep their sign; saturating).
    Nearest-neighbour search over the sorted finite values of the table."""
    x = np.asarray(x, dtype=np.float64)
    flat = np.clip(x.reshape(-1), -MAX_FINITE, MAX_FINITE)
    vals = _TABLE[_FINITE]
    order = np.argsort(vals, kind="stable")
    sv, sc = vals[order], _FINITE[order]          # ascending values (-0 and +0 adjacent)
    hi = np.clip(np.searchsorted(sv, flat, side="left"), 0, len(sv) - 1)
    lo = np.clip(hi - 1, 0, len(sv) - 1)
    dlo, dhi = np.abs(flat - sv[lo]), np.abs(sv[hi] - flat)
    code = np.where(dlo < dhi, sc[lo], sc[hi])
    tie = (dlo == dhi) & (sv[lo] != sv[hi])
    even = np.where((sc[lo] & 1) == 0, sc[lo], sc[hi])
    code = np.where(tie, even, code)
    zero = _TABLE[code] == 0.0                    # rounds to zero: keep the input's sign
    code = np.where(zero, np.where(np.signbit(flat), 0x80, 0x00), code)
    code = np.where(np.isnan(flat), 0x7F, code)
    return code.astype(np.uint8).reshape(x.shape)


def bf16_bits_to_f64(bits: np.ndarray) -> np.ndarray:
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def f64_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Exact for every E4M3 value (3-bit mantissa, exponents -9..8 fit bf16)."""
    return (np.asarray(x, dtype=np.float32).view(np.uint32) >> 16).astype(np.uint16)


def quantize_bf16_bits(bits: np.ndarray):
    """bf16 K/V rows -> (E4M3 codes, the dequantized values as bf16 bits)."""
    codes = encode(bf16_bits_to_f64(bits))
    return codes, f64_to_bf16_bits(decode(codes))
