"""bfloat16 codec written out from the format definition (NEXT-3 bf16 math mode).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

bfloat16 = the upper 16 bits of an IEEE 754 binary32: sign(1) exponent(8)
mantissa(7); the same exponent range as binary32 (max finite
(2 - 2^-7) * 2^127), 8 significant bits.  Rounding from binary32 is
round-to-nearest-even on the discarded low 16 bits; overflow rounds to infinity,
NaN stays NaN.  PAPER.md:134 discusses the fp16 range hazard; bf16 trades
precision for binary32's range (reading Q29 in DESIGN.md: the bf16 mode applies
the same rounding points R0-R15 with bf16 in place of fp16).

``rbf16`` rounds float64 -> binary32 (RNE) -> bfloat16 (RNE) and returns
float64, matching the GPU's fp32-accumulate-then-__float2bfloat16_rn path.
"""
from __future__ import annotations

import numpy as np

MAX_FINITE = float(np.float32(np.uint32(0x7F7F0000).view(np.float32)))


def decode(bits) -> np.ndarray:
    """Exact float32 value of 16-bit bfloat16 patterns (array of uint16)."""
    b = np.asarray(bits, dtype=np.uint32) & 0xFFFF
    return (b << 16).astype(np.uint32).view(np.float32)


def encode_f32(x) -> np.ndarray:
    """RNE encoding of float32 values into bfloat16 bit patterns (uint16)."""
    u = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    nan = np.isnan(np.asarray(x, dtype=np.float32))
    lsb = (u >> 16) & 1
    r = ((u + 0x7FFF + lsb) >> 16) & 0xFFFF          # ties to the even upper half
    r = np.where(nan, (u >> 16) | 0x0040, r)          # quiet NaN, sign kept
    return r.astype(np.uint16)


def rbf16(x) -> np.ndarray:
    """Round to bfloat16 via binary32 (RNE at each step), return float64."""
    f = np.asarray(x, dtype=np.float64).astype(np.float32)
    return decode(encode_f32(f)).astype(np.float64)
