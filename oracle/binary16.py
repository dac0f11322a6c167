"""IEEE 754 binary16 codec written out from the format definition.

PAPER.md:134: "Half-precision floating point format (10-bit mantissa and
5-bit exponent) has a numerical range of (0.00006,65504)".  SPEC.md:51-68:
round-to-nearest-even, overflow to signed infinity, subnormals supported.

``decode`` / ``encode`` are the bit-level definition (pinned exhaustively
against numpy.float16 in tests).  ``r16`` / ``r32`` are the rounding helpers
the oracle uses at the pinned rounding points.  ``r16`` rounds through
float32 (x -> fp32 -> fp16), matching the GPU's fp32-accumulate-then-RNE
path; rounding fp64 straight to fp16 can differ by double rounding.
"""
from __future__ import annotations

import math

import numpy as np

MAX_FINITE = 65504.0
MIN_NORMAL = 2.0 ** -14
MIN_SUBNORMAL = 2.0 ** -24


def decode(bits: int) -> float:
    """Exact real value of a 16-bit pattern: sign(1) exponent(5) mantissa(10)."""
    bits &= 0xFFFF
    sign = -1.0 if bits & 0x8000 else 1.0
    e = (bits >> 10) & 0x1F
    m = bits & 0x3FF
    if e == 0x1F:
        return sign * math.inf if m == 0 else math.nan
    if e == 0:                                  # zero / subnormal: m * 2^-24
        return sign * m * MIN_SUBNORMAL
    return sign * (1.0 + m / 1024.0) * 2.0 ** (e - 15)


def encode(x: float) -> int:
    """Round-to-nearest-even encoding of a real number (overflow -> inf)."""
    if math.isnan(x):
        return 0x7E00
    sign = 0x8000 if math.copysign(1.0, x) < 0 else 0
    a = abs(x)
    if math.isinf(a):
        return sign | 0x7C00
    # quantum (ulp) of the binade [2^e, 2^(e+1)) containing a: 2^(e-10);
    # the subnormal range shares the quantum of the lowest binade, 2^-24
    if a < MIN_NORMAL:
        q = MIN_SUBNORMAL
    else:
        _, E = math.frexp(a)                    # a = f * 2^E, f in [0.5, 1)
        q = 2.0 ** (E - 1 - 10)
    n = a / q                                   # exact (power-of-two divisor)
    k = math.floor(n)
    frac = n - k
    if frac > 0.5 or (frac == 0.5 and (k & 1)):
        k += 1
    v = k * q
    if v > MAX_FINITE:
        return sign | 0x7C00
    if v < MIN_NORMAL:                          # subnormal or zero: v = m * 2^-24
        return sign | int(round(v / MIN_SUBNORMAL))
    e = int(math.floor(math.log2(v)))
    m = int(round((v / 2.0 ** e - 1.0) * 1024))
    if m == 1024:
        e, m = e + 1, 0
    return sign | ((e + 15) << 10) | m


def r32(x):
    """Round to binary32 (RNE) and return as float64."""
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float64)


def r16(x):
    """Round to binary16 via binary32 (RNE at each step), return float64."""
    return np.asarray(x, dtype=np.float64).astype(np.float32).astype(np.float16).astype(np.float64)


def count_nonfinite(x) -> int:
    return int(np.count_nonzero(~np.isfinite(np.asarray(x))))
