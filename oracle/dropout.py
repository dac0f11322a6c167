"""Variational recurrent dropout masks (NEXT-3; "recurrent dropout").

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Reading Q16b: one Bernoulli(keep) mask per (training step, layer,
sequence, unit), fixed over the time steps of the sequence (variational form),
applied to the recurrent input only: the recurrent GEMM of layer l at step t
reads h~_{t-1} = fp16(fp32(h_{t-1}) * scale) on kept units and 0 elsewhere,
scale = fp32(1 / keep); the next layer and the head see the unmasked h.

The mask is a counter-based hash that the CUDA path implements independently
from the same definition (all arithmetic mod 2^32):
    mix32(x)  = x ^= x >> 16; x *= 0x7FEB352D; x ^= x >> 15; x *= 0x846CA68B; x ^= x >> 16
    k1 = mix32(seed ^ mix32(step))
    k2 = mix32(k1 ^ (layer * 0x9E3779B9))
    k3 = mix32(k2 ^ (seq * 0x85EBCA6B))
    r  = mix32(k3 ^ (unit * 0xC2B2AE35))
    kept  iff  r < thr,  thr = floor(keep * 2^32)   (keep < 1)
`seq` is the sequence's index in the global batch (worker r's sequence b has
index r * B_r + b under the contiguous split), `step` the number of completed
updates before this step.
"""
from __future__ import annotations

import numpy as np

M32 = np.uint64(0xFFFFFFFF)


def _u(x):
    return np.asarray(x, dtype=np.uint64) & M32


def mix32(x):
    x = _u(x)
    x = x ^ (x >> np.uint64(16))
    x = (x * np.uint64(0x7FEB352D)) & M32
    x = x ^ (x >> np.uint64(15))
    x = (x * np.uint64(0x846CA68B)) & M32
    x = x ^ (x >> np.uint64(16))
    return x


def threshold(keep: float) -> int:
    if not (0.0 < keep < 1.0):
        raise ValueError("keep must be in (0, 1) for a mask")
    return int(np.floor(keep * 2.0 ** 32))


def scale(keep: float) -> float:
    """fp32(1 / keep), the factor kept units are multiplied by."""
    return float(np.float32(1.0 / keep))


def mask(seed: int, step: int, layer: int, seqs, hidden: int, keep: float) -> np.ndarray:
    """{0, 1} float64 mask [len(seqs)][hidden] (one row per sequence, fixed over t)."""
    k1 = mix32(_u(seed) ^ mix32(step))
    k2 = mix32(k1 ^ ((_u(layer) * np.uint64(0x9E3779B9)) & M32))
    seqs = _u(np.asarray(seqs))[:, None]
    k3 = mix32(k2 ^ ((seqs * np.uint64(0x85EBCA6B)) & M32))
    units = _u(np.arange(hidden))[None, :]
    r = mix32(k3 ^ ((units * np.uint64(0xC2B2AE35)) & M32))
    return (r < np.uint64(threshold(keep))).astype(np.float64)
