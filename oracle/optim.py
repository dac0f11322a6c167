"""Gradient averaging and the global weight update.

Step 4 (:94): aggregate the workers' gradients and average them.
Step 5 (:95): update optimizer state and global weights.
Eqs. 1-2 (:101-102), SGD with momentum, paper form (reading Q9: lambda
inside the momentum buffer):
    H_k = m * H_{k-1} - lambda * dW
    W_k = W_{k-1} + H_k
The loss scale alpha is removed after averaging (reading Q6):
    dW = (sum_r g_r) / (N * alpha)
Adam (reading Q15; :98 "allows using any optimizers") per Kingma & Ba with
bias correction; no paper pin beyond its closed forms.

Two flavours:
  * float64 reference (``average``, ``sgdm``, ``adam``) with r32 applied to
    stored state (update precision fp32, :144);
  * ``fused_avg_update_f32``: the exact float32 operation sequence the fused
    average+update kernel is specified to perform (R14/R15 in DESIGN.md) --
    rank-ordered fp32 sum, one multiply by fp32(1/(N*alpha)), separately
    rounded multiplies / adds, RNE recast to fp16.  NumPy float32 ufuncs are
    IEEE single precision with round-to-nearest-even, so this is the
    bit-exact expected value for that kernel on the same inputs.
"""
from __future__ import annotations

import numpy as np

from .binary16 import r32

F32 = np.float32


def average(grads, N: int, alpha: float) -> np.ndarray:
    """float64: (sum_r g_r) / (N * alpha)."""
    s = np.zeros_like(np.asarray(grads[0], np.float64))
    for g in grads:
        s = s + np.asarray(g, np.float64)
    return s / (N * alpha)


def quorum(fraction: float, N: int) -> int:
    """Partial collection ("collecting a fraction of gradients (normally at
    90-95%) before proceeding to averaging"): proceed once ceil(f*N)
    contributions have arrived."""
    assert 0.0 < fraction <= 1.0
    return max(1, min(N, int(np.ceil(fraction * N - 1e-9))))


def partial_average(grads, contributors, alpha: float) -> np.ndarray:
    """float64: the average over the contributors that arrived ("returns
    their sum and the count so the caller averages by the actual contributor count;
    late arrivals are discarded for this step"): sum_{r in S} g_r / (|S| * alpha)."""
    S = sorted(contributors)
    return average([grads[r] for r in S], len(S), alpha)


def sgdm(W, H, dW, lam: float, m: float):
    """Eqs. 1-2 with fp32 state (r32)."""
    H = r32(m * H - lam * dW)
    W = r32(W + H)
    return W, H


def adam(W, m1, v, dW, lam: float, k: int, b1=0.9, b2=0.999, eps=1e-8):
    """Kingma & Ba with bias correction, step index k >= 1, fp32 state."""
    m1 = r32(b1 * m1 + (1 - b1) * dW)
    v = r32(b2 * v + (1 - b2) * dW * dW)
    mhat = m1 / (1 - b1 ** k)
    vhat = v / (1 - b2 ** k)
    W = r32(W - lam * mhat / (np.sqrt(vhat) + eps))
    return W, m1, v


def scalars_f32(N: int, alpha: float, lam: float, m: float):
    """Host-side scalar preparation: each computed in float64, rounded once."""
    return F32(1.0 / (N * alpha)), F32(lam), F32(m)


def l2_term_f32(g, W, l2x2, mixed: bool):
    """g + fp32(2*l2) * w_work, each op rounded to fp32; w_work is the working
    weight the step's fprop used: fp16(W) in mixed mode (R1), W in FP32 mode."""
    if not l2x2:
        return g
    Wf = np.asarray(W, F32)
    wk = Wf.astype(np.float16).astype(F32) if mixed else Wf
    return (g + (F32(l2x2) * wk).astype(F32)).astype(F32)


def fused_avg_update_f32(grads, W, H, inv_scale, lam, m, l2x2=0.0, mixed=True):
    """float32 emulation of the fused average + SGD-m update.

    grads: list (rank order) of fp16 or fp32 arrays; W, H: float32 arrays.
    l2x2 = fp32(2*l2) adds the L2 gradient (``l2_term_f32``) after the descale.
    Returns (W', H', w16', nonfinite_count).
    """
    s = np.asarray(grads[0]).astype(F32)
    for g in grads[1:]:
        s = (s + np.asarray(g).astype(F32)).astype(F32)
    g = (s * F32(inv_scale)).astype(F32)
    g = l2_term_f32(g, W, l2x2, mixed)
    t1 = (F32(m) * np.asarray(H, F32)).astype(F32)
    t2 = (F32(lam) * g).astype(F32)
    Hn = (t1 - t2).astype(F32)
    Wn = (np.asarray(W, F32) + Hn).astype(F32)
    nonfinite = int(sum(np.count_nonzero(~np.isfinite(np.asarray(gr))) for gr in grads))
    return Wn, Hn, Wn.astype(np.float16), nonfinite


def adam_consts_f32(lam, k, b1=0.9, b2=0.999, eps=1e-8):
    return dict(lam=F32(lam), b1=F32(b1), omb1=F32(1.0 - b1), b2=F32(b2), omb2=F32(1.0 - b2),
                c1=F32(1.0 / (1.0 - b1 ** k)), c2=F32(1.0 / (1.0 - b2 ** k)), eps=F32(eps))


def fused_avg_adam_f32(grads, W, m1, v, inv_scale, c, l2x2=0.0, mixed=True):
    """float32 emulation of the fused average + Adam update (same op order
    as the kernel: every product and sum separately rounded)."""
    s = np.asarray(grads[0]).astype(F32)
    for gr in grads[1:]:
        s = (s + np.asarray(gr).astype(F32)).astype(F32)
    g = (s * F32(inv_scale)).astype(F32)
    g = l2_term_f32(g, W, l2x2, mixed)
    m1n = ((c["b1"] * np.asarray(m1, F32)).astype(F32) + (c["omb1"] * g).astype(F32)).astype(F32)
    gg = (g * g).astype(F32)
    vn = ((c["b2"] * np.asarray(v, F32)).astype(F32) + (c["omb2"] * gg).astype(F32)).astype(F32)
    mhat = (m1n * c["c1"]).astype(F32)
    vhat = (vn * c["c2"]).astype(F32)
    den = (np.sqrt(vhat).astype(F32) + c["eps"]).astype(F32)
    upd = (mhat / den).astype(F32)
    stp = (c["lam"] * upd).astype(F32)
    Wn = (np.asarray(W, F32) - stp).astype(F32)
    nonfinite = int(sum(np.count_nonzero(~np.isfinite(np.asarray(gr))) for gr in grads))
    return Wn, m1n, vn, Wn.astype(np.float16), nonfinite


def dynamic_loss_scale(alpha: float, good: int, nonfinite: int, interval: int, factor: float = 2.0,
                       min_alpha: float = 1.0):
    """Dynamic loss scaling (NEXT-3; PAPER.md:134 names fp16 overflow as the hazard
    the static alpha of :177 leaves open; reading Q14b in DESIGN.md).

    A step whose gradients contain a non-finite fp16 value is skipped (weights and
    optimizer state unchanged) and alpha is divided by ``factor`` (not below
    ``min_alpha``); after ``interval`` consecutive finite steps alpha is multiplied
    by ``factor``.  Returns (alpha', good', skipped)."""
    if nonfinite:
        return max(alpha / factor, min_alpha), 0, True
    good += 1
    if good >= interval:
        return alpha * factor, 0, False
    return alpha, good, False

