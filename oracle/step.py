"""One synchronous data-parallel training step over N simulated workers
(PAPER.md:89-97 steps 3-6), run sequentially in one process.

  step 3: every worker r runs fprop + bprop on its mini-batch m_r
  step 4: gradients aggregated and averaged (÷N, ÷alpha -- reading Q6)
  step 5: optimizer update of the global weights (Eqs. 1-2 or Adam)
  step 6: the updated weights are what every worker uses next step
          (mixed mode: the fp16 copy of the fp32 master, R1)

The global batch is split contiguously: worker r gets rows
[r*B/N, (r+1)*B/N).  The learning rate is passed in (``schedule``
computes it); the oracle does not decide N-dependence itself.

Partial collection: ``contributors`` lists the
workers whose gradients arrived in time; the step averages exactly those
(``optim.partial_average``) and discards the rest.

L2 regularisation ("application of L2 regularization"; SPEC.md:171
"loss = alpha*mean hinge + alpha*l2*||W||^2"; reading Q16 in DESIGN.md): the
penalty l2 * sum(w^2) runs over every parameter w of the working weights used
by this step's fprop (R1), is part of the reported loss, and its gradient
2*l2*w is added to the averaged data gradient (the alpha it would carry inside
the scaled loss cancels in the descale, so it is added after step 4).
"""
from __future__ import annotations

from typing import Dict, Optional

import numpy as np

from . import dropout as dropout_mod
from . import lstm, optim
from .bfloat16 import rbf16
from .binary16 import count_nonfinite, r16


def working_weights(master: np.ndarray, mode: str) -> np.ndarray:
    """R1: the weights used by fprop/bprop (fp16 copy of the master in mixed mode)."""
    if mode == "bf16":
        return rbf16(master)
    return r16(master) if mode == "mixed" else np.asarray(master, np.float64)


def worker_grads(cfg, wflat, x, targets, alpha, mode, abs_terms=None, drop=None, relu_active=None):
    """Steps 3 for one worker: returns (L_r scaled, flat gradient, y)."""
    P = lstm.unpack(cfg, wflat)
    L, y, cache = lstm.forward(cfg, P, x, targets, alpha, mode, drop, relu_active)
    G = lstm.backward(cfg, P, cache, alpha, mode, abs_terms)
    return L, lstm.pack(cfg, G), y


def train_step(cfg, master, state: Dict[str, np.ndarray], x_global, t_global, N: int,
               alpha: float, lam: float, mode: str, optimizer: str = "sgdm",
               momentum: float = 0.9, adam_k: int = 1,
               grads_override: Optional[list] = None, l2: float = 0.0, skip_nonfinite: bool = False,
               dropout: Optional[dict] = None, contributors: Optional[list] = None):
    """Returns a dict with loss (unscaled mean over workers), per-worker
    gradients (carrying alpha), the averaged gradient, new master/state,
    the fp16 working copy and the non-finite count."""
    B = x_global.shape[0]
    assert B % N == 0
    b = B // N
    w = working_weights(master, mode)
    losses, grads, abs_terms = [], [], []
    for r in range(N):
        sl = slice(r * b, (r + 1) * b)
        at = {}
        drop = None
        if dropout is not None and dropout["keep"] < 1.0:
            # recurrent dropout (oracle/dropout.py): masks keyed by the global sequence index
            seqs = np.arange(r * b, (r + 1) * b)
            drop = {"scale": dropout_mod.scale(dropout["keep"]),
                    "masks": [dropout_mod.mask(dropout["seed"], dropout["step"], l, seqs, cfg.hidden, dropout["keep"])
                              for l in range(cfg.n_layers)]}
        L, g, _ = worker_grads(cfg, w, x_global[sl], t_global[sl], alpha, mode, at, drop)
        losses.append(L)
        grads.append(g)
        abs_terms.append(at)
    if grads_override is not None:
        grads = grads_override
    if contributors is None:
        nonfinite = sum(count_nonfinite(g) for g in grads)
        avg = optim.average(grads, N, alpha)
    else:  # partial collection: only the contributors that arrived are averaged
        nonfinite = sum(count_nonfinite(grads[r]) for r in contributors)
        avg = optim.partial_average(grads, contributors, alpha)
    if l2:
        avg = avg + 2.0 * l2 * w
    if skip_nonfinite and nonfinite:
        # dynamic loss scaling (optim.dynamic_loss_scale): the step is skipped
        W, new_state = np.asarray(master, np.float64), dict(state)
    elif optimizer == "sgdm":
        W, H = optim.sgdm(master, state["H"], avg, lam, momentum)
        new_state = {"H": H}
    else:
        W, m1, v = optim.adam(master, state["m1"], state["v"], avg, lam, adam_k)
        new_state = {"m1": m1, "v": v}
    return {
        "loss": float(np.sum(losses) / (N * alpha)) + (float(l2 * np.dot(w, w)) if l2 else 0.0),
        "losses_scaled": losses,
        "grads": grads,
        "abs_terms": abs_terms,
        "avg": avg,
        "master": W,
        "state": new_state,
        "w16": rbf16(W) if mode == "bf16" else r16(W),
        "nonfinite": nonfinite,
    }
