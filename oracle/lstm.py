"""One worker's forward pass, scaled hinge loss and BPTT (PAPER.md:60-82,
:177-180), in float64 with optional fp16/fp32 rounding at the pinned points.

Model (Fig. 2 :64-80 and the readings in DESIGN.md):
  [embedding (C3)] -> L stacked LSTM layers -> head
  head = per-step FC(ReLU) -> Linear(1)   (C2, Fig. 2, reading Q4)
       | per-step Linear(1)               (C1, C4, reading Q24)
       | last-step Linear(1)              (C3, reading Q23)

LSTM cell ("gates ... implemented using the logistic
function"; standard equations, no peepholes, one bias per gate, gate order
i, f, g, o -- reading Q1):
  a   = W x_t + U h_{t-1} + b
  i = sigma(a_i)  f = sigma(a_f)  g = tanh(a_g)  o = sigma(a_o)
  c_t = f * c_{t-1} + i * g          (no activation on the recurrent path, :62)
  h_t = o * tanh(c_t)
with h_{-1} = c_{-1} = 0 per sequence (reading Q3).

Loss, Eq. 6 (:179): L = alpha * max(0, 1 - t*y), averaged over the worker's
terms (reading Q5); alpha multiplies the loss "before evaluating partial
derivatives on the bprop step" (:177), so every gradient carries alpha.

Modes
  "fp64"  : no rounding at all (used by the finite-difference pins)
  "fp32"  : the paper's FP32 baseline (:147); no rounding inside fwd/bwd
  "mixed" : FP16 math (:142) with rounding points:
            R4 saved gates fp16, R5 c fp32, R6 h fp16, R7 FC output fp16,
            R9 dz fp16, R10 dA fp16, R12 parameter gradients fp16 (one RNE
            of the float64 accumulation).  R0 (inputs) and R1 (weights) are
            fp16 by construction of the caller.
  "bf16"  : the same rounding points with bfloat16 in place of fp16 (NEXT-3 bf16
            math mode, reading Q29; oracle/bfloat16.py); R5 c stays fp32.
"""
from __future__ import annotations

from typing import Dict, List

import numpy as np

from .bfloat16 import rbf16
from .binary16 import r16, r32

MODES = ("fp64", "fp32", "mixed", "bf16")
LOWP = ("mixed", "bf16")     # modes with 16-bit rounding points


# ----------------------------------------------------------------------------
# canonical parameter layout (include/hdp.h, hdp_load_params):
#   [E]? then per layer W_l [4h][I_l], U_l [4h][h], b_l [4h]; then
#   [F [fc][h], fb [fc]]?, wo [fc or h], bo [1]
# ----------------------------------------------------------------------------

def layout(cfg) -> List[tuple]:
    h = cfg.hidden
    out = []
    if cfg.vocab > 0:
        out.append(("E", (cfg.vocab, cfg.embed_dim)))
    in_dims = [cfg.embed_dim if cfg.vocab > 0 else cfg.input_dim] + [h] * (cfg.n_layers - 1)
    for l in range(cfg.n_layers):
        out += [(f"W{l}", (4 * h, in_dims[l])), (f"U{l}", (4 * h, h)), (f"b{l}", (4 * h,))]
    if cfg.fc_hidden > 0:
        out += [("F", (cfg.fc_hidden, h)), ("fb", (cfg.fc_hidden,)), ("wo", (cfg.fc_hidden,))]
    else:
        out += [("wo", (h,))]
    out += [("bo", (1,))]
    return out


def count(cfg) -> int:
    return int(sum(int(np.prod(s)) for _, s in layout(cfg)))


def unpack(cfg, flat) -> Dict[str, np.ndarray]:
    flat = np.asarray(flat, dtype=np.float64)
    assert flat.size == count(cfg), (flat.size, count(cfg))
    out, off = {}, 0
    for name, shape in layout(cfg):
        n = int(np.prod(shape))
        out[name] = flat[off:off + n].reshape(shape)
        off += n
    return out


def pack(cfg, d: Dict[str, np.ndarray]) -> np.ndarray:
    return np.concatenate([np.asarray(d[name], np.float64).reshape(-1) for name, _ in layout(cfg)])


def _sigmoid(a):
    return 1.0 / (1.0 + np.exp(-a))


def _q16(mode):
    """The 16-bit rounding of the mode's rounding points (identity in fp32 / fp64)."""
    return r16 if mode == "mixed" else rbf16 if mode == "bf16" else (lambda v: v)


# ----------------------------------------------------------------------------
# forward
# ----------------------------------------------------------------------------

def forward(cfg, P: Dict[str, np.ndarray], x, targets, alpha: float, mode: str, drop=None, relu_active=None):
    """fprop + scaled loss for one worker's mini-batch.

    drop (optional, NEXT-3 recurrent dropout, oracle/dropout.py): {"masks": [per layer
    {0,1} [B][h]], "scale": fp32(1/keep)}; layer l's recurrent GEMM then reads
    h~_{t-1} = r16(h_{t-1} * scale) on kept units, 0 elsewhere (R6d).

    relu_active (optional, bool [T][B][fc]): the FC head's ReLU decision per unit, where
    the caller fixes the branch of a pre-activation that lies within rounding of 0
    (both branches are correct results there, DESIGN.md R-relu); default zpre > 0.

    x: float [B][T][I] (fp16-representable, R0) or int tokens [B][T] (C3).
    targets: {-1,+1} [B][T] (per-step heads) or [B] (last-step head).
    Returns (L, y, cache) with L = alpha * mean hinge (Eq. 6) and y the
    network output ([T][B] or [B]).
    """
    assert mode in MODES
    q = _q16(mode)
    h = cfg.hidden
    T = cfg.seq
    if cfg.vocab > 0:
        tok = np.asarray(x)
        B = tok.shape[0]
        Xin = P["E"][tok.T]                      # [T][B][E]  (rows of E, R1)
    else:
        xx = np.asarray(x, dtype=np.float64)
        B = xx.shape[0]
        Xin = np.transpose(xx, (1, 0, 2))        # time-major [T][B][I]
    layers = []
    for l in range(cfg.n_layers):
        W, U, b = P[f"W{l}"], P[f"U{l}"], P[f"b{l}"]
        h_prev = np.zeros((B, h))
        c_prev = np.zeros((B, h))
        gates = np.zeros((T, B, 4 * h))
        C = np.zeros((T, B, h))
        H = np.zeros((T, B, h))
        Hin = np.zeros((T, B, h))                # recurrent input of each step (h~_{t-1})
        for t in range(T):
            h_in = h_prev if drop is None else q(h_prev * drop["scale"]) * drop["masks"][l]
            Hin[t] = h_in
            a = Xin[t] @ W.T + h_in @ U.T + b
            i = _sigmoid(a[:, 0:h])
            f = _sigmoid(a[:, h:2 * h])
            g = np.tanh(a[:, 2 * h:3 * h])
            o = _sigmoid(a[:, 3 * h:4 * h])
            c = f * c_prev + i * g
            if mode in LOWP:
                c = r32(c)                       # R5
            hh = q(o * np.tanh(c))               # R6
            gates[t] = q(np.concatenate([i, f, g, o], axis=1))   # R4 (saved)
            C[t] = c
            H[t] = hh
            h_prev, c_prev = hh, c
        layers.append({"X": Xin, "gates": gates, "C": C, "H": H, "Hin": Hin,
                       "rmask": None if drop is None else drop["masks"][l] * drop["scale"]})
        Xin = H
    Htop = Xin
    cache = {"layers": layers, "B": B, "tokens": np.asarray(x) if cfg.vocab > 0 else None}
    if cfg.fc_hidden > 0:
        zpre = Htop @ P["F"].T + P["fb"]         # [T][B][fc]
        act = zpre > 0.0 if relu_active is None else np.asarray(relu_active, bool)
        z = q(np.where(act, zpre, 0.0))          # R7: ReLU
        y = z @ P["wo"] + P["bo"][0]             # [T][B]
        cache.update(zpre=zpre, z=z, act=act)
    elif cfg.head_last_step:
        y = Htop[T - 1] @ P["wo"] + P["bo"][0]   # [B]
    else:
        y = Htop @ P["wo"] + P["bo"][0]          # [T][B]
    tt = np.asarray(targets, dtype=np.float64)
    tt = tt if cfg.head_last_step else tt.T      # align with y
    margin = 1.0 - tt * y
    L = alpha * np.mean(np.maximum(0.0, margin))  # Eq. 6, mean over terms
    cache.update(y=y, t=tt, margin=margin, Htop=Htop)
    return L, y, cache


# ----------------------------------------------------------------------------
# backward (BPTT)
# ----------------------------------------------------------------------------

def backward(cfg, P: Dict[str, np.ndarray], cache, alpha: float, mode: str,
             abs_terms: Dict[str, np.ndarray] = None) -> Dict[str, np.ndarray]:
    """Gradients of L = alpha * mean hinge w.r.t. every parameter block.

    In mixed mode each returned gradient is rounded once to fp16 (R12); the
    caller counts non-finite values.  If ``abs_terms`` is a dict, it receives
    for the bias-type blocks (b_l, fb, bo) the sum of the absolute values of
    the B*T terms each element sums -- the scale of any finite-precision
    evaluation's rounding error for those sums (diagnostic only; the
    gradients are unchanged).
    """
    q = _q16(mode)
    h = cfg.hidden
    T = cfg.seq
    B = cache["B"]
    y, tt, margin, Htop = cache["y"], cache["t"], cache["margin"], cache["Htop"]
    n_terms = y.size
    # d/dy of alpha*mean(max(0, 1 - t y)): -alpha t / n on active terms;
    # subgradient 0 at the kink (reading Q5)
    dy = np.where(margin > 0.0, -alpha * tt / n_terms, 0.0)
    G: Dict[str, np.ndarray] = {}
    G["bo"] = np.array([dy.sum()])
    if abs_terms is not None:
        abs_terms["bo"] = np.array([np.abs(dy).sum()])
    if cfg.fc_hidden > 0:
        z, zpre = cache["z"], cache["zpre"]
        G["wo"] = dy.reshape(-1) @ z.reshape(-1, z.shape[-1])
        dz = q(dy[..., None] * P["wo"][None, None, :] * cache["act"])   # R9 (ReLU' = 1 on active units)
        G["F"] = dz.reshape(-1, dz.shape[-1]).T @ Htop.reshape(-1, h)
        G["fb"] = dz.sum(axis=(0, 1))
        if abs_terms is not None:
            abs_terms["fb"] = np.abs(dz).sum(axis=(0, 1))
        dH_above = dz @ P["F"]                   # [T][B][h], R11 (not rounded)
    elif cfg.head_last_step:
        G["wo"] = dy @ Htop[T - 1]
        dH_above = np.zeros((T, B, h))
        dH_above[T - 1] = dy[:, None] * P["wo"][None, :]
    else:
        G["wo"] = dy.reshape(-1) @ Htop.reshape(-1, h)
        dH_above = dy[..., None] * P["wo"][None, None, :]
    for l in reversed(range(cfg.n_layers)):
        Lc = cache["layers"][l]
        W, U = P[f"W{l}"], P[f"U{l}"]
        gates, C, H, X = Lc["gates"], Lc["C"], Lc["H"], Lc["X"]
        dA_all = np.zeros((T, B, 4 * h))
        dh_rec = np.zeros((B, h))
        dc = np.zeros((B, h))
        for t in reversed(range(T)):
            i, f = gates[t][:, 0:h], gates[t][:, h:2 * h]
            g, o = gates[t][:, 2 * h:3 * h], gates[t][:, 3 * h:4 * h]
            c_t = C[t]
            c_prev = C[t - 1] if t > 0 else np.zeros((B, h))
            dh = dH_above[t] + dh_rec
            tc = np.tanh(c_t)
            dc = dc + dh * o * (1.0 - tc * tc)
            dA = np.concatenate([dc * g * i * (1.0 - i),
                                 dc * c_prev * f * (1.0 - f),
                                 dc * i * (1.0 - g * g),
                                 dh * tc * o * (1.0 - o)], axis=1)
            dA = q(dA)                           # R10
            dA_all[t] = dA
            dh_rec = dA @ U                      # R11
            if Lc["rmask"] is not None:          # gradient of h~_{t-1} -> h_{t-1}
                dh_rec = dh_rec * Lc["rmask"]
            dc = dc * f
        Hprev = Lc["Hin"]                        # h~_{t-1} (= h_{t-1} without dropout; zeros at t = 0)
        # sums over (t, b) written as one matrix product each
        dA2 = dA_all.reshape(-1, 4 * h)
        G[f"W{l}"] = dA2.T @ X.reshape(-1, X.shape[-1])
        G[f"U{l}"] = dA2.T @ Hprev.reshape(-1, h)
        G[f"b{l}"] = dA_all.sum(axis=(0, 1))
        if abs_terms is not None:
            abs_terms[f"b{l}"] = np.abs(dA_all).sum(axis=(0, 1))
        if l > 0:
            dH_above = dA_all @ W                # dX of layer l -> layer l-1
        elif cfg.vocab > 0:
            dX0 = dA_all @ W                     # [T][B][E]
            dE = np.zeros_like(P["E"])
            tok = cache["tokens"]
            np.add.at(dE, tok.T.reshape(-1), dX0.reshape(-1, dX0.shape[-1]))
            G["E"] = dE
    if mode in LOWP:
        G = {k: q(v) for k, v in G.items()}      # R12
    return G
