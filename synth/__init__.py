"""Seeded synthetic inputs shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no LSTM, no loss, no update,
no schedule).  It only describes the five configurations of
``BASELINE.json`` as plain data and draws seeded random inputs with the
shapes and structure of the paper's workloads:

* JET-shaped multi-channel 1 ms time series (Fig. 2
  "(256,128,9)", App. A :266-281 "about 10% of shots ends in a disruption"),
  per-channel standardisation in fp32, stored as fp16.
* IMDB-shaped token sequences (labels split evenly).
* Dense N(0,1) inputs for the tiny (C1) and the ~70M stacked (C4) configs.
* Random parameter initialisation, "Initialize the network parameters
  randomly" (step 1): U(-1/sqrt(fan_in), +1/sqrt(fan_in)) per
  block, forget-gate bias 1, other biases 0, rounded to
  fp16-representable values so that fp32 master == fp16 working copy at k=0.

Seeds: data 1912, init 286, rank r's throughput
stream 1912 + 1000*r.

The canonical (unpadded) parameter layout is the C-ABI's host format
(include/hdp.h, hdp_load_params):  [E (vocab x embed)]?  then per layer l:
W_l [4h][I_l], U_l [4h][h], b_l [4h] with gate blocks in the order i, f, g, o
(row r = gate*h + unit); then the head: [F [fc][h], f_b [fc]]?, w_o [fc or h],
b_o [1].  ``param_blocks`` lists it.
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Tuple

import numpy as np

DATA_SEED = 1912
INIT_SEED = 286


@dataclasses.dataclass(frozen=True)
class ModelConfig:
    """Shape description of one LSTM model (no arithmetic)."""
    name: str
    n_layers: int
    input_dim: int          # I of layer 0 (ignored when vocab > 0; embed_dim is used)
    hidden: int             # h
    seq: int                # T
    batch: int              # per-rank batch beta_0 used by the bench
    fc_hidden: int = 0      # 0 = no FC layer (C2 has FC 200 + ReLU, Fig. 2)
    head_last_step: bool = False   # C3: one output per sequence at t = T-1
    vocab: int = 0          # >0: token input through an embedding (C3)
    embed_dim: int = 0
    alpha: float = 10.0     # loss scale, "loss scaling factor: 10.0"
    lambda0: float = 4e-4
    gamma: float = 0.8      # SPEC.md:269 default
    n_half: float = 100.0   # SPEC.md:242 examples
    momentum: float = 0.9   # SPEC.md:269 default
    max_eff_lr: float = 0.1

    @property
    def layer_input_dims(self) -> List[int]:
        first = self.embed_dim if self.vocab > 0 else self.input_dim
        return [first] + [self.hidden] * (self.n_layers - 1)

    def with_(self, **kw) -> "ModelConfig":
        return dataclasses.replace(self, **kw)


# BASELINE.json configs[0..3]; C5 is a flat update sweep (no model).
CONFIGS: Dict[str, ModelConfig] = {
    "C1": ModelConfig("C1-tiny", n_layers=1, input_dim=8, hidden=32, seq=16, batch=4,
                      lambda0=0.01),
    "C2": ModelConfig("C2-jet", n_layers=2, input_dim=9, hidden=200, seq=128, batch=128,
                      fc_hidden=200, lambda0=4e-4),
    "C3": ModelConfig("C3-imdb", n_layers=2, input_dim=0, hidden=256, seq=256, batch=128,
                      head_last_step=True, vocab=20000, embed_dim=128, lambda0=0.02),
    "C4": ModelConfig("C4-stacked", n_layers=4, input_dim=2048, hidden=2048, seq=128, batch=256,
                      lambda0=4e-4),
}
C1_SIM_WORKERS = 2
C1_GLOBAL_BATCH = 8


def param_blocks(cfg: ModelConfig) -> List[Tuple[str, Tuple[int, ...], str]]:
    """Canonical block list: (name, shape, kind) with kind in
    {'embed','W','U','b','F','fb','wo','bo'}."""
    h = cfg.hidden
    out: List[Tuple[str, Tuple[int, ...], str]] = []
    if cfg.vocab > 0:
        out.append(("E", (cfg.vocab, cfg.embed_dim), "embed"))
    for l, i_l in enumerate(cfg.layer_input_dims):
        out.append((f"W{l}", (4 * h, i_l), "W"))
        out.append((f"U{l}", (4 * h, h), "U"))
        out.append((f"b{l}", (4 * h,), "b"))
    if cfg.fc_hidden > 0:
        out.append(("F", (cfg.fc_hidden, h), "F"))
        out.append(("fb", (cfg.fc_hidden,), "fb"))
        out.append(("wo", (cfg.fc_hidden,), "wo"))
    else:
        out.append(("wo", (h,), "wo"))
    out.append(("bo", (1,), "bo"))
    return out


def n_params(cfg: ModelConfig) -> int:
    return int(sum(int(np.prod(s)) for _, s, _ in param_blocks(cfg)))


def _fp16_representable(a: np.ndarray) -> np.ndarray:
    return a.astype(np.float16).astype(np.float32)


def init_params(cfg: ModelConfig, seed: int = INIT_SEED) -> np.ndarray:
    """Flat fp32 vector in the canonical layout."""
    rng = np.random.Generator(np.random.PCG64(seed))
    h = cfg.hidden
    parts = []
    for name, shape, kind in param_blocks(cfg):
        if kind in ("W", "U", "F", "wo", "embed"):
            fan_in = shape[-1] if len(shape) == 2 else shape[0]
            lim = 1.0 / np.sqrt(fan_in)
            parts.append(rng.uniform(-lim, lim, size=shape).ravel())
        elif kind == "b":
            b = np.zeros(shape)
            b[h:2 * h] = 1.0          # forget-gate bias = 1 (gate order i, f, g, o)
            parts.append(b)
        else:
            parts.append(np.zeros(shape).ravel())
    return _fp16_representable(np.concatenate(parts))


# ----------------------------------------------------------------------------
# Inputs
# ----------------------------------------------------------------------------

def dense_batch(B: int, T: int, I: int, seed: int, pos_frac: float = 0.25,
                end_window: bool = False) -> Tuple[np.ndarray, np.ndarray]:
    """C1 / C4: x ~ N(0,1) [B][T][I] as fp16; targets in {-1,+1} int8 [B][T].

    end_window=False: iid +1 with probability pos_frac (C1, 25%).
    end_window=True : a fraction pos_frac of sequences is positive on a final
    window of 10..40 steps, -1 elsewhere (C4, 10%).
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    x = rng.standard_normal((B, T, I)).astype(np.float16)
    if not end_window:
        t = np.where(rng.random((B, T)) < pos_frac, 1, -1).astype(np.int8)
    else:
        t = -np.ones((B, T), np.int8)
        pos = rng.random(B) < pos_frac
        for b in np.nonzero(pos)[0]:
            w = int(rng.integers(10, 41))
            t[b, max(0, T - w):] = 1
    return x, t


def jet_batch(B: int, T: int, D: int, seed: int) -> Tuple[np.ndarray, np.ndarray]:
    """C2, JET-shaped: D channels at 1 ms (App. A :266-281).

    Per channel an AR(1) process x_t = 0.95 x_{t-1} + 0.3 eps_t plus a slow
    linear drift; 10% of sequences are "disruptive" (App. A "about 10%"):
    a linear ramp on 3 random channels over the last 50..120 steps.  Targets
    are +1 on the ramp steps of disruptive sequences, -1 elsewhere (SPEC.md:205
    horizon idea).  Per-channel standardisation in fp32, then
    fp16.
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    eps = rng.standard_normal((B, T, D))
    x = np.zeros((B, T, D))
    for t in range(T):
        x[:, t] = (0.95 * x[:, t - 1] if t > 0 else 0.0) + 0.3 * eps[:, t]
    drift = rng.normal(0.0, 0.01, size=(B, 1, D)) * np.arange(T)[None, :, None]
    x = x + drift
    tgt = -np.ones((B, T), np.int8)
    n_dis = max(1, int(round(0.10 * B)))
    dis = rng.choice(B, size=n_dis, replace=False)
    for b in dis:
        L = int(rng.integers(50, min(120, T) + 1)) if T >= 50 else T
        ch = rng.choice(D, size=min(3, D), replace=False)
        ramp = np.linspace(0.0, 3.0, L)
        for c in ch:
            x[b, T - L:, c] += ramp * rng.choice([-1.0, 1.0])
        tgt[b, T - L:] = 1
    x32 = x.astype(np.float32)
    mu = x32.mean(axis=(0, 1), keepdims=True, dtype=np.float32)
    sd = x32.std(axis=(0, 1), keepdims=True, dtype=np.float32)
    sd = np.where(sd > 0, sd, np.float32(1.0))
    xs = ((x32 - mu) / sd).astype(np.float32)
    return xs.astype(np.float16), tgt


# JET channels of App. A that carry the synthetic precursors of
# jet_precursor_batch: l_i (internal inductance), MLA (locked-mode amplitude), P_rad
# (radiated power) -- indices in the App. A order
PRECURSOR_CHANNELS = (3, 5, 6)


def jet_precursor_batch(B: int, T: int, D: int, seed: int, disruptive_frac: float = 0.1,
                        amplitude: float = 3.0, lead=(60, 100)) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    """JET-analog chunks with a LEARNABLE disruption precursor (NEXT-4 convergence runs).

    Background as in jet_batch: per channel AR(1) x_t = 0.95 x_{t-1} + 0.3 eps_t plus a
    slow linear drift.  A chunk is disruptive with probability ``disruptive_frac``
    (App. A :279 "about 10%"; training chunks may be class-balanced); a disruptive chunk
    ends in the disruption (t_disrupt = T) and carries a rising ramp of ``amplitude`` on
    the PRECURSOR_CHANNELS over its last L ~ U[lead] steps (so at least lead[0] - 30 ramp
    steps precede the 30 ms alarm cutoff).  Targets are +1 on the ramp
    steps, -1 elsewhere.  Standardisation uses fixed constants of the
    generator (mean 0, scale 1.2) so every batch sees the same transform; fp16 storage.
    Returns x fp16 [B][T][D], targets int8 [B][T], disruptive bool [B]."""
    rng = np.random.Generator(np.random.PCG64(seed))
    eps = rng.standard_normal((B, T, D))
    x = np.zeros((B, T, D))
    for t in range(T):
        x[:, t] = (0.95 * x[:, t - 1] if t > 0 else 0.0) + 0.3 * eps[:, t]
    x = x + rng.normal(0.0, 0.01, size=(B, 1, D)) * np.arange(T)[None, :, None]
    tgt = -np.ones((B, T), np.int8)
    dis = rng.random(B) < disruptive_frac
    chans = [c for c in PRECURSOR_CHANNELS if c < D]
    for b in np.nonzero(dis)[0]:
        L = int(rng.integers(lead[0], min(lead[1], T) + 1))
        for c in chans:
            x[b, T - L:, c] += np.linspace(0.0, amplitude, L)
        tgt[b, T - L:] = 1
    xs = (x.astype(np.float32) / np.float32(1.2)).astype(np.float16)
    return xs, tgt, dis


IMDB_LEXICON = 50


def imdb_batch(B: int, T: int, vocab: int, seed: int) -> Tuple[np.ndarray, np.ndarray]:
    """C3, IMDB-shaped token sequences (App. B :285-293).

    Token ids ~ Zipf(a=1.2) clipped to [1, vocab-1]; lengths ~
    lognormal(ln 180, 0.6) clipped to [10, 2500], pre-padded / truncated to T
    with id 0 (so t = T-1 is always a real token); labels +-1 split evenly;
    planted signal: 3% of tokens drawn from a 50-id positive or negative
    lexicon according to the label.  (Length and Zipf parameters are
    assumptions; the paper gives none.)
    Returns tokens int32 [B][T] and labels int8 [B].
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    labels = np.where(np.arange(B) % 2 == 0, 1, -1).astype(np.int8)
    rng.shuffle(labels)
    toks = np.zeros((B, T), np.int32)
    lengths = np.clip(np.exp(rng.normal(np.log(180.0), 0.6, size=B)), 10, 2500).astype(int)
    pos_lex = np.arange(100, 100 + IMDB_LEXICON)
    neg_lex = np.arange(200, 200 + IMDB_LEXICON)
    for b in range(B):
        n = min(int(lengths[b]), T)
        z = np.minimum(rng.zipf(1.2, size=n), vocab - 1).astype(np.int32)
        plant = rng.random(n) < 0.03
        lex = pos_lex if labels[b] > 0 else neg_lex
        z[plant] = rng.choice(lex, size=int(plant.sum()))
        toks[b, T - n:] = z
    return toks, labels


def model_batch(cfg: ModelConfig, B: int, seed: int):
    """Inputs for one (global or per-rank) batch of ``cfg``.

    Returns (x, targets) where x is fp16 [B][T][I] or int32 tokens [B][T],
    targets int8 [B][T] (per-step heads) or [B] (last-step head).
    """
    T = cfg.seq
    if cfg.vocab > 0:
        return imdb_batch(B, T, cfg.vocab, seed)
    if cfg.fc_hidden > 0:
        return jet_batch(B, T, cfg.input_dim, seed)
    if cfg.name.startswith("C4"):
        return dense_batch(B, T, cfg.input_dim, seed, pos_frac=0.10, end_window=True)
    return dense_batch(B, T, cfg.input_dim, seed, pos_frac=0.25)


def update_sweep_inputs(n_elems: int, n_ranks: int, seed: int, wire_fp32: bool = False):
    """C5 inputs: per-rank gradients g ~ N(0, 0.05^2) (already x alpha) with one
    element in 1e6 set to +-30000 (finite, near the fp16 range); master ~
    U(-0.1, 0.1); momentum H ~ N(0, 1e-3^2)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    gdt = np.float32 if wire_fp32 else np.float16
    grads = []
    for r in range(n_ranks):
        g = rng.normal(0.0, 0.05, size=n_elems)
        k = max(1, n_elems // 1_000_000)
        idx = rng.integers(0, n_elems, size=k)
        g[idx] = rng.choice([-30000.0, 30000.0], size=k)
        grads.append(g.astype(gdt))
    master = rng.uniform(-0.1, 0.1, size=n_elems).astype(np.float32)
    mom = rng.normal(0.0, 1e-3, size=n_elems).astype(np.float32)
    return grads, master, mom
