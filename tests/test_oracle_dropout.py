"""Pins for the recurrent-dropout oracle (NEXT-3; oracle/dropout.py,
reading Q16b): finite differences with the masks held fixed, the keep = 1
identity, and the statistics of the counter-based mask."""
import numpy as np
import pytest

import synth
from oracle import dropout, lstm, step


def _tiny(kind):
    if kind == "fc":
        return synth.ModelConfig("t-fc", n_layers=2, input_dim=3, hidden=5, seq=5, batch=3, fc_hidden=3)
    return synth.ModelConfig("t-lin", n_layers=2, input_dim=3, hidden=5, seq=5, batch=3)


def _near_kink(cfg, cache):
    if np.min(np.abs(cache["margin"])) < 1e-3:
        return True
    return bool(cfg.fc_hidden and np.min(np.abs(cache["zpre"])) < 1e-3)


@pytest.mark.parametrize("kind", ["lin", "fc"])
def test_bptt_with_recurrent_dropout_matches_central_differences(kind):
    cfg = _tiny(kind)
    keep = 0.6
    drop = {"scale": dropout.scale(keep),
            "masks": [dropout.mask(7, 3, l, np.arange(cfg.batch), cfg.hidden, keep) for l in range(cfg.n_layers)]}
    assert all(0 < m.mean() < 1 for m in drop["masks"])          # some units dropped, some kept
    seed = 0
    while True:
        rng = np.random.default_rng(500 + seed)
        flat = rng.uniform(-0.6, 0.6, lstm.count(cfg))
        x = rng.standard_normal((cfg.batch, cfg.seq, cfg.input_dim))
        t = np.where(rng.random((cfg.batch, cfg.seq)) < 0.5, 1, -1).astype(np.int8)
        L, _, cache = lstm.forward(cfg, lstm.unpack(cfg, flat), x, t, 10.0, "fp64", drop)
        if not _near_kink(cfg, cache):
            break
        seed += 1
    G = lstm.pack(cfg, lstm.backward(cfg, lstm.unpack(cfg, flat), cache, 10.0, "fp64"))
    eps = 1e-5
    fd = np.zeros_like(flat)
    for k in range(flat.size):
        d = np.zeros_like(flat)
        d[k] = eps
        fd[k] = (lstm.forward(cfg, lstm.unpack(cfg, flat + d), x, t, 10.0, "fp64", drop)[0] -
                 lstm.forward(cfg, lstm.unpack(cfg, flat - d), x, t, 10.0, "fp64", drop)[0]) / (2 * eps)
    floor = 1e-9 * max(1.0, abs(L))
    assert np.all(np.abs(G - fd) <= 1e-6 * np.abs(G) + floor)
    # the masks matter: without them the gradient is different
    L0, _, c0 = lstm.forward(cfg, lstm.unpack(cfg, flat), x, t, 10.0, "fp64")
    G0 = lstm.pack(cfg, lstm.backward(cfg, lstm.unpack(cfg, flat), c0, 10.0, "fp64"))
    assert np.max(np.abs(G0 - G)) > 1e-3 * np.max(np.abs(G))


def test_keep_one_is_no_dropout():
    cfg = _tiny("fc").with_(batch=4)
    rng = np.random.default_rng(1)
    w = rng.uniform(-0.5, 0.5, lstm.count(cfg))
    x = rng.standard_normal((4, cfg.seq, cfg.input_dim))
    t = np.where(rng.random((4, cfg.seq)) < 0.5, 1, -1).astype(np.int8)
    a = step.train_step(cfg, w, {"H": np.zeros_like(w)}, x, t, 2, 10.0, 0.1, "mixed")
    b = step.train_step(cfg, w, {"H": np.zeros_like(w)}, x, t, 2, 10.0, 0.1, "mixed",
                        dropout={"keep": 1.0, "seed": 5, "step": 0})
    assert np.array_equal(a["master"], b["master"]) and a["loss"] == b["loss"]
    c = step.train_step(cfg, w, {"H": np.zeros_like(w)}, x, t, 2, 10.0, 0.1, "mixed",
                        dropout={"keep": 0.5, "seed": 5, "step": 0})
    assert not np.array_equal(a["master"], c["master"])


def test_mask_statistics_and_keys():
    keep = 0.7
    m = dropout.mask(11, 4, 1, np.arange(2000), 256, keep)
    n = m.size
    assert abs(m.mean() - keep) <= 5 * np.sqrt(keep * (1 - keep) / n)          # Bernoulli(keep)
    assert set(np.unique(m)) <= {0.0, 1.0}
    assert np.array_equal(m, dropout.mask(11, 4, 1, np.arange(2000), 256, keep))  # deterministic
    for other in (dropout.mask(11, 5, 1, np.arange(2000), 256, keep),           # next step
                  dropout.mask(11, 4, 0, np.arange(2000), 256, keep),           # other layer
                  dropout.mask(12, 4, 1, np.arange(2000), 256, keep),           # other seed
                  dropout.mask(11, 4, 1, np.arange(1, 2001), 256, keep)):       # shifted sequences
        agree = np.mean(m == other)                                             # independent draws
        assert abs(agree - (keep ** 2 + (1 - keep) ** 2)) < 0.01
    # the row of a sequence does not depend on which other sequences are in the batch
    assert np.array_equal(dropout.mask(11, 4, 1, [17], 256, keep)[0], m[17])
    assert dropout.scale(0.8) == np.float32(1.25) and dropout.threshold(0.5) == 2 ** 31
