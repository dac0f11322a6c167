"""Recompute the wavefront weight-gradient role's outputs on the host from the
device's own dA / Hs / X0 buffers (one C2 step) to localise a mismatch."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
import synth
from paper_1912_00286_b200 import hdp
sys.path.insert(0, ROOT)
from bench import device_view

cfg = synth.CONFIGS["C2"]
T, B = cfg.seq, cfg.batch
dev = torch.device("cuda:0")
desc = hdp.desc_from_config(cfg, B, hdp.MATH_MIXED16, hdp.WIRE_FP16_A2A, hdp.OPT_SGDM, sim_workers=1)
tr = hdp.Trainer(desc, synth.init_params(cfg), lambda0=cfg.lambda0, alpha=cfg.alpha, gamma=cfg.gamma,
                 n_half=cfg.n_half, momentum=cfg.momentum)
x, t = synth.model_batch(cfg, B, synth.DATA_SEED)
xd = torch.from_numpy(np.ascontiguousarray(x)).to(dev); td = torch.from_numpy(np.ascontiguousarray(t)).to(dev)
s = torch.cuda.current_stream()
hdp.lstm_forward(tr.ctx, xd, td, B, T, 0, None, tr.loss[0:1], s)
hdp.lstm_backward(tr.ctx, 0, s)
torch.cuda.synchronize()
blocks = {b["name"]: b for b in hdp.param_blocks(tr.ctx)}
hp = blocks["U0"]["dev_cols"]; H4 = blocks["U0"]["dev_rows"]; Ip0 = blocks["W0"]["dev_cols"]
print("hp", hp, "4hp", H4, "Ip0", Ip0)
def buf(name, n, ts="<f2"):
    return device_view(hdp.debug_buffer(tr.ctx, 0, name), n, ts, dev).float().cpu().numpy().astype(np.float64)
dA1 = buf("dA", T * B * H4).reshape(T, B, H4)
dA0 = buf("dA2", T * B * H4).reshape(T, B, H4)
Hs = buf("Hs", 2 * (T + 1) * B * hp).reshape(2, T + 1, B, hp)
X0 = buf("X0", T * B * Ip0).reshape(T, B, Ip0)
gptr = hdp.grads_ptr(tr.ctx, 0)
P = sum(b["dev_rows"] * b["dev_cols"] for b in blocks.values())
gall = device_view(gptr, max(b["dev_offset"] + b["dev_rows"] * b["dev_cols"] for b in blocks.values()), "<f2", dev).float().cpu().numpy().astype(np.float64)
def G(name):
    b = blocks[name]
    return gall[b["dev_offset"]:b["dev_offset"] + b["dev_rows"] * b["dev_cols"]].reshape(b["dev_rows"], b["dev_cols"])
print("|dA1|", np.abs(dA1).max(), "|dA0|", np.abs(dA0).max(), "|Hs|", np.abs(Hs).max(), "|X0|", np.abs(X0).max())
exp = {
    "U1": np.einsum("tbr,tbj->rj", dA1, Hs[1, :T]),
    "W1": np.einsum("tbr,tbj->rj", dA1, Hs[0, 1:]),
    "U0": np.einsum("tbr,tbj->rj", dA0, Hs[0, :T]),
    "W0": np.einsum("tbr,tbj->rj", dA0, X0),
    "b1": dA1.sum((0, 1))[:, None],
    "b0": dA0.sum((0, 1))[:, None],
}
for k, e in exp.items():
    g = G(k)
    den = np.abs(e).max() or 1
    print(k, g.shape, e.shape, "err", np.abs(g - e).max() / den, "norm ratio", np.linalg.norm(g) / np.linalg.norm(e))
# hypotheses for U1
g = G("U1")
for name, h in [("h1_t", Hs[1, 1:]), ("h0_{t-1}", Hs[0, :T]), ("h0_t", Hs[0, 1:])]:
    e = np.einsum("tbr,tbj->rj", dA1, h)
    print("U1 vs dA1^T", name, np.abs(g - e).max() / (np.abs(e).max() or 1))
e = np.einsum("tbr,tbj->rj", dA0, Hs[1, :T]); print("U1 vs dA0^T h1_{t-1}", np.abs(g - e).max() / np.abs(e).max())
gb = G("b1")[:, 0] if G("b1").ndim == 2 else G("b1")
print("b1 first 8 got", gb[:8], "exp", exp["b1"][:8, 0])
