"""Compare the wavefront weight-gradient role (HDP_WAVEFRONT_WGRAD=1) with the
K8 GEMMs (=0) on one C2 step: per-block error, norm ratio, worst rows/cols."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
import synth
from oracle import lstm as olstm
from paper_1912_00286_b200 import hdp

cfg = synth.CONFIGS["C2"]
T = int(os.environ.get("DIAG_T", cfg.seq)); cfg = cfg.with_(seq=T)
B = int(os.environ.get("DIAG_B", cfg.batch))
out = {}
for flag in ("0", "1"):
    os.environ["HDP_WAVEFRONT_WGRAD"] = flag
    desc = hdp.desc_from_config(cfg, B, hdp.MATH_MIXED16, hdp.WIRE_FP16_A2A, hdp.OPT_SGDM, sim_workers=1)
    params = synth.init_params(cfg)
    tr = hdp.Trainer(desc, params, lambda0=cfg.lambda0, alpha=cfg.alpha, gamma=cfg.gamma, n_half=cfg.n_half,
                     momentum=cfg.momentum)
    x, t = synth.model_batch(cfg, B, synth.DATA_SEED)
    dev = torch.device("cuda:0")
    xd = torch.from_numpy(np.ascontiguousarray(x)).to(dev); td = torch.from_numpy(np.ascontiguousarray(t)).to(dev)
    s = torch.cuda.current_stream()
    for rep in range(2):
        hdp.lstm_forward(tr.ctx, xd, td, B, T, 0, None, tr.loss[0:1], s)
        hdp.lstm_backward(tr.ctx, 0, s)
        torch.cuda.synchronize()
        g = olstm.unpack(cfg, hdp.read_grads(tr.ctx, 0, tr.n).astype(np.float64))
        out[(flag, rep)] = g
    tr.close()
ref = out[("0", 0)]
for key in [("0", 1), ("1", 0), ("1", 1)]:
    print("==", key)
    for k, r in ref.items():
        gk = out[key][k]
        den = np.max(np.abs(r)) or 1.0
        err = np.max(np.abs(gk - r)) / den
        line = f"  {k:4s} shape {r.shape} err {err:.3e} |g|/|r| {np.linalg.norm(gk) / (np.linalg.norm(r) or 1):.4f}"
        if err > 1e-2 and r.ndim == 2:
            d = np.abs(gk - r)
            rows = np.argsort(-d.max(1))[:6]; cols = np.argsort(-d.max(0))[:6]
            line += f" worst rows {rows.tolist()} cols {cols.tolist()} | nz rows with err>1e-2*den: {int((d.max(1) > 1e-2 * den).sum())}/{r.shape[0]}"
            c = np.corrcoef(gk.ravel(), r.ravel())[0, 1]
            line += f" corr {c:.4f}"
        elif err > 1e-2:
            d = np.abs(gk - r)
            line += f" worst idx {np.argsort(-d)[:8].tolist()} ({int((d > 1e-2 * den).sum())}/{r.size} bad)"
        print(line)
