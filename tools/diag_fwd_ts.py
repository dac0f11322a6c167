"""Compare the forward wavefront's saved activations (Hs, C, gates) between the
TMEM-A instantiation and the generic one (HDP_WAVEFRONT_TS=0) on one C2 batch."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
import synth
from paper_1912_00286_b200 import hdp
from bench import device_view

cfg = synth.CONFIGS["C2"]
T = int(os.environ.get("DIAG_T", 16)); cfg = cfg.with_(seq=T)
B = cfg.batch
dev = torch.device("cuda:0")
out = {}
for flag in ("0", "1"):
    os.environ["HDP_WAVEFRONT_TS"] = flag
    desc = hdp.desc_from_config(cfg, B, hdp.MATH_MIXED16, hdp.WIRE_FP16_A2A, hdp.OPT_SGDM, sim_workers=1)
    tr = hdp.Trainer(desc, synth.init_params(cfg), lambda0=cfg.lambda0, alpha=cfg.alpha, gamma=cfg.gamma,
                     n_half=cfg.n_half, momentum=cfg.momentum)
    x, t = synth.model_batch(cfg, B, synth.DATA_SEED)
    xd = torch.from_numpy(np.ascontiguousarray(x)).to(dev); td = torch.from_numpy(np.ascontiguousarray(t)).to(dev)
    hdp.lstm_forward(tr.ctx, xd, td, B, T, 0, None, tr.loss[0:1], torch.cuda.current_stream())
    torch.cuda.synchronize()
    blocks = {b["name"]: b for b in hdp.param_blocks(tr.ctx)}
    hp = blocks["U0"]["dev_cols"]
    def buf(name, n, ts):
        return device_view(hdp.debug_buffer(tr.ctx, 0, name), n, ts, dev).float().cpu().numpy()
    out[flag] = {"Hs": buf("Hs", 2 * (T + 1) * B * hp, "<f2").reshape(2, T + 1, B, hp),
                 "C": buf("C", 2 * T * B * hp, "<f4").reshape(2, T, B, hp),
                 "gates": buf("gates", 2 * T * B * 4 * hp, "<f2").reshape(2, T, B, 4 * hp),
                 "loss": float(tr.loss[0].item())}
    tr.close()
for k in ("Hs", "C", "gates"):
    a, b = out["0"][k], out["1"][k]
    d = np.abs(a - b)
    print(k, "max diff", d.max(), "max |ref|", np.abs(a).max())
    for l in range(2):
        dl = d[l].reshape(d.shape[1], -1).max(1)
        print(f"  layer {l}: per-t max diff (first 6 t)", np.round(dl[:6], 5).tolist())
    if k == "gates":
        dd = d[0, 1]  # layer 0, t=1
        bad = np.argwhere(dd > 1e-2)
        print("  layer0 t=1 bad (b, gate-row) examples:", bad[:10].tolist(), "count", len(bad))
print("loss", out["0"]["loss"], out["1"]["loss"])
