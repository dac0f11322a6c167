"""Diagnostic: per-block GPU-vs-oracle gradient errors for reduced C3 in FP32 mode."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch, synth
from oracle import lstm as olstm
from paper_1912_00286_b200 import hdp

def run(cfg, B, mixed=False):
    desc = hdp.desc_from_config(cfg, B, hdp.MATH_MIXED16 if mixed else hdp.MATH_FP32, 0, 0, 1)
    p = synth.init_params(cfg)
    tr = hdp.Trainer(desc, p, lambda0=cfg.lambda0, alpha=cfg.alpha)
    x, t = synth.model_batch(cfg, B, synth.DATA_SEED)
    xx = x if cfg.vocab else (x if mixed else x.astype(np.float32))
    xd = torch.from_numpy(np.ascontiguousarray(xx)).cuda(); td = torch.from_numpy(np.ascontiguousarray(t)).cuda()
    hdp.lstm_forward(tr.ctx, xd, td, B, cfg.seq, 0, None, tr.loss[0:1], torch.cuda.current_stream())
    hdp.lstm_backward(tr.ctx, 0, torch.cuda.current_stream())
    torch.cuda.synchronize()
    g = hdp.read_grads(tr.ctx, 0, tr.n).astype(np.float64)
    P = olstm.unpack(cfg, p.astype(np.float64))
    L, y, c = olstm.forward(cfg, P, x, t, cfg.alpha, "mixed" if mixed else "fp32")
    G = olstm.backward(cfg, P, c, cfg.alpha, "mixed" if mixed else "fp32")
    Gg = olstm.unpack(cfg, g)
    print(cfg.name, "T", cfg.seq, "B", B, "loss gpu", tr.loss.item(), "ref", L / cfg.alpha)
    for k in G:
        e = np.abs(Gg[k] - G[k]); den = np.max(np.abs(G[k]))
        i = np.unravel_index(np.argmax(e), e.shape)
        print(f"  {k:3s} err {np.max(e)/den:.2e} max|ref| {den:.3e} worst idx {i} gpu {Gg[k][i]:.6e} ref {G[k][i]:.6e}")
    tr.close()

for seq, B in ((24, 4), (2, 4), (1, 4), (24, 1)):
    run(synth.CONFIGS["C3"].with_(seq=seq), B)
run(synth.CONFIGS["C3"].with_(seq=24, vocab=0, input_dim=128, embed_dim=0), 4)
run(synth.CONFIGS["C1"].with_(n_layers=2, head_last_step=True), 4)
