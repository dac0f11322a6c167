"""Where a training step's time goes between the C-ABI calls: CUDA events on the caller's
stream around hdp_lstm_forward / hdp_lstm_backward / hdp_grad_average_update (each a
captured graph or a short launch sequence), for comparison with the kernel durations of
the launch list -- the difference is launch gaps and serialisation.
    python tools/step_timeline.py [C2|C3|C4] [steps]"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1912_00286_b200 import hdp  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg = synth.CONFIGS[name]
B = cfg.batch
desc = hdp.desc_from_config(cfg, B, hdp.MATH_MIXED16)
tr = hdp.Trainer(desc, synth.init_params(cfg), lambda0=cfg.lambda0, alpha=cfg.alpha, gamma=cfg.gamma,
                 n_half=cfg.n_half, momentum=cfg.momentum)
x, t = synth.model_batch(cfg, B, synth.DATA_SEED)
xd, td = torch.from_numpy(np.ascontiguousarray(x)).cuda(), torch.from_numpy(np.ascontiguousarray(t)).cuda()
s = torch.cuda.current_stream()
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(5):
    hdp.lstm_forward(tr.ctx, xd, td, B, cfg.seq, 0, None, tr.loss[0:1], s)
    hdp.lstm_backward(tr.ctx, 0, s)
    hdp.grad_average_update(tr.ctx, 0, s)
torch.cuda.synchronize()
rec = []
for _ in range(steps):
    flush.zero_()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record(s)
    hdp.lstm_forward(tr.ctx, xd, td, B, cfg.seq, 0, None, tr.loss[0:1], s)
    ev[1].record(s)
    hdp.lstm_backward(tr.ctx, 0, s)
    ev[2].record(s)
    hdp.grad_average_update(tr.ctx, 0, s)
    ev[3].record(s)
    rec.append(ev)
torch.cuda.synchronize()
out = {"config": name, "steps": steps}
for i, k in enumerate(("forward_us", "backward_us", "update_us")):
    out[k] = round(statistics.mean(1e3 * e[i].elapsed_time(e[i + 1]) for e in rec), 1)
out["step_us"] = round(statistics.mean(1e3 * e[0].elapsed_time(e[3]) for e in rec), 1)
print(json.dumps(out))
tr.close()
