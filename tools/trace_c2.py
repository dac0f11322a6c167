"""Phase trace of the C2 wavefront launches (option recur_trace, profile mode):
per-step means of every phase of each role, printed to stderr by recur_trace.cpp.
    python tools/trace_c2.py [B] [T]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1912_00286_b200 import hdp  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
cfg = synth.CONFIGS["C2"]
T = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.seq
desc = hdp.desc_from_config(cfg, B, hdp.MATH_MIXED16)
tr = hdp.Trainer(desc, synth.init_params(cfg), lambda0=cfg.lambda0)
x, t = synth.model_batch(cfg, B, synth.DATA_SEED)
xd, td = torch.from_numpy(x).cuda(), torch.from_numpy(t).cuda()
s = torch.cuda.current_stream()
for _ in range(3):  # warm (graphs)
    tr.step([xd], [td], B, T, stream=s)
torch.cuda.synchronize()
hdp.set_option(None, "recur_trace", 1)
hdp.lib().hdp_profile(tr.ctx, 1)
for _ in range(2):
    print(f"---- traced step (B={B}, T={T})", file=sys.stderr, flush=True)
    tr.step([xd], [td], B, T, stream=s)
    torch.cuda.synchronize()
hdp.lib().hdp_profile(tr.ctx, 0)
hdp.set_option(None, "recur_trace", 0)
tr.close()
