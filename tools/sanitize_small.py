"""Tiny training steps for compute-sanitizer (memcheck) runs on one GPU:
    compute-sanitizer --tool memcheck python tools/sanitize_small.py perstep|wavefront
perstep  : C1 (2 simulated workers, K11 and the one-kernel exchange loopback), the
           per-step GEMM + fused-epilogue path (persistent recurrences off) incl. C3's
           embedding gather / radix-sort backward, 2 steps each;
wavefront: C2 at B = 32, T = 8 through both two-layer wavefront launches, 2 steps."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import synth  # noqa: E402
from parity import kernel_options, run_parity  # noqa: E402

from paper_1912_00286_b200 import hdp  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "perstep"
if which == "perstep":
    with kernel_options(persistent=0):
        for exch in (hdp.EXCH_NCCL, hdp.EXCH_P2P):
            recs = run_parity(synth.CONFIGS["C1"], 8, 2, steps=2, mixed=True, exchange=exch, compare_grads=False)
            print("C1 exchange", exch, "master err", max(recs[-1]["master_err"].values()), flush=True)
        recs = run_parity(synth.CONFIGS["C3"].with_(seq=6), 4, 1, steps=2, mixed=True, compare_grads=False)
        print("C3 per-step master err", max(recs[-1]["master_err"].values()), flush=True)
        recs = run_parity(synth.CONFIGS["C2"].with_(seq=4), 4, 1, steps=1, mixed=True, compare_grads=False)
        print("C2 per-step master err", max(recs[-1]["master_err"].values()), flush=True)
else:
    recs = run_parity(synth.CONFIGS["C2"].with_(seq=8), 32, 1, steps=2, mixed=True, compare_grads=False)
    print("C2 wavefront master err", max(recs[-1]["master_err"].values()), flush=True)
print("sanitize_small done", which, flush=True)
