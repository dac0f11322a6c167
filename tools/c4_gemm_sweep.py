"""Tile / split-K sweep of the tcgen05 GEMM on the C4 per-timestep recurrent
shapes (K2: G_h = h U^T, M=256 N=8192 K=2048; K7: dh_rec = dA U, M=256
N=2048 K=8192 with U read MN-major), L2-warm back-to-back launches as in the
recurrence.  Prints one JSON line per (shape, bn, splits)."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_1912_00286_b200 import hdp


def run(M, N, K, amn, bmn, bn, splits, iters=50):
    A = (torch.randn(M, K, device="cuda") * 0.1).half()
    B = (torch.randn(N, K, device="cuda") * 0.1).half()
    As, lda = (A.T.contiguous(), M) if amn else (A, K)
    Bs, ldb = (B.T.contiguous(), N) if bmn else (B, K)
    C = torch.empty(M, N, device="cuda")
    ws = torch.empty(16 * M * N, device="cuda")
    f = lambda: hdp.gemm_f16(As, lda, amn, Bs, ldb, bmn, M, N, K, C, N, 0, ws=ws, ws_floats=ws.numel(), bn=bn,
                             splits=splits)
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    ref = (A.float() @ B.float().T)
    err = ((C - ref).abs().max() / ref.abs().max()).item()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(iters):
        f()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / iters * 1e3
    return {"M": M, "N": N, "K": K, "amn": amn, "bmn": bmn, "bn": bn, "splits": splits, "us": round(us, 2),
            "tflops": round(2.0 * M * N * K / us / 1e6, 1), "err": err}


if __name__ == "__main__":
    only = os.environ.get("SWEEP_ONLY")
    shapes = [(256, 8192, 2048, 0, 0), (256, 2048, 8192, 0, 1)]
    for (M, N, K, a, b) in shapes:
        for bn in (64, 128, 256):
            for sp in (1, 2, 3, 4, 6, 8, 16):
                if only and f"{bn}/{sp}" not in only.split(","):
                    continue
                try:
                    print(json.dumps(run(M, N, K, a, b, bn, sp)), flush=True)
                except Exception as e:
                    print(json.dumps({"M": M, "bn": bn, "splits": sp, "error": str(e)}), flush=True)
