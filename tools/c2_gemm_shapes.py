"""Per-shape timing of the tcgen05 GEMM on the C2 (JET-shaped) step's
non-recurrent contractions, with the HBM-traffic lower bound of each."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_1912_00286_b200 import hdp



def tstore(X, mn):
    return (X.T.contiguous(), X.shape[0]) if mn else (X, X.shape[1])


R, H4, H, I, F = 16384, 832, 208, 16, 208
SHAPES = {  # name: (M, N, K, a_mn, b_mn)
    "K1 Gx0 = X0 W0^T": (R, H4, I, 0, 0),
    "head Z = H Fw^T": (R, F, H, 0, 0),
    "head dF = dz^T H": (F, H, R, 1, 1),
    "head dH = dz Fw": (R, H, F, 0, 1),
    "K8 dW0 = dA0^T X0": (H4, I, R, 1, 1),
    "K8 dU0 = dA0^T H0": (H4, H, R, 1, 1),
    "C3 K1 Gx0 = E X0": (32768, 1024, 128, 0, 0),
    "C3 K9 dX0 = dA0 W0": (32768, 128, 1024, 0, 1),
}


def run(M, N, K, amn, bmn, bn, splits, iters=50):
    A = torch.randn(M, K, device="cuda").half(); B = torch.randn(N, K, device="cuda").half()
    As, lda = tstore(A, amn); Bs, ldb = tstore(B, bmn)
    C = torch.empty(M, N, device="cuda")
    ws = torch.empty(16 * M * N, device="cuda")
    f = lambda st: hdp.gemm_f16(As, lda, amn, Bs, ldb, bmn, M, N, K, C, N, 0, ws=ws, ws_floats=ws.numel(), bn=bn,
                                splits=splits, stream=st)
    s0 = torch.cuda.current_stream()
    for _ in range(3): f(s0)
    torch.cuda.synchronize()
    # device time only: the launches are replayed from a CUDA graph (host overhead excluded)
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    with torch.cuda.stream(cs):
        with torch.cuda.graph(g, stream=cs):
            for _ in range(iters): f(cs)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    g.replay()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e3


for name, (M, N, K, a, b) in SHAPES.items():
    ideal_us = (2 * (M * K + N * K) + 4 * M * N) / 7.0e12 * 1e6
    for bn in (0, 128, 256):
        for splits in ((0,) if K < 4096 else (0, 16)):
            try:
                us = run(M, N, K, a, b, bn, splits)
                print(json.dumps({"shape": name, "M": M, "N": N, "K": K, "bn": bn, "splits": splits, "us": round(us, 2),
                                  "hbm_bound_us": round(ideal_us, 2)}), flush=True)
            except Exception as e:
                print(json.dumps({"shape": name, "bn": bn, "splits": splits, "error": str(e)[:200]}), flush=True)
