"""Microbenchmark of the tcgen05 GEMM (hdp_gemm_f16) on the C4 contraction
shapes, against torch.matmul (cuBLAS) on the same fp16 operands."""
import os, sys, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_1912_00286_b200 import hdp

def tstore(X, mn):
    return (X.T.contiguous(), X.shape[0]) if mn else (X, X.shape[1])

def bench(M, N, K, amn, bmn, bn=0, splits=0, iters=20):
    A = torch.randn(M, K, device="cuda").half(); B = torch.randn(N, K, device="cuda").half()
    As, lda = tstore(A, amn); Bs, ldb = tstore(B, bmn)
    C = torch.empty(M, N, device="cuda")
    ws = torch.empty(16 * M * N, device="cuda")
    f = lambda: hdp.gemm_f16(As, lda, amn, Bs, ldb, bmn, M, N, K, C, N, 0, ws=ws, ws_floats=ws.numel(), bn=bn, splits=splits)
    for _ in range(3): f()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(iters): f()
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / iters
    g = lambda: torch.matmul(A, B.T)
    for _ in range(3): g()
    e0.record()
    for _ in range(iters): g()
    e1.record(); torch.cuda.synchronize()
    ms_cublas = e0.elapsed_time(e1) / iters
    fl = 2.0 * M * N * K
    return {"M": M, "N": N, "K": K, "amn": amn, "bmn": bmn, "bn": bn, "splits": splits, "us": ms * 1e3,
            "tflops": fl / ms / 1e9, "cublas_tflops": fl / ms_cublas / 1e9}

shapes = [(8192, 8192, 8192, 0, 0), (32768, 8192, 2048, 0, 0), (256, 8192, 2048, 0, 0), (256, 2048, 8192, 0, 1),
          (8192, 2048, 32768, 1, 1), (32768, 2048, 8192, 0, 1), (128, 832, 208, 0, 0)]
for (M, N, K, a, b) in shapes:
    for bn in (0, 64, 128, 256):
        try:
            print(json.dumps(bench(M, N, K, a, b, bn=bn)), flush=True)
        except Exception as e:
            print(json.dumps({"M": M, "N": N, "K": K, "bn": bn, "error": str(e)}), flush=True)
