"""Do the C4 per-step GEMMs of different layers gain from running concurrently?
Times NL x (64 / NL) launches of the K2 shape (256 x 8192 x 2048, BN = 128) and of the
K7 shape (256 x 2048 x 8192, BN = 256, 8 K-splits) captured in one CUDA graph, the NL
chains on NL streams with a separate U (and split-K scratch) per stream -- the
concurrency a layer-diagonal schedule of the per-step path would give.
python tools/concurrent_gemm.py  ->  one JSON line per (shape, NL)"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_1912_00286_b200 import hdp  # noqa: E402

TOTAL = 64
SHAPES = {"K2": (256, 8192, 2048, 0, 0, 128, 1), "K7": (256, 2048, 8192, 0, 1, 256, 8)}


def run(name, NL):
    M, N, K, amn, bmn, bn, splits = SHAPES[name]
    A = [torch.randn(M, K, device="cuda").half() for _ in range(NL)]
    B = [(torch.randn(K, N, device="cuda") if bmn else torch.randn(N, K, device="cuda")).half() for _ in range(NL)]
    C = [torch.empty(M, N, device="cuda") for _ in range(NL)]
    ws = [torch.empty(splits * M * N + 16, device="cuda") for _ in range(NL)]
    streams = [torch.cuda.Stream() for _ in range(NL)]

    def body():
        main = torch.cuda.current_stream()
        for s in streams:
            s.wait_stream(main)
        for i in range(TOTAL // NL):
            for l in range(NL):
                hdp.gemm_f16(A[l], K, amn, B[l], N if bmn else K, bmn, M, N, K, C[l], N, 0, ws=ws[l],
                             ws_floats=ws[l].numel(), bn=bn, splits=splits, stream=streams[l])
        for s in streams:
            main.wait_stream(s)

    body()  # warm (plans, tensor maps)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream()
    with torch.cuda.stream(cap):
        with torch.cuda.graph(g, stream=cap):
            body()
    torch.cuda.synchronize()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / reps / TOTAL
    tf = 2.0 * M * N * K / (us * 1e-6) / 1e12
    print(json.dumps({"shape": name, "streams": NL, "us_per_gemm": round(us, 2), "tflops": round(tf, 1)}), flush=True)


if __name__ == "__main__":
    for name in SHAPES:
        for NL in (1, 2, 4):
            run(name, NL)
