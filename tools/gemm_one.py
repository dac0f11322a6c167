"""One GEMM shape through hdp_gemm_f16, a few launches (for ncu captures):
python tools/gemm_one.py M N K a_mn b_mn [iters] [bn] [splits]
e.g. the C4 per-step shapes: K2 256 8192 2048 0 0 3 128 1; K7 256 2048 8192 0 1 3 256 8"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_1912_00286_b200 import hdp

M, N, K, amn, bmn = (int(v) for v in sys.argv[1:6])
iters = int(sys.argv[6]) if len(sys.argv) > 6 else 3
bn = int(sys.argv[7]) if len(sys.argv) > 7 else 0
splits = int(sys.argv[8]) if len(sys.argv) > 8 else 0
A = (torch.randn(K, M, device="cuda") if amn else torch.randn(M, K, device="cuda")).half()
B = (torch.randn(K, N, device="cuda") if bmn else torch.randn(N, K, device="cuda")).half()
C = torch.empty(M, N, device="cuda")
ws = torch.empty(16 * M * N if M * N <= (1 << 24) else 1, device="cuda")
for _ in range(iters):
    hdp.gemm_f16(A, M if amn else K, amn, B, N if bmn else K, bmn, M, N, K, C, N, 0, ws=ws, ws_floats=ws.numel(),
                 bn=bn, splits=splits)
torch.cuda.synchronize()
print("ok", M, N, K, amn, bmn, bn, splits)
