"""GPU unit tests of the hand-written sm_100a kernels, called through the
C-ABI: the tcgen05 gate-contraction GEMM in every operand layout the LSTM
step uses (vs a float64 matmul of the same fp16 operands) and the fused
average + update kernel K11 (bit-exact vs the oracle's float32 emulation)."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from oracle import optim as ooptim  # noqa: E402


@pytest.fixture(scope="module")
def hdp():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1912_00286_b200 import hdp as h
    return h


def _store(X, mn_major, pad=8):
    """Store logical X [rows][K] either K-major ([rows][K]) or MN-major ([K][rows])
    with a padded leading dimension; returns (tensor, ld)."""
    R, K = X.shape
    if not mn_major:
        ld = (K + 7) // 8 * 8 + pad
        buf = torch.zeros(R, ld, dtype=X.dtype, device=X.device)
        buf[:, :K] = X
    else:
        ld = (R + 7) // 8 * 8 + pad
        buf = torch.zeros(K, ld, dtype=X.dtype, device=X.device)
        buf[:, :R] = X.T
    return buf, ld


SHAPES = [
    (128, 64, 64),      # one tile
    (200, 130, 100),    # ragged M, N, K tails
    (1, 8, 8),          # degenerate
    (128, 832, 208),    # recurrent K2 at C2 (B x 4h x h)
    (128, 208, 832),    # recurrent backward K7 at C2
    (2048, 832, 16),    # input projection K1 (K = padded I = 16)
    (832, 208, 4096),   # weight gradient K8 (split-K)
    (640, 512, 384),
]


@pytest.mark.parametrize("a_mn", [0, 1])
@pytest.mark.parametrize("b_mn", [0, 1])
@pytest.mark.parametrize("shape", SHAPES)
def test_gemm_layouts(hdp, a_mn, b_mn, shape):
    M, N, K = shape
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N * 3 + K + a_mn * 2 + b_mn)
    A = torch.randn(M, K, generator=g, device="cuda").half()
    B = torch.randn(N, K, generator=g, device="cuda").half()
    ref = (A.double() @ B.double().T)
    As, lda = _store(A, a_mn)
    Bs, ldb = _store(B, b_mn)
    ws = torch.empty(16 * M * N, dtype=torch.float32, device="cuda")
    C = torch.full((M, N), float("nan"), dtype=torch.float32, device="cuda")
    hdp.gemm_f16(As, lda, a_mn, Bs, ldb, b_mn, M, N, K, C, N, 0, ws=ws, ws_floats=ws.numel())
    torch.cuda.synchronize()
    err = (C.double() - ref).abs().max().item() / max(ref.abs().max().item(), 1e-30)
    assert err < 1e-5, err


@pytest.mark.parametrize("bn", [64, 128, 256])
@pytest.mark.parametrize("splits", [1, 3])
def test_gemm_tiles_and_splits(hdp, bn, splits):
    M, N, K = 300, 520, 700
    g = torch.Generator(device="cuda").manual_seed(bn + splits)
    A = torch.randn(M, K, generator=g, device="cuda").half()
    B = torch.randn(N, K, generator=g, device="cuda").half()
    ref = A.double() @ B.double().T
    ws = torch.empty(splits * M * N, dtype=torch.float32, device="cuda")
    for a_mn in (0, 1):
        for b_mn in (0, 1):
            As, lda = _store(A, a_mn)
            Bs, ldb = _store(B, b_mn)
            C = torch.zeros(M, N, dtype=torch.float32, device="cuda")
            hdp.gemm_f16(As, lda, a_mn, Bs, ldb, b_mn, M, N, K, C, N, 0, ws=ws, ws_floats=ws.numel(), bn=bn,
                         splits=splits)
            torch.cuda.synchronize()
            err = (C.double() - ref).abs().max().item() / ref.abs().max().item()
            assert err < 1e-5, (a_mn, b_mn, err)


def test_gemm_epilogues(hdp):
    M, N, K = 256, 192, 96
    g = torch.Generator(device="cuda").manual_seed(11)
    A = torch.randn(M, K, generator=g, device="cuda").half()
    B = torch.randn(N, K, generator=g, device="cuda").half()
    bias_n = torch.randn(N, generator=g, device="cuda")
    bias_m = torch.randn(M, generator=g, device="cuda")
    ref = (A.float() @ B.float().T)
    # bias on n + ReLU, fp16 output (RNE)
    C16 = torch.zeros(M, N, dtype=torch.float16, device="cuda")
    hdp.gemm_f16(A, K, 0, B, K, 0, M, N, K, C16, N, 2, bias=bias_n, relu=1)
    # transposed fp32 store with bias on m
    CT = torch.zeros(N, M, dtype=torch.float32, device="cuda")
    hdp.gemm_f16(A, K, 0, B, K, 0, M, N, K, CT, M, 1, bias=bias_m, bias_on_m=1)
    # accumulate into an existing fp32 output
    C = torch.ones(M, N, dtype=torch.float32, device="cuda")
    hdp.gemm_f16(A, K, 0, B, K, 0, M, N, K, C, N, 0, accumulate=1)
    torch.cuda.synchronize()
    r16 = torch.relu(ref + bias_n).half()
    assert (C16.float() - r16.float()).abs().max().item() <= 1e-2 * r16.float().abs().max().item()
    assert torch.allclose(CT, (ref + bias_m[:, None]).T, rtol=1e-4, atol=1e-4)
    assert torch.allclose(C, ref + 1.0, rtol=1e-4, atol=1e-4)


@pytest.mark.parametrize("a_mn", [0, 1])
@pytest.mark.parametrize("b_mn", [0, 1])
def test_gemm_f32_simt(hdp, a_mn, b_mn):
    M, N, K = 70, 45, 33
    g = torch.Generator(device="cuda").manual_seed(5)
    A = torch.randn(M, K, generator=g, device="cuda", dtype=torch.float64).float()
    B = torch.randn(N, K, generator=g, device="cuda", dtype=torch.float64).float()
    As, lda = _store(A, a_mn)
    Bs, ldb = _store(B, b_mn)
    C = torch.zeros(M, N, dtype=torch.float32, device="cuda")
    hdp.gemm_f32(As, lda, a_mn, Bs, ldb, b_mn, M, N, K, C, N, 0)
    torch.cuda.synchronize()
    ref = A.double() @ B.double().T
    assert (C.double() - ref).abs().max().item() <= 1e-6 * ref.abs().max().item()


# ------------------------------------------------------------------ K11

@pytest.mark.parametrize("nsrc", [1, 2, 4, 8])
@pytest.mark.parametrize("count", [8, 1000, (1 << 20) + 64])
@pytest.mark.parametrize("wire_f32", [False, True])
def test_k11_sgdm_bit_exact(hdp, nsrc, count, wire_f32):
    import synth
    grads, W, H = synth.update_sweep_inputs(count, nsrc, seed=count + nsrc, wire_fp32=wire_f32)
    lam, m, alpha = 3.7037037e-4, 0.9, 10.0
    inv, lam32, m32 = ooptim.scalars_f32(nsrc, alpha, lam, m)
    Wr, Hr, w16r, nfr = ooptim.fused_avg_update_f32(grads, W, H, inv, lam32, m32)
    g_dev = torch.from_numpy(np.concatenate(grads)).cuda()
    W_dev = torch.from_numpy(W.copy()).cuda()
    H_dev = torch.from_numpy(H.copy()).cuda()
    w16 = torch.zeros(count, dtype=torch.float16, device="cuda")
    nf = torch.zeros(1, dtype=torch.int32, device="cuda")
    hdp.fused_avg_update(g_dev, count, nsrc, wire_f32, count, W_dev, H_dev, None, w16, None, float(inv),
                         float(lam32), float(m32), hdp.OPT_SGDM, None, nf)
    torch.cuda.synchronize()
    assert np.array_equal(W_dev.cpu().numpy().view(np.uint32), Wr.view(np.uint32))
    assert np.array_equal(H_dev.cpu().numpy().view(np.uint32), Hr.view(np.uint32))
    assert np.array_equal(w16.cpu().numpy().view(np.uint16), w16r.view(np.uint16))
    assert nf.item() == nfr == 0


def test_k11_adam_bit_exact(hdp):
    import synth
    count, nsrc = 4096 + 8, 3
    grads, W, _ = synth.update_sweep_inputs(count, nsrc, seed=77)
    rng = np.random.default_rng(1)
    m1 = rng.normal(0, 1e-3, count).astype(np.float32)
    v = np.abs(rng.normal(0, 1e-4, count)).astype(np.float32)
    k = 5
    c = ooptim.adam_consts_f32(1e-3, k)
    inv = np.float32(1.0 / (nsrc * 10.0))
    Wr, m1r, vr, w16r, _ = ooptim.fused_avg_adam_f32(grads, W, m1, v, inv, c)
    g_dev = torch.from_numpy(np.concatenate(grads)).cuda()
    W_dev, m_dev, v_dev = (torch.from_numpy(a.copy()).cuda() for a in (W, m1, v))
    w16 = torch.zeros(count, dtype=torch.float16, device="cuda")
    hdp.fused_avg_update(g_dev, count, nsrc, False, count, W_dev, m_dev, v_dev, w16, None, float(inv),
                         float(c["lam"]), 0.0, hdp.OPT_ADAM, (0.9, 0.999, 1e-8, k), None)
    torch.cuda.synchronize()
    assert np.array_equal(W_dev.cpu().numpy().view(np.uint32), Wr.view(np.uint32))
    assert np.array_equal(m_dev.cpu().numpy().view(np.uint32), m1r.view(np.uint32))
    assert np.array_equal(v_dev.cpu().numpy().view(np.uint32), vr.view(np.uint32))
    assert np.array_equal(w16.cpu().numpy().view(np.uint16), w16r.view(np.uint16))


def test_k11_counts_nonfinite(hdp):
    count = 64
    g = np.zeros((2, count), np.float16)
    g[0, 3] = np.inf
    g[1, 7] = np.nan
    g[1, 9] = -np.inf
    W = np.zeros(count, np.float32)
    nf = torch.zeros(1, dtype=torch.int32, device="cuda")
    hdp.fused_avg_update(torch.from_numpy(g.reshape(-1)).cuda(), count, 2, False, count, torch.zeros(count).cuda(),
                         torch.zeros(count).cuda(), None, None, None, 0.05, 0.1, 0.9, hdp.OPT_SGDM, None, nf)
    torch.cuda.synchronize()
    assert nf.item() == 3 == ooptim.fused_avg_update_f32(list(g), W, W, 0.05, 0.1, 0.9)[3]


@pytest.mark.parametrize("mixed", [True, False])
@pytest.mark.parametrize("opt", ["sgdm", "adam"])
def test_k11_l2_bit_exact(hdp, mixed, opt):
    # NEXT-3 L2 term inside K11: g = s*inv + fp32(2 l2) * w_work, w_work = fp16(W) when a
    # w16 copy is written (mixed, R1) else W -- bit-exact vs the float32 emulation
    import synth
    count, nsrc = 8192 + 8, 2
    grads, W, H = synth.update_sweep_inputs(count, nsrc, seed=91)
    W = (W * 20).astype(np.float32)    # weights large enough that the decay term matters
    l2x2 = np.float32(2 * 0.01)
    inv = np.float32(1.0 / (nsrc * 10.0))
    g_dev = torch.from_numpy(np.concatenate(grads)).cuda()
    W_dev = torch.from_numpy(W.copy()).cuda()
    S1 = torch.from_numpy(H.copy()).cuda()
    w16 = torch.zeros(count, dtype=torch.float16, device="cuda") if mixed else None
    w32 = None if mixed else torch.zeros(count, dtype=torch.float32, device="cuda")
    if opt == "sgdm":
        _, lam32, m32 = ooptim.scalars_f32(nsrc, 10.0, 0.05, 0.9)
        Wr, S1r, _, _ = ooptim.fused_avg_update_f32(grads, W, H, inv, lam32, m32, l2x2=l2x2, mixed=mixed)
        hdp.fused_avg_update(g_dev, count, nsrc, False, count, W_dev, S1, None, w16, w32, float(inv), float(lam32),
                             float(m32), hdp.OPT_SGDM, None, None, l2x2=float(l2x2))
    else:
        v = np.abs(np.random.default_rng(2).normal(0, 1e-4, count)).astype(np.float32)
        c = ooptim.adam_consts_f32(1e-3, 3)
        Wr, S1r, vr, _, _ = ooptim.fused_avg_adam_f32(grads, W, H, v, inv, c, l2x2=l2x2, mixed=mixed)
        v_dev = torch.from_numpy(v.copy()).cuda()
        hdp.fused_avg_update(g_dev, count, nsrc, False, count, W_dev, S1, v_dev, w16, w32, float(inv),
                             float(c["lam"]), 0.0, hdp.OPT_ADAM, (0.9, 0.999, 1e-8, 3), None, l2x2=float(l2x2))
    torch.cuda.synchronize()
    assert np.array_equal(W_dev.cpu().numpy().view(np.uint32), Wr.view(np.uint32))
    assert np.array_equal(S1.cpu().numpy().view(np.uint32), S1r.view(np.uint32))
    # the L2 term changed the result (the check bites)
    if opt == "sgdm":
        W0, _, _, _ = ooptim.fused_avg_update_f32(grads, W, H, inv, lam32, m32)
        assert not np.array_equal(W0, Wr)


@pytest.mark.parametrize("cg,bn,amn,bmn", [(2, 128, 0, 0), (2, 256, 0, 1), (2, 256, 1, 1), (2, 128, 1, 0)])
def test_gemm_cta_pair_and_multicast_variants(hdp, cg, bn, amn, bmn):
    # opt-in GEMM variants: CTA pairs (cta_group::2, 256-row tiles) and A
    # multicast across 4-CTA clusters; ragged M and N, against an fp64 reference
    for env, val in (("gemm_cta_group", cg), ("gemm_cluster_n", 4)):
        hdp.set_option(None, env, val)
        M, N, K = 304, 1000, 320   # ragged against 128 / 256-row tiles; 16-B aligned rows
        A = (torch.randn(M, K, device="cuda") * 0.1).half()
        B = (torch.randn(N, K, device="cuda") * 0.1).half()
        Bs, ldb = (B.T.contiguous(), N) if bmn else (B, K)
        As, lda = (A.T.contiguous(), M) if amn else (A, K)
        C = torch.empty(M, N, device="cuda")
        ws = torch.empty(16 * M * N, device="cuda")
        hdp.gemm_f16(As, lda, amn, Bs, ldb, bmn, M, N, K, C, N, 0, ws=ws, ws_floats=ws.numel(), bn=bn, splits=2)
        torch.cuda.synchronize()
        ref = A.double() @ B.double().T
        hdp.set_option(None, env, hdp.KERNEL_OPTION_DEFAULTS[env])
        assert (C.double() - ref).abs().max().item() <= 1e-5 * ref.abs().max().item(), env


def _dev_f16(ptr, n):
    """host copy of n fp16 values of library-owned device memory (CUDA array interface)"""
    class _CAI:
        __cuda_array_interface__ = {"shape": (n,), "typestr": "<f2", "data": (ptr, False), "version": 3}
    return torch.as_tensor(_CAI(), device="cuda").cpu().numpy()


def test_recurrent_dropout_masks_bit_exact(hdp):
    # the CUDA mask hash (csrc/dropout.cuh) against the oracle's (oracle/dropout.py), bit for
    # bit: after one forward, h~_t = fp16(fp32(h_t) * fp32(1/keep)) on kept units, 0 elsewhere
    import synth
    from oracle import dropout as odrop
    cfg = synth.CONFIGS["C1"].with_(n_layers=2)
    B, keep, seed = 4, 0.7, 4321
    desc = hdp.desc_from_config(cfg, B, hdp.MATH_MIXED16, sim_workers=2)
    tr = hdp.Trainer(desc, synth.init_params(cfg), lambda0=cfg.lambda0)
    try:
        hdp.set_recurrent_dropout(tr.ctx, keep, seed)
        x, t = synth.model_batch(cfg, 2 * B, synth.DATA_SEED)
        T, hp, L = cfg.seq, 32, cfg.n_layers
        sc = np.float32(odrop.scale(keep))
        for slot in (0, 1):
            xs = torch.from_numpy(np.ascontiguousarray(x[slot * B:(slot + 1) * B])).cuda()
            ts = torch.from_numpy(np.ascontiguousarray(t[slot * B:(slot + 1) * B])).cuda()
            hdp.lstm_forward(tr.ctx, xs, ts, B, T, slot, None, tr.loss[slot:slot + 1])
            torch.cuda.synchronize()
            h = _dev_f16(hdp.debug_buffer(tr.ctx, slot, "Hs"), L * (T + 1) * B * hp).reshape(L, T + 1, B, hp)
            # Hst: per layer (T_max + 1) * B_max rows; here T = T_max and B = B_max
            h_t = _dev_f16(hdp.debug_buffer(tr.ctx, slot, "Hst"), L * (T + 1) * B * hp).reshape(L, T + 1, B, hp)
            for l in range(L):
                m = odrop.mask(seed, 0, l, np.arange(slot * B, (slot + 1) * B), cfg.hidden, keep)  # [B][h]
                assert 0 < m.mean() < 1
                exp = np.where(m[None] > 0, (h[l, 1:, :, :cfg.hidden].astype(np.float32) * sc).astype(np.float16),
                               np.float16(0))
                got = h_t[l, 1:, :, :cfg.hidden]
                assert np.array_equal(got.view(np.uint16), exp.view(np.uint16)), (slot, l)
                assert not np.any(h_t[l, 0])                     # h~_{-1} = 0
    finally:
        tr.close()
