"""Pins for oracle.schedule and oracle.optim
(PAPER.md:94-103): closed forms, SPEC worked examples, invariants."""
import numpy as np
import pytest

from oracle import optim, schedule


def test_lr_golden(golden):
    for lam0, N, n, gamma, e, expected in golden("lr_schedule.txt"):
        got = schedule.rate_for_epoch(float(lam0), int(N), float(n), float(gamma), int(e))
        assert got == pytest.approx(float(expected), rel=1e-15, abs=0), (lam0, N, n, gamma, e)


def test_halving_at_n():
    # PAPER.md:119 "equal to the number of workers at which it is halved"
    for lam0 in (1e-4, 4e-4, 1e-3):
        for n in (2, 8, 50, 100):
            assert schedule.base_rate(lam0, n, n, max_eff=1e9) == pytest.approx(lam0 / 2, rel=1e-15)


def test_clip_invariant_and_monotone():
    # base_rate * N <= 0.1; strictly decreasing in N and epoch
    for lam0 in (4e-4, 1e-3, 0.02, 0.05, 0.5):
        prev = None
        for N in range(1, 1025):
            r = schedule.base_rate(lam0, N, 100.0)
            assert r * N <= 0.1 * (1 + 1e-15)
            if prev is not None:
                assert r < prev
            prev = r
        rates = [schedule.rate_for_epoch(lam0, 8, 100.0, 0.8, e) for e in range(10)]
        assert all(a > b for a, b in zip(rates, rates[1:]))
    # gamma = 1 => constant
    assert len({schedule.rate_for_epoch(4e-4, 4, 100.0, 1.0, e) for e in range(5)}) == 1


def test_sgdm_golden(golden):
    W0 = np.array([0.5])
    W, H = W0.copy(), np.zeros(1)
    for k, Hk, dWk in golden("sgdm_example.txt"):
        W, H = optim.sgdm(W, H, np.ones(1), lam=0.1, m=0.9)
        assert H[0] == pytest.approx(float(Hk), rel=1e-6)
        assert (W - W0)[0] == pytest.approx(float(dWk), rel=1e-6)


def test_sgdm_special_cases():
    rng = np.random.default_rng(0)
    W = rng.standard_normal(100).astype(np.float32).astype(np.float64)
    H = rng.standard_normal(100).astype(np.float32).astype(np.float64)
    g = rng.standard_normal(100)
    # m = 0 -> plain SGD
    W1, H1 = optim.sgdm(W, H, g, lam=0.01, m=0.0)
    assert np.array_equal(H1, optim.r32(-0.01 * g))
    assert np.array_equal(W1, optim.r32(W + H1))
    # lambda = 0 -> W unchanged apart from the momentum term, H = m H
    W2, H2 = optim.sgdm(W, np.zeros(100), g, lam=0.0, m=0.9)
    assert np.array_equal(W2, W) and np.all(H2 == 0)


def test_average_divides_by_N_alpha():
    gs = [np.full(4, 10.0), np.full(4, 30.0)]
    assert np.allclose(optim.average(gs, 2, 10.0), 2.0)
    # SPEC.md:193 descale example g = [10, -20], alpha = 10 -> [1, -2]
    assert np.array_equal(optim.average([np.array([10.0, -20.0])], 1, 10.0), [1.0, -2.0])


def test_fused_f32_emulation_vs_fp64():
    rng = np.random.default_rng(3)
    n, N, alpha = 10000, 4, 10.0
    gs = [rng.normal(0, 0.05, n).astype(np.float16) for _ in range(N)]
    W = rng.uniform(-0.1, 0.1, n).astype(np.float32)
    H = rng.normal(0, 1e-3, n).astype(np.float32)
    lam, m = 3.7e-4, 0.9
    inv, lam32, m32 = optim.scalars_f32(N, alpha, lam, m)
    Wn, Hn, w16, nf = optim.fused_avg_update_f32(gs, W, H, inv, lam32, m32)
    avg = optim.average([g.astype(np.float64) for g in gs], N, alpha)
    Hr = 0.9 * H.astype(np.float64) - lam * avg
    Wr = W.astype(np.float64) + Hr
    assert nf == 0
    assert np.max(np.abs(Hn - Hr)) <= 1e-6 * np.max(np.abs(Hr))
    assert np.max(np.abs(Wn - Wr)) <= 1e-6 * np.max(np.abs(Wr))
    assert np.array_equal(w16, Wn.astype(np.float16))


def test_fused_f32_hand_example():
    # two ranks, alpha = 10: g = (20 + 10) / 20 = 1.5; H = 0.9*0 - 0.1*1.5 = -0.15; W = 1 - 0.15
    gs = [np.array([20.0], np.float16), np.array([10.0], np.float16)]
    inv, lam, m = optim.scalars_f32(2, 10.0, 0.1, 0.9)
    Wn, Hn, w16, nf = optim.fused_avg_update_f32(gs, np.array([1.0], np.float32), np.zeros(1, np.float32), inv, lam, m)
    assert Hn[0] == np.float32(-0.15) or abs(Hn[0] + 0.15) < 1e-7
    assert abs(Wn[0] - 0.85) < 1e-7
    # a non-finite contribution is counted
    gs.append(np.array([np.inf], np.float16))
    assert optim.fused_avg_update_f32(gs, Wn, Hn, inv, lam, m)[3] == 1


def test_adam_first_step_closed_form():
    # with bias correction, step 1 has mhat = g, vhat = g^2:
    # W1 = W0 - lambda * g / (|g| + eps)   (Kingma & Ba, reading Q15)
    rng = np.random.default_rng(5)
    g = rng.standard_normal(50)
    W0 = np.zeros(50)
    W1, m1, v = optim.adam(W0, np.zeros(50), np.zeros(50), g, lam=1e-3, k=1)
    ref = -1e-3 * g / (np.abs(g) + 1e-8)
    assert np.allclose(W1, ref, rtol=1e-6, atol=0)


def test_adam_constant_gradient_closed_form():
    # a constant gradient g makes the bias-corrected moments exact at every step:
    # m_k = (1 - b1^k) g and v_k = (1 - b2^k) g^2 (geometric sums of the recurrences),
    # so mhat = g, vhat = g^2 and W_k = W_0 - k * lambda * g / (|g| + eps) for k = 1..5.
    # A wrong decay (e.g. (1 - b1) * m instead of b1 * m) breaks this from k = 2 on.
    rng = np.random.default_rng(7)
    g = rng.choice([-1.0, 1.0], 64) * rng.uniform(0.5, 2.0, 64)
    W, m1, v = np.zeros(64), np.zeros(64), np.zeros(64)
    lam, eps = 1e-3, 1e-8
    for k in range(1, 6):
        W, m1, v = optim.adam(W, m1, v, g, lam=lam, k=k, eps=eps)
        assert np.allclose(m1, (1 - 0.9 ** k) * g, rtol=1e-6, atol=0), k
        assert np.allclose(v, (1 - 0.999 ** k) * g * g, rtol=1e-6, atol=0), k
        assert np.allclose(W, -k * lam * g / (np.abs(g) + eps), rtol=1e-6, atol=0), k


def test_adam_impulse_closed_form():
    # g_1 = g, then g_k = 0: m_k = b1^(k-1) (1 - b1) g, v_k = b2^(k-1) (1 - b2) g^2, so
    #   mhat_k = b1^(k-1) (1 - b1) / (1 - b1^k) * g,  sqrt(vhat_k) = sqrt(b2^(k-1) (1 - b2) / (1 - b2^k)) |g|
    # and (eps negligible against |g| = 1) the k-th step moves W by
    #   -lambda sign(g) * [b1^(k-1)(1-b1)/(1-b1^k)] / sqrt(b2^(k-1)(1-b2)/(1-b2^k)).
    # Hand values for b1 = 0.9, b2 = 0.999: k = 2: (0.09/0.19) / sqrt(0.000999/0.001999)
    #   = 0.4736842 / 0.7069298 = 0.6700583; k = 3: (0.081/0.271) / sqrt(0.000998001/0.002997001)
    #   = 0.2988930 / 0.5770614 = 0.5179570
    lam = 1e-2
    W, m1, v = np.zeros(2), np.zeros(2), np.zeros(2)
    g = np.array([1.0, -1.0])
    W1, m1, v = optim.adam(W, m1, v, g, lam=lam, k=1)
    assert np.allclose(W1, -lam * g, rtol=1e-6)
    W2, m1, v = optim.adam(W1, m1, v, np.zeros(2), lam=lam, k=2)
    assert np.allclose(W2 - W1, -lam * 0.6700583 * g, rtol=2e-6)
    W3, m1, v = optim.adam(W2, m1, v, np.zeros(2), lam=lam, k=3)
    assert np.allclose(W3 - W2, -lam * 0.5179570 * g, rtol=2e-6)


def test_adam_f32_emulation_vs_fp64():
    rng = np.random.default_rng(6)
    n, N, alpha = 5000, 2, 10.0
    gs = [rng.normal(0, 0.05, n).astype(np.float16) for _ in range(N)]
    W = rng.uniform(-0.1, 0.1, n).astype(np.float32)
    m1 = rng.normal(0, 1e-3, n).astype(np.float32)
    v = np.abs(rng.normal(0, 1e-4, n)).astype(np.float32)
    lam, k = 1e-3, 3
    c = optim.adam_consts_f32(lam, k)
    Wn, m1n, vn, _, _ = optim.fused_avg_adam_f32(gs, W, m1, v, np.float32(1.0 / (N * alpha)), c)
    avg = optim.average([g.astype(np.float64) for g in gs], N, alpha)
    Wr, m1r, vr = optim.adam(W.astype(np.float64), m1.astype(np.float64), v.astype(np.float64), avg, lam, k)
    assert np.max(np.abs(Wn - Wr)) <= 1e-6 * np.max(np.abs(Wr))
    assert np.max(np.abs(m1n - m1r)) <= 1e-6 * np.max(np.abs(m1r))


def test_fused_f32_l2_term_vs_fp64():
    # the L2 gradient 2*l2*w_work is added after the descale; w_work = fp16(W) in mixed
    # mode (R1) -- float32 emulation within 1e-6 of the float64 update
    rng = np.random.default_rng(5)
    n, N, alpha, l2 = 4096, 2, 10.0, 1e-3
    gs = [rng.normal(0, 0.05, n).astype(np.float16) for _ in range(N)]
    W = rng.uniform(-0.5, 0.5, n).astype(np.float32)
    H = np.zeros(n, np.float32)
    inv, lam, m = optim.scalars_f32(N, alpha, 0.05, 0.9)
    for mixed in (True, False):
        Wn, Hn, _, _ = optim.fused_avg_update_f32(gs, W, H, inv, lam, m, l2x2=np.float32(2 * l2), mixed=mixed)
        wk = W.astype(np.float16).astype(np.float64) if mixed else W.astype(np.float64)
        g = optim.average([x.astype(np.float64) for x in gs], N, alpha) + 2 * l2 * wk
        Hr = -0.05 * g
        assert np.max(np.abs(Hn - Hr)) <= 1e-6 * np.max(np.abs(Hr))
        assert np.max(np.abs(Wn - (W + Hr))) <= 1e-6
    # l2x2 = 0 is the plain update, bit for bit
    a = optim.fused_avg_update_f32(gs, W, H, inv, lam, m)
    b = optim.fused_avg_update_f32(gs, W, H, inv, lam, m, l2x2=0.0)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_dynamic_loss_scale_closed_form_trajectory():
    # halve on a non-finite step (and skip it), double after `interval` finite steps
    seq = [1, 1, 0, 0, 0, 1, 0, 0, 0, 0]
    a, g = 80.0, 0
    alphas, skips = [], []
    for nf in seq:
        a, g, sk = optim.dynamic_loss_scale(a, g, nf, interval=3)
        alphas.append(a)
        skips.append(sk)
    assert alphas == [40.0, 20.0, 20.0, 20.0, 40.0, 20.0, 20.0, 20.0, 40.0, 40.0]
    assert skips == [bool(x) for x in seq]
    # floor at min_alpha
    assert optim.dynamic_loss_scale(1.5, 0, 5, 10)[0] == 1.0
    # alpha * 2^k stays exact in fp32 (10 * 2^k)
    assert np.float32(10.0 * 2 ** 20) / np.float32(2 ** 20) == np.float32(10.0)


def test_skipped_step_leaves_state_unchanged():
    import synth
    from oracle import lstm, step
    cfg = synth.ModelConfig("t", n_layers=1, input_dim=3, hidden=4, seq=4, batch=2)
    rng = np.random.default_rng(0)
    w = rng.uniform(-0.5, 0.5, lstm.count(cfg))
    x = rng.standard_normal((2, 4, 3))
    t = np.where(rng.random((2, 4)) < 0.5, 1, -1).astype(np.int8)
    H = rng.normal(0, 1e-3, w.size)
    # alpha so large that the fp16 gradients overflow (R12)
    out = step.train_step(cfg, w, {"H": H}, x, t, 1, 1e12, 0.1, "mixed", skip_nonfinite=True)
    assert out["nonfinite"] > 0
    assert np.array_equal(out["master"], w) and np.array_equal(out["state"]["H"], H)
    ok = step.train_step(cfg, w, {"H": H}, x, t, 1, 10.0, 0.1, "mixed", skip_nonfinite=True)
    assert ok["nonfinite"] == 0 and not np.array_equal(ok["master"], w)


def test_library_lr_matches_golden(golden):
    """hdp_lr (include/hdp.h) on a host-only context (device -1: no CUDA) reproduces
    every row of the golden schedule, the clip rows included.  N is
    the context's world size (flat model, one worker per rank)."""
    import ctypes
    from paper_1912_00286_b200 import hdp
    L = hdp.lib()
    for lam0, N, n, gamma, e, expected in golden("lr_schedule.txt"):
        h = ctypes.c_void_p()
        assert L.hdp_init(int(N), 0, None, -1, ctypes.byref(h)) == 0
        try:
            desc = hdp.ModelDesc(n_layers=0, sim_workers=1, flat_params=4096)
            hdp.configure(h.value, desc)
            hdp.set_lr_schedule(h.value, float(lam0), float(gamma), float(n))
            assert hdp.lr(h.value, int(e)) == pytest.approx(float(expected), rel=1e-15, abs=0), (lam0, N, n, gamma, e)
            assert hdp.lr(h.value, -1) < 0
        finally:
            hdp.destroy(h.value)


def test_partial_collection_spec_examples():
    # f = 1 -> all N; N = 10, f = 0.9, one straggler -> count 9, sum over
    # the 9; N = 2, f = 0.95 -> ceil(1.9) = 2 (a full barrier)
    assert optim.quorum(1.0, 7) == 7
    assert optim.quorum(0.9, 10) == 9
    assert optim.quorum(0.95, 2) == 2
    assert optim.quorum(0.5, 2) == 1 and optim.quorum(0.75, 4) == 3 and optim.quorum(0.01, 8) == 1
    rng = np.random.default_rng(11)
    gs = [rng.standard_normal(5) for _ in range(10)]
    arrived = [r for r in range(10) if r != 6]             # rank 6 is the straggler
    got = optim.partial_average(gs, arrived, alpha=10.0)
    assert np.allclose(got * 9 * 10.0, sum(gs[r] for r in arrived), rtol=1e-14)
    # every contributor present: identical to the plain average
    assert np.array_equal(optim.partial_average(gs, range(10), 10.0), optim.average(gs, 10, 10.0))
    # duplicated gradients: the partial average equals any single one (the count divides)
    same = [gs[0]] * 4
    assert np.allclose(optim.partial_average(same, [0, 2, 3], 1.0), gs[0], rtol=1e-15)
