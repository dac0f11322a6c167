"""The NEXT-2 one-kernel exchange (csrc/p2p_exchange.cu: A9 all-to-all + A10
fused average / update + A11 all-gather, PAPER.md:94-96 steps 4-6) on ONE GPU:
desc.exchange = HDP_EXCH_P2P at world 1 runs the kernel as a loopback whose
peers are the simulated workers' gradient slots and whose all-gather writes
sim_workers weight copies.  Its arithmetic must equal K11's bit for bit (same
rank-ordered fp32 sum, same operation sequence), every copy must equal the
working weights, and the result must match the oracle within the north_star
tolerance.  Plus the boundary's error paths added with it."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import synth  # noqa: E402

from parity import run_parity  # noqa: E402


@pytest.fixture(scope="module")
def hdp():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1912_00286_b200 import hdp as h
    return h


def _max(d):
    return max(d.values())


CASES = [
    # (config, global batch, simulated workers, seq override, optimizer, l2)
    ("C1", 8, 2, None, "sgdm", 0.0),
    ("C1", 16, 4, None, "sgdm", 0.0),
    ("C1", 24, 8, None, "adam", 0.0),
    ("C1", 8, 2, None, "sgdm", 0.05),
    ("C2", 64, 2, 16, "sgdm", 0.0),    # 2-layer wavefront kernels + FC head
    ("C3", 16, 2, 12, "sgdm", 0.0),    # embedding bucket
    ("C3", 32, 8, 8, "sgdm", 0.0),     # C3 at N = 8 workers (SURVEY §8(c) parity plan), 8 weight copies
    ("C2", 64, 4, 12, "sgdm", 0.0),    # 4 workers of B = 16: the wavefront kernels' smallest batch group
]


@pytest.mark.parametrize("name,gb,nw,seq,opt,l2", CASES)
def test_loopback_bit_identical_to_k11_and_oracle(hdp, name, gb, nw, seq, opt, l2):
    cfg = synth.CONFIGS[name].with_(lambda0=0.05, n_half=1e9)   # stress rate: the update is visible
    if seq:
        cfg = cfg.with_(seq=seq)
    kw = dict(steps=3, mixed=True, optimizer=opt, l2=l2, keep_state=True, compare_grads=False)
    k11 = run_parity(cfg, gb, nw, exchange=hdp.EXCH_NCCL, **kw)
    p2p = run_parity(cfg, gb, nw, exchange=hdp.EXCH_P2P, **kw)
    for a, b in zip(k11, p2p):
        assert np.array_equal(a["gpu_master"], b["gpu_master"]), a["step"]   # bit for bit
        assert np.array_equal(a["gpu_w"], b["gpu_w"]), a["step"]
        assert b["copies_equal"], b["step"]                                  # the all-gather stores
        assert b["w_matches_master"]
        assert b["nonfinite_gpu"] == 0
        assert abs(b["loss_gpu"] - b["loss_ref"]) <= 1e-2 * max(1.0, abs(b["loss_ref"]))
    assert _max(p2p[-1]["master_err"]) <= 2e-2, p2p[-1]["master_err"]
    if opt == "sgdm":
        # (Adam normalises every element's step to ~lambda, so near-zero gradients whose
        # fp16 rounding differs from the oracle's move by a full step: no update bound)
        assert _max(p2p[-1]["dmaster_err"]) <= 5e-2, p2p[-1]["dmaster_err"]


@pytest.mark.parametrize("exchange", [1, 2])
def test_dynamic_loss_scale_both_exchanges(hdp, exchange):
    """Dynamic loss scaling (reading Q14b) through K11 and through the loopback kernel:
    the same skip decisions and alpha trajectory as the oracle's rule, and the two
    exchanges agree bit for bit."""
    from oracle import optim as ooptim
    from oracle import schedule as osched
    from oracle import step as ostep
    from parity import block_errors
    cfg = synth.CONFIGS["C1"]
    N, Bg = 2, 8
    B = Bg // N
    alpha0, interval, steps = 10.0 * 2.0 ** 16, 2, 8
    params = synth.init_params(cfg)
    desc = hdp.desc_from_config(cfg, B, hdp.MATH_MIXED16, sim_workers=N, exchange=exchange)
    tr = hdp.Trainer(desc, params, lambda0=0.05, alpha=alpha0, gamma=cfg.gamma, n_half=1e9, momentum=cfg.momentum)
    dev = torch.device("cuda:0")
    master, state = params.astype(np.float64), {"H": np.zeros(tr.n)}
    a_ref, good, skips_ref, skips_gpu = alpha0, 0, [], []
    try:
        hdp.set_dynamic_loss_scale(tr.ctx, interval)
        for k in range(steps):
            x, t = synth.model_batch(cfg, Bg, synth.DATA_SEED + k)
            xs = [torch.from_numpy(np.ascontiguousarray(x[r * B:(r + 1) * B])).to(dev) for r in range(N)]
            ts = [torch.from_numpy(np.ascontiguousarray(t[r * B:(r + 1) * B])).to(dev) for r in range(N)]
            nf = tr.step(xs, ts, B, cfg.seq, epoch=0, stream=torch.cuda.current_stream(), sync=True)
            skips_gpu.append(nf > 0)
            lam = float(np.float32(osched.rate_for_epoch(0.05, N, 1e9, cfg.gamma, 0)))
            ref = ostep.train_step(cfg, master, state, x, t, N, a_ref, lam, "mixed", skip_nonfinite=True)
            a_ref, good, sk = ooptim.dynamic_loss_scale(a_ref, good, ref["nonfinite"], interval)
            skips_ref.append(sk)
            master, state = ref["master"], ref["state"]
        a_gpu, nskip = hdp.loss_scale_state(tr.ctx)
        got = hdp.gather_master(tr.ctx, tr.n)
    finally:
        tr.close()
    assert skips_gpu == skips_ref, (skips_gpu, skips_ref)
    assert any(skips_ref) and not all(skips_ref)
    assert nskip == sum(skips_ref) and a_gpu == np.float32(a_ref)
    assert max(block_errors(cfg, got.astype(np.float64), master).values()) <= 2e-2
    test_dynamic_loss_scale_both_exchanges.results[exchange] = got


test_dynamic_loss_scale_both_exchanges.results = {}


def test_dynamic_loss_scale_c2_fused_head(hdp):
    """Dynamic loss scaling through the C2 path (two-layer wavefronts, the fused FC head
    reading the device alpha for dy, its column sums and dH): the oracle's skip decisions
    and alpha trajectory, and the master weights after the run."""
    from oracle import optim as ooptim
    from oracle import schedule as osched
    from oracle import step as ostep
    from parity import block_errors
    cfg = synth.CONFIGS["C2"].with_(seq=12)
    N, Bg = 2, 32
    B = Bg // N
    alpha0, interval, steps = 10.0 * 2.0 ** 14, 2, 6
    params = synth.init_params(cfg)
    desc = hdp.desc_from_config(cfg, B, hdp.MATH_MIXED16, sim_workers=N)
    tr = hdp.Trainer(desc, params, lambda0=0.05, alpha=alpha0, gamma=cfg.gamma, n_half=1e9, momentum=cfg.momentum)
    dev = torch.device("cuda:0")
    master, state = params.astype(np.float64), {"H": np.zeros(tr.n)}
    a_ref, good, skips_ref, skips_gpu = alpha0, 0, [], []
    try:
        hdp.set_dynamic_loss_scale(tr.ctx, interval)
        for k in range(steps):
            x, t = synth.model_batch(cfg, Bg, synth.DATA_SEED + k)
            xs = [torch.from_numpy(np.ascontiguousarray(x[r * B:(r + 1) * B])).to(dev) for r in range(N)]
            ts = [torch.from_numpy(np.ascontiguousarray(t[r * B:(r + 1) * B])).to(dev) for r in range(N)]
            nf = tr.step(xs, ts, B, cfg.seq, epoch=0, stream=torch.cuda.current_stream(), sync=True)
            skips_gpu.append(nf > 0)
            lam = float(np.float32(osched.rate_for_epoch(0.05, N, 1e9, cfg.gamma, 0)))
            ref = ostep.train_step(cfg, master, state, x, t, N, a_ref, lam, "mixed", skip_nonfinite=True)
            a_ref, good, sk = ooptim.dynamic_loss_scale(a_ref, good, ref["nonfinite"], interval)
            skips_ref.append(sk)
            master, state = ref["master"], ref["state"]
        a_gpu, nskip = hdp.loss_scale_state(tr.ctx)
        got = hdp.gather_master(tr.ctx, tr.n)
    finally:
        tr.close()
    assert skips_gpu == skips_ref, (skips_gpu, skips_ref)
    assert any(skips_ref)
    assert nskip == sum(skips_ref) and a_gpu == np.float32(a_ref)
    assert max(block_errors(cfg, got.astype(np.float64), master).values()) <= 2e-2


def test_dynamic_loss_scale_exchanges_agree(hdp):
    r = test_dynamic_loss_scale_both_exchanges.results
    if len(r) < 2:
        pytest.skip("needs both parametrisations of test_dynamic_loss_scale_both_exchanges")
    assert np.array_equal(r[1], r[2])


def test_exchange_mode_errors(hdp):
    cfg = synth.CONFIGS["C1"]
    ctx = hdp.init(1, 0, None, 0)
    try:
        with pytest.raises(hdp.HDPError) as e:   # FP32 math has no fp16 wire
            hdp.configure(ctx, hdp.desc_from_config(cfg, 4, hdp.MATH_FP32, sim_workers=2, exchange=hdp.EXCH_P2P))
        assert e.value.code == hdp.HDP_ERR_UNSUPPORTED
        with pytest.raises(hdp.HDPError) as e:   # one worker: nothing to exchange
            hdp.configure(ctx, hdp.desc_from_config(cfg, 4, hdp.MATH_MIXED16, sim_workers=1, exchange=hdp.EXCH_P2P))
        assert e.value.code == hdp.HDP_ERR_UNSUPPORTED
        with pytest.raises(hdp.HDPError) as e:
            hdp.configure(ctx, hdp.desc_from_config(cfg, 4, hdp.MATH_MIXED16, sim_workers=2, exchange=7))
        assert e.value.code == hdp.HDP_ERR_ARG
    finally:
        hdp.destroy(ctx)


def test_adam_with_dynamic_loss_scale_rejected(hdp):
    cfg = synth.CONFIGS["C1"]
    desc = hdp.desc_from_config(cfg, 4, hdp.MATH_MIXED16, hdp.WIRE_FP16_A2A, hdp.OPT_ADAM, sim_workers=2)
    tr = hdp.Trainer(desc, synth.init_params(cfg), lambda0=cfg.lambda0)
    try:
        with pytest.raises(hdp.HDPError) as e:
            hdp.set_dynamic_loss_scale(tr.ctx, 2)
        assert e.value.code == hdp.HDP_ERR_UNSUPPORTED
        hdp.set_dynamic_loss_scale(tr.ctx, 0)      # static alpha stays allowed
    finally:
        tr.close()


@pytest.mark.parametrize("bad", [-1, 20000])
def test_out_of_range_token_reported(hdp, bad):
    """Token ids outside [0, vocab) (hdp.h contract): no out-of-bounds access, the
    next synchronised update reports HDP_ERR_ARG and the context is poisoned."""
    cfg = synth.CONFIGS["C3"].with_(seq=8)
    B = 4
    desc = hdp.desc_from_config(cfg, B, hdp.MATH_MIXED16)
    tr = hdp.Trainer(desc, synth.init_params(cfg), lambda0=cfg.lambda0)
    dev = torch.device("cuda:0")
    try:
        x, t = synth.model_batch(cfg, B, synth.DATA_SEED)
        x = np.array(x, copy=True)
        x[2, 5] = bad
        xs = torch.from_numpy(x).to(dev)
        ts = torch.from_numpy(np.ascontiguousarray(t)).to(dev)
        s = torch.cuda.current_stream()
        hdp.lstm_forward(tr.ctx, xs, ts, B, cfg.seq, 0, None, tr.loss[0:1], s)
        hdp.lstm_backward(tr.ctx, 0, s)
        with pytest.raises(hdp.HDPError) as e:
            hdp.grad_average_update(tr.ctx, 0, s, sync=True)
        assert e.value.code == hdp.HDP_ERR_ARG and "token ids" in str(e.value)
        with pytest.raises(hdp.HDPError) as e:
            hdp.lstm_forward(tr.ctx, xs, ts, B, cfg.seq, 0, None, tr.loss[0:1], s)
        assert e.value.code == hdp.HDP_ERR_STATE
        # reloading the parameters clears the poison; valid tokens train normally
        hdp.load_params(tr.ctx, synth.init_params(cfg))
        x[2, 5] = 7
        xs = torch.from_numpy(x).to(dev)
        hdp.lstm_forward(tr.ctx, xs, ts, B, cfg.seq, 0, None, tr.loss[0:1], s)
        hdp.lstm_backward(tr.ctx, 0, s)
        assert hdp.grad_average_update(tr.ctx, 0, s, sync=True) == 0
    finally:
        tr.close()


@pytest.mark.parametrize("nw,frac,straggler,expect", [(4, 0.75, 0b0100, 0b1011), (2, 0.5, 0b01, 0b10),
                                                      (4, 1.0, 0b0010, 0b1111)])
def test_partial_collection_loopback(hdp, nw, frac, straggler, expect):
    """NEXT-2 partial collection in the loopback: the
    simulated contributor(s) in `straggler` publish readiness 3 ms late, so with quorum
    ceil(f*N) < N the decision is exactly the others; the update averages only them
    (divided by their count), against the oracle's step over the same contributors.
    f = 1 keeps the lock-step (the straggler is waited for)."""
    from oracle import schedule as osched
    from oracle import step as ostep
    from parity import block_errors
    cfg = synth.CONFIGS["C1"].with_(lambda0=0.05, n_half=1e9)
    Bg = 4 * nw
    B = Bg // nw
    params = synth.init_params(cfg)
    desc = hdp.desc_from_config(cfg, B, hdp.MATH_MIXED16, sim_workers=nw, exchange=hdp.EXCH_P2P)
    tr = hdp.Trainer(desc, params, lambda0=cfg.lambda0, alpha=cfg.alpha, gamma=cfg.gamma, n_half=cfg.n_half,
                     momentum=cfg.momentum)
    dev = torch.device("cuda:0")
    master, state = params.astype(np.float64), {"H": np.zeros(tr.n)}
    try:
        hdp.set_option(tr.ctx, "partial_fraction", frac)
        hdp.set_option(tr.ctx, "straggler_mask", straggler)
        hdp.set_option(tr.ctx, "straggler_us", 3000)
        for k in range(3):
            x, t = synth.model_batch(cfg, Bg, synth.DATA_SEED + k)
            xs = [torch.from_numpy(np.ascontiguousarray(x[r * B:(r + 1) * B])).to(dev) for r in range(nw)]
            ts = [torch.from_numpy(np.ascontiguousarray(t[r * B:(r + 1) * B])).to(dev) for r in range(nw)]
            assert tr.step(xs, ts, B, cfg.seq, epoch=0, stream=torch.cuda.current_stream(), sync=True) == 0
            mask, count = hdp.partial_state(tr.ctx)
            assert mask == expect and count == bin(expect).count("1"), (mask, count)
            contributors = [r for r in range(nw) if (mask >> r) & 1]
            lam = float(np.float32(osched.rate_for_epoch(cfg.lambda0, nw, cfg.n_half, cfg.gamma, 0)))
            ref = ostep.train_step(cfg, master, state, x, t, nw, cfg.alpha, lam, "mixed",
                                   contributors=None if frac == 1.0 else contributors)
            got = hdp.gather_master(tr.ctx, tr.n).astype(np.float64)
            assert max(block_errors(cfg, got, ref["master"]).values()) <= 2e-2
            assert max(block_errors(cfg, got - master, ref["master"] - master).values()) <= 5e-2
            master, state = ref["master"], ref["state"]
    finally:
        tr.close()


def test_partial_collection_option_errors(hdp):
    cfg = synth.CONFIGS["C1"]
    desc = hdp.desc_from_config(cfg, 4, hdp.MATH_MIXED16, sim_workers=2, exchange=hdp.EXCH_NCCL)
    tr = hdp.Trainer(desc, synth.init_params(cfg), lambda0=cfg.lambda0)
    try:
        with pytest.raises(hdp.HDPError) as e:      # K11 path: no partial collection
            hdp.set_option(tr.ctx, "partial_fraction", 0.5)
        assert e.value.code == hdp.HDP_ERR_UNSUPPORTED
        hdp.set_option(tr.ctx, "partial_fraction", 1.0)  # lock-step is always fine
        for bad in (0.0, 1.5, -1.0):
            with pytest.raises(hdp.HDPError):
                hdp.set_option(tr.ctx, "partial_fraction", bad)
        with pytest.raises(hdp.HDPError):
            hdp.set_option(tr.ctx, "no_such_option", 1)
    finally:
        tr.close()
