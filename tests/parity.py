"""Shared helpers of the GPU parity tests: run the CUDA path through the
C-ABI (paper_1912_00286_b200.hdp) and the oracle on the same seeded inputs
and compare them with the north_star metrics:

  e(P) = max|P_gpu - P_ref| / max|P_ref|   per named parameter block.
"""
from __future__ import annotations

import contextlib

import numpy as np

import synth
from oracle import lstm as olstm
from oracle import schedule as osched
from oracle import step as ostep


def block_errors(cfg, got: np.ndarray, ref: np.ndarray, abs_terms: dict = None) -> dict:
    """e(P) = max|P_gpu - P_ref| / scale(P), scale = max|P_ref|.

    For the bias-type gradients (sums of B*T back-propagated terms) the scale
    is max(max|P_ref|, max_j sum_i |term_ij|) when ``abs_terms`` is given:
    an fp32 sum's rounding error is bounded by gamma_n * sum|terms|, not by
    |sum| (reading R-cond); with balanced labels these sums cancel
    by orders of magnitude at initialisation."""
    g = olstm.unpack(cfg, got)
    r = olstm.unpack(cfg, ref)
    out = {}
    for k in r:
        den = np.max(np.abs(r[k]))
        if abs_terms is not None and k in abs_terms:
            den = max(den, float(np.max(abs_terms[k])))
        num = np.max(np.abs(g[k] - r[k]))
        out[k] = float(num / den) if den > 0 else float(num)
    return out


@contextlib.contextmanager
def kernel_options(**kw):
    """Process-wide kernel switches (hdp_set_option) for the duration of a block,
    restored to the library defaults afterwards."""
    from paper_1912_00286_b200 import hdp
    for k, v in kw.items():
        hdp.set_option(None, k, v)
    try:
        yield
    finally:
        for k in kw:
            hdp.set_option(None, k, hdp.KERNEL_OPTION_DEFAULTS[k])


def _bf16_of(a):
    """float32 values rounded to bfloat16 (RNE), via torch (test-side helper)."""
    import torch
    return torch.from_numpy(np.asarray(a, np.float32)).to(torch.bfloat16).float().numpy()


def _copy_dev(dst, src_ptr: int, nbytes: int):
    """Device-to-device copy from a raw library pointer into a torch tensor."""
    import ctypes
    import torch
    if not hasattr(_copy_dev, "rt"):
        _copy_dev.rt = ctypes.CDLL("libcudart.so.12")   # the runtime torch loaded
    cudart = _copy_dev.rt
    torch.cuda.synchronize()
    rc = cudart.cudaMemcpy(ctypes.c_void_p(dst.data_ptr()), ctypes.c_void_p(src_ptr), ctypes.c_size_t(nbytes), 3)
    assert rc == 0, rc


def run_parity(cfg, global_batch: int, n_workers: int, steps: int, mixed: bool, lambda0=None, alpha=None,
               optimizer="sgdm", seed=synth.DATA_SEED, epochs=None, compare_grads=True, l2=0.0, dropout=None,
               exchange=0, keep_state=False, bf16=False):
    """Returns a list of per-step records with GPU-vs-oracle errors.
    exchange: hdp.EXCH_* (EXCH_P2P at 1 GPU = the NVLink kernel's loopback).
    keep_state: also return the GPU master / weights of every step (bit comparisons).
    bf16: the bf16 math mode (HDP_MATH_BF16, oracle mode "bf16"); inputs rounded to bf16."""
    import torch

    from paper_1912_00286_b200 import hdp

    alpha = cfg.alpha if alpha is None else alpha
    lambda0 = cfg.lambda0 if lambda0 is None else lambda0
    mode = "bf16" if bf16 else "mixed" if mixed else "fp32"
    B = global_batch // n_workers
    desc = hdp.desc_from_config(cfg, B, hdp.MATH_BF16 if bf16 else hdp.MATH_MIXED16 if mixed else hdp.MATH_FP32,
                                hdp.WIRE_FP16_A2A, hdp.OPT_SGDM if optimizer == "sgdm" else hdp.OPT_ADAM,
                                sim_workers=n_workers, exchange=exchange)
    params = synth.init_params(cfg)
    tr = hdp.Trainer(desc, params, lambda0=lambda0, alpha=alpha, gamma=cfg.gamma, n_half=cfg.n_half,
                     momentum=cfg.momentum, l2=l2)
    n = tr.n
    if dropout is not None:                     # (keep, seed): NEXT-3 recurrent dropout
        hdp.set_recurrent_dropout(tr.ctx, dropout[0], dropout[1])
    master = params.astype(np.float64)
    state = {"H": np.zeros(n)} if optimizer == "sgdm" else {"m1": np.zeros(n), "v": np.zeros(n)}
    recs = []
    dev = torch.device("cuda:0")
    try:
        for k in range(steps):
            epoch = (epochs[k] if epochs is not None else 0)
            x, t = synth.model_batch(cfg, global_batch, seed + k)
            if (bf16 or not mixed) and cfg.vocab == 0:
                x = x.astype(np.float32)
            xs, ts = [], []
            for r in range(n_workers):
                sl = slice(r * B, (r + 1) * B)
                xt = torch.from_numpy(np.ascontiguousarray(x[sl]))
                if bf16 and cfg.vocab == 0:
                    xt = xt.to(torch.bfloat16)                       # R0: bf16 inputs
                xs.append(xt.to(dev))
                ts.append(torch.from_numpy(np.ascontiguousarray(t[sl])).to(dev))
            stream = torch.cuda.current_stream()
            for r in range(n_workers):
                hdp.lstm_forward(tr.ctx, xs[r], ts[r], B, cfg.seq, r, None, tr.loss[r:r + 1], stream)
                hdp.lstm_backward(tr.ctx, r, stream)
            torch.cuda.synchronize()
            gpu_grads = [hdp.read_grads(tr.ctx, r, n) for r in range(n_workers)] if compare_grads else None
            gpu_losses = tr.loss.cpu().numpy().astype(np.float64)
            nonfinite = hdp.grad_average_update(tr.ctx, epoch, stream, sync=True)
            torch.cuda.synchronize()
            gpu_master = hdp.gather_master(tr.ctx, n)
            gpu_w = hdp.read_weights(tr.ctx, n)
            lam = osched.rate_for_epoch(lambda0, n_workers, cfg.n_half, cfg.gamma, epoch, cfg.max_eff_lr)
            lam32 = float(np.float32(lam))
            if bf16 and cfg.vocab == 0:
                from oracle.bfloat16 import rbf16
                x = rbf16(x)
            ref = ostep.train_step(cfg, master, state, x, t, n_workers, alpha, lam32, mode, optimizer,
                                   cfg.momentum, adam_k=k + 1, l2=l2,
                                   dropout=None if dropout is None else
                                   {"keep": dropout[0], "seed": dropout[1], "step": k})
            rec = {
                "step": k,
                "loss_gpu": float(np.mean(gpu_losses)),
                "loss_ref": ref["loss"],
                "nonfinite_gpu": nonfinite,
                "nonfinite_ref": ref["nonfinite"],
                "master_err": block_errors(cfg, gpu_master.astype(np.float64), ref["master"]),
                "dmaster_err": block_errors(cfg, gpu_master.astype(np.float64) - params,
                                            ref["master"] - params),
                "w_matches_master": bool(np.array_equal(
                    gpu_w, _bf16_of(gpu_master) if bf16 else
                    gpu_master.astype(np.float16).astype(np.float32) if mixed else gpu_master)),
            }
            if keep_state:
                rec["gpu_master"], rec["gpu_w"] = gpu_master, gpu_w
                if exchange == hdp.EXCH_P2P and n_workers > 1:
                    P = tr.sizes.n_params_padded
                    wc = torch.empty((n_workers - 1) * P, dtype=torch.float16, device=dev)
                    _copy_dev(wc, hdp.debug_buffer(tr.ctx, 0, "Wcopy"), wc.numel() * 2)
                    wbase = torch.empty(P, dtype=torch.float16, device=dev)
                    _copy_dev(wbase, hdp.weights_ptr(tr.ctx), P * 2)
                    rec["copies_equal"] = bool(all(torch.equal(wc[i * P:(i + 1) * P], wbase)
                                                   for i in range(n_workers - 1)))
            if compare_grads:
                rec["grad_err"] = [block_errors(cfg, gpu_grads[r].astype(np.float64), ref["grads"][r],
                                                ref["abs_terms"][r]) for r in range(n_workers)]
                rec["grad_err_plain"] = [block_errors(cfg, gpu_grads[r].astype(np.float64), ref["grads"][r])
                                         for r in range(n_workers)]
            recs.append(rec)
            # both sides continue from their own state (trajectory comparison)
            master, state = ref["master"], ref["state"]
    finally:
        tr.close()
    _log_errors(recs)
    return recs


def _log_errors(recs):
    """Observed errors of a parity run, appended to gpurun_out/parity_errors.jsonl
    with the current test's name (evidence for the tolerances; not an assertion)."""
    import json
    import os
    if not recs:
        return
    mx = lambda d: max(d.values())  # noqa: E731
    row = {"case": os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0], "steps": len(recs),
           "max_grad_err": max((mx(g) for r in recs for g in r.get("grad_err", [])), default=None),
           "max_grad_err_plain": max((mx(g) for r in recs for g in r.get("grad_err_plain", [])), default=None),
           "max_master_err": max(mx(r["master_err"]) for r in recs),
           "max_dmaster_err": max(mx(r["dmaster_err"]) for r in recs),
           "max_loss_diff": max(abs(r["loss_gpu"] - r["loss_ref"]) for r in recs)}
    d = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
    os.makedirs(d, exist_ok=True)
    with open(os.path.join(d, "parity_errors.jsonl"), "a") as f:
        f.write(json.dumps(row) + "\n")
