"""Multi-GPU parity worker (launched by tests/test_gpu_multi.py through
torchrun, one process per GPU, NCCL).  Each rank trains on its contiguous
shard of the global batch through libhdp; rank 0 runs the oracle with N
simulated workers on the same global batch and compares.  Every step also
checks that the fp16 working weights are bit-identical on all ranks
(SPEC.md:332, :385)."""
import hashlib
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import synth  # noqa: E402
from paper_1912_00286_b200 import hdp  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    cfg_name = os.environ.get("HDP_MP_CFG", "C1")
    mixed = os.environ.get("HDP_MP_MIXED", "1") == "1"
    wire = int(os.environ.get("HDP_MP_WIRE", "0"))
    steps = int(os.environ.get("HDP_MP_STEPS", "3"))
    gb = int(os.environ.get("HDP_MP_GB", "8"))
    seq = int(os.environ.get("HDP_MP_SEQ", "0"))
    l2 = float(os.environ.get("HDP_MP_L2", "0"))           # NEXT-3 L2 (reading Q16)
    dyn = int(os.environ.get("HDP_MP_DYN", "0"))           # NEXT-3 dynamic loss scale interval (Q14b)
    lam0 = float(os.environ.get("HDP_MP_LAMBDA0", "0"))
    keep = float(os.environ.get("HDP_MP_KEEP", "1"))       # NEXT-3 recurrent dropout (Q16b)
    exch = int(os.environ.get("HDP_MP_EXCH", "0"))         # hdp.EXCH_* (0 auto = NVLink kernel for fp16 a2a)
    partial = float(os.environ.get("HDP_MP_PARTIAL", "1"))  # NEXT-2 partial collection fraction
    straggler = int(os.environ.get("HDP_MP_STRAGGLER", "0"))  # ranks that publish readiness 3 ms late
    cfg = synth.CONFIGS[cfg_name]
    if seq:
        cfg = cfg.with_(seq=seq)
    if lam0:
        cfg = cfg.with_(lambda0=lam0, n_half=1e9)
    alpha = float(os.environ.get("HDP_MP_ALPHA", str(cfg.alpha)))
    B = gb // world
    obj = [hdp.nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    desc = hdp.desc_from_config(cfg, B, hdp.MATH_MIXED16 if mixed else hdp.MATH_FP32, wire, hdp.OPT_SGDM, 1,
                                exchange=exch)
    params = synth.init_params(cfg)
    tr = hdp.Trainer(desc, params if rank == 0 else None, lambda0=cfg.lambda0, alpha=alpha, gamma=cfg.gamma,
                     n_half=cfg.n_half, momentum=cfg.momentum, world=world, rank=rank, uid=obj[0], device=local,
                     l2=l2)
    if dyn:
        hdp.set_dynamic_loss_scale(tr.ctx, dyn)
    if keep < 1.0:
        hdp.set_recurrent_dropout(tr.ctx, keep, 99)
    if partial < 1.0 or straggler:
        hdp.set_option(tr.ctx, "partial_fraction", partial)
        hdp.set_option(tr.ctx, "straggler_mask", straggler)
        hdp.set_option(tr.ctx, "straggler_us", 3000)
    a_ref, good = alpha, 0
    from oracle import optim as ooptim
    n = tr.n
    dev = torch.device(f"cuda:{local}")
    stream = torch.cuda.current_stream(dev)
    recs = []
    master_ref = params.astype(np.float64)
    master_prev = params.astype(np.float64)
    state = {"H": np.zeros(n)}
    from oracle import schedule as osched
    from oracle import step as ostep
    from parity import block_errors
    for k in range(steps):
        x, t = synth.model_batch(cfg, gb, synth.DATA_SEED + k)
        if not mixed and cfg.vocab == 0:
            x = x.astype(np.float32)
        xs = torch.from_numpy(np.ascontiguousarray(x[rank * B:(rank + 1) * B])).to(dev)
        ts = torch.from_numpy(np.ascontiguousarray(t[rank * B:(rank + 1) * B])).to(dev)
        hdp.lstm_forward(tr.ctx, xs, ts, B, cfg.seq, 0, None, tr.loss[0:1], stream)
        hdp.lstm_backward(tr.ctx, 0, stream)
        torch.cuda.synchronize()
        g_mine = hdp.read_grads(tr.ctx, 0, n)           # this rank's fp16 gradients (carry alpha)
        g_all = [None] * world
        dist.all_gather_object(g_all, g_mine)
        nf = hdp.grad_average_update(tr.ctx, 0, stream, sync=True)
        torch.cuda.synchronize()
        pmask, pcount = hdp.partial_state(tr.ctx)
        loss = torch.tensor([tr.loss.item()], device=dev)
        dist.all_reduce(loss)
        master = hdp.gather_master(tr.ctx, n)
        w = hdp.read_weights(tr.ctx, n)
        hs = [None] * world
        dist.all_gather_object(hs, hashlib.sha256(w.tobytes()).hexdigest())
        if rank == 0:
            lam = float(np.float32(osched.rate_for_epoch(cfg.lambda0, world, cfg.n_half, cfg.gamma, 0)))
            ref = ostep.train_step(cfg, master_ref, state, x, t, world, a_ref, lam, "mixed" if mixed else "fp32",
                                   l2=l2, skip_nonfinite=bool(dyn),
                                   dropout={"keep": keep, "seed": 99, "step": k} if keep < 1.0 else None,
                                   contributors=[r for r in range(world) if (pmask >> r) & 1] if partial < 1.0
                                   else None)
            skip_ref = False
            if dyn:
                a_ref, good, skip_ref = ooptim.dynamic_loss_scale(a_ref, good, ref["nonfinite"], dyn)
            recs.append({"step": k, "loss_gpu": loss.item() / world, "loss_ref": ref["loss"], "nonfinite": nf,
                         "skip_gpu": bool(dyn and nf > 0), "skip_ref": bool(skip_ref), "alpha_ref": a_ref,
                         "weights_identical": len(set(hs)) == 1,
                         "exchange_kind": hdp.exchange_kind(tr.ctx),
                         "partial_mask": pmask, "partial_count": pcount,
                         "master_sha": hashlib.sha256(master.tobytes()).hexdigest(),
                         "master_err": block_errors(cfg, master.astype(np.float64), ref["master"]),
                         # the step's update: (master_k - master_{k-1}) on both sides (not vacuous at small lambda)
                         "dmaster_err": block_errors(cfg, master.astype(np.float64) - master_prev,
                                                     ref["master"] - master_ref),
                         # every rank's own gradients against the oracle's worker r (R-cond metric)
                         "grad_err": [block_errors(cfg, g_all[r].astype(np.float64), ref["grads"][r],
                                                   ref["abs_terms"][r]) for r in range(world)]})
            master_prev = master.astype(np.float64)
            master_ref, state = ref["master"], ref["state"]
    if dyn and rank == 0 and recs:
        recs[-1]["alpha_gpu"] = hdp.loss_scale_state(tr.ctx)[0]
    tr.close()
    if rank == 0:
        print("MPRESULT " + json.dumps(recs), flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
