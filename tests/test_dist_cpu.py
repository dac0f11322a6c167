"""World-size-2 multi-process tests of the host-side logic on CPU (gloo).

* every rank computes the same device layout / bucket sharding for world = 2
  (host-only libhdp contexts, device = -1) and the shards partition each
  bucket;
* the NCCL unique id produced by rank 0 reaches every rank intact through
  torch.distributed (the path bench.py uses);
* the owner-sharded exchange protocol of hdp_grad_average_update (all-to-all
  of fp16 gradient shards, rank-ordered fp32 sum + update at the owner,
  allgather of the fp16 weights, reading Q7) gives weights
  bit-identical on all ranks and bit-identical to a single owner summing all
  contributions -- emulated with the oracle's float32 K11 sequence over gloo.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import synth
        from oracle import lstm as olstm
        from oracle import optim as ooptim
        from paper_1912_00286_b200 import hdp

        res = {}
        # ---- layout agreement
        ctx = hdp.init(world, rank, None, -1)
        cfg = synth.CONFIGS["C2"]
        sizes = hdp.configure(ctx, hdp.desc_from_config(cfg, 16))
        blocks = hdp.param_blocks(ctx)
        allb = [None] * world
        dist.all_gather_object(allb, (sizes.n_params_padded, blocks))
        res["layout_equal"] = all(a == allb[0] for a in allb)
        buckets = {}
        for b in blocks:
            buckets.setdefault(b["bucket"], []).append(b)
        res["shards_ok"] = sizes.n_params_padded % (64 * world) == 0
        hdp.set_lr_schedule(ctx, cfg.lambda0)
        res["lr"] = hdp.lr(ctx, 0)
        hdp.destroy(ctx)
        # ---- uid shipping
        obj = [hdp.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        allu = [None] * world
        dist.all_gather_object(allu, obj[0])
        res["uid_ok"] = len(obj[0]) == 128 and all(u == allu[0] for u in allu)
        # ---- owner-sharded exchange protocol on real oracle gradients (C1, mixed)
        c1 = synth.CONFIGS["C1"]
        params = synth.init_params(c1).astype(np.float64)
        x, t = synth.model_batch(c1, 8, synth.DATA_SEED)
        b = 8 // world
        P = olstm.unpack(c1, params)
        L, _, cache = olstm.forward(c1, P, x[rank * b:(rank + 1) * b], t[rank * b:(rank + 1) * b], c1.alpha, "mixed")
        g = olstm.pack(c1, olstm.backward(c1, P, cache, c1.alpha, "mixed")).astype(np.float16)
        n = g.size
        pad = (-n) % (8 * world)
        g = np.concatenate([g, np.zeros(pad, np.float16)])
        W = np.concatenate([params.astype(np.float32), np.zeros(pad, np.float32)])
        H = np.zeros_like(W)
        shard = g.size // world
        inv, lam, m = ooptim.scalars_f32(world, c1.alpha, 5e-3, 0.9)
        # all-to-all emulated with all_gather: owner `rank` takes shard `rank` of every rank, rank-ordered
        gathered = [torch.zeros(g.size, dtype=torch.float16) for _ in range(world)]
        dist.all_gather(gathered, torch.from_numpy(g))
        mine = [gr.numpy()[rank * shard:(rank + 1) * shard] for gr in gathered]
        sl = slice(rank * shard, (rank + 1) * shard)
        Wn, Hn, w16, nf = ooptim.fused_avg_update_f32(mine, W[sl], H[sl], inv, lam, m)
        full = [torch.zeros(shard, dtype=torch.float16) for _ in range(world)]
        dist.all_gather(full, torch.from_numpy(w16))
        w_all = torch.cat(full).numpy()
        # single owner over the full vector, same contributions
        Wr, Hr, w16r, _ = ooptim.fused_avg_update_f32([gr.numpy() for gr in gathered], W, H, inv, lam, m)
        res["bit_identical_to_single_owner"] = bool(np.array_equal(w_all.view(np.uint16), w16r.view(np.uint16)))
        allw = [None] * world
        dist.all_gather_object(allw, w_all.tobytes())
        res["ranks_identical"] = all(a == allw[0] for a in allw)
        res["nonfinite"] = nf
        q.put((rank, res))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, {"error": traceback.format_exc() + repr(e)}))
    finally:
        dist.destroy_process_group()


def test_world2_gloo_host_logic():
    lib = os.path.join(ROOT, "paper_1912_00286_b200", "libhdp.so")
    if not os.path.exists(lib):
        import __graft_entry__
        __graft_entry__.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for r, res in out.items():
        assert "error" not in res, res.get("error")
        assert res["layout_equal"] and res["shards_ok"] and res["uid_ok"], res
        assert res["bit_identical_to_single_owner"] and res["ranks_identical"], res
        assert res["nonfinite"] == 0
        assert res["lr"] == pytest.approx(4e-4 / 1.02, rel=1e-15)
