"""Cross-stream timeline of one training step (the overlap evidence nsys would give; nsys is
not in this image): the library's live profiler (hdp_profile: an event pair around every
launch, eager) plus hdp_profile_timeline, which reports each launch's class, stream and
start / end.  Prints, on rank 0, a text Gantt chart (one row per kernel class and stream)
and how much of the exchange / update time overlaps the backward still running on the
caller's stream.  Eager launches are slower than the graphs the bench replays, so the
absolute times are inflated; the ordering and overlap are what this shows.

    python tools/overlap_timeline.py [C2|C3|C4]                          (1 GPU)
    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \\
        tools/overlap_timeline.py C4                                      (2 GPUs)
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_1912_00286_b200 import hdp  # noqa: E402

TAGS = ["input", "K1", "K2", "K3", "head_fwd", "head_bwd", "K6", "K7", "K8", "K9", "K10", "update/exchange",
        "comm", "recur_fwd", "recur_bwd"]
LANES = {0: "caller", 1: "exchange", 2: "head-side"}


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C4"
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    uid = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
        obj = [hdp.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    cfg = synth.CONFIGS[name]
    B = cfg.batch
    desc = hdp.desc_from_config(cfg, B, hdp.MATH_MIXED16)
    tr = hdp.Trainer(desc, synth.init_params(cfg) if rank == 0 else None, lambda0=cfg.lambda0, alpha=cfg.alpha,
                     gamma=cfg.gamma, n_half=cfg.n_half, momentum=cfg.momentum, world=world, rank=rank, uid=uid,
                     device=local)
    x, t = synth.model_batch(cfg, B, synth.DATA_SEED + rank)
    xd = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    td = torch.from_numpy(np.ascontiguousarray(t)).cuda()
    s = torch.cuda.current_stream()

    def step():
        hdp.lstm_forward(tr.ctx, xd, td, B, cfg.seq, 0, None, tr.loss[0:1], s)
        hdp.lstm_backward(tr.ctx, 0, s)
        hdp.grad_average_update(tr.ctx, 0, s)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    lib = hdp.lib()
    lib.hdp_profile(tr.ctx, 1)
    lib.hdp_profile_read(tr.ctx, None, None, 1)
    step()
    rec = hdp.profile_timeline(tr.ctx)
    lib.hdp_profile_read(tr.ctx, None, None, 1)
    lib.hdp_profile(tr.ctx, 0)
    torch.cuda.synchronize()
    tr.close()
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
    if rank != 0:
        return
    # rows: (lane, tag) -> intervals
    rows = {}
    for tag, lane, a, b in rec:
        rows.setdefault((lane, tag), []).append((a, b))
    t_end = max(b for _, _, _, b in rec)
    W = 100
    lines = [f"{name} dp{world}: one step, eager (per-launch events), {len(rec)} launches, {t_end:.2f} ms"]
    for (lane, tag), iv in sorted(rows.items()):
        bar = [" "] * W
        for a, b in iv:
            for k in range(int(a / t_end * (W - 1)), int(b / t_end * (W - 1)) + 1):
                bar[k] = "#"
        lab = f"{LANES.get(lane, f'layer-{lane - 3}'):9s} {TAGS[tag] if tag < len(TAGS) else tag:16s}"
        lines.append(f"{lab} |{''.join(bar)}| {sum(b - a for a, b in iv):8.3f} ms")
    # overlap of the exchange lane with the backward on the caller's lane
    bwd_tags = {5, 6, 7, 8, 9, 10, 14}
    busy = sorted((a, b) for tag, lane, a, b in rec if lane == 0 and tag in bwd_tags)
    xch = [(a, b) for tag, lane, a, b in rec if lane == 1 and tag in (11, 12)]
    bwd_end = max((b for _, b in busy), default=0.0)
    tot = sum(b - a for a, b in xch)
    before = sum(max(0.0, min(b, bwd_end) - a) for a, b in xch)
    lines.append(f"exchange / update launches: {len(xch)}, {tot:.3f} ms; {before:.3f} ms of it "
                 f"({100 * before / tot if tot else 0:.0f} %) runs before the backward's last launch ends "
                 f"(+{bwd_end:.3f} ms)")
    txt = "\n".join(lines)
    print(txt)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", f"overlap_{name}_n{world}.txt"), "w") as f:
        f.write(txt + "\n")
    with open(os.path.join(ROOT, "gpurun_out", f"overlap_{name}_n{world}.json"), "w") as f:
        json.dump([{"class": TAGS[t] if t < len(TAGS) else t, "lane": LANES.get(l, f"layer-{l - 3}"), "t0_ms": a,
                    "t1_ms": b} for t, l, a, b in rec], f)


if __name__ == "__main__":
    main()
