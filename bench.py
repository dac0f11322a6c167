"""Benchmark of the data-parallel mixed-precision LSTM training step
(arXiv 1912.00286) on B200 -- the driver contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2|C3|C4|C5] [--impl hdp|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...            (N > 1)

A step = forward + BPTT + bucketed exchange + fused average/update of one
per-rank mini-batch (all §8(a) rows), through libhdp's C-ABI.  Prints ONE
JSON line on rank 0.  Default workload: C2 (JET-shaped, BASELINE.json
configs[1]): 2-layer LSTM h=200, FC 200 + ReLU, T=128, 128 sequences per
rank, fp16 math with loss scaling, fp32 master weights.

Timing: W warm-up steps; then K steps, each bracketed by CUDA events on the
launching stream with an L2 flush (256 MiB memset, outside the events)
between steps; barrier + synchronize on both sides; max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

# the JSON line must be the only thing on stdout: NCCL's version banner (printed at
# communicator init when NCCL_DEBUG asks for it) would precede it
if os.environ.get("NCCL_DEBUG", "").upper() in ("", "VERSION", "INFO", "TRACE") and not os.environ.get("HDP_KEEP_NCCL_DEBUG"):
    os.environ["NCCL_DEBUG"] = "WARN"

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "LSTM training samples/s at 1/2/4/8 B200; avg+update GB/s vs HBM peak"

# kernel classes of include/hdp.h (HDP_K_*)
KCLASS = ["input", "gemm_x(K1)", "gemm_h(K2)", "cell_fwd(K3)", "head_fwd(K4)", "head_bwd(K5)", "cell_bwd(K6)",
          "gemm_dh(K7)", "gemm_dw(K8)", "gemm_dx(K9)", "embed_bwd(K10)", "update(K11)", "comm(A9/A11)",
          "recur_fwd(K2+K3)", "recur_bwd(K6+K7)"]


def peaks():
    p = {"hbm_gbs": 6456.2, "bf16_tflops": 1660.9, "bf16_tflops_sustained": 1415.3, "src": "fallback"}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            m = json.load(f)
        p.update({k: m[k] for k in ("hbm_gbs", "bf16_tflops", "bf16_tflops_sustained") if k in m})
        p["src"] = "measured"
    except Exception:
        p["src"] = "fallback (B200_PROFILING.md)"
    return p


class Clocks:
    """SM clock + throttle-reason sampling DURING the timed region
    (B200_PROFILING.md clocks line).  NVML is polled every ~2 ms from a
    background thread that starts before the region; only samples taken between
    start() and stop() count, so short regions still get several samples.
    Falls back to nvidia-smi -lms when NVML is unavailable."""

    REASONS = [("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake_slowdown", "nvmlClocksEventReasonHwPowerBrakeSlowdown")]

    def __init__(self, index):
        import threading
        self.samples, self.t0, self.t1, self.h, self.err = [], None, None, None, None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            if vis:
                ids = [x.strip() for x in vis.split(",")]
                if index < len(ids) and ids[index].isdigit():
                    index = int(ids[index])
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.mx = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
        except Exception as e:  # noqa: BLE001
            self.err = f"nvml: {e}"
            return
        self.stop_ev = threading.Event()
        self.th = threading.Thread(target=self._run, daemon=True)
        self.th.start()
        while not self.samples and self.th.is_alive():
            time.sleep(0.001)

    def _run(self):
        nv = self.nv
        get_r = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or nv.nvmlDeviceGetCurrentClocksThrottleReasons
        while not self.stop_ev.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
                r = get_r(self.h)
            except Exception:  # noqa: BLE001
                break
            self.samples.append((time.perf_counter(), float(sm), int(r)))
            time.sleep(0.002)

    def start(self):
        self.t0 = time.perf_counter()

    def stop(self):
        self.t1 = time.perf_counter()
        if self.h is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [self.err or "nvml unavailable"], "samples": 0}
        time.sleep(0.005)  # one more sample past the end
        self.stop_ev.set()
        self.th.join()
        t0 = self.t0 if self.t0 is not None else 0.0
        inside = [x for x in self.samples if t0 <= x[0] <= self.t1 + 0.003]
        if not inside:  # region shorter than one poll: nearest sample after start
            inside = [x for x in self.samples if x[0] >= t0][:1]
        reasons = set()
        for _, _, r in inside:
            for name, const in self.REASONS:
                bit = getattr(self.nv, const, None)
                if bit is not None and (r & bit):
                    reasons.add(name)
        sm = [x[1] for x in inside]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.mx, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvml"}


def committed_traffic(workload, kclass):
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of this kernel
    class, from one committed `ncu --set full` capture (profiles/traffic.json),
    or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f)[workload][kclass]["traffic_bytes_per_launch"]
    except Exception:  # noqa: BLE001
        return None


def algorithmic_work(cfg, B, world, prof=None):
    """Per-launch algorithmic work of each kernel class:
    flops for contractions (unpadded shapes), HBM bytes for the elementwise /
    update kernels.  Returns {class: (kind, per_launch_amount)}.

    With the 2-layer wavefront (one recur_fwd and one recur_bwd launch per step,
    read from the live profile's launch counts) a launch covers both layers'
    recurrences plus the work fused into it: the layer-1 input projection, the
    layer-0 one when no K1 launch remains, the dX1 projection and, when no K8
    launch remains, the A8 weight gradients of both layers."""
    h, T, L = cfg.hidden, cfg.seq, cfg.n_layers
    I0 = cfg.embed_dim if cfg.vocab else cfg.input_dim
    ins = [I0] + [h] * (L - 1)
    w = {}
    rec = 2.0 * B * 4 * h * h * (T - 1)          # one layer's U h_{t-1} (or U^T dA) over t = 1..T-1
    w["gemm_h(K2)"] = ("flop", 2.0 * B * 4 * h * h)
    w["gemm_dh(K7)"] = ("flop", 2.0 * B * 4 * h * h)
    w["gemm_x(K1)"] = ("flop", sum(2.0 * B * T * 4 * h * i for i in ins) / L)
    w["gemm_dw(K8)"] = ("flop", sum(2.0 * 4 * h * (i + h) * B * T for i in ins) / (3 * L))  # dW, dU, db launches
    w["gemm_dx(K9)"] = ("flop", 2.0 * B * T * 4 * h * h)
    w["recur_fwd(K2+K3)"] = ("flop", rec)   # one launch = all T steps of a layer
    w["recur_bwd(K6+K7)"] = ("flop", rec)
    prof = prof or {}
    if L == 2 and prof.get("recur_fwd(K2+K3)", {}).get("launches_per_step") == 1:
        f = 2 * rec + 2.0 * B * T * 4 * h * h                       # R0 + R1 + P (layer-1 projection)
        if "gemm_x(K1)" not in prof:
            f += 2.0 * B * T * 4 * h * I0                             # fused layer-0 projection
        w["recur_fwd(K2+K3)"] = ("flop", f)
    if L == 2 and prof.get("recur_bwd(K6+K7)", {}).get("launches_per_step") == 1:
        f = 2 * rec + 2.0 * B * T * 4 * h * h                       # Q1 + Q0 + X (dX1 = dA1 W1)
        if "gemm_dw(K8)" not in prof:
            f += sum(2.0 * 4 * h * (i + h) * B * T for i in ins)      # W role: dU, dW of both layers
        w["recur_bwd(K6+K7)"] = ("flop", f)
    w["cell_fwd(K3)"] = ("byte", 50.0 * B * h)   # Gx 16 + Gh 16 + c_prev 4 + gates 8 + c 4 + h 2
    w["cell_bwd(K6)"] = ("byte", 40.0 * B * h)   # dHa 4 + dh_rec 4 + gates 8 + c 4 + c_prev 4 + dc 8 + dA 8
    return w


def latency_floor(cfg, kclass):
    """Dependency-chain floor of a recurrence launch: T + 2 steps of
    (tcgen05 MMA chain + one DSMEM hand-off), both measured by the micro-benchmarks in
    profiles/r02_latency_floor.json; the cell epilogue is not in it (a lower bound).
    The MMA part scales with the K-steps for h_p other than the measured 208."""
    try:
        with open(os.path.join(ROOT, "profiles", "r02_latency_floor.json")) as f:
            m = json.load(f)["model"]
    except Exception:  # noqa: BLE001
        return None
    hp = (cfg.hidden + 15) // 16 * 16
    key = "backward step (Q roles)" if kclass.startswith("recur_bwd") else "forward step (R roles)"
    step_ns = m[key]["mma_ns"] * hp / 208.0 + m[key]["hop_ns"]
    steps = cfg.seq + 2
    return {"per_step_ns": round(step_ns, 1), "steps": steps, "floor_us": steps * step_ns / 1e3,
            "model": "(T + 2) x (MMA chain + DSMEM hop), epilogue excluded",
            "source": "profiles/r02_latency_floor.json (tools/micro on B200)"}


def run_hdp(args, rank, world, local_rank):
    import numpy as np
    import torch

    import synth
    from paper_1912_00286_b200 import hdp

    dev = torch.device(f"cuda:{local_rank}")
    torch.cuda.set_device(dev)
    cfg = synth.CONFIGS[args.config]
    B = args.batch or cfg.batch
    uid = None
    if world > 1:
        import torch.distributed as dist
        obj = [hdp.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    desc = hdp.desc_from_config(cfg, B, hdp.MATH_MIXED16, hdp.WIRE_FP16_A2A, hdp.OPT_SGDM, 1)
    params = synth.init_params(cfg) if rank == 0 else None
    tr = hdp.Trainer(desc, params, lambda0=cfg.lambda0, alpha=cfg.alpha, gamma=cfg.gamma, n_half=cfg.n_half,
                     momentum=cfg.momentum, world=world, rank=rank, uid=uid, device=local_rank)
    exchange = hdp.EXCHANGE_KINDS.get(hdp.exchange_kind(tr.ctx), "?")
    x, t = synth.model_batch(cfg, B, synth.DATA_SEED + 1000 * rank)
    xd = torch.from_numpy(np.ascontiguousarray(x)).to(dev)
    td = torch.from_numpy(np.ascontiguousarray(t)).to(dev)
    xh = torch.from_numpy(np.ascontiguousarray(x)).pin_memory()
    th = torch.from_numpy(np.ascontiguousarray(t)).pin_memory()
    loss_h = torch.zeros(1, dtype=torch.float32).pin_memory()
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # > 126 MB L2

    def step(xx, tt, epoch=0):
        hdp.lstm_forward(tr.ctx, xx, tt, B, cfg.seq, 0, None, tr.loss[0:1], stream)
        hdp.lstm_backward(tr.ctx, 0, stream)
        hdp.grad_average_update(tr.ctx, epoch, stream)

    def barrier():
        torch.cuda.synchronize(dev)
        if world > 1:
            import torch.distributed as dist
            dist.barrier()

    def max_over_ranks(v):
        if world == 1:
            return v
        import torch.distributed as dist
        tv = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(tv, op=dist.ReduceOp.MAX)
        return tv.item()

    for _ in range(args.warmup):
        step(xd, td)
    barrier()

    # ---------------- timed region (device-resident inputs)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    clk = Clocks(local_rank)
    k0 = hdp.lib().hdp_kernel_launches(tr.ctx)
    barrier()
    clk.start()
    for k in range(args.steps):
        flush.zero_()
        evs[k][0].record(stream)
        step(xd, td)
        evs[k][1].record(stream)
    barrier()
    clocks = clk.stop()
    launches = hdp.lib().hdp_kernel_launches(tr.ctx) - k0
    step_ms = [a.elapsed_time(b) for a, b in evs]
    ms = max_over_ranks(statistics.mean(step_ms))
    loss_dev = tr.loss.item()

    # ---------------- e2e: host (pinned) buffers through the C-ABI, loss read back every step
    e_evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    barrier()
    for k in range(args.steps):
        flush.zero_()
        e_evs[k][0].record(stream)
        step(xh, th)
        loss_h.copy_(tr.loss[0:1], non_blocking=True)
        e_evs[k][1].record(stream)
    barrier()
    e2e_ms = max_over_ranks(statistics.mean([a.elapsed_time(b) for a, b in e_evs]))

    # ---------------- live per-kernel-class profile (eager, CUDA events around each launch)
    nk = len(KCLASS)
    ms_by = (__import__("ctypes").c_double * nk)()
    n_by = (__import__("ctypes").c_longlong * nk)()
    hdp.lib().hdp_profile(tr.ctx, 1)
    hdp.lib().hdp_profile_read(tr.ctx, ms_by, n_by, 1)
    prof_steps = 2
    for _ in range(prof_steps):
        step(xd, td)
    hdp.lib().hdp_profile_read(tr.ctx, ms_by, n_by, 1)
    hdp.lib().hdp_profile(tr.ctx, 0)
    barrier()
    prof = {KCLASS[i]: {"ms_per_step": ms_by[i] / prof_steps, "launches_per_step": n_by[i] / prof_steps}
            for i in range(nk) if n_by[i]}
    tr.close()

    if rank != 0:
        return None
    pk = peaks()
    work = algorithmic_work(cfg, B, world, prof)
    cand = {k: v for k, v in prof.items() if k in work}
    dom = max(cand, key=lambda k: cand[k]["ms_per_step"])
    kind, per_launch = work[dom]
    avg_launch_ms = cand[dom]["ms_per_step"] / cand[dom]["launches_per_step"]
    if kind == "flop":
        achieved = per_launch / (avg_launch_ms * 1e-3) / 1e12
        peak = pk["bf16_tflops_sustained"]
        roof = {"bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "traffic": None}
    else:
        achieved = per_launch / (avg_launch_ms * 1e-3) / 1e9
        peak = pk["hbm_gbs"]
        roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": None}
    roof["traffic"] = committed_traffic(cfg.name, dom)
    if dom in ("recur_bwd(K6+K7)", "recur_fwd(K2+K3)"):
        lf = latency_floor(cfg, dom)
        if lf:
            roof["latency_floor"] = lf
            roof["latency_floor_frac"] = lf["floor_us"] / (avg_launch_ms * 1e3)
    roof.update({"kernel": dom, "peak_src": pk["src"] + (" sustained" if kind == "flop" else ""),
                 "avg_launch_us": avg_launch_ms * 1e3, "per_launch": per_launch,
                 "per_launch_unit": "flop" if kind == "flop" else "byte",
                 "share_of_step": cand[dom]["ms_per_step"] / sum(v["ms_per_step"] for v in prof.values())})
    samples = B * world
    x_bytes = int(xh.numel() * xh.element_size())
    t_bytes = int(th.numel() * th.element_size())
    out = {
        "metric": METRIC,
        "value": samples / (ms * 1e-3),
        "unit": "samples/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "f16",
        "data": "synthetic (seeded JET-shaped / IMDB-shaped / dense generators, random init)",
        "config": {"workload": cfg.name, "per_rank_batch": B, "global_batch": samples, "seq_len": cfg.seq,
                   "hidden": cfg.hidden, "layers": cfg.n_layers, "fc_hidden": cfg.fc_hidden,
                   "parallelism": f"dp{world}", "math": "fp16 (fp32 accumulate, fp32 master)",
                   "wire": "fp16", "exchange": exchange, "optimizer": "sgd-momentum", "loss_scale": cfg.alpha,
                   "recurrence": ("two-layer wavefront launches (forward, backward)"
                                  if cfg.n_layers == 2 and cfg.hidden <= 256 else
                                  "per-step GEMMs with fused cell epilogues; layer-diagonal forward in chunks of "
                                  f"{hdp.get_option('layer_pipe')} steps"),
                   "l2_cache": "flushed between timed steps (256 MiB memset, outside the events)",
                   "l2_regularisation": 0.0, "recurrent_dropout_keep": 1.0, "loss_scale_mode": "static"},
        "e2e": {"value": samples / (e2e_ms * 1e-3), "unit": "samples/s", "h2d_bytes_per_step": x_bytes + t_bytes,
                "d2h_bytes_per_step": 4},
        "gpu_launches": int(launches),
        "roofline": roof,
        "clocks": clocks,
        "loss_last": loss_dev,
        "profile_ms_per_step": {k: round(v["ms_per_step"], 4) for k, v in prof.items()},
    }
    return out


class _CAI:
    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3}


def device_view(ptr, n, typestr, dev):
    """torch view of library-owned device memory (no copy)."""
    import torch
    return torch.as_tensor(_CAI(ptr, n, typestr), device=dev)


def run_c5(args, rank, world, local_rank):
    """C5: fused fp16 gradient average + weight update sweep (BASELINE.json
    configs[4]) through hdp_grad_average_update on a flat parameter vector:
    per size, exchange (all-to-all) + K11 + allgather, timed per step with
    CUDA events; K11 alone from the live profiler."""
    import ctypes

    import numpy as np
    import torch

    import synth
    from paper_1912_00286_b200 import hdp

    dev = torch.device(f"cuda:{local_rank}")
    torch.cuda.set_device(dev)

    def fresh_uid():  # a NCCL unique id is single-use: one per communicator
        if world == 1:
            return None
        import torch.distributed as dist
        obj = [hdp.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return obj[0]

    sizes_mib = [int(v) for v in args.sizes.split(",")]
    wire = {"fp16": hdp.WIRE_FP16_A2A, "fp16sum": hdp.WIRE_FP16_NCCLSUM, "fp32": hdp.WIRE_FP32}[args.wire]
    gsz = 4 if wire == hdp.WIRE_FP32 else 2
    nsim = 1 if world > 1 else max(1, args.sim)
    stream = torch.cuda.current_stream(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    rows = []
    clk = Clocks(local_rank)
    clk.start()
    for mib in sizes_mib:
        S = (mib << 20) // 2          # fp16 gradient elements
        desc = hdp.ModelDesc(n_layers=0, max_batch=1, max_seq=1, math=hdp.MATH_MIXED16, wire=wire,
                             optimizer=hdp.OPT_SGDM, sim_workers=nsim, flat_params=S)
        ctx = hdp.init(world, rank, fresh_uid(), local_rank)
        sz = hdp.configure(ctx, desc)
        arena = torch.empty(sz.arena_bytes + 256, dtype=torch.uint8, device=dev)
        base = arena.data_ptr() + ((-arena.data_ptr()) % 256)
        hdp.bind(ctx, base, sz.arena_bytes)
        rng = np.random.default_rng(1912 + rank)
        hdp.load_params(ctx, rng.uniform(-0.1, 0.1, S).astype(np.float32) if rank == 0 else None, 0)
        hdp.set_lr_schedule(ctx, 4e-4)
        hdp.set_loss_scale(ctx, 10.0)
        P = sz.n_params_padded
        for sl in range(nsim):
            dst = device_view(hdp.grads_ptr(ctx, sl), P, "<f2" if gsz == 2 else "<f4", dev)
            dst.copy_((torch.randn(P, device=dev) * 0.05).to(dst.dtype))
        for _ in range(args.warmup):
            hdp.grad_average_update(ctx, 0, stream)
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        torch.cuda.synchronize(dev)
        for k in range(args.steps):
            flush.zero_()
            evs[k][0].record(stream)
            hdp.grad_average_update(ctx, 0, stream)
            evs[k][1].record(stream)
        torch.cuda.synchronize(dev)
        ms = statistics.mean(a.elapsed_time(b) for a, b in evs)
        ms_by = (ctypes.c_double * len(KCLASS))()
        n_by = (ctypes.c_longlong * len(KCLASS))()
        hdp.lib().hdp_profile(ctx, 1)
        hdp.lib().hdp_profile_read(ctx, ms_by, n_by, 1)
        for _ in range(3):
            flush.zero_()
            hdp.grad_average_update(ctx, 0, stream)
        hdp.lib().hdp_profile_read(ctx, ms_by, n_by, 1)
        hdp.lib().hdp_profile(ctx, 0)
        kind = hdp.exchange_kind(ctx)
        k11_ms = ms_by[11] / 3.0                       # per step (K11, or the one-kernel exchange)
        k11_launch_ms = ms_by[11] / max(1, n_by[11])
        comm_ms = ms_by[12] / 3.0                      # NCCL collectives (0 on the one-kernel path)
        own = P // world
        nsrc = world if (world > 1 and wire != hdp.WIRE_FP16_NCCLSUM and wire != hdp.WIRE_FP32) else (1 if world > 1 else nsim)
        if kind == 2:
            nsrc = world
        # HBM bytes of the update arithmetic per rank (contributions + W, H read/write + fp16 w)
        k11_bytes = own * (nsrc * gsz + 18)
        # NVLink bytes per rank per direction: the owned shard's contributions from the N-1
        # peers (gradient wire) + the N-1 peers' fp16 weight shards (all-gather / peer stores)
        nvl_bytes = (world - 1) / world * P * (gsz + 2) if world > 1 else 0
        xch_ms = k11_ms if kind == 2 else comm_ms     # the time the NVLink traffic has to fit in
        rows.append({"mib": mib, "elements": P, "step_ms": ms, "exchange": hdp.EXCHANGE_KINDS.get(kind, "?"),
                     "k11_ms": k11_ms, "comm_ms": comm_ms,
                     "k11_gbs": k11_bytes / (k11_ms * 1e-3) / 1e9 if kind != 2 else None,
                     "k11_launch_us": k11_launch_ms * 1e3, "k11_bytes": k11_bytes,
                     "nvlink_bytes_per_direction": nvl_bytes,
                     "busbw_gbs": (nvl_bytes / (xch_ms * 1e-3) / 1e9) if world > 1 and xch_ms > 0 else None,
                     "busbw_step_gbs": (nvl_bytes / (ms * 1e-3) / 1e9) if world > 1 else None})
        hdp.destroy(ctx)
        del arena
        torch.cuda.synchronize(dev)
    clocks = clk.stop()
    if rank != 0:
        return None
    pk = peaks()
    big = rows[-1]
    out = {"metric": METRIC, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": big["step_ms"], "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
           "dtype": "f32 (fp16 wire)" if gsz == 2 else "f32 (fp32 wire)", "data": "synthetic gradients N(0, 0.05^2)",
           "config": {"workload": "C5-avg-update", "sizes_mib": sizes_mib, "wire": args.wire,
                      "contributions": nsim if world == 1 else world, "parallelism": f"dp{world}",
                      "exchange": big["exchange"], "l2_cache": "flushed between timed steps"},
           "sweep": rows, "clocks": clocks, "gpu_launches": None}
    if world == 1:
        # one GPU: the fused average + update is HBM-bound (the metric's "avg+update GB/s vs HBM peak")
        out.update({"value": big["k11_gbs"], "unit": "GB/s",
                    "roofline": {"bound": "hbm", "achieved": big["k11_gbs"], "peak": pk["hbm_gbs"], "unit": "GB/s",
                                 "frac": big["k11_gbs"] / pk["hbm_gbs"], "traffic": None, "kernel": "update(K11)",
                                 "peak_src": pk["src"], "avg_launch_us": big["k11_launch_us"],
                                 "per_launch": big["k11_bytes"], "per_launch_unit": "byte"}})
    else:
        # N GPUs: what binds is NVLink -- bytes per rank per direction over the exchange time,
        # against the measured peer-copy rate (B200_PROFILING.md: 770 GB/s; 900 nominal)
        bw = big["busbw_gbs"]
        out.update({"value": bw, "unit": "GB/s (NVLink per GPU per direction)",
                    "roofline": {"bound": "nvlink", "achieved": bw, "peak": 770.0, "unit": "GB/s",
                                 "frac": bw / 770.0 if bw else None, "traffic": None,
                                 "kernel": "exch_update" if "kernel" in big["exchange"] else "nccl",
                                 "peak_src": "measured peer copy per direction (B200_PROFILING.md), 900 nominal",
                                 "per_launch": big["nvlink_bytes_per_direction"], "per_launch_unit": "byte",
                                 "frac_of_nominal_900": bw / 900.0 if bw else None}})
    return out


def host_cpu():
    """CPU model and the cores this process may run on (for the cpu_baseline lines)."""
    model = "unknown"
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    try:
        cores = len(os.sched_getaffinity(0))
    except Exception:  # noqa: BLE001
        cores = os.cpu_count()
    return model, cores


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        return max([i.get("num_threads", 1) for i in threadpool_info()] + [1])
    except Exception:  # noqa: BLE001
        return os.cpu_count()


def cpu_baseline(args, seconds=15.0, max_steps=4):
    """The oracle as it stands, on the host cores, on a bounded sample."""
    import numpy as np

    import synth
    from oracle import step as ostep
    threads = blas_threads()
    model, cores = host_cpu()
    cfg = synth.CONFIGS[args.config]
    B = args.batch or cfg.batch
    if args.config == "C4":
        B = min(B, 4)
    master = synth.init_params(cfg).astype(np.float64)
    x, t = synth.model_batch(cfg, B, synth.DATA_SEED)
    n, t0 = 0, time.perf_counter()
    state = {"H": np.zeros_like(master)}
    while n < max_steps:
        out = ostep.train_step(cfg, master, state, x, t, 1, cfg.alpha, float(np.float32(cfg.lambda0 / 1.01)),
                               "mixed")
        master, state = out["master"], out["state"]
        n += 1
        if time.perf_counter() - t0 > seconds:
            break
    dt = time.perf_counter() - t0
    return {"value": n * B / dt, "unit": "samples/s", "cores": threads, "kind": "oracle",
            "sample": f"{n} oracle.step.train_step of {cfg.name} ({B} sequences x T={cfg.seq}, mixed mode, N=1) "
                      f"in {dt:.1f} s",
            "cpu": model, "host_cores": cores,
            "threads_note": "cores = BLAS threads of the matrix products; elementwise phases single-threaded"}


def run_reference(args):
    """--impl reference: the oracle (NumPy fp64 with fp16 rounding points) on the host."""
    import numpy as np

    import synth
    from oracle import step as ostep
    cfg = synth.CONFIGS[args.config]
    Bs = {"C1": 8, "C2": 8, "C3": 4, "C4": 1}.get(args.config, 8)   # bounded sample per step
    cfgs = cfg if args.config != "C4" else cfg.with_(seq=16)
    master = synth.init_params(cfgs).astype(np.float64)
    x, t = synth.model_batch(cfgs, Bs, synth.DATA_SEED)
    state = {"H": np.zeros_like(master)}

    def one():
        nonlocal master, state
        out = ostep.train_step(cfgs, master, state, x, t, 1, cfg.alpha, 4e-4, "mixed")
        master, state = out["master"], out["state"]

    for _ in range(args.warmup):
        one()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        one()
    dt = time.perf_counter() - t0
    threads = blas_threads()
    model, cores = host_cpu()
    v = Bs * args.steps / dt
    sample = f"{Bs} sequences of {cfgs.name} (T={cfgs.seq}) per step, oracle.step.train_step, mixed mode"
    return {"impl": "reference", "metric": METRIC, "value": v, "unit": "samples/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": cfg.name, "per_rank_batch": Bs, "seq_len": cfgs.seq,
                                              "parallelism": "host"},
            "cpu_baseline": {"value": v, "unit": "samples/s", "cores": threads, "kind": "oracle", "sample": sample,
                             "cpu": model, "host_cores": cores},
            "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    # the JSON line must be the only thing on stdout: NCCL / torch.distributed banners
    # (e.g. "NCCL version ..." at communicator creation) go to stderr instead
    real_stdout = os.fdopen(os.dup(1), "w")
    sys.stdout.flush()
    os.dup2(2, 1)
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C2", choices=["C1", "C2", "C3", "C4", "C5"])
    ap.add_argument("--sizes", default="1,4,16,64,256,1024", help="C5 sweep sizes in MiB of fp16 gradient")
    ap.add_argument("--wire", default="fp16", choices=["fp16", "fp16sum", "fp32"], help="C5 wire format")
    ap.add_argument("--sim", type=int, default=1, help="C5 at N=1: simulated contributions")
    ap.add_argument("--batch", type=int, default=0, help="per-rank batch (default: the config's)")
    ap.add_argument("--impl", default="hdp", choices=["hdp", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--option", action="append", default=[],
                    help="kernel switch name=value (hdp_set_option; ablations, default = the measured best)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args)), file=real_stdout, flush=True)
        return

    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local_rank}"))
    if args.option:
        from paper_1912_00286_b200 import hdp
        for kv in args.option:
            k, v = kv.split("=")
            hdp.set_option(None, k, float(v))
    out = run_c5(args, rank, world, local_rank) if args.config == "C5" else run_hdp(args, rank, world, local_rank)
    if args.option:
        out["config"]["options"] = dict(kv.split("=") for kv in args.option)
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline and args.config != "C5":
            out["cpu_baseline"] = cpu_baseline(args)
        print(json.dumps(out), file=real_stdout, flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
