"""Thin Python binding of libhdp.so (include/hdp.h) -- argument marshalling only.

Every step of the training path runs in the library's CUDA kernels; this
module converts Python values to C arguments and raises ``HDPError`` on a
negative return code.  There is no CPU fallback: if ``libhdp.so`` is missing
the import fails loudly.  PyTorch is used (by ``Trainer``) only to allocate
the device arena and to obtain CUDA stream handles.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import List, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhdp.so")

HDP_OK, HDP_ERR_ARG, HDP_ERR_CUDA, HDP_ERR_NCCL, HDP_ERR_NONFINITE, HDP_ERR_STATE, HDP_ERR_UNSUPPORTED = \
    0, -1, -2, -3, -4, -5, -6
MATH_FP32, MATH_MIXED16, MATH_BF16 = 0, 1, 2
WIRE_FP16_A2A, WIRE_FP16_NCCLSUM, WIRE_FP32 = 0, 1, 2
OPT_SGDM, OPT_ADAM = 0, 1
EXCH_AUTO, EXCH_NCCL, EXCH_P2P, EXCH_TASK0 = 0, 1, 2, 3

EXPORTED = [
    "hdp_nccl_unique_id", "hdp_init", "hdp_destroy", "hdp_last_error", "hdp_configure", "hdp_bind",
    "hdp_num_blocks", "hdp_exchange_kind", "hdp_param_block", "hdp_load_params", "hdp_gather_master", "hdp_read_weights",
    "hdp_read_grads", "hdp_set_lr_schedule", "hdp_lr", "hdp_set_loss_scale", "hdp_set_l2", "hdp_set_dynamic_loss_scale", "hdp_set_recurrent_dropout",
    "hdp_loss_scale_state", "hdp_lstm_forward",
    "hdp_lstm_backward", "hdp_grad_average_update", "hdp_weights_ptr", "hdp_grads_ptr", "hdp_master_ptr",
    "hdp_fused_avg_update", "hdp_gemm_f16", "hdp_gemm_f32", "hdp_profile", "hdp_profile_read",
    "hdp_kernel_launches", "hdp_debug_buffer", "hdp_set_option", "hdp_get_option", "hdp_partial_state", "hdp_profile_timeline",
]
NTAGS = 15


class HDPError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"hdp error {code}: {msg}")
        self.code = code


class ModelDesc(C.Structure):
    _fields_ = [("n_layers", C.c_int), ("input_dim", C.c_int), ("hidden", C.c_int), ("fc_hidden", C.c_int),
                ("head_last_step", C.c_int), ("vocab", C.c_int), ("embed_dim", C.c_int),
                ("max_batch", C.c_int), ("max_seq", C.c_int), ("math", C.c_int), ("wire", C.c_int),
                ("optimizer", C.c_int), ("sim_workers", C.c_int), ("flat_params", C.c_longlong),
                ("exchange", C.c_int)]


class Sizes(C.Structure):
    _fields_ = [("n_params", C.c_longlong), ("n_params_padded", C.c_longlong), ("n_buckets", C.c_longlong),
                ("arena_bytes", C.c_longlong)]


class Block(C.Structure):
    _fields_ = [("name", C.c_char * 16), ("canon_offset", C.c_longlong), ("rows", C.c_longlong),
                ("cols", C.c_longlong), ("dev_offset", C.c_longlong), ("dev_rows", C.c_longlong),
                ("dev_cols", C.c_longlong), ("bucket", C.c_int)]


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libhdp.so not built at {LIB_PATH}: run __graft_entry__.build() "
                          "(no CPU fallback exists)")
    lib = C.CDLL(LIB_PATH)
    vp, i, ll, d, f = C.c_void_p, C.c_int, C.c_longlong, C.c_double, C.c_float
    sig = {
        "hdp_nccl_unique_id": ([C.c_char_p], i),
        "hdp_init": ([i, i, C.c_char_p, i, C.POINTER(vp)], i),
        "hdp_destroy": ([vp], i),
        "hdp_last_error": ([], C.c_char_p),
        "hdp_configure": ([vp, C.POINTER(ModelDesc), C.POINTER(Sizes)], i),
        "hdp_bind": ([vp, vp, ll], i),
        "hdp_num_blocks": ([vp], i),
        "hdp_exchange_kind": ([vp], i),
        "hdp_param_block": ([vp, i, C.POINTER(Block)], i),
        "hdp_load_params": ([vp, vp, i], i),
        "hdp_gather_master": ([vp, vp], i),
        "hdp_read_weights": ([vp, vp], i),
        "hdp_read_grads": ([vp, i, vp], i),
        "hdp_set_lr_schedule": ([vp, d, d, d, d, d, d, d, d], i),
        "hdp_lr": ([vp, i], d),
        "hdp_set_loss_scale": ([vp, f], i),
        "hdp_set_l2": ([vp, d], i),
        "hdp_set_dynamic_loss_scale": ([vp, i], i),
        "hdp_set_recurrent_dropout": ([vp, d, C.c_uint], i),
        "hdp_loss_scale_state": ([vp, C.POINTER(f), C.POINTER(i)], i),
        "hdp_lstm_forward": ([vp, vp, vp, i, i, i, vp, vp, vp], i),
        "hdp_lstm_backward": ([vp, i, vp], i),
        "hdp_grad_average_update": ([vp, i, vp, C.POINTER(i)], i),
        "hdp_weights_ptr": ([vp], vp),
        "hdp_grads_ptr": ([vp, i], vp),
        "hdp_master_ptr": ([vp], vp),
        "hdp_debug_buffer": ([vp, i, C.c_char_p], vp),
        "hdp_fused_avg_update": ([vp, ll, i, i, ll, vp, vp, vp, vp, vp, f, f, f, i, vp, vp, f, vp], i),
        "hdp_gemm_f16": ([vp, ll, i, vp, ll, i, i, i, i, vp, ll, i, vp, i, i, i, vp, ll, i, i, vp], i),
        "hdp_gemm_f32": ([vp, ll, i, vp, ll, i, i, i, i, vp, ll, i, vp, i, i, i, vp], i),
        "hdp_profile": ([vp, i], i),
        "hdp_profile_read": ([vp, vp, vp, i], i),
        "hdp_kernel_launches": ([vp], ll),
        "hdp_set_option": ([vp, C.c_char_p, d], i),
        "hdp_partial_state": ([vp, C.POINTER(C.c_uint), C.POINTER(i)], i),
        "hdp_get_option": ([C.c_char_p, C.POINTER(d)], i),
        "hdp_profile_timeline": ([vp, C.POINTER(i), C.POINTER(i), C.POINTER(d), C.POINTER(d), i, C.POINTER(i)], i),
    }
    for name, (args, res) in sig.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    return lib


_lib = _load()


def lib():
    return _lib


def last_error() -> str:
    return (_lib.hdp_last_error() or b"").decode()


def _ck(rc):
    if rc != HDP_OK:
        raise HDPError(rc, last_error())
    return rc


def _ptr(x) -> Optional[int]:
    """Raw address of a torch tensor / numpy array / int / None."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    if hasattr(x, "data_ptr"):
        return x.data_ptr()
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    raise TypeError(type(x))


def _stream(s) -> Optional[int]:
    if s is None:
        return None
    if isinstance(s, int):
        return s
    return s.cuda_stream


# ------------------------------------------------------------------ C-ABI, same names
def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _ck(_lib.hdp_nccl_unique_id(buf))
    return buf.raw


def init(world: int, rank: int, uid: Optional[bytes] = None, device: int = 0) -> int:
    h = C.c_void_p()
    _ck(_lib.hdp_init(world, rank, uid, device, C.byref(h)))
    return h.value


def destroy(ctx: int):
    _ck(_lib.hdp_destroy(ctx))


def configure(ctx: int, desc: ModelDesc) -> Sizes:
    s = Sizes()
    _ck(_lib.hdp_configure(ctx, C.byref(desc), C.byref(s)))
    return s


def bind(ctx: int, arena, nbytes: int):
    _ck(_lib.hdp_bind(ctx, _ptr(arena), nbytes))


EXCHANGE_KINDS = {0: "K11 over local gradient slots", 1: "NCCL all-to-all + K11 + all-gather",
                  2: "one-kernel NVLink exchange (peer loads/stores)", 3: "one-kernel exchange, 1-GPU loopback",
                  4: "task-0 ablation (gather to rank 0, full update, broadcast)"}


def exchange_kind(ctx: int) -> int:
    return _lib.hdp_exchange_kind(ctx)


def param_blocks(ctx: int) -> List[dict]:
    out = []
    for k in range(_lib.hdp_num_blocks(ctx)):
        b = Block()
        _ck(_lib.hdp_param_block(ctx, k, C.byref(b)))
        out.append({f: (getattr(b, f).decode() if f == "name" else getattr(b, f)) for f, _ in Block._fields_})
    return out


def load_params(ctx: int, params: Optional[np.ndarray], root: int = 0):
    if params is not None:
        params = np.ascontiguousarray(params, dtype=np.float32)
    _ck(_lib.hdp_load_params(ctx, _ptr(params), root))


def gather_master(ctx: int, n: int) -> np.ndarray:
    out = np.zeros(n, np.float32)
    _ck(_lib.hdp_gather_master(ctx, _ptr(out)))
    return out


def read_weights(ctx: int, n: int) -> np.ndarray:
    out = np.zeros(n, np.float32)
    _ck(_lib.hdp_read_weights(ctx, _ptr(out)))
    return out


def read_grads(ctx: int, slot: int, n: int) -> np.ndarray:
    out = np.zeros(n, np.float32)
    _ck(_lib.hdp_read_grads(ctx, slot, _ptr(out)))
    return out


def set_lr_schedule(ctx, lambda0, gamma=0.8, n_half=100.0, max_eff_lr=0.1, momentum=0.9, adam_b1=0.9,
                    adam_b2=0.999, adam_eps=1e-8):
    _ck(_lib.hdp_set_lr_schedule(ctx, lambda0, gamma, n_half, max_eff_lr, momentum, adam_b1, adam_b2, adam_eps))


def lr(ctx: int, epoch: int) -> float:
    return _lib.hdp_lr(ctx, epoch)


def set_loss_scale(ctx: int, alpha: float):
    _ck(_lib.hdp_set_loss_scale(ctx, alpha))


def set_l2(ctx: int, l2: float):
    _ck(_lib.hdp_set_l2(ctx, l2))


def set_recurrent_dropout(ctx: int, keep: float, seed: int = 0):
    _ck(_lib.hdp_set_recurrent_dropout(ctx, keep, seed))


def set_dynamic_loss_scale(ctx: int, growth_interval: int):
    _ck(_lib.hdp_set_dynamic_loss_scale(ctx, growth_interval))


def loss_scale_state(ctx: int):
    """(alpha, skipped_steps) -- synchronises the device."""
    a, k = C.c_float(), C.c_int()
    _ck(_lib.hdp_loss_scale_state(ctx, C.byref(a), C.byref(k)))
    return a.value, k.value


# process-wide kernel switches and their defaults (csrc/options.h, hdp_set_option)
KERNEL_OPTION_DEFAULTS = {"persistent": 1, "wavefront": 1, "wavefront_fusex": 1, "wavefront_wgrad": 1,
                          "wavefront_tmem": 1, "recur_nbg": 0, "gemm_cta_group": 0,
                          "gemm_cluster_n": 0, "pdl": 0, "k7_bn": 0, "k7_splits": 0, "recur_trace": 0,
                          "layer_pipe": 16, "head_fused": 1, "k7_cluster": 0, "fwd_pdl": 0}


def set_option(ctx, name: str, value: float):
    """hdp_set_option: context options (ctx) or process-wide kernel switches (ctx may be None)."""
    _ck(_lib.hdp_set_option(ctx, name.encode(), float(value)))


def get_option(name: str) -> int:
    """hdp_get_option: current value of a process-wide kernel switch."""
    v = C.c_double()
    _ck(_lib.hdp_get_option(name.encode(), C.byref(v)))
    return int(v.value)


def profile_timeline(ctx, cap=100000):
    """hdp_profile_timeline: [(tag, lane, t0_ms, t1_ms)] of the profiled launches so far."""
    tags, lanes = (C.c_int * cap)(), (C.c_int * cap)()
    t0, t1 = (C.c_double * cap)(), (C.c_double * cap)()
    n = C.c_int()
    _ck(_lib.hdp_profile_timeline(ctx, tags, lanes, t0, t1, cap, C.byref(n)))
    return [(tags[i], lanes[i], t0[i], t1[i]) for i in range(min(n.value, cap))]


def partial_state(ctx):
    """(contributor mask, count) of the last partial-collection decision."""
    m, n = C.c_uint(), C.c_int()
    _ck(_lib.hdp_partial_state(ctx, C.byref(m), C.byref(n)))
    return m.value, n.value


def lstm_forward(ctx, x, targets, B, T, slot=0, y_out=None, loss_out=None, stream=None):
    _ck(_lib.hdp_lstm_forward(ctx, _ptr(x), _ptr(targets), B, T, slot, _ptr(y_out), _ptr(loss_out),
                              _stream(stream)))


def lstm_backward(ctx, slot=0, stream=None):
    _ck(_lib.hdp_lstm_backward(ctx, slot, _stream(stream)))


def grad_average_update(ctx, epoch=0, stream=None, sync=False) -> Optional[int]:
    if sync:
        n = C.c_int(0)
        rc = _lib.hdp_grad_average_update(ctx, epoch, _stream(stream), C.byref(n))
        if rc not in (HDP_OK, HDP_ERR_NONFINITE):
            _ck(rc)
        if rc == HDP_ERR_NONFINITE:
            raise HDPError(rc, last_error())
        return n.value
    _ck(_lib.hdp_grad_average_update(ctx, epoch, _stream(stream), None))
    return None


def weights_ptr(ctx) -> int:
    return _lib.hdp_weights_ptr(ctx)


def grads_ptr(ctx, slot=0) -> int:
    return _lib.hdp_grads_ptr(ctx, slot)


def debug_buffer(ctx, slot: int, name: str) -> int:
    return _lib.hdp_debug_buffer(ctx, slot, name.encode())


def master_ptr(ctx) -> int:
    return _lib.hdp_master_ptr(ctx)


def fused_avg_update(grads, src_stride, nsrc, grads_f32, count, W, S1, S2=None, w16=None, w32=None,
                     inv_scale=1.0, lr=0.0, momentum=0.0, optimizer=OPT_SGDM, adam=None, nonfinite=None,
                     stream=None, l2x2=0.0):
    adam_arr = None
    if adam is not None:
        adam_arr = (C.c_double * 4)(*adam)
    _ck(_lib.hdp_fused_avg_update(_ptr(grads), src_stride, nsrc, int(grads_f32), count, _ptr(W), _ptr(S1),
                                  _ptr(S2), _ptr(w16), _ptr(w32), inv_scale, lr, momentum, optimizer,
                                  C.cast(adam_arr, C.c_void_p) if adam_arr is not None else None,
                                  _ptr(nonfinite), l2x2, _stream(stream)))


def gemm_f16(A, lda, a_mn, B, ldb, b_mn, M, N, K, Cout, ldc, c_mode=0, bias=None, bias_on_m=0, relu=0,
             accumulate=0, ws=None, ws_floats=0, bn=0, splits=0, stream=None):
    _ck(_lib.hdp_gemm_f16(_ptr(A), lda, a_mn, _ptr(B), ldb, b_mn, M, N, K, _ptr(Cout), ldc, c_mode, _ptr(bias),
                          bias_on_m, relu, accumulate, _ptr(ws), ws_floats, bn, splits, _stream(stream)))


def gemm_f32(A, lda, a_mn, B, ldb, b_mn, M, N, K, Cout, ldc, c_mode=0, bias=None, bias_on_m=0, relu=0,
             accumulate=0, stream=None):
    _ck(_lib.hdp_gemm_f32(_ptr(A), lda, a_mn, _ptr(B), ldb, b_mn, M, N, K, _ptr(Cout), ldc, c_mode, _ptr(bias),
                          bias_on_m, relu, accumulate, _stream(stream)))


# ------------------------------------------------------------------ convenience
def desc_from_config(cfg, max_batch: int, math: int = MATH_MIXED16, wire: int = WIRE_FP16_A2A,
                     optimizer: int = OPT_SGDM, sim_workers: int = 1, exchange: int = EXCH_AUTO) -> ModelDesc:
    """Build a ModelDesc from a synth.ModelConfig-like object (shape fields only)."""
    return ModelDesc(n_layers=cfg.n_layers, input_dim=cfg.input_dim, hidden=cfg.hidden, fc_hidden=cfg.fc_hidden,
                     head_last_step=int(cfg.head_last_step), vocab=cfg.vocab, embed_dim=cfg.embed_dim,
                     max_batch=max_batch, max_seq=cfg.seq, math=math, wire=wire, optimizer=optimizer,
                     sim_workers=sim_workers, flat_params=0, exchange=exchange)


class Trainer:
    """One rank's training context: allocates the arena with torch, loads the
    parameters, sets the schedule.  ``step`` = forward + backward on every
    slot + grad_average_update (all in libhdp)."""

    def __init__(self, desc: ModelDesc, params: Optional[np.ndarray], lambda0: float, alpha: float = 10.0,
                 gamma: float = 0.8, n_half: float = 100.0, momentum: float = 0.9, world: int = 1, rank: int = 0,
                 uid: Optional[bytes] = None, device: int = 0, max_eff_lr: float = 0.1, l2: float = 0.0):
        import torch
        self.torch = torch
        self.ctx = init(world, rank, uid, device)
        self.desc = desc
        self.sizes = configure(self.ctx, desc)
        self.arena = torch.empty(self.sizes.arena_bytes + 256, dtype=torch.uint8, device=f"cuda:{device}")
        base = self.arena.data_ptr()
        off = (-base) % 256
        bind(self.ctx, base + off, self.sizes.arena_bytes)
        self.n = self.sizes.n_params
        load_params(self.ctx, params, 0)
        set_lr_schedule(self.ctx, lambda0, gamma, n_half, max_eff_lr, momentum)
        set_loss_scale(self.ctx, alpha)
        if l2:
            set_l2(self.ctx, l2)
        self.loss = torch.zeros(max(1, desc.sim_workers), dtype=torch.float32, device=f"cuda:{device}")

    def step(self, xs, ts, B, T, epoch=0, stream=None, sync=False):
        """xs / ts: one input per slot (device or pinned-host tensors)."""
        for s in range(self.desc.sim_workers if self.desc.sim_workers > 0 else 1):
            lstm_forward(self.ctx, xs[s], ts[s], B, T, s, None, self.loss[s:s + 1], stream)
            lstm_backward(self.ctx, s, stream)
        return grad_average_update(self.ctx, epoch, stream, sync)

    def close(self):
        if self.ctx:
            destroy(self.ctx)
            self.ctx = None
