"""Host-side mirror of the reference ProxyKV scoring / mapper / prune API over
the B200 C ABI (include/pkv_capi.h).

Names, argument meaning and error behaviour follow the reference
(/root/reference/proj/include/proxykv/{pruning,mapper}.hpp) so the parity tests
read like the reference's own tests. Device memory is torch-allocated
(plumbing); every computation runs in libpkv_b200.so's sm_100a kernels.
There is no CPU fallback: without a B200 every compute call raises
NoDeviceError.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import _lib
from ._lib import (BadMagicError, ConfigError, CudaError, IoError, NoDeviceError, PayloadLengthError, PkvError,
                   PkvValueError, ShapeError, TruncatedFileError, VersionMismatchError, check, lib)

__all__ = [
    "Context", "PruneMask", "MaskApplication", "ModelGeometry", "MapperConfig", "Mapper", "Pruner",
    "retention_count", "topk_select", "topk_indices", "topk_mask", "apply_mask", "compact_kv", "select_compact", "score", "score_lse",
    "proxy_prefill_attention", "packed_decode_attention", "paged_decode_attention", "compact_kv_paged", "topk_overlap_device", "captured_mass_device",
    "spearman_device", "slice_metrics_device", "MetricAccumulator", "MetricReport",
    "LossConfig", "LossReport", "loss_total", "MapperTrainer",
    "layer_pair", "window_offsets", "mapper_init_params", "ShapeError", "PkvValueError", "ConfigError",
    "CudaError", "NoDeviceError", "PkvError", "SCORE_REDUCE_MAX", "SCORE_REDUCE_SUM", "SCORE_CAUSAL",
    "MAPPER_FP16", "MAPPER_FP16X2", "MAPPER_FP16X3", "MAPPER_FP16F8", "SHARD_LAYER", "SHARD_HEAD", "ShardPlan", "shard_plan",
    "Comm", "shard_exchange_schedule", "write_trace", "read_trace", "write_checkpoint", "read_checkpoint", "IoError", "BadMagicError",
    "VersionMismatchError", "TruncatedFileError", "PayloadLengthError",
]

SCORE_REDUCE_MAX = 0
SCORE_REDUCE_SUM = 1
SCORE_CAUSAL = 2
MAPPER_FP16 = 1
MAPPER_FP16X2 = 2
MAPPER_FP16X3 = 3
MAPPER_FP16W2 = 4
MAPPER_FP16X3F = 5
MAPPER_FP16F8 = 6
SHARD_LAYER = 0
SHARD_HEAD = 1
COMM_ID_BYTES = 128


def _torch():
    import torch
    return torch


def _ptr(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _stream(stream) -> Optional[int]:
    torch = _torch()
    if stream is None:
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


class Context:
    """pkv_ctx: one per device (and host thread)."""

    _default = {}

    def __init__(self, device: int = 0):
        h = ctypes.c_void_p()
        check(lib().pkv_ctx_create(device, ctypes.byref(h)))
        self.h = h
        self.device = device

    @classmethod
    def default(cls, device: int = 0) -> "Context":
        if device not in cls._default:
            cls._default[device] = Context(device)
        return cls._default[device]

    def launches(self) -> int:
        return int(lib().pkv_ctx_launch_count(self.h))

    def __del__(self):
        h = getattr(self, "h", None)
        if h and _lib._lib is not None:
            _lib._lib.pkv_ctx_destroy(h)
            self.h = None


# ------------------------------------------------------------------ select --
def retention_count(rho: float, n: int) -> int:
    """pruning.cpp:14-18."""
    k = ctypes.c_int64()
    check(lib().pkv_retention_count(float(rho), int(n), ctypes.byref(k)))
    return k.value


def topk_select(scores, k: int, *, want_mask: bool = True, want_idx: bool = True, ctx: Context = None,
                stream=None):
    """Device Top-K: scores fp32 cuda tensor [..., n] -> (mask u8 [..., n] | None, idx i32 [slices, k] | None)."""
    torch = _torch()
    ctx = ctx or Context.default(scores.device.index or 0)
    if scores.dtype not in (torch.float32, torch.float64) or not scores.is_cuda:
        raise ShapeError("topk_select expects a float32 or float64 CUDA tensor")
    s = scores.contiguous()
    n = s.shape[-1]
    slices = s.numel() // n if n else 0
    mask = torch.empty(s.shape, dtype=torch.uint8, device=s.device) if want_mask else None
    idx = torch.empty((slices, max(int(k), 0)), dtype=torch.int32, device=s.device) if want_idx else None
    fn = lib().pkv_topk_select_f64 if s.dtype == torch.float64 else lib().pkv_topk_select
    check(fn(ctx.h, _ptr(s), slices, n, int(k), _ptr(mask), _ptr(idx), _stream(stream)))
    return mask, idx


def topk_indices(values: np.ndarray, k: int, ctx: Context = None) -> np.ndarray:
    """pruning.cpp:20-35 on a host fp64 row: the k best (ties to the lower index), ascending."""
    ctx = ctx or Context.default()
    v = np.ascontiguousarray(values, np.float64).reshape(-1)
    out = np.zeros(max(int(k), 0), np.int64)
    check(lib().pkv_topk_indices_host(ctx.h, v.ctypes.data, v.size, int(k), out.ctypes.data))
    return out


@dataclass
class PruneMask:
    """pruning.hpp:22-30."""
    shape: Tuple[int, ...]
    bits: np.ndarray
    retention_ratio: float = 1.0
    k: int = 0
    idx_asc: Optional[np.ndarray] = None  # [slices, k], from the GPU select

    def token_count(self) -> int:
        return self.shape[-1]

    def slice_count(self) -> int:
        return int(np.prod(self.shape)) // self.shape[-1]


def topk_mask(scores: np.ndarray, rho: float, ctx: Context = None) -> PruneMask:
    """pruning.cpp:37-56 with host scores (the reference signature): GPU radix select,
    mask bits and ascending indices copied back. fp64 input (the reference's
    ScoreTensor) is ranked on 64-bit keys, fp32 input on 32-bit keys: exact
    either way, never narrowed."""
    torch = _torch()
    s = np.asarray(scores)
    if s.ndim == 0:
        raise ShapeError("topk_mask needs a shaped tensor")
    n = s.shape[-1]
    k = retention_count(rho, n)
    dt = np.float32 if s.dtype == np.float32 else np.float64
    dev = torch.from_numpy(np.ascontiguousarray(s, dtype=dt)).cuda()
    mask, idx = topk_select(dev, k, ctx=ctx)
    torch.cuda.synchronize()
    return PruneMask(tuple(s.shape), mask.cpu().numpy(), rho, k, idx.cpu().numpy())


@dataclass
class MaskApplication:
    """pruning.hpp:48-53."""
    retained: List[np.ndarray] = field(default_factory=list)
    dropped_per_slice: int = 0
    bytes_saved_per_head: int = 0
    bytes_saved_total: int = 0


def apply_mask(mask: PruneMask, head_dim: int, bytes_per_elem: int = 2) -> MaskApplication:
    """pruning.cpp:197-215: retained indices (ascending, produced on the GPU by the
    select kernel's ordered compaction) and the byte accounting."""
    if mask.idx_asc is None:
        raise PkvValueError("apply_mask needs a PruneMask produced by topk_mask (GPU indices)")
    n, slices = mask.token_count(), mask.slice_count()
    app = MaskApplication([mask.idx_asc[s].astype(np.int64) for s in range(slices)])
    app.dropped_per_slice = n - mask.k
    app.bytes_saved_per_head = app.dropped_per_slice * head_dim * bytes_per_elem * 2
    app.bytes_saved_total = app.bytes_saved_per_head * slices
    return app


def topk_overlap_device(mask_a, mask_b, k: int, *, ctx: Context = None, stream=None):
    """pruning.cpp:91-108 on the device: per-slice |a ∩ b| / k (fp64 cuda tensor)."""
    torch = _torch()
    ctx = ctx or Context.default(mask_a.device.index or 0)
    n = mask_a.shape[-1]
    slices = mask_a.numel() // n
    out = torch.empty(slices, dtype=torch.float64, device=mask_a.device)
    check(lib().pkv_topk_overlap(ctx.h, _ptr(mask_a.contiguous()), _ptr(mask_b.contiguous()), slices, n, int(k),
                                 _ptr(out), _stream(stream)))
    return out


def captured_mass_device(mask_pred, y, k: int, *, ctx: Context = None, stream=None):
    """pruning.cpp:58-80 on the device: per-slice captured-mass ratio (fp64 cuda tensor)."""
    torch = _torch()
    ctx = ctx or Context.default(y.device.index or 0)
    n = y.shape[-1]
    slices = y.numel() // n
    out = torch.empty(slices, dtype=torch.float64, device=y.device)
    check(lib().pkv_captured_mass(ctx.h, _ptr(mask_pred.contiguous()), _ptr(y.contiguous()), slices, n, int(k),
                                  _ptr(out), _stream(stream)))
    return out


def spearman_device(a, b, *, ctx: Context = None, stream=None):
    """pruning.cpp:173-186 on the device: per-slice Spearman correlation of two
    fp32 cuda tensors [..., n] with average ranks on ties (fp64 cuda tensor)."""
    torch = _torch()
    ctx = ctx or Context.default(a.device.index or 0)
    if a.shape != b.shape:
        raise ShapeError(f"spearman shapes differ: {tuple(a.shape)} vs {tuple(b.shape)}")
    n = a.shape[-1]
    slices = a.numel() // n
    out = torch.empty(slices, dtype=torch.float64, device=a.device)
    check(lib().pkv_spearman(ctx.h, _ptr(a.contiguous()), _ptr(b.contiguous()), slices, n, _ptr(out),
                             _stream(stream)))
    return out


def slice_metrics_device(y_pred, y_true, rho: float, *, ctx: Context = None, stream=None):
    """One MetricAccumulator::add sample (pruning.cpp:218-247) on the device:
    (captured mass, Top-K overlap, Spearman) per slice, fp64 cuda tensors."""
    torch = _torch()
    ctx = ctx or Context.default(y_pred.device.index or 0)
    if y_pred.shape != y_true.shape:
        raise ShapeError(f"metric shapes differ: {tuple(y_pred.shape)} vs {tuple(y_true.shape)}")
    n = y_pred.shape[-1]
    slices = y_pred.numel() // n
    k = retention_count(rho, n)
    outs = [torch.empty(slices, dtype=torch.float64, device=y_pred.device) for _ in range(3)]
    check(lib().pkv_slice_metrics(ctx.h, _ptr(y_pred.contiguous()), _ptr(y_true.contiguous()), slices, n, k,
                                  _ptr(outs[0]), _ptr(outs[1]), _ptr(outs[2]), _stream(stream)))
    return tuple(outs)


@dataclass
class MetricReport:
    """pruning.hpp MetricReport: means over samples per (layer, head) and overall."""
    rho: float
    captured_mass: float
    topk_overlap: float
    spearman: float
    per_slice_mass: list
    per_slice_overlap: list
    per_slice_spearman: list


class MetricAccumulator:
    """MetricAccumulator (pruning.cpp:218-275) with the per-sample work on the
    device (pkv_slice_metrics); only the running sums are host arithmetic.
    add() takes [B, L, H, N] or [L, H, N] fp32 cuda tensors."""

    def __init__(self, rho: float, *, ctx: Context = None):
        self.rho = float(rho)
        self.ctx = ctx
        self._sums = None
        self._counts = None
        self._slices = 0

    def add(self, y_pred, y_true, stream=None):
        torch = _torch()
        if y_pred.shape != y_true.shape:
            raise ShapeError(f"metric shapes differ: {tuple(y_pred.shape)} vs {tuple(y_true.shape)}")
        if y_pred.dim() not in (3, 4):
            raise ShapeError(f"metrics expect [B, L, H, N] or [L, H, N], got {tuple(y_pred.shape)}")
        b = y_pred.shape[0] if y_pred.dim() == 4 else 1
        lh = y_pred.numel() // y_pred.shape[-1] // b
        if self._slices == 0:
            self._slices = lh
            self._sums = torch.zeros(3, lh, dtype=torch.float64, device=y_pred.device)
            self._counts = 0
        if lh != self._slices:
            raise ShapeError("inconsistent (layer, head) slice count across samples")
        m, o, s = slice_metrics_device(y_pred, y_true, self.rho, ctx=self.ctx, stream=stream)
        # samples are added in batch order, slice key = i % lh (pruning.cpp:240-245)
        self._sums += torch.stack([m, o, s]).view(3, b, lh).sum(dim=1)
        self._counts += b

    def report(self) -> MetricReport:
        if self._slices == 0:
            raise PkvValueError("no samples accumulated")
        per = (self._sums / float(self._counts)).cpu().numpy()
        lh = float(self._slices)
        return MetricReport(self.rho, float(sum(per[0].tolist()) / lh), float(sum(per[1].tolist()) / lh),
                            float(sum(per[2].tolist()) / lh), per[0].tolist(), per[1].tolist(), per[2].tolist())


@dataclass
class LossConfig:
    """loss.hpp LossConfig (same fields, same defaults)."""
    lambda_mse: float = 20.0
    lambda_bin: float = 10.0
    lambda_fine: float = 3.0
    lambda_global: float = 2.0
    lambda_cos: float = 0.5
    ratios: Sequence[float] = (0.05, 0.1, 0.15, 0.2, 0.3, 0.4, 0.5)
    gamma: float = 1.0
    epsilon: float = 0.1
    mse_exponent: float = 1.5
    margin: float = 1.0
    clip_lo: float = 1.0
    clip_hi: float = 5.0
    pair_filter_frac: float = 0.01
    topk_ratio_for_rank: float = 0.2
    max_pairs: int = 4096


class _CLossConfig(ctypes.Structure):
    _fields_ = [("lambda_mse", ctypes.c_double), ("lambda_bin", ctypes.c_double), ("lambda_fine", ctypes.c_double),
                ("lambda_global", ctypes.c_double), ("lambda_cos", ctypes.c_double),
                ("ratios", ctypes.POINTER(ctypes.c_double)), ("n_ratios", ctypes.c_int64),
                ("gamma", ctypes.c_double), ("epsilon", ctypes.c_double), ("mse_exponent", ctypes.c_double),
                ("margin", ctypes.c_double), ("clip_lo", ctypes.c_double), ("clip_hi", ctypes.c_double),
                ("pair_filter_frac", ctypes.c_double), ("topk_ratio_for_rank", ctypes.c_double),
                ("max_pairs", ctypes.c_int64)]


class _CLossReport(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in ("bin", "mse", "fine", "global_", "cos", "weighted_bin", "weighted_mse",
                                               "weighted_fine", "weighted_global", "weighted_cos", "total",
                                               "s_max")] + \
               [(n, ctypes.c_int64) for n in ("fine_used", "fine_filtered", "global_used", "global_filtered",
                                              "cos_floor_hits")]


@dataclass
class LossReport:
    """loss.hpp LossReport (total_tensor -> the gradient returned beside it)."""
    bin: float
    mse: float
    fine: float
    global_: float
    cos: float
    weighted_bin: float
    weighted_mse: float
    weighted_fine: float
    weighted_global: float
    weighted_cos: float
    total: float
    s_max: float
    fine_used: int
    fine_filtered: int
    global_used: int
    global_filtered: int
    cos_floor_hits: int


def loss_total(logits, y, cfg: LossConfig = None, seed: int = 0, *, want_grad: bool = True, ctx: Context = None,
               stream=None):
    """loss_total (loss.cpp:324-374) on the device: fp32 cuda logits / scores
    of one shape -> (LossReport, d total / d logits as an fp64 cuda tensor or
    None). The pair samples are the reference's own for the same seed."""
    torch = _torch()
    cfg = cfg or LossConfig()
    ctx = ctx or Context.default(logits.device.index or 0)
    if logits.shape != y.shape:
        raise ShapeError(f"loss_total shapes differ: {tuple(logits.shape)} vs {tuple(y.shape)}")
    if logits.dtype != torch.float32 or y.dtype != torch.float32 or not logits.is_cuda:
        raise ShapeError("loss_total expects float32 CUDA tensors")
    ratios = (ctypes.c_double * max(1, len(cfg.ratios)))(*cfg.ratios)
    c = _CLossConfig(cfg.lambda_mse, cfg.lambda_bin, cfg.lambda_fine, cfg.lambda_global, cfg.lambda_cos,
                     ctypes.cast(ratios, ctypes.POINTER(ctypes.c_double)) if len(cfg.ratios) else None,
                     len(cfg.ratios), cfg.gamma, cfg.epsilon, cfg.mse_exponent, cfg.margin, cfg.clip_lo, cfg.clip_hi,
                     cfg.pair_filter_frac, cfg.topk_ratio_for_rank, int(cfg.max_pairs))
    shape = (ctypes.c_int64 * logits.dim())(*logits.shape)
    rep = _CLossReport()
    grad = torch.empty(logits.shape, dtype=torch.float64, device=logits.device) if want_grad else None
    check(lib().pkv_loss_total(ctx.h, _ptr(logits.contiguous()), _ptr(y.contiguous()), shape, logits.dim(),
                               ctypes.byref(c), ctypes.c_uint64(seed), ctypes.byref(rep),
                               _ptr(grad) if want_grad else None, _stream(stream)))
    return LossReport(*[getattr(rep, f[0]) for f in _CLossReport._fields_]), grad


class MapperTrainer:
    """GPU training of the HybridAxialMapper (pkv_trainer): the reference's training
    forward_pair (mapper.cpp:274-342, BN on batch statistics) and the reverse sweep
    of its tape from d loss / d logits to the parameter gradients (blob layout)."""

    def __init__(self, geom: ModelGeometry, cfg: MapperConfig, blob: np.ndarray = None, *, seed: int = 0,
                 ctx: Context = None):
        self.geom, self.cfg = geom, cfg
        self.ctx = ctx or Context.default()
        if blob is None:
            blob = mapper_init_params(geom, cfg, seed)
        blob = np.ascontiguousarray(blob, np.float64)
        h = ctypes.c_void_p()
        check(lib().pkv_trainer_create(self.ctx.h, geom.as5(), cfg.as12(), blob.ctypes.data, blob.size,
                                       ctypes.byref(h)))
        self.h = h
        npar, tot = ctypes.c_int64(), ctypes.c_int64()
        check(lib().pkv_trainer_param_count(h, ctypes.byref(npar), ctypes.byref(tot)))
        self.n_params, self.n_total = npar.value, tot.value

    def __del__(self):
        h = getattr(self, "h", None)
        if h and _lib._lib is not None:
            _lib._lib.pkv_trainer_destroy(h)
            self.h = None

    def forward(self, x, stream=None):
        """x fp32 cuda [B, H_s, n] -> logits fp32 [B, H_l, n] (training mode; keeps activations)."""
        torch = _torch()
        B, hs, n = x.shape
        if hs != self.geom.proxy_heads:
            raise ShapeError(f"input has {hs} proxy heads, geometry expects {self.geom.proxy_heads}")
        x = x.contiguous()
        y = torch.empty((B, self.geom.target_heads, n), dtype=torch.float32, device=x.device)
        check(lib().pkv_trainer_forward(self.h, _ptr(x), B, n, _ptr(y), _stream(stream)))
        return y

    def backward(self, dlogits, grad=None, stream=None):
        """d loss / d logits (fp64 cuda, the last forward's shape) -> parameter gradients
        (fp64 cuda [n_params], accumulated into `grad` when given)."""
        torch = _torch()
        if grad is None:
            grad = torch.zeros(self.n_params, dtype=torch.float64, device=dlogits.device)
        check(lib().pkv_trainer_backward(self.h, _ptr(dlogits.contiguous()), _ptr(grad), _stream(stream)))
        return grad

    def blob(self) -> np.ndarray:
        """Parameters + BN running statistics (pkv_mapper_init_params layout)."""
        out = np.zeros(self.n_total, np.float64)
        check(lib().pkv_trainer_blob(self.h, out.ctypes.data))
        return out


def compact_kv(k_in, v_in, idx_asc, *, ctx: Context = None, stream=None, out=None):
    """Packed gather of retained rows: k_in/v_in [S, n, d] (2-byte) cuda, idx_asc i32 [S, k]."""
    torch = _torch()
    ctx = ctx or Context.default(k_in.device.index or 0)
    S, n, d = k_in.shape
    k = idx_asc.shape[1]
    if out is None:
        ko = torch.empty((S, k, d), dtype=k_in.dtype, device=k_in.device)
        vo = torch.empty((S, k, d), dtype=v_in.dtype, device=v_in.device)
    else:
        ko, vo = out
    check(lib().pkv_compact_kv(ctx.h, _ptr(k_in), _ptr(v_in), _ptr(idx_asc), S, n, k, d, k_in.element_size(),
                               _ptr(ko), _ptr(vo), _stream(stream)))
    return ko, vo


def select_compact(scores, k_in, v_in, k: int, *, ctx: Context = None, stream=None, out=None):
    """Top-K select then the packed gather in one call (pkv_select_compact): scores fp32 [S, n],
    k_in/v_in [S, n, d] cuda -> (idx_asc i32 [S, k], k_out, v_out [S, k, d])."""
    torch = _torch()
    ctx = ctx or Context.default(scores.device.index or 0)
    S, n, d = k_in.shape
    if tuple(scores.shape) != (S, n) or scores.dtype != torch.float32 or not scores.is_contiguous():
        raise ShapeError("select_compact expects contiguous float32 scores [S, n] matching k_in")
    if out is None:
        idx = torch.empty((S, k), dtype=torch.int32, device=scores.device)
        ko = torch.empty((S, k, d), dtype=k_in.dtype, device=k_in.device)
        vo = torch.empty((S, k, d), dtype=v_in.dtype, device=v_in.device)
    else:
        idx, ko, vo = out
    check(lib().pkv_select_compact(ctx.h, _ptr(scores), S, n, k, _ptr(k_in), _ptr(v_in), d, k_in.element_size(),
                                   _ptr(idx), _ptr(ko), _ptr(vo), _stream(stream)))
    return idx, ko, vo


# ----------------------------------------------------------------- scoring --
def score(q, k, *, reduce: str = "max", causal: bool = False, lse=None, ctx: Context = None, stream=None, out=None):
    """Proxy scoring: q bf16 [L, Hq, Nq, d], k bf16 [L, Hkv, Nk, d] -> X fp32 [L, Hkv, Nk]."""
    torch = _torch()
    ctx = ctx or Context.default(q.device.index or 0)
    L, hq, nq, d = q.shape
    _, hkv, nk, _ = k.shape
    flags = (SCORE_REDUCE_SUM if reduce == "sum" else SCORE_REDUCE_MAX) | (SCORE_CAUSAL if causal else 0)
    x = out if out is not None else torch.empty((L, hkv, nk), dtype=torch.float32, device=q.device)
    check(lib().pkv_score(ctx.h, _ptr(q), _ptr(k), L, hq, hkv, nq, nk, d, flags, _ptr(lse), _ptr(x),
                          _stream(stream)))
    return x


def proxy_prefill_attention(q, k, v, *, causal: bool = True, want_out: bool = True, ctx: Context = None,
                            stream=None):
    """Proxy prefill attention (bf16): returns (O bf16 [L, Hq, Nq, d] | None, lse fp32 [L, Hq, Nq]); the LSE is
    what `score(..., lse=...)` takes to skip its first pass."""
    torch = _torch()
    ctx = ctx or Context.default(q.device.index or 0)
    L, hq, nq, d = q.shape
    _, hkv, nk, _ = k.shape
    o = torch.empty_like(q) if want_out else None
    lse = torch.empty((L, hq, nq), dtype=torch.float32, device=q.device)
    check(lib().pkv_proxy_prefill_attention(ctx.h, _ptr(q), _ptr(k), _ptr(v), L, hq, hkv, nq, nk, d,
                                            SCORE_CAUSAL if causal else 0, _ptr(o), _ptr(lse), _stream(stream)))
    return o, lse


def packed_decode_attention(q, k_packed, v_packed, *, scale: float = None, ctx: Context = None, stream=None,
                            out=None):
    """Decode over the packed cache: q bf16 [L, Hq, d], k/v_packed bf16 [L, Hkv, K, d] -> fp32 [L, Hq, d]."""
    torch = _torch()
    ctx = ctx or Context.default(q.device.index or 0)
    L, hq, d = q.shape
    _, hkv, K, _ = k_packed.shape
    o = out if out is not None else torch.empty((L, hq, d), dtype=torch.float32, device=q.device)
    sc = float(scale) if scale is not None else 1.0 / d ** 0.5
    check(lib().pkv_packed_decode_attention(ctx.h, _ptr(q), _ptr(k_packed), _ptr(v_packed), L, hq, hkv, K, d, sc,
                                            _ptr(o), _stream(stream)))
    return o


def paged_decode_attention(q, k_pool, v_pool, block_table, seq_lens, *, max_len: int = None, scale: float = None,
                           ctx: Context = None, stream=None, out=None):
    """Decode over a paged cache: q bf16 [L, Hq, d]; k/v_pool bf16 [pages, page, d];
    block_table i32 [L, Hkv, max_blocks]; seq_lens i32 [L, Hkv] -> fp32 [L, Hq, d]."""
    torch = _torch()
    ctx = ctx or Context.default(q.device.index or 0)
    L, hq, d = q.shape
    _, hkv, mb = block_table.shape
    page = k_pool.shape[1]
    ml = int(max_len) if max_len is not None else int(seq_lens.max().item())
    o = out if out is not None else torch.empty((L, hq, d), dtype=torch.float32, device=q.device)
    sc = float(scale) if scale is not None else 1.0 / d ** 0.5
    check(lib().pkv_paged_decode_attention(ctx.h, _ptr(q), _ptr(k_pool), _ptr(v_pool), _ptr(block_table.contiguous()),
                                           _ptr(seq_lens.contiguous()), L, hq, hkv, mb, page, max(ml, 1), d, sc,
                                           _ptr(o), _stream(stream)))
    return o


def compact_kv_paged(k_in, v_in, idx_asc, block_table, k_pool, v_pool, *, ctx: Context = None, stream=None):
    """Gather retained rows into pages: k_in/v_in [S, n, d] (2-byte) cuda, idx_asc
    i32 [S, k], block_table i32 [S, max_blocks], pools [pages, page, d]."""
    ctx = ctx or Context.default(k_in.device.index or 0)
    S, n, d = k_in.shape
    k = idx_asc.shape[1]
    check(lib().pkv_compact_kv_paged(ctx.h, _ptr(k_in), _ptr(v_in), _ptr(idx_asc), S, n, k, d, k_in.element_size(),
                                     _ptr(block_table.contiguous()), block_table.shape[-1], k_pool.shape[1],
                                     _ptr(k_pool), _ptr(v_pool), _stream(stream)))
    return k_pool, v_pool


def score_lse(q, k, *, causal: bool = False, ctx: Context = None, stream=None):
    torch = _torch()
    ctx = ctx or Context.default(q.device.index or 0)
    L, hq, nq, d = q.shape
    _, hkv, nk, _ = k.shape
    out = torch.empty((L, hq, nq), dtype=torch.float32, device=q.device)
    check(lib().pkv_score_lse(ctx.h, _ptr(q), _ptr(k), L, hq, hkv, nq, nk, d, SCORE_CAUSAL if causal else 0,
                              _ptr(out), _stream(stream)))
    return out


# ------------------------------------------------------------------ mapper --
@dataclass
class ModelGeometry:
    """mapper.hpp:16-25."""
    target_layers: int = 32
    target_heads: int = 32
    proxy_layers: int = 16
    proxy_heads: int = 32
    head_dim: int = 128

    def as5(self):
        return (ctypes.c_int64 * 5)(self.target_layers, self.target_heads, self.proxy_layers, self.proxy_heads,
                                    self.head_dim)


@dataclass
class MapperConfig:
    """mapper.hpp:35-55 (stage modes 'active' | 'bypass')."""
    d_time: int = 512
    encoder_layers: int = 6
    encoder_heads: int = 8
    ffn_mult: int = 4
    d_head: int = 64
    crop_len: int = 2048
    stride: int = 1024
    synthetic_heads: int = 0
    stage_conv: str = "active"
    stage_encoder: str = "active"
    stage_cross: str = "active"
    normalize_input: bool = False

    def as12(self):
        m = {"active": 0, "bypass": 1}
        for s in (self.stage_conv, self.stage_encoder, self.stage_cross):
            if s not in m:
                raise ConfigError(f"unknown stage mode '{s}' (expected active|bypass)")
        return (ctypes.c_int64 * 12)(self.d_time, self.encoder_layers, self.encoder_heads, self.ffn_mult,
                                     self.d_head, self.crop_len, self.stride, self.synthetic_heads,
                                     m[self.stage_conv], m[self.stage_encoder], m[self.stage_cross],
                                     int(self.normalize_input))


def layer_pair(target_layer: int, geom: ModelGeometry) -> int:
    """mapper.cpp:44-49."""
    out = ctypes.c_int64()
    check(lib().pkv_layer_pair(int(target_layer), geom.as5(), ctypes.byref(out)))
    return out.value


def window_offsets(n: int, crop: int, stride: int) -> List[int]:
    """mapper.cpp:66-79."""
    cnt = ctypes.c_int64()
    check(lib().pkv_window_offsets(n, crop, stride, None, 0, ctypes.byref(cnt)))
    buf = (ctypes.c_int64 * max(cnt.value, 1))()
    check(lib().pkv_window_offsets(n, crop, stride, buf, cnt.value, ctypes.byref(cnt)))
    return list(buf[:cnt.value])


def mapper_init_params(geom: ModelGeometry, cfg: MapperConfig, seed: int) -> np.ndarray:
    """MapperParams::init (mapper.cpp:97-164) as the flat fp64 parameter blob."""
    cnt = ctypes.c_int64()
    check(lib().pkv_mapper_init_params(geom.as5(), cfg.as12(), seed, None, ctypes.byref(cnt)))
    blob = np.zeros(cnt.value, np.float64)
    check(lib().pkv_mapper_init_params(geom.as5(), cfg.as12(), seed, blob.ctypes.data, ctypes.byref(cnt)))
    return blob


class Mapper:
    """Device-resident HybridAxialMapper (pkv_mapper)."""

    def __init__(self, geom: ModelGeometry, cfg: MapperConfig, blob: np.ndarray = None, *, seed: int = 0,
                 precision: int = MAPPER_FP16X3, ctx: Context = None):
        self.geom, self.cfg = geom, cfg
        self.ctx = ctx or Context.default()
        if blob is None:
            blob = mapper_init_params(geom, cfg, seed)
        blob = np.ascontiguousarray(blob, np.float64)
        h = ctypes.c_void_p()
        check(lib().pkv_mapper_create(self.ctx.h, geom.as5(), cfg.as12(), blob.ctypes.data, blob.size,
                                      precision, ctypes.byref(h)))
        self.h = h

    @classmethod
    def from_checkpoint(cls, path: str, *, precision: int = MAPPER_FP16X3, ctx: "Context" = None) -> "Mapper":
        """A trained mapper (SPEC.md:198 checkpoint) on the device."""
        geom, cfg, blob = read_checkpoint(path)
        return cls(geom, cfg, blob, precision=precision, ctx=ctx)

    def __del__(self):
        h = getattr(self, "h", None)
        if h and _lib._lib is not None:
            _lib._lib.pkv_mapper_destroy(h)
            self.h = None

    def forward_full(self, x_all, stream=None, out=None):
        """x_all fp32 cuda [B, L_s, H_s, N] -> [B, L_l, H_l, N]."""
        torch = _torch()
        B, ls, hs, n = x_all.shape
        x = x_all.contiguous()
        y = out if out is not None else torch.empty((B, self.geom.target_layers, self.geom.target_heads, n),
                                                    dtype=torch.float32, device=x.device)
        check(lib().pkv_mapper_forward_full(self.h, _ptr(x), B, n, _ptr(y), _stream(stream)))
        return y

    def sliding_forward(self, x, stream=None):
        """x fp32 cuda [B, H_s, N] -> [B, H_l, N] (forward_pair when N <= crop_len)."""
        torch = _torch()
        B, hs, n = x.shape
        x = x.contiguous()
        y = torch.empty((B, self.geom.target_heads, n), dtype=torch.float32, device=x.device)
        check(lib().pkv_mapper_sliding_forward(self.h, _ptr(x), B, n, _ptr(y), _stream(stream)))
        return y

    def forward_pair(self, x, stream=None, trace: Optional[dict] = None):
        """forward_pair (mapper.cpp:274-342): x fp32 cuda [B, H_s, n <= crop_len] -> [B, H_l, n]; with
        `trace` a dict, trace["cross_attention"] = the Stage-3 attention [B, n, H_l, H_syn] (StageTrace)."""
        torch = _torch()
        B, hs, n = x.shape
        x = x.contiguous()
        y = torch.empty((B, self.geom.target_heads, n), dtype=torch.float32, device=x.device)
        attn = None
        if trace is not None and self.cfg.stage_cross == "active":
            syn = self.cfg.synthetic_heads or self.geom.proxy_heads
            attn = torch.empty((B, n, self.geom.target_heads, syn), dtype=torch.float32, device=x.device)
        check(lib().pkv_mapper_forward_pair(self.h, _ptr(x), B, n, _ptr(y), _ptr(attn), _stream(stream)))
        if trace is not None and attn is not None:
            trace["cross_attention"] = attn
        return y

    def forward_pair_host(self, x: np.ndarray, trace: Optional[dict] = None) -> np.ndarray:
        """The reference calling convention: fp64 host [B, H_s, n] -> fp64 host [B, H_l, n]."""
        x = np.ascontiguousarray(x, np.float64)
        B, hs, n = x.shape
        y = np.zeros((B, self.geom.target_heads, n))
        attn = None
        if trace is not None and self.cfg.stage_cross == "active":
            syn = self.cfg.synthetic_heads or self.geom.proxy_heads
            attn = np.zeros((B, n, self.geom.target_heads, syn))
        check(lib().pkv_mapper_forward_pair_host(self.h, x.ctypes.data, B, n, y.ctypes.data,
                                                 attn.ctypes.data if attn is not None else None))
        if attn is not None:
            trace["cross_attention"] = attn
        return y

    def sliding_forward_host(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        B, hs, n = x.shape
        y = np.zeros((B, self.geom.target_heads, n))
        check(lib().pkv_mapper_sliding_forward_host(self.h, x.ctypes.data, B, n, y.ctypes.data))
        return y

    def forward_full_host(self, x_all: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x_all, np.float64)
        B, ls, hs, n = x.shape
        y = np.zeros((B, self.geom.target_layers, self.geom.target_heads, n))
        check(lib().pkv_mapper_forward_full_host(self.h, x.ctypes.data, B, n, y.ctypes.data))
        return y


@dataclass(frozen=True)
class ShardPlan:
    """What one rank owns of one context (pkv_shard_plan; 0-based, half-open):
    it selects and compacts target slices [t_lo, t_hi) x heads [h_lo, h_hi),
    scores and maps proxy layers [p_lo, p_hi) and produces the mapped scores of
    target layers [a, b) (all heads)."""
    t_lo: int
    t_hi: int
    h_lo: int
    h_hi: int
    p_lo: int
    p_hi: int
    a: int
    b: int


def shard_plan(geom: ModelGeometry, world: int, rank: int, mode: int = SHARD_LAYER) -> ShardPlan:
    """Host logic only (no device): the multi-GPU partition of SURVEY §8e."""
    out = (ctypes.c_int64 * 8)()
    check(lib().pkv_shard_plan(geom.as5(), world, rank, mode, out))
    return ShardPlan(*[int(v) for v in out])


def shard_exchange_schedule(geom: ModelGeometry, world: int, rank: int, N: int) -> np.ndarray:
    """The head-group exchange of rank `rank` as int64 ops [n, 5] = (kind 0 send / 1 recv, peer,
    element offset, element count, tag = target layer) — exactly what the NCCL exchange issues
    (pkv_shard_exchange_schedule; host logic only)."""
    cnt = ctypes.c_int64()
    check(lib().pkv_shard_exchange_schedule(geom.as5(), world, rank, N, None, 0, ctypes.byref(cnt)))
    ops = np.zeros((max(cnt.value, 1), 5), np.int64)
    check(lib().pkv_shard_exchange_schedule(geom.as5(), world, rank, N, ops.ctypes.data, cnt.value,
                                            ctypes.byref(cnt)))
    return ops[:cnt.value]


class Comm:
    """pkv_comm: NCCL communicator for head-group sharding. `uid` is the
    PKV_COMM_ID_BYTES id from Comm.unique_id() on rank 0, distributed by the
    caller (e.g. torch.distributed.broadcast_object_list)."""

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(COMM_ID_BYTES)
        check(lib().pkv_comm_unique_id(buf))
        return buf.raw

    def __init__(self, ctx: Context, world: int, rank: int, uid: bytes):
        h = ctypes.c_void_p()
        check(lib().pkv_comm_create(ctx.h, world, rank, ctypes.create_string_buffer(uid, COMM_ID_BYTES),
                                    ctypes.byref(h)))
        self.h = h
        self.world = world
        self.rank = rank

    def __del__(self):
        h = getattr(self, "h", None)
        if h and _lib._lib is not None:
            _lib._lib.pkv_comm_destroy(h)
            self.h = None


class Pruner:
    """pkv_pruner: score -> map -> select -> compact for one context shape.
    With `shard=(mode, world, rank)` (and `comm` for SHARD_HEAD) the pruner
    handles this rank's part of the context; buffers are then shard-local
    (see pkv_pruner_create_sharded and `self.plan`)."""

    def __init__(self, mapper: Mapper, Hq: int, dp: int, dt: int, N: int, rho: float, *, reduce: str = "max",
                 causal: bool = False, shard: Optional[Tuple[int, int, int]] = None, comm: Optional[Comm] = None):
        self.mapper = mapper
        flags = (SCORE_REDUCE_SUM if reduce == "sum" else SCORE_REDUCE_MAX) | (SCORE_CAUSAL if causal else 0)
        h = ctypes.c_void_p()
        if shard is None:
            check(lib().pkv_pruner_create(mapper.ctx.h, mapper.h, Hq, dp, dt, N, float(rho), flags, ctypes.byref(h)))
            self.plan = ShardPlan(0, mapper.geom.target_layers, 0, mapper.geom.target_heads, 0,
                                  mapper.geom.proxy_layers, 0, mapper.geom.target_layers)
        else:
            mode, world, rank = shard
            check(lib().pkv_pruner_create_sharded(mapper.ctx.h, mapper.h, Hq, dp, dt, N, float(rho), flags, mode,
                                                  world, rank, comm.h if comm is not None else None,
                                                  ctypes.byref(h)))
            self.plan = shard_plan(mapper.geom, world, rank, mode)
        self.comm = comm
        self.h = h
        self.k = int(lib().pkv_pruner_k(h))
        self.N = N

    def __del__(self):
        h = getattr(self, "h", None)
        if h and _lib._lib is not None:
            _lib._lib.pkv_pruner_destroy(h)
            self.h = None

    def profile(self, runs: int):
        """Record stage-boundary CUDA events during the next `runs` device-resident runs."""
        check(lib().pkv_pruner_profile(self.h, int(runs)))

    def profile_read(self):
        """Per profiled run: ms of (LSE pass, pooled pass, map, select, compaction)."""
        cap = 4096
        buf = (ctypes.c_double * (cap * 5))()
        n = ctypes.c_int64()
        check(lib().pkv_pruner_profile_read(self.h, buf, cap, ctypes.byref(n)))
        return [tuple(buf[r * 5:(r + 1) * 5]) for r in range(n.value)]

    def run(self, q, kp, kt, vt, k_out, v_out, idx_out=None, scores_out=None, stream=None):
        check(lib().pkv_pruner_run(self.h, _ptr(q), _ptr(kp), _ptr(kt), _ptr(vt), _ptr(k_out), _ptr(v_out),
                                   _ptr(idx_out), _ptr(scores_out), _stream(stream)))

    def exchange(self, y_local, y_recv, stream=None):
        """Head-group sharding: the NCCL exchange step alone (y_local [b-a, H_l, N] -> y_recv [L_l, nh, N])."""
        check(lib().pkv_pruner_exchange(self.h, _ptr(y_local), _ptr(y_recv), _stream(stream)))

    def run_lse(self, q, kp, lse, kt, vt, k_out, v_out, idx_out=None, scores_out=None, stream=None):
        """Paper regime: the row LSE [L_s, Hq, N] from the proxy's prefill attention
        (proxy_prefill_attention), so scoring is the pooled pass alone."""
        check(lib().pkv_pruner_run_lse(self.h, _ptr(q), _ptr(kp), _ptr(lse.contiguous()), _ptr(kt), _ptr(vt),
                                       _ptr(k_out), _ptr(v_out), _ptr(idx_out), _ptr(scores_out), _stream(stream)))

    def run_dual(self, q, kp, kt, vt, k_out, v_out, idx_out=None, scores_out=None, *, proxy_stream, target_stream):
        """Scoring + mapping on proxy_stream, select + compaction on target_stream."""
        check(lib().pkv_pruner_run_dual(self.h, _ptr(q), _ptr(kp), _ptr(kt), _ptr(vt), _ptr(k_out), _ptr(v_out),
                                        _ptr(idx_out), _ptr(scores_out), _stream(proxy_stream),
                                        _stream(target_stream)))

    def run_two_device(self, target_ctx: "Context", q, kp, kt, vt, k_out, v_out, idx_out=None, scores_out=None, *,
                       proxy_stream=None, target_stream=None):
        """Paper regime: score + map on this pruner's device (q, kp there), Ŷ peer-copied to
        target_ctx's device, select + compaction there (kt, vt, outputs there)."""
        check(lib().pkv_pruner_run_two_device(self.h, target_ctx.h, _ptr(q), _ptr(kp), _ptr(kt), _ptr(vt),
                                              _ptr(k_out), _ptr(v_out), _ptr(idx_out), _ptr(scores_out),
                                              _stream(proxy_stream), _stream(target_stream)))

    def run_host(self, q, kp, kt, vt, k_out, v_out, idx_out=None, stream=None):
        """Host (ideally pinned) torch tensors in and out; copies happen inside the call."""
        check(lib().pkv_pruner_run_host(self.h, _ptr(q), _ptr(kp), _ptr(kt), _ptr(vt), _ptr(k_out), _ptr(v_out),
                                        _ptr(idx_out), _stream(stream)))


# ------------------------------------------------------------ file formats --
def write_trace(path: str, x: np.ndarray, y: np.ndarray, meta: str = "") -> None:
    """PKVT trace: x fp32 [S, B, L_s, H_s, N], y fp32 [S, B, L_l, H_l, N]."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    y = np.ascontiguousarray(y, dtype=np.float32)
    if x.ndim != 5 or y.ndim != 5 or x.shape[0] != y.shape[0] or x.shape[1] != y.shape[1] or x.shape[4] != y.shape[4]:
        raise ShapeError(f"trace expects x [S,B,L_s,H_s,N] and y [S,B,L_l,H_l,N], got {x.shape} and {y.shape}")
    S, B, Ls, Hs, N = x.shape
    g = (ctypes.c_int64 * 6)(Ls, Hs, y.shape[2], y.shape[3], N, B)
    check(lib().pkv_trace_write(path.encode(), g, S, x.ctypes.data, y.ctypes.data, meta.encode()))


def read_trace(path: str) -> Tuple[np.ndarray, np.ndarray]:
    g = (ctypes.c_int64 * 6)()
    n = ctypes.c_int64()
    check(lib().pkv_trace_read_header(path.encode(), g, ctypes.byref(n)))
    Ls, Hs, Ll, Hl, N, B = (int(v) for v in g)
    x = np.empty((n.value, B, Ls, Hs, N), np.float32)
    y = np.empty((n.value, B, Ll, Hl, N), np.float32)
    check(lib().pkv_trace_read(path.encode(), x.ctypes.data, y.ctypes.data))
    return x, y


def write_checkpoint(path: str, geom: ModelGeometry, cfg: MapperConfig, blob: np.ndarray) -> None:
    """Mapper checkpoint of a pkv_mapper_init_params-layout fp64 blob."""
    b = np.ascontiguousarray(blob, dtype=np.float64)
    check(lib().pkv_checkpoint_write(path.encode(), geom.as5(), cfg.as12(), b.ctypes.data, b.size))


def read_checkpoint(path: str) -> Tuple[ModelGeometry, MapperConfig, np.ndarray]:
    g = (ctypes.c_int64 * 5)()
    c = (ctypes.c_int64 * 12)()
    n = ctypes.c_int64()
    check(lib().pkv_checkpoint_read(path.encode(), g, c, None, ctypes.byref(n)))
    blob = np.empty(n.value, np.float64)
    check(lib().pkv_checkpoint_read(path.encode(), g, c, blob.ctypes.data, ctypes.byref(n)))
    modes = ("active", "bypass")
    cfg = MapperConfig(d_time=c[0], encoder_layers=c[1], encoder_heads=c[2], ffn_mult=c[3], d_head=c[4],
                       crop_len=c[5], stride=c[6], synthetic_heads=c[7], stage_conv=modes[c[8]],
                       stage_encoder=modes[c[9]], stage_cross=modes[c[10]], normalize_input=bool(c[11]))
    return ModelGeometry(*[int(v) for v in g]), cfg, blob
