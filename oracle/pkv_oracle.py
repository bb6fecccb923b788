"""CPU restatement of the ProxyKV pruning hot path — the parity ORACLE.

TEST INFRASTRUCTURE ONLY. Only tests/, ``__graft_entry__.smoke()`` and
``bench.py``'s cpu_baseline / ``--impl reference`` legs may import this module,
and only as the checker or the timed CPU baseline — never as the product. The
product (``paper_2605_16360_b200``) has no CPU fallback.

Two layers:

* ``libpkvoracle.so`` (oracle/pkv_oracle.c): plain-C restatement of select,
  apply_mask, compaction, scoring, the reference RNG and ``MapperParams::init``.
* numpy fp64 restatement of the HybridAxialMapper forward
  (``/root/reference/proj/src/mapper.cpp:274-398`` over ``ops.cpp``).

``RefLib`` wraps ``oracle/_ref/libpkvref.so`` — the reference's own C++ sources
compiled by oracle/Makefile — used to pin the restatement (tests/test_oracle.py)
and as the ``kind: "reference"`` CPU baseline.

Citations are ``path:line`` into /root/reference/.
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DIR = os.path.join(HERE, "_ref")

_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)
_f32p = ctypes.POINTER(ctypes.c_float)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_u16p = ctypes.POINTER(ctypes.c_uint16)
_i32p = ctypes.POINTER(ctypes.c_int32)
_u64p = ctypes.POINTER(ctypes.c_uint64)


def _ptr(a: np.ndarray, t):
    return a.ctypes.data_as(t)


class OracleError(Exception):
    pass


# --------------------------------------------------------------- C oracle --
_olib = None


def olib():
    """Loads oracle/_ref/libpkvoracle.so (built by oracle/Makefile)."""
    global _olib
    if _olib is None:
        path = os.path.join(REF_DIR, "libpkvoracle.so")
        if not os.path.exists(path):
            raise OracleError(f"{path} missing: run `make -C oracle oracle`")
        lib = ctypes.CDLL(path)
        lib.pkvo_retention_count.argtypes = [ctypes.c_double, ctypes.c_int64, _i64p]
        lib.pkvo_topk_select_f32.argtypes = [_f32p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _u8p, _i32p]
        lib.pkvo_compact_kv.argtypes = [_u16p, _u16p, _i32p] + [ctypes.c_int64] * 4 + [_u16p, _u16p]
        lib.pkvo_compact_kv.restype = None
        lib.pkvo_score_head.argtypes = [_u16p, _u16p] + [ctypes.c_int64] * 4 + [ctypes.c_int, ctypes.c_int, _f32p]
        lib.pkvo_score_head.restype = None
        lib.pkvo_score_lse.argtypes = [_u16p, _u16p] + [ctypes.c_int64] * 3 + [ctypes.c_int, _f32p]
        lib.pkvo_score_lse.restype = None
        lib.pkvo_mapper_init.argtypes = [_i64p, _i64p, ctypes.c_uint64, _f64p]
        lib.pkvo_mapper_init.restype = ctypes.c_int64
        lib.pkvo_rng_uniform.argtypes = [ctypes.c_uint64, ctypes.c_double, ctypes.c_double, ctypes.c_int64, _f64p]
        lib.pkvo_rng_uniform.restype = None
        lib.pkvo_rng_normal.argtypes = [ctypes.c_uint64, ctypes.c_int64, _f64p]
        lib.pkvo_rng_normal.restype = None
        lib.pkvo_rng_below.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64, _u64p]
        lib.pkvo_rng_below.restype = None
        _olib = lib
    return _olib


def retention_count(rho: float, n: int) -> int:
    """pruning.cpp:14-18 — ceil(rho * n) in double; ValueError outside (0, 1]."""
    k = ctypes.c_int64()
    if olib().pkvo_retention_count(float(rho), int(n), ctypes.byref(k)) != 0:
        raise ValueError(f"retention ratio must be in (0, 1], got {rho} (n={n})")
    return k.value


def topk_select(scores: np.ndarray, k: int) -> Tuple[np.ndarray, np.ndarray]:
    """pruning.cpp:20-56 + 197-215 restated: returns (mask u8 [..., n], idx_asc i32 [slices, k])."""
    s = np.ascontiguousarray(scores, dtype=np.float32)
    n = s.shape[-1]
    slices = s.size // n
    mask = np.zeros(s.shape, np.uint8)
    idx = np.zeros((slices, k), np.int32)
    rc = olib().pkvo_topk_select_f32(_ptr(s, _f32p), slices, n, k, _ptr(mask, _u8p), _ptr(idx, _i32p))
    if rc == 2:
        raise ValueError(f"top-k count {k} out of range for length {n}")
    if rc == 3:
        raise ValueError("NaN score")
    return mask, idx


def compact_kv(k_bits: np.ndarray, v_bits: np.ndarray, idx_asc: np.ndarray) -> Tuple[np.ndarray, np.ndarray]:
    """Packed gather in apply_mask order. k_bits/v_bits: uint16 [slices, n, d]."""
    kb = np.ascontiguousarray(k_bits, dtype=np.uint16)
    vb = np.ascontiguousarray(v_bits, dtype=np.uint16)
    ix = np.ascontiguousarray(idx_asc, dtype=np.int32)
    slices, n, d = kb.shape
    k = ix.shape[1]
    ko = np.zeros((slices, k, d), np.uint16)
    vo = np.zeros((slices, k, d), np.uint16)
    olib().pkvo_compact_kv(_ptr(kb, _u16p), _ptr(vb, _u16p), _ptr(ix, _i32p), slices, n, k, d, _ptr(ko, _u16p), _ptr(vo, _u16p))
    return ko, vo


def score(q_bits: np.ndarray, k_bits: np.ndarray, reduce: str = "max", causal: bool = False) -> np.ndarray:
    """Proxy scoring restated (north-star max-pool).

    q_bits: uint16 bf16 [L, Hq, Nq, d]; k_bits: uint16 bf16 [L, Hkv, Nk, d] -> X fp32 [L, Hkv, Nk].
    """
    L, hq, nq, d = q_bits.shape
    _, hkv, nk, _ = k_bits.shape
    g = hq // hkv
    out = np.zeros((L, hkv, nk), np.float32)
    lib = olib()
    for l in range(L):
        for h in range(hkv):
            q = np.ascontiguousarray(q_bits[l, h * g:(h + 1) * g], dtype=np.uint16)
            kk = np.ascontiguousarray(k_bits[l, h], dtype=np.uint16)
            x = np.zeros(nk, np.float32)
            lib.pkvo_score_head(_ptr(q, _u16p), _ptr(kk, _u16p), g, nq, nk, d, 0 if reduce == "sum" else 1,
                                1 if causal else 0, _ptr(x, _f32p))
            out[l, h] = x
    return out


def score_lse(q_bits: np.ndarray, k_bits: np.ndarray, causal: bool = False) -> np.ndarray:
    """Row LSE per query head: q [L, Hq, Nq, d], k [L, Hkv, Nk, d] -> [L, Hq, Nq] fp32."""
    L, hq, nq, d = q_bits.shape
    _, hkv, nk, _ = k_bits.shape
    g = hq // hkv
    out = np.zeros((L, hq, nq), np.float32)
    for l in range(L):
        for h in range(hq):
            q = np.ascontiguousarray(q_bits[l, h], dtype=np.uint16)
            kk = np.ascontiguousarray(k_bits[l, h // g], dtype=np.uint16)
            x = np.zeros(nq, np.float32)
            olib().pkvo_score_lse(_ptr(q, _u16p), _ptr(kk, _u16p), nq, nk, d, 1 if causal else 0, _ptr(x, _f32p))
            out[l, h] = x
    return out


# ------------------------------------------------------------ bf16 helpers --
def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16 bit patterns (uint16)."""
    u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    return r


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint32) << 16).view(np.float32)


# ------------------------------------------------------------------ mapper --
@dataclass
class Geometry:
    """ModelGeometry, mapper.hpp:16-25."""
    target_layers: int = 32
    target_heads: int = 32
    proxy_layers: int = 16
    proxy_heads: int = 32
    head_dim: int = 128

    def as5(self) -> List[int]:
        return [self.target_layers, self.target_heads, self.proxy_layers, self.proxy_heads, self.head_dim]


@dataclass
class MapperConfig:
    """MapperConfig, mapper.hpp:35-55 (stage modes: 'active' | 'bypass')."""
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

    def conv_mid(self) -> int:
        return self.d_time // 2 if self.d_time // 2 > 0 else 1

    def syn(self, g: Geometry) -> int:
        return self.synthetic_heads if self.synthetic_heads > 0 else g.proxy_heads

    def as12(self) -> List[int]:
        m = {"active": 0, "bypass": 1}
        return [self.d_time, self.encoder_layers, self.encoder_heads, self.ffn_mult, self.d_head, self.crop_len,
                self.stride, self.synthetic_heads, m[self.stage_conv], m[self.stage_encoder], m[self.stage_cross],
                int(self.normalize_input)]


def param_layout(g: Geometry, c: MapperConfig) -> List[Tuple[str, Tuple[int, ...]]]:
    """named_parameters() + named_buffers() order and shapes (mapper.cpp:166-225, 97-164)."""
    hs, dt, mid, dh = g.proxy_heads, c.d_time, c.conv_mid(), c.d_head
    syn, ffn = c.syn(g), c.ffn_mult * c.d_time
    out: List[Tuple[str, Tuple[int, ...]]] = []
    if c.stage_conv == "active":
        out += [("stem.conv1.w", (mid, hs, 3)), ("stem.conv1.b", (mid,)), ("stem.bn1.gamma", (mid,)),
                ("stem.bn1.beta", (mid,)), ("stem.conv2.w", (dt, mid, 3)), ("stem.conv2.b", (dt,)),
                ("stem.bn2.gamma", (dt,)), ("stem.bn2.beta", (dt,))]
    else:
        out += [("stem.bypass.w", (dt, hs, 1)), ("stem.bypass.b", (dt,))]
    if c.stage_encoder == "active":
        for i in range(c.encoder_layers):
            p = f"encoder.{i}."
            for m in ("q", "k", "v", "o"):
                out += [(p + f"attn.w{m}", (dt, dt)), (p + f"attn.b{m}", (dt,))]
            out += [(p + "ln1.gamma", (dt,)), (p + "ln1.beta", (dt,)), (p + "ln2.gamma", (dt,)),
                    (p + "ln2.beta", (dt,)), (p + "ffn1.w", (dt, ffn)), (p + "ffn1.b", (ffn,)),
                    (p + "ffn2.w", (ffn, dt)), (p + "ffn2.b", (dt,))]
    if c.stage_cross == "active":
        out += [("cross.key.w", (dt, syn * dh)), ("cross.key.b", (syn * dh,))]
    out += [("cross.value.w", (dt, syn * dh)), ("cross.value.b", (syn * dh,))]
    if c.stage_cross == "active":
        out += [("cross.queries", (g.target_heads, dh))]
    out += [("cross.out.w", (dh, 1)), ("cross.out.b", (1,))]
    if c.stage_conv == "active":
        out += [("stem.bn1.running_mean", (mid,)), ("stem.bn1.running_var", (mid,)),
                ("stem.bn2.running_mean", (dt,)), ("stem.bn2.running_var", (dt,))]
    return out


def mapper_init_blob(g: Geometry, c: MapperConfig, seed: int) -> np.ndarray:
    """MapperParams::init (mapper.cpp:97-164) restated in C: flat fp64 blob in layout order."""
    g5 = np.array(g.as5(), np.int64)
    c12 = np.array(c.as12(), np.int64)
    n = olib().pkvo_mapper_init(_ptr(g5, _i64p), _ptr(c12, _i64p), seed, None)
    blob = np.zeros(n, np.float64)
    olib().pkvo_mapper_init(_ptr(g5, _i64p), _ptr(c12, _i64p), seed, _ptr(blob, _f64p))
    return blob


def unpack_blob(g: Geometry, c: MapperConfig, blob: np.ndarray) -> Dict[str, np.ndarray]:
    params: Dict[str, np.ndarray] = {}
    pos = 0
    for name, shape in param_layout(g, c):
        n = int(np.prod(shape))
        params[name] = np.asarray(blob[pos:pos + n], np.float64).reshape(shape)
        pos += n
    if pos != blob.size:
        raise OracleError(f"blob has {blob.size} values, layout expects {pos}")
    return params


@dataclass
class MapperParams:
    geometry: Geometry
    config: MapperConfig
    p: Dict[str, np.ndarray] = field(default_factory=dict)

    @staticmethod
    def init(g: Geometry, c: MapperConfig, seed: int) -> "MapperParams":
        return MapperParams(g, c, unpack_blob(g, c, mapper_init_blob(g, c, seed)))


def layer_pair(target_layer: int, g: Geometry) -> int:
    """mapper.cpp:44-49: ceil(l_l * L_s / L_l) in integer arithmetic (1-based)."""
    if not (1 <= target_layer <= g.target_layers):
        raise ValueError(f"target layer {target_layer} out of range [1, {g.target_layers}]")
    return (target_layer * g.proxy_layers + g.target_layers - 1) // g.target_layers


def sinusoidal_pe(n: int, d_time: int) -> np.ndarray:
    """mapper.cpp:51-64 (element-wise, same pow/sin/cos calls as the reference)."""
    if d_time <= 0 or d_time % 2:
        raise ValueError(f"positional encoding width must be even, got {d_time}")
    pe = np.zeros((n, d_time))
    omega = np.array([math.pow(10000.0, -2.0 * i / d_time) for i in range(d_time // 2)])
    pos = np.arange(n, dtype=np.float64)[:, None]
    arg = pos * omega[None, :]
    pe[:, 0::2] = np.sin(arg)
    pe[:, 1::2] = np.cos(arg)
    return pe


def window_offsets(n: int, crop: int, stride: int) -> List[int]:
    """mapper.cpp:66-79: stride-spaced windows plus a right-aligned tail."""
    if n <= 0 or crop <= 0 or stride <= 0:
        raise ValueError("window parameters must be positive")
    if n <= crop:
        return [0]
    offs = list(range(0, n - crop + 1, stride))
    if offs[-1] + crop < n:
        offs.append(n - crop)
    return offs


def _erf(x: np.ndarray) -> np.ndarray:
    from scipy.special import erf
    return erf(x)


def _gelu(x):
    """ops.cpp:225-234, exact erf form."""
    return 0.5 * x * (1.0 + _erf(x * 0.7071067811865475244))


def _conv1d(x, w, b, pad):
    """ops.cpp:582-629: cross-correlation, zero padding. x [B, Cin, n], w [Cout, Cin, k]."""
    B, cin, n = x.shape
    cout, _, k = w.shape
    n_out = n + 2 * pad - k + 1
    xp = np.zeros((B, cin, n + 2 * pad))
    xp[:, :, pad:pad + n] = x
    col = np.stack([xp[:, :, t:t + n_out] for t in range(k)], axis=2)  # [B, Cin, k, n_out]
    col = col.reshape(B, cin * k, n_out)
    out = np.einsum("oc,bcn->bon", w.reshape(cout, cin * k), col, optimize=True)
    return out + b[None, :, None]


def _bn_eval(x, g, b, rm, rv, eps=1e-5):
    """ops.cpp:852-875 eval branch: (x - mean) * (1/sqrt(var + eps)) * gamma + beta."""
    ic = 1.0 / np.sqrt(rv + eps)
    return (x - rm[None, :, None]) * ic[None, :, None] * g[None, :, None] + b[None, :, None]


def _layernorm(x, g, b, eps=1e-5):
    """ops.cpp:721-754."""
    mu = x.mean(axis=-1, keepdims=True)
    c = x - mu
    var = (c * c).mean(axis=-1, keepdims=True)
    inv = 1.0 / np.sqrt(var + eps)
    return g * (c * inv) + b


def _softmax(x, axis):
    """ops.cpp:670-700."""
    m = x.max(axis=axis, keepdims=True)
    e = np.exp(x - m)
    return e / e.sum(axis=axis, keepdims=True)


def _encoder_attention(h, P, pre, heads):
    """mapper.cpp:254-270: non-causal MHA over [B, n, D], scale 1/sqrt(dh)."""
    B, n, d = h.shape
    dh = d // heads

    def split(t):
        return t.reshape(B, n, heads, dh).transpose(0, 2, 1, 3)

    q = split(h @ P[pre + "attn.wq"] + P[pre + "attn.bq"])
    k = split(h @ P[pre + "attn.wk"] + P[pre + "attn.bk"])
    v = split(h @ P[pre + "attn.wv"] + P[pre + "attn.bv"])
    s = (q @ k.transpose(0, 1, 3, 2)) * (1.0 / math.sqrt(dh))
    a = _softmax(s, 3)
    ctx = (a @ v).transpose(0, 2, 1, 3).reshape(B, n, d)
    return ctx @ P[pre + "attn.wo"] + P[pre + "attn.bo"]


def forward_pair(x: np.ndarray, mp: MapperParams, trace: Optional[dict] = None) -> np.ndarray:
    """mapper.cpp:274-342 (eval): x [B, H_s, n] -> raw logits [B, H_l, n]."""
    g, c, P = mp.geometry, mp.config, mp.p
    x = np.asarray(x, np.float64)
    if x.ndim != 3:
        raise ValueError(f"forward_pair input must be [B, H_s, N], got {list(x.shape)}")
    if x.shape[1] != g.proxy_heads:
        raise ValueError(f"input has {x.shape[1]} proxy heads, geometry expects {g.proxy_heads}")
    if x.shape[2] > c.crop_len:
        raise ValueError(f"input length {x.shape[2]} exceeds crop_len {c.crop_len}; long inputs go through sliding_forward")
    B, _, n = x.shape
    if c.normalize_input:
        x = x / np.maximum(x.mean(axis=2, keepdims=True), 1e-12)
    if c.stage_conv == "active":
        z = _gelu(_bn_eval(_conv1d(x, P["stem.conv1.w"], P["stem.conv1.b"], 1), P["stem.bn1.gamma"],
                           P["stem.bn1.beta"], P["stem.bn1.running_mean"], P["stem.bn1.running_var"]))
        z = _gelu(_bn_eval(_conv1d(z, P["stem.conv2.w"], P["stem.conv2.b"], 1), P["stem.bn2.gamma"],
                           P["stem.bn2.beta"], P["stem.bn2.running_mean"], P["stem.bn2.running_var"]))
    else:
        z = _conv1d(x, P["stem.bypass.w"], P["stem.bypass.b"], 0)
    z = z.transpose(0, 2, 1)
    if c.stage_encoder == "active":
        z = z + sinusoidal_pe(n, c.d_time)
        for i in range(c.encoder_layers):
            pre = f"encoder.{i}."
            z = z + _encoder_attention(_layernorm(z, P[pre + "ln1.gamma"], P[pre + "ln1.beta"]), P, pre,
                                       c.encoder_heads)
            h = _layernorm(z, P[pre + "ln2.gamma"], P[pre + "ln2.beta"])
            z = z + (_gelu(h @ P[pre + "ffn1.w"] + P[pre + "ffn1.b"]) @ P[pre + "ffn2.w"] + P[pre + "ffn2.b"])
    else:
        z = z + z.mean(axis=1, keepdims=True)
    syn, dh = c.syn(g), c.d_head
    values = (z @ P["cross.value.w"] + P["cross.value.b"]).reshape(B, n, syn, dh)
    if c.stage_cross == "active":
        keys = (z @ P["cross.key.w"] + P["cross.key.b"]).reshape(B, n, syn, dh)
        s = np.einsum("hd,bnsd->bnhs", P["cross.queries"], keys) * (1.0 / math.sqrt(dh))
        a = _softmax(s, 3)
        if trace is not None:
            trace["cross_attention"] = a
        heads = a @ values
    else:
        heads = np.broadcast_to(values.mean(axis=2, keepdims=True), (B, n, g.target_heads, dh))
    logits = (heads @ P["cross.out.w"] + P["cross.out.b"]).reshape(B, n, g.target_heads)
    return logits.transpose(0, 2, 1).copy()


def sliding_forward(x: np.ndarray, mp: MapperParams) -> np.ndarray:
    """mapper.cpp:344-377: ascending-offset accumulation, then /coverage count."""
    c = mp.config
    n = x.shape[2]
    if n <= c.crop_len:
        return forward_pair(x, mp)
    B, hl = x.shape[0], mp.geometry.target_heads
    acc = np.zeros((B, hl, n))
    counts = np.zeros(n)
    for off in window_offsets(n, c.crop_len, c.stride):
        acc[:, :, off:off + c.crop_len] += forward_pair(x[:, :, off:off + c.crop_len], mp)
        counts[off:off + c.crop_len] += 1.0
    return acc / counts


def forward_full(x_all: np.ndarray, mp: MapperParams) -> np.ndarray:
    """mapper.cpp:379-398: [B, L_s, H_s, N] -> [B, L_l, H_l, N]. Shared proxy layers are computed
    once (bit-identical to recomputation, test_mapper.cpp:283-291)."""
    g = mp.geometry
    if x_all.ndim != 4 or x_all.shape[1] != g.proxy_layers or x_all.shape[2] != g.proxy_heads:
        raise ValueError(f"forward_full input must be [B, {g.proxy_layers}, {g.proxy_heads}, N], got {list(x_all.shape)}")
    cache: Dict[int, np.ndarray] = {}
    outs = []
    for ll in range(1, g.target_layers + 1):
        ls = layer_pair(ll, g)
        if ls not in cache:
            cache[ls] = sliding_forward(x_all[:, ls - 1], mp)
        outs.append(cache[ls])
    return np.stack(outs, axis=1)


def topk_overlap_per_slice(mask_a: np.ndarray, mask_b: np.ndarray, k: int) -> np.ndarray:
    """pruning.cpp:91-108."""
    n = mask_a.shape[-1]
    a = mask_a.reshape(-1, n).astype(bool)
    b = mask_b.reshape(-1, n).astype(bool)
    return (a & b).sum(axis=1) / float(k)


def average_ranks(v: np.ndarray) -> np.ndarray:
    """pruning.cpp:122-140: 1-based ranks along the last axis, ties sharing the
    mean of their positions (a stable sort; -0.0 == +0.0 as in a double compare)."""
    v = np.asarray(v, np.float64) + 0.0  # folds -0.0 onto +0.0
    n = v.shape[-1]
    flat = v.reshape(-1, n)
    out = np.empty_like(flat)
    for s in range(flat.shape[0]):
        order = np.argsort(flat[s], kind="stable")
        sv = flat[s][order]
        head = np.r_[True, sv[1:] != sv[:-1]]
        start = np.maximum.accumulate(np.where(head, np.arange(n), 0))
        tail = np.r_[sv[1:] != sv[:-1], True]
        end = np.minimum.accumulate(np.where(tail, np.arange(n), n)[::-1])[::-1]
        out[s, order] = 0.5 * (start + end) + 1.0
    return out.reshape(v.shape)


def spearman_per_slice(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """pruning.cpp:142-186: Pearson of the average ranks per slice; 1 when both
    slices are constant, 0 when exactly one is."""
    n = a.shape[-1]
    if a.shape != b.shape:
        raise ValueError("spearman shapes differ")
    if n < 2:
        raise ValueError("spearman needs at least two tokens per slice")
    ra = average_ranks(a).reshape(-1, n)
    rb = average_ranks(b).reshape(-1, n)
    out = np.empty(ra.shape[0])
    for s in range(ra.shape[0]):
        da, db = ra[s] - ra[s].mean(), rb[s] - rb[s].mean()
        saa, sbb = (da * da).sum(), (db * db).sum()
        if saa == 0.0 and sbb == 0.0:
            out[s] = 1.0
        elif saa == 0.0 or sbb == 0.0:
            out[s] = 0.0
        else:
            out[s] = (da * db).sum() / np.sqrt(saa * sbb)
    return out


# ---------------------------------------------------- compiled reference ----
class RefLib:
    """ctypes view of oracle/_ref/libpkvref.so: the UNMODIFIED reference compiled here."""

    def __init__(self, path: Optional[str] = None):
        path = path or os.path.join(REF_DIR, "libpkvref.so")
        if not os.path.exists(path):
            raise OracleError(f"{path} missing: run `make -C oracle` where /root/reference exists")
        L = ctypes.CDLL(path)
        L.pkvref_last_error.restype = ctypes.c_char_p
        L.pkvref_retention_count.argtypes = [ctypes.c_double, ctypes.c_int64, _i64p]
        L.pkvref_topk_indices.argtypes = [_f64p, ctypes.c_int64, ctypes.c_int64, _i64p]
        L.pkvref_topk_mask.argtypes = [_f64p, _i64p, ctypes.c_int, ctypes.c_double, _u8p, _i64p]
        L.pkvref_apply_mask.argtypes = [_u8p, _i64p, ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                        _i64p, _i64p, _i64p, _i64p]
        L.pkvref_topk_overlap_per_slice.argtypes = [_u8p, _u8p, _i64p, ctypes.c_int, ctypes.c_int64,
                                                    ctypes.c_int64, _f64p]
        L.pkvref_layer_pair.argtypes = [ctypes.c_int64, _i64p, _i64p]
        L.pkvref_window_offsets.argtypes = [ctypes.c_int64] * 3 + [_i64p, ctypes.c_int64, _i64p]
        L.pkvref_sinusoidal_pe.argtypes = [ctypes.c_int64, ctypes.c_int64, _f64p]
        L.pkvref_mapper_create.argtypes = [_i64p, _i64p, ctypes.c_uint64, ctypes.POINTER(ctypes.c_void_p)]
        L.pkvref_mapper_destroy.argtypes = [ctypes.c_void_p]
        L.pkvref_mapper_destroy.restype = None
        L.pkvref_mapper_tensor_count.argtypes = [ctypes.c_void_p]
        L.pkvref_mapper_tensor.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_char_p, ctypes.c_int, _i64p,
                                           ctypes.POINTER(ctypes.c_int), _f64p]
        for fn in ("pkvref_forward_pair", "pkvref_sliding_forward"):
            getattr(L, fn).argtypes = [ctypes.c_void_p, _f64p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64, _f64p]
        L.pkvref_forward_full.argtypes = [ctypes.c_void_p, _f64p] + [ctypes.c_int64] * 4 + [_f64p]
        L.pkvref_rng_create.argtypes = [ctypes.c_uint64]
        L.pkvref_rng_create.restype = ctypes.c_void_p
        L.pkvref_rng_destroy.argtypes = [ctypes.c_void_p]
        L.pkvref_rng_destroy.restype = None
        L.pkvref_rng_uniform.argtypes = [ctypes.c_void_p, ctypes.c_double, ctypes.c_double]
        L.pkvref_rng_uniform.restype = ctypes.c_double
        L.pkvref_rng_below.argtypes = [ctypes.c_void_p, ctypes.c_uint64]
        L.pkvref_rng_below.restype = ctypes.c_uint64
        L.pkvref_rng_normal.argtypes = [ctypes.c_void_p]
        L.pkvref_rng_normal.restype = ctypes.c_double
        self.L = L

    def _check(self, rc: int):
        if rc == 0:
            return
        msg = self.L.pkvref_last_error().decode()
        if rc == 1:
            raise OracleError("ShapeError: " + msg)
        if rc == 2:
            raise ValueError(msg)
        raise OracleError(msg)

    def retention_count(self, rho, n):
        k = ctypes.c_int64()
        self._check(self.L.pkvref_retention_count(rho, n, ctypes.byref(k)))
        return k.value

    def topk_mask(self, scores: np.ndarray, rho: float) -> Tuple[np.ndarray, int]:
        s = np.ascontiguousarray(scores, np.float64)
        shape = np.array(s.shape, np.int64)
        bits = np.zeros(s.shape, np.uint8)
        k = ctypes.c_int64()
        self._check(self.L.pkvref_topk_mask(_ptr(s, _f64p), _ptr(shape, _i64p), s.ndim, rho, _ptr(bits, _u8p),
                                            ctypes.byref(k)))
        return bits, k.value

    def captured_mass_per_slice(self, pred_bits: np.ndarray, k: int, y: np.ndarray) -> np.ndarray:
        """The reference's captured_mass_per_slice (pruning.cpp:58-80)."""
        yy = np.ascontiguousarray(y, np.float64)
        pb = np.ascontiguousarray(pred_bits, np.uint8)
        shape = np.array(yy.shape, np.int64)
        out = np.zeros(yy.size // yy.shape[-1], np.float64)
        self.L.pkvref_captured_mass_per_slice.argtypes = [_u8p, ctypes.c_int64, _f64p, _i64p, ctypes.c_int, _f64p]
        self._check(self.L.pkvref_captured_mass_per_slice(_ptr(pb, _u8p), k, _ptr(yy, _f64p), _ptr(shape, _i64p),
                                                          yy.ndim, _ptr(out, _f64p)))
        return out

    def spearman_per_slice(self, a: np.ndarray, b: np.ndarray) -> np.ndarray:
        """The reference's spearman_per_slice (pruning.cpp:173-186)."""
        aa = np.ascontiguousarray(a, np.float64)
        bb = np.ascontiguousarray(b, np.float64)
        shape = np.array(aa.shape, np.int64)
        out = np.zeros(aa.size // aa.shape[-1], np.float64)
        self.L.pkvref_spearman_per_slice.argtypes = [_f64p, _f64p, _i64p, ctypes.c_int, _f64p]
        self._check(self.L.pkvref_spearman_per_slice(_ptr(aa, _f64p), _ptr(bb, _f64p), _ptr(shape, _i64p), aa.ndim,
                                                     _ptr(out, _f64p)))
        return out

    def loss_total(self, logits: np.ndarray, y: np.ndarray, cfg, seed: int, want_grad: bool = True):
        """The reference's loss_total (loss.cpp:324-374) and, through its tape,
        d total / d logits. cfg: any object with LossConfig's field names."""
        z = np.ascontiguousarray(logits, np.float64)
        yy = np.ascontiguousarray(y, np.float64)
        shape = np.array(z.shape, np.int64)
        cf = np.array([cfg.lambda_mse, cfg.lambda_bin, cfg.lambda_fine, cfg.lambda_global, cfg.lambda_cos, cfg.gamma,
                       cfg.epsilon, cfg.mse_exponent, cfg.margin, cfg.clip_lo, cfg.clip_hi, cfg.pair_filter_frac,
                       cfg.topk_ratio_for_rank], np.float64)
        ratios = np.ascontiguousarray(cfg.ratios, np.float64)
        rep = np.zeros(12, np.float64)
        cnt = np.zeros(5, np.int64)
        grad = np.zeros_like(z) if want_grad else None
        self.L.pkvref_loss_total.argtypes = [_f64p, _f64p, _i64p, ctypes.c_int, _f64p, _f64p, ctypes.c_int64,
                                             ctypes.c_int64, ctypes.c_uint64, _f64p, _i64p, ctypes.c_void_p]
        self._check(self.L.pkvref_loss_total(_ptr(z, _f64p), _ptr(yy, _f64p), _ptr(shape, _i64p), z.ndim,
                                             _ptr(cf, _f64p), _ptr(ratios, _f64p), len(ratios), int(cfg.max_pairs),
                                             seed, _ptr(rep, _f64p), _ptr(cnt, _i64p),
                                             grad.ctypes.data if want_grad else None))
        names = ["bin", "mse", "fine", "global", "cos", "weighted_bin", "weighted_mse", "weighted_fine",
                 "weighted_global", "weighted_cos", "total", "s_max"]
        out = dict(zip(names, rep.tolist()))
        out.update(fine_used=int(cnt[0]), fine_filtered=int(cnt[1]), global_used=int(cnt[2]),
                   global_filtered=int(cnt[3]), cos_floor_hits=int(cnt[4]))
        return out, grad

    def mapper_train_grad(self, m: "RefMapper", x: np.ndarray, dlogits: np.ndarray):
        """Training-mode forward_pair + the tape's reverse sweep of Σ dlogits ⊙ logits
        (ref_capi.cpp pkvref_mapper_train_grad): (logits, parameter gradients in
        named_parameters() order, concatenated). Updates m's BN running statistics."""
        xx = np.ascontiguousarray(x, np.float64)
        b, hs, n = xx.shape
        dl = np.ascontiguousarray(dlogits, np.float64)
        logits = np.zeros_like(dl)
        nparam = sum(t.size for name, t in m.tensors() if not name.endswith(("running_mean", "running_var")))
        grads = np.zeros(nparam, np.float64)
        self.L.pkvref_mapper_train_grad.argtypes = [ctypes.c_void_p, _f64p, ctypes.c_int64, ctypes.c_int64,
                                                    ctypes.c_int64, _f64p, _f64p, _f64p]
        self._check(self.L.pkvref_mapper_train_grad(m.h, _ptr(xx, _f64p), b, hs, n, _ptr(dl, _f64p),
                                                    _ptr(logits, _f64p), _ptr(grads, _f64p)))
        return logits, grads

    def apply_mask(self, bits: np.ndarray, k: int, head_dim: int, bytes_per_elem: int = 2):
        b = np.ascontiguousarray(bits, np.uint8)
        shape = np.array(b.shape, np.int64)
        slices = b.size // b.shape[-1]
        idx = np.zeros((slices, k), np.int64)
        d, bh, bt = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        self._check(self.L.pkvref_apply_mask(_ptr(b, _u8p), _ptr(shape, _i64p), b.ndim, k, head_dim, bytes_per_elem,
                                             _ptr(idx, _i64p), ctypes.byref(d), ctypes.byref(bh), ctypes.byref(bt)))
        return idx, d.value, bh.value, bt.value

    def layer_pair(self, ll: int, g: Geometry) -> int:
        g5 = np.array(g.as5(), np.int64)
        out = ctypes.c_int64()
        self._check(self.L.pkvref_layer_pair(ll, _ptr(g5, _i64p), ctypes.byref(out)))
        return out.value

    def window_offsets(self, n, crop, stride):
        buf = np.zeros(4096, np.int64)
        cnt = ctypes.c_int64()
        self._check(self.L.pkvref_window_offsets(n, crop, stride, _ptr(buf, _i64p), buf.size, ctypes.byref(cnt)))
        return buf[:cnt.value].tolist()

    def sinusoidal_pe(self, n, d):
        out = np.zeros((n, d))
        self._check(self.L.pkvref_sinusoidal_pe(n, d, _ptr(out, _f64p)))
        return out

    def rng(self, seed: int) -> "RefRng":
        return RefRng(self, seed)

    def mapper(self, g: Geometry, c: MapperConfig, seed: int) -> "RefMapper":
        return RefMapper(self, g, c, seed)


class RefRng:
    """The reference's Rng (rng.hpp:25-87) through libpkvref.so."""

    def __init__(self, ref: RefLib, seed: int):
        self.ref = ref
        self.h = ref.L.pkvref_rng_create(seed)

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.L.pkvref_rng_destroy(self.h)
            self.h = None

    def uniform(self, lo: float = 0.0, hi: float = 1.0) -> float:
        return self.ref.L.pkvref_rng_uniform(self.h, lo, hi)

    def below(self, n: int) -> int:
        return self.ref.L.pkvref_rng_below(self.h, n)

    def normal(self) -> float:
        return self.ref.L.pkvref_rng_normal(self.h)


class RefMapper:
    def __init__(self, ref: RefLib, g: Geometry, c: MapperConfig, seed: int):
        self.ref, self.g, self.c = ref, g, c
        g5 = np.array(g.as5(), np.int64)
        c12 = np.array(c.as12(), np.int64)
        h = ctypes.c_void_p()
        ref._check(ref.L.pkvref_mapper_create(_ptr(g5, _i64p), _ptr(c12, _i64p), seed, ctypes.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.ref.L.pkvref_mapper_destroy(self.h)
            self.h = None

    def tensors(self) -> List[Tuple[str, np.ndarray]]:
        L = self.ref.L
        out = []
        for i in range(L.pkvref_mapper_tensor_count(self.h)):
            name = ctypes.create_string_buffer(128)
            shape = np.zeros(8, np.int64)
            rank = ctypes.c_int()
            self.ref._check(L.pkvref_mapper_tensor(self.h, i, name, 128, _ptr(shape, _i64p), ctypes.byref(rank), None))
            shp = tuple(int(s) for s in shape[:rank.value])
            vals = np.zeros(int(np.prod(shp)), np.float64)
            self.ref._check(L.pkvref_mapper_tensor(self.h, i, name, 128, _ptr(shape, _i64p), ctypes.byref(rank),
                                                   _ptr(vals, _f64p)))
            out.append((name.value.decode(), vals.reshape(shp)))
        return out

    def blob(self) -> np.ndarray:
        return np.concatenate([t.ravel() for _, t in self.tensors()])

    def forward_pair(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        B, hs, n = x.shape
        out = np.zeros((B, self.g.target_heads, n))
        self.ref._check(self.ref.L.pkvref_forward_pair(self.h, _ptr(x, _f64p), B, hs, n, _ptr(out, _f64p)))
        return out

    def train_grad(self, x: np.ndarray, dlogits: np.ndarray):
        """(logits, parameter gradients) of one training step; see RefLib.mapper_train_grad."""
        return self.ref.mapper_train_grad(self, x, dlogits)

    def sliding_forward(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float64)
        B, hs, n = x.shape
        out = np.zeros((B, self.g.target_heads, n))
        self.ref._check(self.ref.L.pkvref_sliding_forward(self.h, _ptr(x, _f64p), B, hs, n, _ptr(out, _f64p)))
        return out

    def forward_full(self, x_all: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x_all, np.float64)
        B, ls, hs, n = x.shape
        out = np.zeros((B, self.g.target_layers, self.g.target_heads, n))
        self.ref._check(self.ref.L.pkvref_forward_full(self.h, _ptr(x, _f64p), B, ls, hs, n, _ptr(out, _f64p)))
        return out


def ref_available() -> bool:
    return os.path.exists(os.path.join(REF_DIR, "libpkvref.so"))
