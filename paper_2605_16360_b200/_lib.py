"""ctypes binding of libpkv_b200.so (include/pkv_capi.h).

This is exactly the binding a reference-side maintainer would add
(INTEGRATION.md): plain pointers and sizes, status codes mapped onto the
reference exception taxonomy (proj/include/proxykv/common.hpp:13-52).
The library is loaded from the package directory (built in-tree by
``__graft_entry__.build()``); a missing library is an error, never a fallback.
"""
from __future__ import annotations

import builtins
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libpkv_b200.so")


class PkvError(RuntimeError):
    """proxykv::Error (common.hpp:13)."""


class ShapeError(PkvError):
    """proxykv::ShapeError (common.hpp:17)."""


class PkvValueError(PkvError, builtins.ValueError):
    """proxykv::ValueError (common.hpp:21)."""


class ConfigError(PkvError):
    """proxykv::ConfigError (common.hpp:29)."""


class CudaError(PkvError):
    """CUDA runtime / launch failure inside the B200 path."""


class NoDeviceError(PkvError):
    """No sm_100 device: the B200 path has no CPU fallback."""


class IoError(PkvError):
    """proxykv::IoError (common.hpp:33)."""


class BadMagicError(IoError):
    """proxykv::BadMagicError (common.hpp:38)."""


class VersionMismatchError(IoError):
    """proxykv::VersionMismatchError (common.hpp:42)."""


class TruncatedFileError(IoError):
    """proxykv::TruncatedFileError (common.hpp:46)."""


class PayloadLengthError(IoError):
    """proxykv::PayloadLengthError (common.hpp:50)."""


_STATUS = {1: ShapeError, 2: PkvValueError, 3: CudaError, 4: CudaError, 5: ConfigError, 6: NoDeviceError, 7: IoError,
           8: BadMagicError, 9: VersionMismatchError, 10: TruncatedFileError, 11: PayloadLengthError}

_c_i64 = ctypes.c_int64
_c_i64p = ctypes.POINTER(ctypes.c_int64)
_c_vp = ctypes.c_void_p
_c_u32 = ctypes.c_uint32
_c_dbl = ctypes.c_double

# name -> (restype, argtypes). Every symbol include/pkv_capi.h declares.
SIGNATURES = {
    "pkv_abi_version": (ctypes.c_int, []),
    "pkv_last_error": (ctypes.c_char_p, []),
    "pkv_sm100_device_count": (ctypes.c_int, []),
    "pkv_ctx_create": (ctypes.c_int, [ctypes.c_int, ctypes.POINTER(_c_vp)]),
    "pkv_ctx_destroy": (None, [_c_vp]),
    "pkv_ctx_launch_count": (_c_i64, [_c_vp]),
    "pkv_retention_count": (ctypes.c_int, [_c_dbl, _c_i64, _c_i64p]),
    "pkv_topk_select": (ctypes.c_int, [_c_vp, _c_vp, _c_i64, _c_i64, _c_i64, _c_vp, _c_vp, _c_vp]),
    "pkv_topk_select_f64": (ctypes.c_int, [_c_vp, _c_vp, _c_i64, _c_i64, _c_i64, _c_vp, _c_vp, _c_vp]),
    "pkv_topk_indices_host": (ctypes.c_int, [_c_vp, _c_vp, _c_i64, _c_i64, _c_vp]),
    "pkv_topk_overlap_host": (ctypes.c_int, [_c_vp, _c_vp, _c_vp, _c_i64, _c_i64, _c_i64, _c_vp]),
    "pkv_mapper_forward_pair": (ctypes.c_int, [_c_vp, _c_vp, _c_i64, _c_i64, _c_vp, _c_vp, _c_vp]),
    "pkv_mapper_forward_pair_host": (ctypes.c_int, [_c_vp, _c_vp, _c_i64, _c_i64, _c_vp, _c_vp]),
    "pkv_mapper_sliding_forward_host": (ctypes.c_int, [_c_vp, _c_vp, _c_i64, _c_i64, _c_vp]),
    "pkv_mapper_forward_full_host": (ctypes.c_int, [_c_vp, _c_vp, _c_i64, _c_i64, _c_vp]),
    "pkv_topk_mask_host": (ctypes.c_int, [_c_vp, _c_vp, _c_i64, _c_i64, _c_dbl, _c_vp, _c_i64p]),
    "pkv_topk_overlap": (ctypes.c_int, [_c_vp, _c_vp, _c_vp, _c_i64, _c_i64, _c_i64, _c_vp, _c_vp]),
    "pkv_captured_mass": (ctypes.c_int, [_c_vp, _c_vp, _c_vp, _c_i64, _c_i64, _c_i64, _c_vp, _c_vp]),
    "pkv_compact_kv_paged": (ctypes.c_int, [_c_vp, _c_vp, _c_vp, _c_vp, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_vp,
                                            _c_i64, _c_i64, _c_vp, _c_vp, _c_vp]),
    "pkv_paged_decode_attention": (ctypes.c_int, [_c_vp, _c_vp, _c_vp, _c_vp, _c_vp, _c_vp, _c_i64, _c_i64, _c_i64,
                                                  _c_i64, _c_i64, _c_i64, _c_i64, ctypes.c_double, _c_vp, _c_vp]),
    "pkv_pruner_run_two_device": (ctypes.c_int, [_c_vp] * 12),
    "pkv_pruner_run_lse": (ctypes.c_int, [_c_vp] * 11),
    "pkv_spearman": (ctypes.c_int, [_c_vp, _c_vp, _c_vp, _c_i64, _c_i64, _c_vp, _c_vp]),
    "pkv_pruner_profile": (ctypes.c_int, [_c_vp, _c_i64]),
    "pkv_pruner_profile_read": (ctypes.c_int, [_c_vp, _c_vp, _c_i64, _c_i64p]),
    "pkv_trainer_create": (ctypes.c_int, [_c_vp, _c_i64p, _c_i64p, _c_vp, _c_i64, ctypes.POINTER(_c_vp)]),
    "pkv_trainer_destroy": (None, [_c_vp]),
    "pkv_trainer_param_count": (ctypes.c_int, [_c_vp, _c_i64p, _c_i64p]),
    "pkv_trainer_forward": (ctypes.c_int, [_c_vp, _c_vp, _c_i64, _c_i64, _c_vp, _c_vp]),
    "pkv_trainer_backward": (ctypes.c_int, [_c_vp, _c_vp, _c_vp, _c_vp]),
    "pkv_trainer_blob": (ctypes.c_int, [_c_vp, _c_vp]),
    "pkv_trainer_forward_host": (ctypes.c_int, [_c_vp, _c_vp, _c_i64, _c_i64, _c_vp]),
    "pkv_trainer_backward_host": (ctypes.c_int, [_c_vp, _c_vp, _c_vp]),
    "pkv_loss_total": (ctypes.c_int, [_c_vp, _c_vp, _c_vp, _c_vp, ctypes.c_int, _c_vp, ctypes.c_uint64, _c_vp, _c_vp,
                                      _c_vp]),
    "pkv_slice_metrics": (ctypes.c_int, [_c_vp, _c_vp, _c_vp, _c_i64, _c_i64, _c_i64, _c_vp, _c_vp, _c_vp, _c_vp]),
    "pkv_select_compact": (ctypes.c_int, [_c_vp, _c_vp, _c_i64, _c_i64, _c_i64, _c_vp, _c_vp, _c_i64, _c_i64, _c_vp,
                                          _c_vp, _c_vp, _c_vp]),
    "pkv_compact_kv": (ctypes.c_int, [_c_vp, _c_vp, _c_vp, _c_vp, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _c_vp,
                                      _c_vp, _c_vp]),
    "pkv_score": (ctypes.c_int, [_c_vp, _c_vp, _c_vp] + [_c_i64] * 6 + [_c_u32, _c_vp, _c_vp, _c_vp]),
    "pkv_score_lse": (ctypes.c_int, [_c_vp, _c_vp, _c_vp] + [_c_i64] * 6 + [_c_u32, _c_vp, _c_vp]),
    "pkv_proxy_prefill_attention": (ctypes.c_int, [_c_vp, _c_vp, _c_vp, _c_vp] + [_c_i64] * 6 + [_c_u32, _c_vp, _c_vp,
                                                                                              _c_vp]),
    "pkv_layer_pair": (ctypes.c_int, [_c_i64, _c_i64p, _c_i64p]),
    "pkv_window_offsets": (ctypes.c_int, [_c_i64, _c_i64, _c_i64, _c_i64p, _c_i64, _c_i64p]),
    "pkv_mapper_init_params": (ctypes.c_int, [_c_i64p, _c_i64p, ctypes.c_uint64, _c_vp, _c_i64p]),
    "pkv_mapper_create": (ctypes.c_int, [_c_vp, _c_i64p, _c_i64p, _c_vp, _c_i64, _c_u32, ctypes.POINTER(_c_vp)]),
    "pkv_mapper_destroy": (None, [_c_vp]),
    "pkv_mapper_forward_full": (ctypes.c_int, [_c_vp, _c_vp, _c_i64, _c_i64, _c_vp, _c_vp]),
    "pkv_mapper_sliding_forward": (ctypes.c_int, [_c_vp, _c_vp, _c_i64, _c_i64, _c_vp, _c_vp]),
    "pkv_pruner_create": (ctypes.c_int, [_c_vp, _c_vp, _c_i64, _c_i64, _c_i64, _c_i64, _c_dbl, _c_u32,
                                         ctypes.POINTER(_c_vp)]),
    "pkv_pruner_destroy": (None, [_c_vp]),
    "pkv_pruner_k": (_c_i64, [_c_vp]),
    "pkv_pruner_run": (ctypes.c_int, [_c_vp] * 10),
    "pkv_pruner_run_host": (ctypes.c_int, [_c_vp] * 9),
    "pkv_pruner_run_dual": (ctypes.c_int, [_c_vp] * 11),
    "pkv_packed_decode_attention": (ctypes.c_int, [_c_vp, _c_vp, _c_vp, _c_vp] + [_c_i64] * 5 + [_c_dbl, _c_vp,
                                                                                                _c_vp]),
    "pkv_shard_plan": (ctypes.c_int, [_c_i64p, ctypes.c_int, ctypes.c_int, _c_u32, _c_i64p]),
    "pkv_shard_exchange_schedule": (ctypes.c_int, [_c_i64p, ctypes.c_int, ctypes.c_int, _c_i64, _c_vp, _c_i64,
                                                   _c_i64p]),
    "pkv_pruner_exchange": (ctypes.c_int, [_c_vp, _c_vp, _c_vp, _c_vp]),
    "pkv_trace_write": (ctypes.c_int, [ctypes.c_char_p, _c_i64p, _c_i64, _c_vp, _c_vp, ctypes.c_char_p]),
    "pkv_trace_read_header": (ctypes.c_int, [ctypes.c_char_p, _c_i64p, _c_i64p]),
    "pkv_trace_read": (ctypes.c_int, [ctypes.c_char_p, _c_vp, _c_vp]),
    "pkv_checkpoint_write": (ctypes.c_int, [ctypes.c_char_p, _c_i64p, _c_i64p, _c_vp, _c_i64]),
    "pkv_checkpoint_read": (ctypes.c_int, [ctypes.c_char_p, _c_i64p, _c_i64p, _c_vp, _c_i64p]),
    "pkv_comm_unique_id": (ctypes.c_int, [_c_vp]),
    "pkv_comm_create": (ctypes.c_int, [_c_vp, ctypes.c_int, ctypes.c_int, _c_vp, ctypes.POINTER(_c_vp)]),
    "pkv_comm_destroy": (None, [_c_vp]),
    "pkv_pruner_create_sharded": (ctypes.c_int, [_c_vp, _c_vp, _c_i64, _c_i64, _c_i64, _c_i64, _c_dbl, _c_u32,
                                                 _c_u32, ctypes.c_int, ctypes.c_int, _c_vp, ctypes.POINTER(_c_vp)]),
}

_lib = None


def lib() -> ctypes.CDLL:
    """The loaded libpkv_b200.so with argtypes set. Raises if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            try:
                fn = getattr(L, name)
            except AttributeError:  # reported by tests/test_capi.py::test_every_header_symbol_exported
                continue
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def check(status: int) -> None:
    if status == 0:
        return
    msg = lib().pkv_last_error().decode(errors="replace")
    raise _STATUS.get(status, PkvError)(msg)
