"""B200-native (sm_100a) ProxyKV pruning hot path: proxy scoring ->
HybridAxialMapper -> Top-K select -> KV compaction, behind the reference's
scoring / mapper / prune API (see include/pkv_capi.h)."""
from . import proxykv  # noqa: F401
from ._lib import LIB_PATH, check, lib  # noqa: F401
from .proxykv import *  # noqa: F401,F403
