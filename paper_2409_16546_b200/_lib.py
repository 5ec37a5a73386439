"""ctypes binding of libakv.so (the C ABI in include/akv.h).

The product path has no CPU fallback: if the in-tree library is missing or
the GPU is absent, every compute entry point raises.
"""

from __future__ import annotations

import ctypes
import os
import threading

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG, "libakv.so")

HEAD_DIM = 128
PAGE_TOKENS = 256
PAGE_BYTES = 65536
MAX_GROUP = 8
MAX_KSEL = 64
TARGET_UNKNOWN = -(1 << 31)

AKV_OK, AKV_EINVAL, AKV_EUNSUPPORTED, AKV_ECUDA = 0, -1, -2, -3
STATUS_NONFINITE, STATUS_DEGENERATE, STATUS_BAD_Q, STATUS_CAPACITY, STATUS_POSITION = 1, 2, 3, 4, 5

_c = ctypes.c_void_p
_i32 = ctypes.c_int32


class AkvStore(ctypes.Structure):
    _fields_ = [("n_units", _i32), ("head_dim", _i32), ("max_pages", _i32), ("pool_pages", _i32),
                ("k_pool", _c), ("v_pool", _c), ("page_table", _c), ("lengths", _c), ("colmax", _c),
                ("rowmax", _c)]


class AkvCfg(ctypes.Structure):
    _fields_ = [("group", _i32), ("margin_bits", _i32), ("zero_skip", _i32), ("force_tier", _i32),
                ("k_sel", _i32), ("m", _i32), ("strategy", _i32), ("trunc_bits", _i32)]


class AkvStep(ctypes.Structure):
    _fields_ = [(name, _c) for name in (
        "q", "scores", "probs", "page_stats", "o_est", "targets", "sel_bits", "sel_idx", "head_meta",
        "head_metaf", "o_partial", "o", "counters", "unit_bytes", "status", "k_tiers", "v_tiers", "work", "need_bits")]


_lock = threading.Lock()
_lib = None


class AkvError(RuntimeError):
    pass


def lib():
    """Load the in-tree libakv.so (build it with `python -m paper_2409_16546_b200.build`)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise AkvError(f"{LIB_PATH} is missing: run `python -m paper_2409_16546_b200.build` "
                           "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        P = ctypes.POINTER
        L.akv_version.restype = _i32
        L.akv_workspace_bytes.restype = ctypes.c_int64
        L.akv_workspace_bytes.argtypes = [_i32, _i32, _i32]
        L.akv_step_carve.restype = _i32
        L.akv_step_carve.argtypes = [P(AkvStep), _c, _i32, _i32, _i32]
        L.akv_append.restype = _i32
        L.akv_append.argtypes = [P(AkvStore), _c, _c, _i32, _c, _c]
        L.akv_append_at.restype = _i32
        L.akv_append_at.argtypes = [P(AkvStore), _c, _c, _i32, _c, _c]
        L.akv_append_workspace_bytes.restype = ctypes.c_int64
        L.akv_append_workspace_bytes.argtypes = [_i32, _i32]
        L.akv_read_elements.restype = _i32
        L.akv_read_elements.argtypes = [P(AkvStore), _i32, _c, _c, _c, _c, ctypes.c_int64, _c, _c, _c]
        L.akv_append_ws.restype = _i32
        L.akv_append_ws.argtypes = [P(AkvStore), _c, _c, _i32, _c, _c, ctypes.c_int64, _c]
        for name in ("akv_qk", "akv_softmax_select", "akv_pv", "akv_combine", "akv_decode_step"):
            f = getattr(L, name)
            f.restype = _i32
            f.argtypes = [P(AkvStore), P(AkvCfg), P(AkvStep), _i32, _c]
        L.akv_export_planes.restype = _i32
        L.akv_export_planes.argtypes = [P(AkvStore), _i32, _c, _c, _c, _c]
        L.akv_error_histogram.restype = _i32
        L.akv_error_histogram.argtypes = [_c, _c, ctypes.c_int64, _i32, _c, _c]
        _lib = L
        return L


EXPORTED_SYMBOLS = ("akv_version", "akv_workspace_bytes", "akv_step_carve", "akv_append", "akv_append_at",
                    "akv_append_workspace_bytes",
                    "akv_append_ws", "akv_read_elements", "akv_qk",
                    "akv_softmax_select", "akv_pv", "akv_combine", "akv_decode_step", "akv_export_planes",
                    "akv_error_histogram")


def check(rc: int, what: str) -> None:
    if rc != AKV_OK:
        names = {AKV_EINVAL: "AKV_EINVAL", AKV_EUNSUPPORTED: "AKV_EUNSUPPORTED", AKV_ECUDA: "AKV_ECUDA"}
        raise AkvError(f"{what} failed: {names.get(rc, rc)}")
