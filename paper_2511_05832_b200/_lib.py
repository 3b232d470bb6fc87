"""ctypes loader for libhla.so (the C ABI declared in include/hla.h).

Argument marshalling only.  There is deliberately no fallback: if the shared
library is missing or fails to load, every call raises.
"""

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, os.environ.get("HLA_LIB_NAME", "libhla.so"))   # HLA_LIB_NAME: dev trace build

HLA_OK, HLA_ERR_INVALID, HLA_ERR_UNSUPPORTED, HLA_ERR_CAPACITY, HLA_ERR_CUDA = range(5)
STATUS_NAMES = {0: "HLA_OK", 1: "HLA_ERR_INVALID", 2: "HLA_ERR_UNSUPPORTED", 3: "HLA_ERR_CAPACITY",
                4: "HLA_ERR_CUDA"}

# exported symbols of include/hla.h and include/hla_debug.h
EXPORTED = ("hla_hilbert_index", "hla_hilbert_perm", "hla_build_block_mask", "hla_mask_ratios",
            "hla_attn_fwd", "hla_attn_bwd", "hla_attn_bwd_workspace", "hla_attn_bwd_preprocess",
            "hla_attn_bwd_main", "hla_attn_bwd_finalize", "hla_build_bwd_plan", "hla_last_error", "hla_version",
            "hla_debug_umma", "hla_debug_gather4", "hla_debug_mma_rate",
            "hla_debug_tmem_rate", "hla_debug_ex2_rate", "hla_debug_xu_rate", "hla_debug_sync_latency",
            "hla_debug_softmax_rate", "hla_debug_softmax_tile", "hla_debug_load_rate")


class PatternDesc(ctypes.Structure):
    _fields_ = [("grid_h", ctypes.c_int32), ("grid_w", ctypes.c_int32), ("order", ctypes.c_int32),
                ("pattern", ctypes.c_int32), ("win_h", ctypes.c_int32), ("win_w", ctypes.c_int32),
                ("shift", ctypes.c_int32), ("block_q", ctypes.c_int32), ("block_k", ctypes.c_int32)]


class ScoreModC(ctypes.Structure):
    """hla_score_mod (include/hla.h): kind 1 = global RPB."""
    _fields_ = [("kind", ctypes.c_int32), ("rpb", ctypes.c_void_p), ("drpb", ctypes.c_void_p),
                ("seq_to_cell", ctypes.c_void_p)]


class BlockMaskC(ctypes.Structure):
    _fields_ = [("n_qblocks", ctypes.c_int32), ("n_kblocks", ctypes.c_int32), ("capacity", ctypes.c_int64),
                ("row_ptr", ctypes.c_void_p), ("col_idx", ctypes.c_void_p), ("kind", ctypes.c_void_p),
                ("t_row_ptr", ctypes.c_void_p), ("t_col_idx", ctypes.c_void_p), ("t_kind", ctypes.c_void_p),
                ("counts", ctypes.c_void_p),
                ("t_dq", ctypes.c_void_p), ("q_dq_local", ctypes.c_void_p), ("n_dq_nonlocal", ctypes.c_int32),
                ("host_counts", ctypes.c_int64 * 4)]


class HlaError(RuntimeError):
    def __init__(self, fn, status, msg):
        super().__init__("%s -> %s: %s" % (fn, STATUS_NAMES.get(status, status), msg))
        self.status = status


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError("libhla.so not built (%s); run __graft_entry__.build() -- there is no fallback" % LIB_PATH)
    L = ctypes.CDLL(LIB_PATH)
    vp, i32, i64, f32, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_size_t
    pdesc, pmask = ctypes.POINTER(PatternDesc), ctypes.POINTER(BlockMaskC)
    sig = {
        "hla_hilbert_index": [i32, i32, vp, vp, vp],
        "hla_hilbert_perm": [i32, i32, i32, i32, i32, i32, ctypes.POINTER(vp), ctypes.POINTER(vp), vp, vp],
        "hla_build_block_mask": [pdesc, pmask, ctypes.POINTER(i64), vp],
        "hla_mask_ratios": [pdesc, ctypes.POINTER(i64), ctypes.POINTER(ctypes.c_double),
                            ctypes.POINTER(ctypes.c_double)],
        "hla_attn_fwd": [pdesc, pmask, i32, i32, i32, f32, vp, vp, vp, vp, vp, vp, vp, vp, vp],
        "hla_attn_bwd": [pdesc, pmask, i32, i32, i32, f32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp,
                         vp],
        "hla_attn_bwd_preprocess": [i32, i32, i32, i32, f32, vp, vp, vp, vp, pmask, vp, sz, vp],
        "hla_attn_bwd_main": [pdesc, pmask, i32, i32, i32, f32, vp, vp, vp, vp, vp, vp, vp, vp, vp, vp, sz, vp, vp],
        "hla_attn_bwd_finalize": [i32, i32, i32, i32, vp, sz, vp, vp, pmask, vp],
        "hla_build_bwd_plan": [pmask, vp],
        "hla_debug_umma": [vp, vp, vp, i32, i32, i32, i32, i32, i32, vp],
        "hla_debug_gather4": [vp, i64, i32, i32, vp, i32, i32, vp, vp],
        "hla_debug_mma_rate": [i32, i32, i32, i32, i32, vp, vp],
        "hla_debug_tmem_rate": [i32, i32, i32, i32, vp, vp],
        "hla_debug_ex2_rate": [i32, i32, vp, vp, vp],
        "hla_debug_xu_rate": [i32, i32, i32, vp, vp, vp],
        "hla_debug_sync_latency": [i32, i32, vp, vp],
        "hla_debug_softmax_rate": [i32, i32, vp, vp, vp],
        "hla_debug_softmax_tile": [i32, i32, vp, vp, vp],
        "hla_debug_load_rate": [vp, i64, i32, i32, i32, i32, i32, vp, vp],
    }
    for name, args in sig.items():
        if name.startswith("hla_debug_") and not hasattr(L, name):
            continue   # bring-up probes are optional (e.g. an older dev build under HLA_LIB_NAME)
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    L.hla_attn_bwd_workspace.argtypes = [i32, i32, i32, i32]
    L.hla_attn_bwd_workspace.restype = sz
    L.hla_last_error.restype = ctypes.c_char_p
    L.hla_version.restype = ctypes.c_char_p
    _lib = L
    return L


def check(name, status):
    if status != HLA_OK:
        raise HlaError(name, status, lib().hla_last_error().decode())
