"""ctypes loaders for libhla.so (the hot path: the C ABI declared in include/hla.h) and
libhla_debug.so (tcgen05 / TMA bring-up and machine-constant probes, include/hla_debug.h;
never loaded by the product path).

Argument marshalling only.  There is deliberately no fallback: if the shared
library is missing or fails to load, every call raises.
"""

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, os.environ.get("HLA_LIB_NAME", "libhla.so"))   # HLA_LIB_NAME: dev variant builds
DEBUG_LIB_PATH = os.path.join(_HERE, "libhla_debug.so")

HLA_OK, HLA_ERR_INVALID, HLA_ERR_UNSUPPORTED, HLA_ERR_CAPACITY, HLA_ERR_CUDA = range(5)
STATUS_NAMES = {0: "HLA_OK", 1: "HLA_ERR_INVALID", 2: "HLA_ERR_UNSUPPORTED", 3: "HLA_ERR_CAPACITY",
                4: "HLA_ERR_CUDA"}

# exported symbols of include/hla.h (libhla.so) and include/hla_debug.h (libhla_debug.so)
EXPORTED = ("hla_hilbert_index", "hla_hilbert_tiled_index", "hla_hilbert_perm", "hla_build_block_mask", "hla_mask_ratios",
            "hla_attn_fwd", "hla_attn_bwd", "hla_attn_bwd_workspace", "hla_attn_bwd_preprocess",
            "hla_attn_bwd_main", "hla_attn_bwd_finalize", "hla_build_bwd_plan", "hla_build_tile_lists",
            "hla_attn_bwd_fuses_preprocess", "hla_last_error", "hla_version")
DEBUG_EXPORTED = ("hla_debug_umma", "hla_debug_gather4", "hla_debug_mma_rate",
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
                ("host_counts", ctypes.c_int64 * 4),
                ("w_row_ptr", ctypes.c_void_p), ("w_col", ctypes.c_void_p), ("w_kind", ctypes.c_void_p),
                ("wt_row_ptr", ctypes.c_void_p), ("wt_col", ctypes.c_void_p), ("wt_kind", ctypes.c_void_p),
                ("w_capacity", ctypes.c_int64), ("w_counts", ctypes.c_int64 * 4)]


class HlaError(RuntimeError):
    def __init__(self, fn, status, msg):
        super().__init__("%s -> %s: %s" % (fn, STATUS_NAMES.get(status, status), msg))
        self.status = status


_lib = None
_debug_lib = None

_vp, _i32, _i64, _f32, _sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_size_t
_pdesc, _pmask = ctypes.POINTER(PatternDesc), ctypes.POINTER(BlockMaskC)
_SIG = {
    "hla_hilbert_index": [_i32, _i32, _vp, _vp, _vp],
    "hla_hilbert_tiled_index": [_i32, _i32, _vp, _vp, _vp],
    "hla_hilbert_perm": [_i32, _i32, _i32, _i32, _i32, _i32, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _vp, _vp],
    "hla_build_block_mask": [_pdesc, _pmask, ctypes.POINTER(_i64), _vp],
    "hla_mask_ratios": [_pdesc, ctypes.POINTER(_i64), ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)],
    "hla_attn_fwd": [_pdesc, _pmask, _i32, _i32, _i32, _f32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "hla_attn_bwd": [_pdesc, _pmask, _i32, _i32, _i32, _f32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                     _vp, _sz, _vp, _vp],
    "hla_attn_bwd_preprocess": [_i32, _i32, _i32, _i32, _f32, _vp, _vp, _vp, _vp, _pmask, _vp, _sz, _vp],
    "hla_attn_bwd_main": [_pdesc, _pmask, _i32, _i32, _i32, _f32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                          _sz, _vp, _vp],
    "hla_attn_bwd_finalize": [_i32, _i32, _i32, _i32, _vp, _sz, _vp, _vp, _pmask, _vp],
    "hla_build_bwd_plan": [_pmask, _vp],
    "hla_build_tile_lists": [_pmask, ctypes.POINTER(_i64), _vp],
    "hla_attn_bwd_fuses_preprocess": [_pdesc, _pmask, _vp],
}
_DEBUG_SIG = {
    "hla_debug_umma": [_vp, _vp, _vp, _i32, _i32, _i32, _i32, _i32, _i32, _vp],
    "hla_debug_gather4": [_vp, _i64, _i32, _i32, _vp, _i32, _i32, _vp, _vp],
    "hla_debug_mma_rate": [_i32, _i32, _i32, _i32, _i32, _vp, _vp],
    "hla_debug_tmem_rate": [_i32, _i32, _i32, _i32, _vp, _vp],
    "hla_debug_ex2_rate": [_i32, _i32, _vp, _vp, _vp],
    "hla_debug_xu_rate": [_i32, _i32, _i32, _vp, _vp, _vp],
    "hla_debug_sync_latency": [_i32, _i32, _vp, _vp],
    "hla_debug_softmax_rate": [_i32, _i32, _vp, _vp, _vp],
    "hla_debug_softmax_tile": [_i32, _i32, _vp, _vp, _vp],
    "hla_debug_load_rate": [_vp, _i64, _i32, _i32, _i32, _i32, _i32, _vp, _vp],
}


def _load(path, sig, what):
    if not os.path.exists(path):
        raise ImportError("%s not built (%s); run __graft_entry__.build() -- there is no fallback" % (what, path))
    L = ctypes.CDLL(path)
    for name, args in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = ctypes.c_int
    L.hla_last_error.restype = ctypes.c_char_p
    return L


def lib():
    """libhla.so: the hot path (include/hla.h)."""
    global _lib
    if _lib is not None:
        return _lib
    L = _load(LIB_PATH, _SIG, "libhla.so")
    L.hla_attn_bwd_workspace.argtypes = [_i32, _i32, _i32, _i32]
    L.hla_attn_bwd_workspace.restype = _sz
    L.hla_version.restype = ctypes.c_char_p
    _lib = L
    return L


def debug_lib():
    """libhla_debug.so: bring-up / machine-constant probes (include/hla_debug.h); tests and tools only."""
    global _debug_lib
    if _debug_lib is None:
        _debug_lib = _load(DEBUG_LIB_PATH, _DEBUG_SIG, "libhla_debug.so")
    return _debug_lib


def check(name, status, L=None):
    if status != HLA_OK:
        raise HlaError(name, status, (L or (debug_lib() if name.startswith("hla_debug_") else lib())).hla_last_error().decode())
