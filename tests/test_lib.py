"""CPU-side checks of the C ABI library: it loads, exports every symbol the
headers declare, validates arguments host-side (no GPU needed), and computes the
sparsity ratios bit-exactly like the oracle.  Also: no product module imports
the oracle, and the product path has no fallback when libhla.so is missing."""

import ast
import ctypes
import glob
import os
import re

import pytest

from oracle import blocks
from oracle.patterns import Spec

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    return set(re.findall(r"HLA_API\s+[\w\s\*]+?\b(hla_\w+)\s*\(", src))


def test_library_exports_header_symbols():
    """libhla.so exports exactly include/hla.h (the hot path); the bring-up probes of
    include/hla_debug.h live in libhla_debug.so, not in the product library."""
    from paper_2511_05832_b200 import _lib
    L = _lib.lib()
    declared = _declared_symbols("hla.h")
    assert len(declared) >= 10
    for name in declared:
        assert hasattr(L, name), name
    assert set(_lib.EXPORTED) == declared
    for name in _declared_symbols("hla_debug.h"):
        assert not hasattr(L, name), name
    assert "sm_100a" in L.hla_version().decode()
    D = _lib.debug_lib()
    dbg = _declared_symbols("hla_debug.h")
    assert set(_lib.DEBUG_EXPORTED) == dbg and len(dbg) >= 5
    for name in dbg:
        assert hasattr(D, name), name


def test_argument_validation_without_gpu():
    from paper_2511_05832_b200 import _lib, api
    L = _lib.lib()
    n = 1
    arr = (ctypes.c_void_p * n)(16)
    # explicit permutation on a non-2^k grid -> UNSUPPORTED, checked before any CUDA call
    assert L.hla_hilbert_perm(56, 64, 0, 1, 128, 1, arr, arr, None, None) == _lib.HLA_ERR_UNSUPPORTED
    assert b"square" in L.hla_last_error()
    # the index itself covers any grid (generalized curve on the host); no outputs -> no work
    assert L.hla_hilbert_index(48, 56, None, None, None) == _lib.HLA_OK
    assert L.hla_hilbert_index(0, 56, None, None, None) == _lib.HLA_ERR_INVALID
    # window not dividing the grid -> INVALID
    d = api.pattern_desc("WSA", 64, 64, 7, 7)
    m = _lib.BlockMaskC()
    nnz = ctypes.c_int64()
    assert L.hla_build_block_mask(ctypes.byref(d), ctypes.byref(m), ctypes.byref(nnz), None) == _lib.HLA_ERR_INVALID
    # attention limits: tiles of 64 or 128; block 64 runs on the mask's window lists
    d = api.pattern_desc("HWA", 64, 64, 16, 16, block=32)
    m = _lib.BlockMaskC(128, 128, 1, 8, 8, 8, 8, 8, 8, 8)
    st = L.hla_attn_fwd(ctypes.byref(d), ctypes.byref(m), 1, 1, 64, 0.0, 16, 16, 16, 16, 16, None, None, None,
                        None)
    assert st == _lib.HLA_ERR_UNSUPPORTED
    d = api.pattern_desc("HWA", 64, 64, 16, 16, block=64)
    m = _lib.BlockMaskC(64, 64, 1, 8, 8, 8, 8, 8, 8, 8)
    st = L.hla_attn_fwd(ctypes.byref(d), ctypes.byref(m), 1, 1, 64, 0.0, 16, 16, 16, 16, 16, None, None, None,
                        None)
    assert st == _lib.HLA_ERR_INVALID and b"window lists" in L.hla_last_error()
    d = api.pattern_desc("HWA", 64, 64, 16, 16)
    m = _lib.BlockMaskC(32, 32, 1, 8, 8, 8, 8, 8, 8, 8)
    st = L.hla_attn_fwd(ctypes.byref(d), ctypes.byref(m), 1, 1, 128, 0.0, 16, 16, 16, 16, 16, None, None, None,
                        None)
    assert st == _lib.HLA_ERR_UNSUPPORTED
    # score_mod validation (global RPB, reading R19): unknown kind, missing table,
    # Hilbert order without the cell map, backward without a gradient buffer
    for mod, want in ((_lib.ScoreModC(7, 16, 16, 16), _lib.HLA_ERR_UNSUPPORTED),
                      (_lib.ScoreModC(1, None, 16, 16), _lib.HLA_ERR_INVALID),
                      (_lib.ScoreModC(1, 16, 16, None), _lib.HLA_ERR_INVALID)):
        st = L.hla_attn_fwd(ctypes.byref(d), ctypes.byref(m), 1, 1, 64, 0.0, 16, 16, 16, 16, 16, None,
                            ctypes.byref(mod), None, None)
        assert st == want, (mod.kind, st)
    mod = _lib.ScoreModC(1, 16, None, 16)
    st = L.hla_attn_bwd_main(ctypes.byref(d), ctypes.byref(m), 1, 1, 64, 0.0, 16, 16, 16, 16, 16, 16, 16, None,
                             ctypes.byref(mod), 256, 1 << 30, None, None)
    assert st == _lib.HLA_ERR_INVALID and b"drpb" in L.hla_last_error()
    # backward dQ plan: needs a filled mask and its two plan arrays; square tiles only
    m = _lib.BlockMaskC(32, 32, 1, 8, None, 8, 8, 8, 8, 8, 16, 16, -1)
    assert L.hla_build_bwd_plan(ctypes.byref(m), None) == _lib.HLA_ERR_INVALID and b"filled" in L.hla_last_error()
    m = _lib.BlockMaskC(32, 32, 1, 8, 8, 8, 8, 8, 8, 8, None, 16, -1)
    assert L.hla_build_bwd_plan(ctypes.byref(m), None) == _lib.HLA_ERR_INVALID
    m = _lib.BlockMaskC(32, 16, 1, 8, 8, 8, 8, 8, 8, 8, 16, 16, -1)
    assert L.hla_build_bwd_plan(ctypes.byref(m), None) == _lib.HLA_ERR_UNSUPPORTED


def test_tiled_order_validation_without_gpu():
    """HLA_ORDER_HILBERT_TILED (reading R23) is accepted only where it is the same attention:
    host-side checks before any CUDA call, and the layer's selection rule agrees with them."""
    from paper_2511_05832_b200 import _lib, api
    L = _lib.lib()
    assert L.hla_hilbert_tiled_index(4, 4, None, None, None) == _lib.HLA_ERR_UNSUPPORTED
    assert L.hla_hilbert_tiled_index(56, 56, None, None, None) == _lib.HLA_ERR_UNSUPPORTED
    assert L.hla_hilbert_tiled_index(64, 32, None, None, None) == _lib.HLA_ERR_UNSUPPORTED
    assert L.hla_hilbert_tiled_index(64, 64, None, None, None) == _lib.HLA_OK   # no outputs: no work
    m = _lib.BlockMaskC()
    nnz = ctypes.c_int64()
    for kind, g, w, want in (("HSA", 64, 16, _lib.HLA_ERR_UNSUPPORTED), ("HWA", 64, 4, _lib.HLA_ERR_UNSUPPORTED),
                             ("HNA", 64, 8, _lib.HLA_ERR_UNSUPPORTED), ("HWA", 56, 8, _lib.HLA_ERR_UNSUPPORTED)):
        d = api.pattern_desc(kind, g, g, w, w, tiled=True)
        assert L.hla_build_block_mask(ctypes.byref(d), ctypes.byref(m), ctypes.byref(nnz), None) == want, kind
        assert not api.tiled_order_applies(kind, g, g, w, w)
    with pytest.raises(ValueError):
        api.pattern_desc("WSA", 64, 64, 8, 8, tiled=True)      # row-major: not a Hilbert order
    assert api.tiled_order_applies("HWA", 64, 64, 8, 8) and api.tiled_order_applies("HWA", 8, 8, 8, 8)
    assert api.tiled_order_applies("HWA", 128, 128, 16, 16) and not api.tiled_order_applies("HWA", 64, 64, 7, 7)


@pytest.mark.parametrize("kind,H,W,wh,ww,b", [("HWA", 56, 56, 7, 7, 128), ("SA", 56, 56, 7, 7, 128),
                                             ("HNA", 128, 128, 17, 17, 128), ("WSA", 128, 128, 16, 16, 512),
                                             ("HWA", 16, 16, 8, 8, 16)])
def test_mask_ratios_match_oracle_bitwise(kind, H, W, wh, ww, b):
    from paper_2511_05832_b200 import _lib, api
    spec = Spec(kind, H, W, wh, ww)
    st = blocks.stats(blocks.classify_spec(spec, b, b), spec.n_tokens, b, b)
    d = api.pattern_desc(kind, H, W, wh, ww, block=b)
    cnt = (ctypes.c_int64 * 4)(st["nnz"], st["n_full"], st["n_partial"], st["n_empty"])
    e, s = ctypes.c_double(), ctypes.c_double()
    assert _lib.lib().hla_mask_ratios(ctypes.byref(d), cnt, ctypes.byref(e), ctypes.byref(s)) == 0
    assert e.value == st["empty_tile_ratio"] and s.value == st["sparsity"]


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2511_05832_b200")
    for path in glob.glob(os.path.join(pkg, "**", "*.py"), recursive=True):
        tree = ast.parse(open(path).read())
        for node in ast.walk(tree):
            if isinstance(node, ast.Import):
                assert not any(a.name.split(".")[0] == "oracle" for a in node.names), path
            if isinstance(node, ast.ImportFrom):
                assert (node.module or "").split(".")[0] != "oracle", path
    for path in glob.glob(os.path.join(pkg, "csrc", "*")):
        assert not re.search(r'#include\s*["<][^">]*oracle', open(path, errors="ignore").read()), path


def test_missing_library_fails_loudly(monkeypatch):
    from paper_2511_05832_b200 import _lib
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", "/nonexistent/libhla.so")
    with pytest.raises(ImportError):
        _lib.lib()
