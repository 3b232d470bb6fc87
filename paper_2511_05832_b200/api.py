"""Thin Python binding of libhla.so with the C ABI's names (argument marshalling only).

Every step of the path runs in the CUDA kernels behind include/hla.h; PyTorch is
used for device memory, streams and process groups only.  There is no CPU or
PyTorch fallback: if libhla.so is missing, the first call raises.
"""

import ctypes
from dataclasses import dataclass

import torch

from . import _lib
from ._lib import BlockMaskC, PatternDesc, check, lib

ORDER_ROW_MAJOR, ORDER_HILBERT, ORDER_HILBERT_TILED = 0, 1, 2
WINDOW, SLIDE, NEIGHBORHOOD, DENSE, SHIFTED_WINDOW = 0, 1, 2, 3, 4
TO_HILBERT, FROM_HILBERT = 0, 1

# paper names -> (order, pattern family)   (HWA/HSA/HNA/HSWA: P:L39; WSA/SA/NA2D: P:L28)
KINDS = {
    "HWA": (ORDER_HILBERT, WINDOW), "HSA": (ORDER_HILBERT, SLIDE), "HNA": (ORDER_HILBERT, NEIGHBORHOOD),
    "HSWA": (ORDER_HILBERT, SHIFTED_WINDOW), "WSA": (ORDER_ROW_MAJOR, WINDOW), "SA": (ORDER_ROW_MAJOR, SLIDE),
    "NA2D": (ORDER_ROW_MAJOR, NEIGHBORHOOD), "DENSE": (ORDER_ROW_MAJOR, DENSE),
}


def _stream(stream=None, device=None):
    """The launch stream: `stream`, else the current stream of `device` (the tensors' device,
    not whichever device happens to be current)."""
    s = stream if stream is not None else torch.cuda.current_stream(device)
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def pattern_desc(kind, grid_h, grid_w, win_h=1, win_w=1, block=128, shift=0, tiled=False):
    """tiled=True: HLA_ORDER_HILBERT_TILED (HWA with a multiple of 64 tokens per window on a square
    2^k grid: the same attention, 64-token segments relabeled in raster order; include/hla.h)."""
    order, pattern = KINDS[kind]
    if tiled:
        if order != ORDER_HILBERT:
            raise ValueError("tiled order is a Hilbert order: %s is not a Hilbert pattern" % kind)
        order = ORDER_HILBERT_TILED
    return PatternDesc(grid_h, grid_w, order, pattern, win_h, win_w, shift, block, block)


def is_hilbert(desc):
    return desc.order != ORDER_ROW_MAJOR


def tiled_order_applies(kind, grid_h, grid_w, win_h, win_w):
    """The shapes HLA_ORDER_HILBERT_TILED accepts (api_common.cu make_pattern_fields)."""
    return (kind == "HWA" and (win_h * win_w) % 64 == 0 and grid_h == grid_w and grid_h >= 8
            and grid_h & (grid_h - 1) == 0)


@dataclass
class BlockMask:
    """Device CSR block mask (include/hla.h hla_block_mask) plus its host counts."""
    desc: PatternDesc
    row_ptr: torch.Tensor
    col_idx: torch.Tensor
    kind: torch.Tensor
    t_row_ptr: torch.Tensor
    t_col_idx: torch.Tensor
    t_kind: torch.Tensor
    counts: torch.Tensor          # device int64[4]: nnz, n_full, n_partial, n_empty
    host_counts: tuple = None
    t_dq: torch.Tensor = None     # backward dQ plan (hla_build_bwd_plan): uint8 per transposed entry
    q_dq_local: torch.Tensor = None   # uint8 per q-block: 1 = dQ written by the main backward kernel
    n_dq_nonlocal: int = -1
    # block 64: the attention kernels' window lists (hla_build_tile_lists)
    w_row_ptr: torch.Tensor = None
    w_col: torch.Tensor = None
    w_kind: torch.Tensor = None
    wt_row_ptr: torch.Tensor = None
    wt_col: torch.Tensor = None
    wt_kind: torch.Tensor = None
    w_counts: tuple = (0, 0, 0, 0)

    @property
    def c(self):
        hc = (ctypes.c_int64 * 4)(*(self.host_counts or (0, 0, 0, 0)))
        wc = (ctypes.c_int64 * 4)(*self.w_counts)
        cap = self.w_col.numel() if self.w_col is not None else 0
        return BlockMaskC(self.row_ptr.numel() - 1, self.t_row_ptr.numel() - 1, self.col_idx.numel(),
                          self.row_ptr.data_ptr(), self.col_idx.data_ptr(), self.kind.data_ptr(),
                          self.t_row_ptr.data_ptr(), self.t_col_idx.data_ptr(), self.t_kind.data_ptr(),
                          self.counts.data_ptr(), _dp(self.t_dq), _dp(self.q_dq_local), self.n_dq_nonlocal, hc,
                          _dp(self.w_row_ptr), _dp(self.w_col), _dp(self.w_kind), _dp(self.wt_row_ptr),
                          _dp(self.wt_col), _dp(self.wt_kind), cap, wc)

    @property
    def tiles(self):
        """128 x 128 tiles the attention kernels execute per (b, h): the CSR entries at block
        128, the forward windows at block 64."""
        return self.w_counts[0] if self.w_col is not None else self.nnz

    @property
    def nnz(self):
        return self.host_counts[0]

    def ratios(self):
        """(empty_tile_ratio, sparsity) computed by hla_mask_ratios from the integer counts."""
        cnt = (ctypes.c_int64 * 4)(*self.host_counts)
        e, s = ctypes.c_double(), ctypes.c_double()
        check("hla_mask_ratios", lib().hla_mask_ratios(ctypes.byref(self.desc), cnt, ctypes.byref(e), ctypes.byref(s)))
        return e.value, s.value


def _dp(t):
    return t.data_ptr() if t is not None else None


def hla_hilbert_index(grid_h, grid_w, device="cuda", stream=None):
    n = grid_h * grid_w
    s2c = torch.empty(n, dtype=torch.int32, device=device)
    c2s = torch.empty(n, dtype=torch.int32, device=device)
    with torch.cuda.device(s2c.device):
        check("hla_hilbert_index", lib().hla_hilbert_index(grid_h, grid_w, _ptr(s2c), _ptr(c2s),
                                                           _stream(stream, s2c.device)))
    return s2c, c2s


def hla_hilbert_tiled_index(grid_h, grid_w, device="cuda", stream=None):
    """seq_to_cell / cell_to_seq of HLA_ORDER_HILBERT_TILED (include/hla.h)."""
    n = grid_h * grid_w
    s2c = torch.empty(n, dtype=torch.int32, device=device)
    c2s = torch.empty(n, dtype=torch.int32, device=device)
    with torch.cuda.device(s2c.device):
        check("hla_hilbert_tiled_index", lib().hla_hilbert_tiled_index(grid_h, grid_w, _ptr(s2c), _ptr(c2s),
                                                                       _stream(stream, s2c.device)))
    return s2c, c2s


def hla_hilbert_perm(grid_h, grid_w, direction, srcs, dsts=None, stream=None):
    """Permute token rows of up to 4 tensors [B, N, ...] between grid and Hilbert order."""
    srcs = list(srcs)
    if dsts is None:
        dsts = [torch.empty_like(s) for s in srcs]
    B, N = srcs[0].shape[0], srcs[0].shape[1]
    row_bytes = srcs[0][0, 0].numel() * srcs[0].element_size()
    for s, d in zip(srcs, dsts):
        assert s.is_cuda and s.is_contiguous() and d.is_contiguous() and s.shape == d.shape
        assert s.shape[0] == B and s.shape[1] == N and s[0, 0].numel() * s.element_size() == row_bytes
    n = len(srcs)
    src_arr = (ctypes.c_void_p * n)(*[s.data_ptr() for s in srcs])
    dst_arr = (ctypes.c_void_p * n)(*[d.data_ptr() for d in dsts])
    with torch.cuda.device(srcs[0].device):
        check("hla_hilbert_perm", lib().hla_hilbert_perm(grid_h, grid_w, direction, B, row_bytes, n, src_arr, dst_arr,
                                                         None, _stream(stream, srcs[0].device)))
    return dsts


def hla_build_block_mask(desc, device="cuda", stream=None, plan=True):
    """Sizing call, then fill call (both synchronous; built once per shape); then
    (plan=True, square tiles) the backward's dQ plan."""
    N = desc.grid_h * desc.grid_w
    mq = (N + desc.block_q - 1) // desc.block_q
    mk = (N + desc.block_k - 1) // desc.block_k
    i32 = dict(dtype=torch.int32, device=device)
    m = BlockMask(desc, torch.zeros(mq + 1, **i32), torch.empty(0, **i32), torch.empty(0, dtype=torch.uint8, device=device),
                  torch.zeros(mk + 1, **i32), torch.empty(0, **i32), torch.empty(0, dtype=torch.uint8, device=device),
                  torch.zeros(4, dtype=torch.int64, device=device))
    c = m.c
    c.col_idx = None
    nnz = ctypes.c_int64()
    dev = m.row_ptr.device
    with torch.cuda.device(dev):
        check("hla_build_block_mask", lib().hla_build_block_mask(ctypes.byref(desc), ctypes.byref(c),
                                                                 ctypes.byref(nnz), _stream(stream, dev)))
    cap = max(1, nnz.value)
    m.col_idx = torch.empty(cap, **i32)
    m.kind = torch.empty(cap, dtype=torch.uint8, device=device)
    m.t_col_idx = torch.empty(cap, **i32)
    m.t_kind = torch.empty(cap, dtype=torch.uint8, device=device)
    c = m.c
    with torch.cuda.device(dev):
        check("hla_build_block_mask", lib().hla_build_block_mask(ctypes.byref(desc), ctypes.byref(c),
                                                                 ctypes.byref(nnz), _stream(stream, dev)))
    m.host_counts = tuple(int(x) for x in c.host_counts)   # written by the fill call
    if desc.block_q == desc.block_k == 64:
        hla_build_tile_lists(m, stream)      # the attention kernels' windows
    if plan and desc.block_q == desc.block_k:
        hla_build_bwd_plan(m, stream)        # block 64: only when every window is 128-aligned
    return m


def hla_build_tile_lists(mask, stream=None):
    """Window lists of a filled block-64 mask (synchronous; once per mask)."""
    dev = mask.row_ptr.device
    c = mask.c
    n = ctypes.c_int64()
    with torch.cuda.device(dev):
        check("hla_build_tile_lists", lib().hla_build_tile_lists(ctypes.byref(c), ctypes.byref(n), _stream(stream, dev)))
    i32 = dict(dtype=torch.int32, device=dev)
    tq, tk = (mask.row_ptr.numel() - 1 + 1) // 2, (mask.t_row_ptr.numel() - 1 + 1) // 2
    mask.w_row_ptr, mask.wt_row_ptr = torch.zeros(tq + 1, **i32), torch.zeros(tk + 1, **i32)
    mask.w_col, mask.wt_col = torch.empty(n.value, **i32), torch.empty(n.value, **i32)
    mask.w_kind = torch.empty(n.value, dtype=torch.uint8, device=dev)
    mask.wt_kind = torch.empty(n.value, dtype=torch.uint8, device=dev)
    c = mask.c
    with torch.cuda.device(dev):
        check("hla_build_tile_lists", lib().hla_build_tile_lists(ctypes.byref(c), ctypes.byref(n), _stream(stream, dev)))
    mask.w_counts = tuple(int(x) for x in c.w_counts)
    return mask


def hla_build_bwd_plan(mask, stream=None):
    """The backward's dQ chaining plan of a filled mask (synchronous; once per mask)."""
    dev = mask.row_ptr.device
    win = mask.w_row_ptr is not None      # block 64: per window-list entry / 128-row tile
    mask.t_dq = torch.zeros(max(1, (mask.wt_col if win else mask.col_idx).numel()), dtype=torch.uint8, device=dev)
    mask.q_dq_local = torch.zeros((mask.w_row_ptr if win else mask.row_ptr).numel() - 1, dtype=torch.uint8, device=dev)
    c = mask.c
    with torch.cuda.device(dev):
        check("hla_build_bwd_plan", lib().hla_build_bwd_plan(ctypes.byref(c), _stream(stream, dev)))
    mask.n_dq_nonlocal = int(c.n_dq_nonlocal)
    return mask


def score_mod(rpb=None, drpb=None, cells=None):
    """hla_score_mod for the global RPB (reading R19): rpb fp32 [heads, 2H-1, 2W-1],
    drpb its gradient buffer (backward), cells = int32 [N] grid cell of every sequence
    position (hla_hilbert_index for Hilbert patterns; None = row-major identity).
    None when rpb is None (no score modification)."""
    if rpb is None:
        return None
    assert rpb.dtype == torch.float32 and rpb.is_cuda and rpb.is_contiguous()
    if drpb is not None:
        assert drpb.dtype == torch.float32 and drpb.shape == rpb.shape and drpb.is_contiguous()
    return _lib.ScoreModC(1, _ptr(rpb), _ptr(drpb), _ptr(cells))


def _sm(mod):
    return ctypes.byref(mod) if mod is not None else None


def hla_attn_fwd(desc, mask, q, k, v, scale=0.0, o=None, lse=None, tiles_visited=None, seq_to_cell=None,
                 stream=None, mod=None):
    """q, k, v: bf16 [B, N, heads, d] in desc's sequence order -> (o, lse [B, heads, N] fp32).
    seq_to_cell (int32 [N] from hla_hilbert_index): fused reorder -- q, k, v, o in grid order.
    mod: optional score_mod(...) (global RPB)."""
    B, N, H, D = q.shape
    for t in (q, k, v):
        assert t.dtype == torch.bfloat16 and t.is_cuda and t.is_contiguous() and t.shape == q.shape
    if o is None:
        o = torch.empty_like(q)
    if lse is None:
        lse = torch.empty(B, H, N, dtype=torch.float32, device=q.device)
    mc = mask.c
    with torch.cuda.device(q.device):
        check("hla_attn_fwd", lib().hla_attn_fwd(ctypes.byref(desc), ctypes.byref(mc), B, H, D, float(scale),
                                                 _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse), _ptr(seq_to_cell),
                                                 _sm(mod), _ptr(tiles_visited), _stream(stream, q.device)))
    return o, lse


def hla_attn_bwd_workspace(B, H, N, D):
    return int(lib().hla_attn_bwd_workspace(B, H, N, D))


def hla_attn_bwd(desc, mask, q, k, v, o, lse, dout, scale=0.0, dq=None, dk=None, dv=None, workspace=None,
                 tiles_visited=None, seq_to_cell=None, stream=None, mod=None):
    B, N, H, D = q.shape
    dq = torch.empty_like(q) if dq is None else dq
    dk = torch.empty_like(k) if dk is None else dk
    dv = torch.empty_like(v) if dv is None else dv
    nbytes = hla_attn_bwd_workspace(B, H, N, D)
    if workspace is None:
        workspace = torch.empty(nbytes, dtype=torch.uint8, device=q.device)
    mc = mask.c
    with torch.cuda.device(q.device):
        check("hla_attn_bwd", lib().hla_attn_bwd(ctypes.byref(desc), ctypes.byref(mc), B, H, D, float(scale),
                                                 _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse), _ptr(dout),
                                                 _ptr(dq), _ptr(dk), _ptr(dv), _ptr(seq_to_cell), _sm(mod),
                                                 _ptr(workspace), workspace.numel(), _ptr(tiles_visited),
                                                 _stream(stream, q.device)))
    return dq, dk, dv


def hla_attn_bwd_fuses_preprocess(desc, mask, mod=None):
    """True if hla_attn_bwd folds the preprocess into its main kernel (one launch)."""
    mc = mask.c
    return bool(lib().hla_attn_bwd_fuses_preprocess(ctypes.byref(desc), ctypes.byref(mc), _sm(mod)))


def _pm(mask):
    return ctypes.byref(mask.c) if mask is not None else None


def hla_attn_bwd_preprocess(o, dout, lse, workspace, scale=0.0, seq_to_cell=None, stream=None, mask=None):
    """mask: the mask whose dQ plan hla_attn_bwd_main will use (None = no plan)."""
    B, N, H, D = o.shape
    with torch.cuda.device(o.device):
        check("hla_attn_bwd_preprocess", lib().hla_attn_bwd_preprocess(B, H, N, D, float(scale), _ptr(o), _ptr(dout),
                                                                       _ptr(lse), _ptr(seq_to_cell), _pm(mask),
                                                                       _ptr(workspace), workspace.numel(),
                                                                       _stream(stream, o.device)))


def hla_attn_bwd_main(desc, mask, q, k, v, dout, dq, dk, dv, workspace, scale=0.0, tiles_visited=None,
                      seq_to_cell=None, stream=None, mod=None):
    """Requires hla_attn_bwd_preprocess to have filled `workspace` (D, LSE in log2 domain).
    dq receives the rows of the q-blocks the mask's dQ plan marks local (the others come
    from hla_attn_bwd_finalize).  With a global-RPB mod, the table gradient is ACCUMULATED
    into mod's drpb."""
    B, N, H, D = q.shape
    mc = mask.c
    with torch.cuda.device(q.device):
        check("hla_attn_bwd_main", lib().hla_attn_bwd_main(ctypes.byref(desc), ctypes.byref(mc), B, H, D,
                                                           float(scale), _ptr(q), _ptr(k), _ptr(v), _ptr(dout),
                                                           _ptr(dq), _ptr(dk), _ptr(dv), _ptr(seq_to_cell), _sm(mod),
                                                           _ptr(workspace), workspace.numel(), _ptr(tiles_visited),
                                                           _stream(stream, q.device)))


def hla_attn_bwd_finalize(workspace, dq, seq_to_cell=None, stream=None, mask=None):
    """mask: the mask whose dQ plan hla_attn_bwd_main used (None = no plan)."""
    B, N, H, D = dq.shape
    with torch.cuda.device(dq.device):
        check("hla_attn_bwd_finalize", lib().hla_attn_bwd_finalize(B, H, N, D, _ptr(workspace), workspace.numel(),
                                                                   _ptr(dq), _ptr(seq_to_cell), _pm(mask),
                                                                   _stream(stream, dq.device)))


def hla_debug_umma(A, B, M, N, K, a_mn=False, b_mn=False, a_tmem=False, stream=None):
    C = torch.empty(M, N, dtype=torch.float32, device=A.device)
    check("hla_debug_umma", _lib.debug_lib().hla_debug_umma(_ptr(A), _ptr(B), _ptr(C), M, N, K, int(a_mn),
                                                            int(b_mn), int(a_tmem), _stream(stream, A.device)))
    return C


def hla_debug_gather4(src, idx, head, box_h=1, stream=None):
    """src: bf16 [rows, heads, d]; idx: int32[128] row indices -> bf16 [128, d] (TMA gather4 bring-up)."""
    rows, heads, d = src.shape
    out = torch.empty(128, d, dtype=torch.bfloat16, device=src.device)
    check("hla_debug_gather4", _lib.debug_lib().hla_debug_gather4(_ptr(src), rows, heads, d, _ptr(idx), head, box_h,
                                                                  _ptr(out), _stream(stream, src.device)))
    return out


def version():
    return lib().hla_version().decode()
