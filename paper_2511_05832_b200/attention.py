"""HilbertLocalAttention -- the public, allocation-free step API over the C ABI.

One instance = one attention layer shape.  Construction does the once-per-shape
work the paper caches ("the path can be precomputed and cached"): the
block mask is built on the GPU and all intermediate buffers are allocated.
forward() / backward() then only launch libhla kernels (capturable in a CUDA
graph):

  Hilbert patterns (HWA / HSA / HNA / HSWA), tensors given in grid order:
    forward : perm(q,k,v -> Hilbert) ; hla_attn_fwd ; perm(o -> grid)
    backward: perm(dO -> Hilbert) ; hla_attn_bwd ; perm(dq,dk,dv -> grid)
  Row-major baselines (WSA / SA / NA2D / DENSE) run the same attention kernels
  directly on grid order.

With fused=True (default for Hilbert patterns) the reorder is fused into the
attention kernels: they gather Hilbert tiles straight from
the grid-order tensors (TMA .tile::gather4 through the cached seq_to_cell path)
and scatter O / dK / dV / dQ rows back to their grid cells, so a step is
fwd ; bwd_pre ; bwd ; bwd_fin with no permutation passes.  fused=False keeps the
explicit hla_hilbert_perm passes (the paper's "Reshape" step).

dq_plan=True (default) also builds the backward's dQ chaining plan with the mask
(hla_build_bwd_plan): dQ partials of a kv-block pair are summed in TMEM, and q-blocks
whose whole kv list lies in one pair get their dQ written by the main backward kernel
(no fp32 accumulator traffic, no finalize pass when that holds for all of them).

rpb=True adds HWT's global relative position bias (reading R19): a table
`self.rpb` fp32 [heads, 2H-1, 2W-1] (zero-initialised) whose gradient is written to
`self.drpb` by backward() (one memset + the backward kernel's accumulation;
launches_per_step counts the memset).  The kernels hold raw pointers to these two
buffers, so they keep their storage for the layer's lifetime: assigning `layer.rpb = t`
copies t into the table (in place), and `drpb` is read-only.
"""

import torch

from . import api


class HilbertLocalAttention:
    def __init__(self, kind, grid_h, grid_w, win_h=1, win_w=1, batch=1, heads=1, head_dim=64, block=128,
                 shift=0, scale=0.0, device="cuda", fused=True, rpb=False, dq_plan=True, tiled=None):
        self.kind = kind
        self.grid_h, self.grid_w = grid_h, grid_w
        self.N = grid_h * grid_w
        self.shape = (batch, self.N, heads, head_dim)
        self.scale = float(scale)
        # tiled Hilbert order (include/hla.h HLA_ORDER_HILBERT_TILED; R23): the same
        # attention for HWA with 64-token-multiple windows on square 2^k grids; at head_dim 32 the
        # fused loads then move one TMA box per 8 x 8 cell square.  None = where it applies and pays.
        ok = api.tiled_order_applies(kind, grid_h, grid_w, win_h, win_w) and fused and not rpb
        self.tiled = ok and head_dim == 32 if tiled is None else bool(tiled)
        if self.tiled and not ok:
            raise ValueError("tiled order needs fused HWA, a multiple of 64 tokens per window, a square 2^k "
                             "grid >= 8 and no RPB")
        self.desc = api.pattern_desc(kind, grid_h, grid_w, win_h, win_w, block, shift, tiled=self.tiled)
        self.mask = api.hla_build_block_mask(self.desc, device, plan=dq_plan)   # + the backward's dQ plan
        self.hilbert = api.is_hilbert(self.desc)
        bf = dict(dtype=torch.bfloat16, device=device)
        e = lambda: torch.empty(self.shape, **bf)   # noqa: E731
        self.o, self.dq, self.dk, self.dv = e(), e(), e(), e()
        self.lse = torch.empty(batch, heads, self.N, dtype=torch.float32, device=device)
        self.workspace = torch.empty(api.hla_attn_bwd_workspace(batch, heads, self.N, head_dim),
                                     dtype=torch.uint8, device=device)
        self.fused = bool(fused) and self.hilbert
        self.s2c = None
        if self.fused:
            index = api.hla_hilbert_tiled_index if self.tiled else api.hla_hilbert_index
            self.s2c, _ = index(grid_h, grid_w, device)     # the cached path; the sequence order of lse
        elif self.hilbert:
            self.qs, self.ks, self.vs, self.os = e(), e(), e(), e()
            self.dos, self.dqs, self.dks, self.dvs = e(), e(), e(), e()
        self._saved = None
        self._rpb = self._drpb = self.mod = None
        if rpb:
            shape = (heads, 2 * grid_h - 1, 2 * grid_w - 1)
            self._rpb = torch.zeros(shape, dtype=torch.float32, device=device)
            self._drpb = torch.zeros(shape, dtype=torch.float32, device=device)
            cells = None
            if self.hilbert:     # 2D offsets need the sequence -> cell map of the order
                cells = self.s2c if self.s2c is not None else api.hla_hilbert_index(grid_h, grid_w, device)[0]
            self._cells = cells
            self.mod = api.score_mod(self._rpb, self._drpb, cells)
        # backward as one launch when the library folds the preprocess into the main kernel
        self.fused_bwd = api.hla_attn_bwd_fuses_preprocess(self.desc, self.mask, self.mod)

    @property
    def rpb(self):
        """The global-RPB table (None without rpb=True); its storage is fixed for the layer."""
        return self._rpb

    @rpb.setter
    def rpb(self, value):
        if self._rpb is None:
            raise AttributeError("layer built without rpb=True")
        self._rpb.copy_(value)   # in place: the kernels hold this buffer's pointer

    @property
    def drpb(self):
        """Gradient of the RPB table written by backward() (read-only binding)."""
        return self._drpb

    # non-empty tiles of the mask per (b, h): R (P:L102 r_i summed over q-blocks)
    @property
    def nnz(self):
        return self.mask.nnz

    # 128 x 128 tiles the kernels execute per (b, h) and per pass (block 64: windows)
    @property
    def tiles(self):
        return self.mask.tiles

    def forward(self, q, k, v, mark=None):
        """q, k, v: bf16 [B, N, heads, d] in grid (row-major cell) order -> o (grid order).

        mark: optional callable(name) invoked after each launch (bench timing hook)."""
        mark = mark or _nop
        if self.fused:
            api.hla_attn_fwd(self.desc, self.mask, q, k, v, self.scale, self.o, self.lse, seq_to_cell=self.s2c,
                             mod=self.mod)
            mark("fwd")
            self._saved = (q, k, v, self.o)
        elif self.hilbert:
            api.hla_hilbert_perm(self.grid_h, self.grid_w, api.TO_HILBERT, (q, k, v), (self.qs, self.ks, self.vs))
            mark("perm_qkv")
            api.hla_attn_fwd(self.desc, self.mask, self.qs, self.ks, self.vs, self.scale, self.os, self.lse,
                             mod=self.mod)
            mark("fwd")
            api.hla_hilbert_perm(self.grid_h, self.grid_w, api.FROM_HILBERT, (self.os,), (self.o,))
            mark("perm_o")
            self._saved = (self.qs, self.ks, self.vs, self.os)
        else:
            api.hla_attn_fwd(self.desc, self.mask, q, k, v, self.scale, self.o, self.lse, mod=self.mod)
            mark("fwd")
            self._saved = (q, k, v, self.o)
        return self.o

    def backward(self, dout, mark=None):
        """dout: bf16 [B, N, heads, d] in grid order -> (dq, dk, dv) in grid order."""
        mark = mark or _nop
        q, k, v, o = self._saved
        if self.hilbert and not self.fused:
            api.hla_hilbert_perm(self.grid_h, self.grid_w, api.TO_HILBERT, (dout,), (self.dos,))
            mark("perm_do")
            dout_s, dq, dk, dv = self.dos, self.dqs, self.dks, self.dvs
        else:
            dout_s, dq, dk, dv = dout, self.dq, self.dk, self.dv
        if self.fused_bwd:
            # the main kernel forms D / LSE itself (hla_attn_bwd_fuses_preprocess; non-local dQ rows:
            # zeroing before, finalize after, inside the same call)
            api.hla_attn_bwd(self.desc, self.mask, q, k, v, o, self.lse, dout_s, self.scale, dq, dk, dv,
                             self.workspace, seq_to_cell=self.s2c, mod=self.mod)
            mark("bwd")
            return self._grads(mark)
        api.hla_attn_bwd_preprocess(o, dout_s, self.lse, self.workspace, self.scale, seq_to_cell=self.s2c,
                                    mask=self.mask)
        if self._drpb is not None:
            self._drpb.zero_()     # the kernel accumulates the table gradient
        mark("bwd_pre")
        api.hla_attn_bwd_main(self.desc, self.mask, q, k, v, dout_s, dq, dk, dv, self.workspace, self.scale,
                              seq_to_cell=self.s2c, mod=self.mod)
        mark("bwd")
        api.hla_attn_bwd_finalize(self.workspace, dq, seq_to_cell=self.s2c, mask=self.mask)
        mark("bwd_fin")
        return self._grads(mark)

    def _grads(self, mark):
        if self.hilbert and not self.fused:
            api.hla_hilbert_perm(self.grid_h, self.grid_w, api.FROM_HILBERT, (self.dqs, self.dks, self.dvs),
                                 (self.dq, self.dk, self.dv))
            mark("perm_grads")
        return self.dq, self.dk, self.dv

    # kernel launches per step (forward + backward)
    @property
    def launches_per_step(self):
        if self.fused_bwd:   # fwd + the backward's main kernel (+ zeroing / finalize of non-local dQ rows)
            nl = 0 if self.mask.n_dq_nonlocal == 0 else 2
            return 2 + nl + (4 if (self.hilbert and not self.fused) else 0) + (1 if self._rpb is not None else 0)
        fin = 0 if self.mask.n_dq_nonlocal == 0 else 1   # the finalize launches nothing when every dQ is local
        return 3 + fin + (4 if (self.hilbert and not self.fused) else 0) + (1 if self._rpb is not None else 0)

    def step(self, q, k, v, dout, mark=None):
        """One pass of the whole hot path: forward then backward."""
        self.forward(q, k, v, mark)
        return self.backward(dout, mark)


def _nop(_name):
    pass
