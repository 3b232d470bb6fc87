"""GPU parity of the block-sparse attention kernels against the fp64 oracle.

Inputs: hla_synth (seeded, bf16, unit variance; "sharp" = Q x 4), the same
values on both sides.  Bar: max-abs <= 2e-2 and mean-abs <= 2e-3 for O and the
gradients (north_star), LSE max-abs <= 1e-3, skip honesty (tiles executed ==
batch*heads*nnz).  Small cases span several tiles and every pattern; the
BASELINE configs run at full size in the launch configuration bench.py uses,
checked on sampled (b, h) slices and query rows the oracle computes one by one.
"""

import numpy as np
import pytest
import torch

import hla_synth
import paper_2511_05832_b200 as hla
from paper_2511_05832_b200 import api
from oracle import attention as oatt
from oracle import hilbert
from oracle.patterns import Spec
from parity import LSE_MAX_ABS, assert_close, emulated_slice, to_np

pytestmark = pytest.mark.gpu
DEV = "cuda"


def _inputs(B, N, H, d, seed=0, sharp=False):
    return [t.to(DEV) for t in hla_synth.attention_inputs(B, N, H, d, seed=seed, sharp=sharp)]


SMALL = [
    # kind, grid, window, B, heads, d
    ("HWA", 16, 16, 8, 8, 1, 1, 32),       # cfg1
    ("HWA", 32, 32, 8, 8, 2, 3, 64),
    ("HWA", 32, 32, 16, 16, 1, 2, 64),
    ("HSA", 32, 32, 5, 5, 2, 2, 64),
    ("HSA", 32, 32, 16, 16, 1, 2, 32),
    ("HNA", 32, 32, 7, 7, 2, 2, 64),
    ("HSWA", 32, 32, 8, 8, 1, 2, 64),
    ("WSA", 32, 32, 8, 8, 2, 2, 64),
    ("SA", 32, 32, 7, 7, 2, 2, 64),
    ("NA2D", 32, 32, 7, 7, 1, 2, 64),
    ("DENSE", 16, 32, 1, 1, 1, 2, 64),
    ("NA2D", 24, 16, 5, 3, 1, 1, 32),      # non-power-of-two width
    ("WSA", 48, 16, 4, 8, 1, 1, 64),
    # ragged N (N % 128 != 0): phantom rows / columns of the last tile
    ("HWA", 8, 8, 8, 8, 2, 3, 32),         # cfg5 stage 4 (7x7 padded to 8x8: N = 64 < one tile)
    ("HNA", 8, 8, 3, 3, 1, 2, 64),
    ("HSA", 4, 4, 3, 3, 1, 1, 32),         # N = 16
    ("WSA", 56, 56, 7, 7, 1, 2, 64),       # paper shape 56x56, W7 (N = 3136 = 24.5 tiles), row-major
    ("SA", 56, 56, 7, 7, 1, 1, 64),
    ("NA2D", 56, 56, 7, 7, 1, 1, 32),
    ("DENSE", 10, 20, 1, 1, 1, 2, 64),     # N = 200
]


@pytest.mark.parametrize("case", SMALL, ids=lambda c: "%s_%dx%d_w%dx%d_d%d" % (c[0], c[1], c[2], c[3], c[4], c[7]))
@pytest.mark.parametrize("sharp", [False, True])
def test_fwd_small(case, sharp):
    kind, gh, gw, wh, ww, B, H, d = case
    shift = (wh * ww) // 2 if kind == "HSWA" else 0
    N = gh * gw
    q, k, v, _ = _inputs(B, N, H, d, seed=3, sharp=sharp)
    desc = hla.pattern_desc(kind, gh, gw, wh, ww, shift=shift)
    m = hla.hla_build_block_mask(desc, DEV)
    visited = torch.zeros(1, dtype=torch.int64, device=DEV)
    o, lse = hla.hla_attn_fwd(desc, m, q, k, v, tiles_visited=visited)
    torch.cuda.synchronize()
    spec = Spec(kind, gh, gw, wh, ww, shift=shift)
    O_ref, L_ref = oatt.attn_fwd(to_np(q), to_np(k), to_np(v), spec)
    assert_close("O", to_np(o), O_ref)
    assert_close("LSE", to_np(lse), L_ref, max_abs=LSE_MAX_ABS, mean_abs=LSE_MAX_ABS)
    assert int(visited.item()) == B * H * m.nnz


def test_fwd_layer_grid_order_hwa_equals_wsa():
    # finding 4: HWA(256 tokens) on the Hilbert sequence == WSA(16x16) on the grid
    B, H, d, n = 2, 4, 64, 64
    q, k, v, _ = _inputs(B, n * n, H, d, seed=5)
    hwa = hla.HilbertLocalAttention("HWA", n, n, 16, 16, B, H, d, device=DEV)
    wsa = hla.HilbertLocalAttention("WSA", n, n, 16, 16, B, H, d, device=DEV)
    o1 = hwa.forward(q, k, v).clone()
    o2 = wsa.forward(q, k, v).clone()
    torch.cuda.synchronize()
    err = (o1.float() - o2.float()).abs()
    assert err.max().item() <= 2e-2 and err.mean().item() <= 2e-3


# BASELINE configs at full size (bench launch configuration), sampled check
FULL = [
    ("cfg2", "HWA", 64, 64, 16, 16, 16, 8, 64),
    ("cfg2-rm", "WSA", 64, 64, 16, 16, 16, 8, 64),
    ("cfg3", "HSA", 64, 64, 16, 16, 16, 8, 64),
    ("cfg3-rm", "SA", 64, 64, 16, 16, 16, 8, 64),
    ("cfg4", "HNA", 128, 128, 7, 7, 16, 12, 64),
    ("cfg4-rm", "NA2D", 128, 128, 7, 7, 16, 12, 64),
    ("dense", "DENSE", 64, 64, 1, 1, 16, 8, 64),
]


@pytest.mark.parametrize("case", FULL, ids=lambda c: c[0])
def test_fwd_full_size_sampled(case):
    name, kind, gh, gw, wh, ww, B, H, d = case
    N = gh * gw
    q, k, v, _ = _inputs(B, N, H, d, seed=0)
    layer = hla.HilbertLocalAttention(kind, gh, gw, wh, ww, B, H, d, device=DEV)
    o = layer.forward(q, k, v)
    torch.cuda.synchronize()
    assert torch.isfinite(o.float()).all()
    spec = Spec(kind, gh, gw, wh, ww)
    rng = np.random.default_rng(1)
    s2c = hilbert.hilbert_order(gh, gw)[0] if layer.hilbert else np.arange(N)
    for b, h in [(0, 0), (B - 1, H - 1), (int(rng.integers(B)), int(rng.integers(H)))]:
        Q = to_np(q[b, :, h])[s2c]
        K = to_np(k[b, :, h])[s2c]
        V = to_np(v[b, :, h])[s2c]
        rows = np.unique(np.concatenate([np.arange(0, 128), np.arange(N - 128, N), rng.integers(0, N, 256)]))
        O_ref, L_ref = oatt.attn_fwd_slice(Q, K, V, spec, rows=rows)
        got = to_np(o[b, :, h])[s2c][rows]            # layer output is in grid order
        assert_close("%s O[b=%d,h=%d]" % (name, b, h), got, O_ref)
        got_lse = to_np(layer.lse[b, h])[rows]        # LSE stays in sequence order
        assert_close("%s LSE" % name, got_lse, L_ref, max_abs=LSE_MAX_ABS, mean_abs=LSE_MAX_ABS)


@pytest.mark.parametrize("case", SMALL, ids=lambda c: "%s_%dx%d_w%dx%d_d%d" % (c[0], c[1], c[2], c[3], c[4], c[7]))
@pytest.mark.parametrize("sharp", [False, True])
def test_bwd_small(case, sharp):
    kind, gh, gw, wh, ww, B, H, d = case
    shift = (wh * ww) // 2 if kind == "HSWA" else 0
    N = gh * gw
    q, k, v, do = _inputs(B, N, H, d, seed=7, sharp=sharp)
    desc = hla.pattern_desc(kind, gh, gw, wh, ww, shift=shift)
    m = hla.hla_build_block_mask(desc, DEV)
    o, lse = hla.hla_attn_fwd(desc, m, q, k, v)
    visited = torch.zeros(1, dtype=torch.int64, device=DEV)
    dq, dk, dv = hla.hla_attn_bwd(desc, m, q, k, v, o, lse, do, tiles_visited=visited)
    torch.cuda.synchronize()
    spec = Spec(kind, gh, gw, wh, ww, shift=shift)
    dQ, dK, dV = oatt.attn_bwd(to_np(q), to_np(k), to_np(v), to_np(do), spec)
    if not sharp:
        for name, got, ref in (("dQ", dq, dQ), ("dK", dk, dK), ("dV", dv, dV)):
            assert_close(name, to_np(got), ref)            # the north_star bound
    else:
        # DESIGN.md reading R16: the north_star bound is absolute for the workload recipe
        # (unit-variance inputs).  The sharp stress input (Q x 4, outside the paper's
        # workloads) scales the gradients up to ~5x; its bound is the error of the bf16
        # rounding model (tests/parity.py emulated_slice: fp64 with the kernels' rounding
        # points) against the same fp64 oracle, times 1.25.
        emu = {n: np.zeros_like(r) for n, r in (("dQ", dQ), ("dK", dK), ("dV", dV))}
        s2c = np.arange(N)
        for b in range(B):
            for h in range(H):
                _, eq, ek, ev = emulated_slice(*(to_np(t[b, :, h]) for t in (q, k, v, do)), spec)
                emu["dQ"][b, :, h], emu["dK"][b, :, h], emu["dV"][b, :, h] = eq, ek, ev
        for name, got, ref in (("dQ", dq, dQ), ("dK", dk, dK), ("dV", dv, dV)):
            e_gpu = np.abs(to_np(got) - ref)
            e_emu = np.abs(emu[name] - ref)
            assert e_gpu.max() <= 1.25 * e_emu.max() + 1e-3, (name, e_gpu.max(), e_emu.max())
            assert e_gpu.mean() <= 1.25 * e_emu.mean() + 1e-4, (name, e_gpu.mean(), e_emu.mean())
    assert int(visited.item()) == B * H * m.nnz


CFG5 = [(64, 3), (32, 6), (16, 12), (8, 24)]   # HWT-T stages: grid (56/28/14/7 padded), heads


@pytest.mark.parametrize("g,H", CFG5, ids=lambda v: str(v))
def test_cfg5_stage(g, H):
    """BASELINE cfg5: HWT-T stack stage (window 49 -> 64 tokens = 8x8, d32), forward and
    backward through the layer API (fused reorder), one slice checked in full."""
    B, d = 4, 32
    N = g * g
    q, k, v, do = _inputs(B, N, H, d, seed=21)
    layer = hla.HilbertLocalAttention("HWA", g, g, 8, 8, B, H, d, device=DEV)
    assert layer.tiled          # d = 32, 64-token windows: the tiled order and square-box loads
    o = layer.forward(q, k, v).clone()
    dq, dk, dv = (t.clone() for t in layer.backward(do))
    torch.cuda.synchronize()
    spec = Spec("HWA", g, g, 8, 8)
    s2c = hilbert.hilbert_order(g, g)[0]
    b, h = B - 1, H - 1
    Q, K, V, DO = (to_np(t[b, :, h])[s2c] for t in (q, k, v, do))
    dQ, dK, dV, O, _ = oatt.attn_bwd_slice(Q, K, V, DO, spec)
    for name, got, ref in (("O", o, O), ("dQ", dq, dQ), ("dK", dk, dK), ("dV", dv, dV)):
        assert_close("cfg5 g%d %s" % (g, name), to_np(got[b, :, h])[s2c], ref)


@pytest.mark.parametrize("g,w,B,H,d,blk", [(64, 8, 4, 3, 32, 64), (64, 8, 2, 3, 32, 128), (32, 16, 2, 2, 32, 64),
                                          (16, 8, 3, 2, 32, 128), (64, 16, 2, 2, 64, 128), (8, 8, 2, 2, 32, 64),
                                          (32, 8, 2, 2, 64, 64), (16, 8, 2, 3, 64, 128)])
def test_tiled_order_vs_oracle_and_hilbert_order(g, w, B, H, d, blk):
    """HLA_ORDER_HILBERT_TILED (reading R23) through the layer: O, dQ, dK, dV equal the fp64
    oracle of the paper's Hilbert-order HWA on every checked slice, agree with the same layer in
    Hilbert order to bf16 rounding, and the LSE (kept in the tiled sequence order) is the oracle's
    LSE relabeled.  d = 32 runs the square-box loads, d = 64 the gather4 loads over the tiled table."""
    N = g * g
    q, k, v, do = _inputs(B, N, H, d, seed=23)
    til = hla.HilbertLocalAttention("HWA", g, g, w, w, B, H, d, block=blk, device=DEV, tiled=True)
    hil = hla.HilbertLocalAttention("HWA", g, g, w, w, B, H, d, block=blk, device=DEV, tiled=False)
    r1 = [t.clone() for t in (til.forward(q, k, v),) + til.backward(do)]
    r2 = [t.clone() for t in (hil.forward(q, k, v),) + hil.backward(do)]
    torch.cuda.synchronize()
    assert til.tiled and not hil.tiled
    for a, b in zip(r1, r2):
        assert (a.float() - b.float()).abs().max().item() <= 2e-2 * max(b.float().abs().max().item(), 1.0)
    spec = Spec("HWA", g, g, w, w)
    h2c, _ = hilbert.hilbert_order(g, g)
    t2c, _ = hilbert.hilbert_tiled_order(g, g)
    _, c2h = hilbert.hilbert_order(g, g)
    for b, h in [(0, 0), (B - 1, H - 1)]:
        Q, K, V, DO = (to_np(t[b, :, h])[h2c] for t in (q, k, v, do))
        dQ, dK, dV, O, L = oatt.attn_bwd_slice(Q, K, V, DO, spec)
        for name, got, ref in zip(("O", "dQ", "dK", "dV"), r1, (O, dQ, dK, dV)):
            assert_close("tiled g%d b%d %s" % (g, blk, name), to_np(got[b, :, h])[h2c], ref)
        got_lse = to_np(til.lse[b, h])           # position t of the tiled order = cell t2c[t]
        assert_close("tiled LSE", got_lse, L[c2h[t2c]], max_abs=LSE_MAX_ABS, mean_abs=LSE_MAX_ABS)


FULL_BWD = [c for c in FULL if c[0] in ("cfg2", "cfg2-rm", "cfg3", "cfg3-rm", "cfg4", "cfg4-rm")]


@pytest.mark.parametrize("kind,g,w,B,H,d", [("HWA", 64, 16, 4, 8, 64), ("HSA", 64, 16, 2, 3, 64),
                                             ("HNA", 128, 7, 1, 4, 64), ("HWA", 16, 8, 1, 1, 32),
                                             ("HNA", 32, 5, 2, 2, 32), ("HSWA", 32, 8, 2, 2, 64)])
def test_fused_reorder_matches_explicit_permutation(kind, g, w, B, H, d):
    """Fused reorder (TMA gather4 loads + scattered epilogues) == explicit
    hla_hilbert_perm passes: O, dK, dV bit-identical (same tiles, same order);
    dQ within atomics-order rounding."""
    q, k, v, do = _inputs(B, g * g, H, d, seed=11)
    shift = (w * w) // 2 if kind == "HSWA" else 0
    fused = hla.HilbertLocalAttention(kind, g, g, w, w, B, H, d, shift=shift, device=DEV, fused=True, tiled=False)
    plain = hla.HilbertLocalAttention(kind, g, g, w, w, B, H, d, shift=shift, device=DEV, fused=False)
    r1 = [t.clone() for t in (fused.forward(q, k, v),) + fused.backward(do)]
    r2 = [t.clone() for t in (plain.forward(q, k, v),) + plain.backward(do)]
    torch.cuda.synchronize()
    assert plain.launches_per_step == fused.launches_per_step + 4 and fused.launches_per_step in (2, 3, 4)
    assert torch.equal(r1[0], r2[0])                       # O
    assert torch.equal(fused.lse, plain.lse)
    assert torch.equal(r1[2], r2[2]) and torch.equal(r1[3], r2[3])   # dK, dV
    assert (r1[1].float() - r2[1].float()).abs().max().item() <= 2e-3   # dQ (fp32 atomics order)


@pytest.mark.parametrize("case", FULL_BWD, ids=lambda c: c[0])
def test_step_full_size_sampled(case):
    """Full hot-path step through the public layer API (perm -> fwd -> unperm ->
    perm dO -> bwd -> unperm), exactly what bench.py times; one (b, h) slice is
    checked completely against the fp64 oracle and every slice against the
    backward invariants sum_k dK = 0 and sum_k dV = sum_q dO."""
    name, kind, gh, gw, wh, ww, B, H, d = case
    N = gh * gw
    q, k, v, do = _inputs(B, N, H, d, seed=0)
    layer = hla.HilbertLocalAttention(kind, gh, gw, wh, ww, B, H, d, device=DEV)
    dq, dk, dv = layer.step(q, k, v, do)
    torch.cuda.synchronize()
    for t in (dq, dk, dv):
        assert torch.isfinite(t.float()).all()
    # invariants on every slice: sum_k dK = 0, sum_k dV = sum_q dO (exact for the
    # fp64 oracle).  On the GPU, bf16 rounding of the dS / P MMA operands leaves a
    # residual ~ sqrt(N) * rms * 2^-8 per column; bound it at 8x that.
    tol = 8 * np.sqrt(N) * float(dk.float().pow(2).mean().sqrt()) * 2 ** -8
    assert dk.float().sum(1).abs().max().item() <= tol
    assert (dv.float().sum(1) - do.float().sum(1)).abs().max().item() <= tol
    spec = Spec(kind, gh, gw, wh, ww)
    s2c = hilbert.hilbert_order(gh, gw)[0] if layer.hilbert else np.arange(N)
    b, h = B - 1, H // 2
    Q, K, V, DO = (to_np(t[b, :, h])[s2c] for t in (q, k, v, do))
    dQ, dK, dV, _, _ = oatt.attn_bwd_slice(Q, K, V, DO, spec, chunk=512)
    assert_close("%s dQ" % name, to_np(dq[b, :, h])[s2c], dQ)
    assert_close("%s dK" % name, to_np(dk[b, :, h])[s2c], dK)
    assert_close("%s dV" % name, to_np(dv[b, :, h])[s2c], dV)


# ------------------------------------------------------------- global RPB (R19, R20)
RPB_CASES = [
    # kind, grid, window, B, heads, d, fused
    ("HWA", 32, 8, 2, 2, 64, True),
    ("HSWA", 32, 8, 1, 3, 32, True),       # HWT's second block of a pair, d32 (cfg5 family)
    ("HNA", 32, 5, 1, 2, 64, False),       # explicit permutation path
    ("WSA", 32, 8, 2, 2, 64, True),        # row-major: identity cell map
    ("WSA", 56, 7, 1, 1, 32, True),        # 56x56 (paper shape), ragged last tile
    ("HWA", 56, 7, 1, 2, 32, True),        # generalized Hilbert 56x56 (fused), ragged last tile
    ("HSWA", 28, 7, 2, 6, 32, True),       # cfg5 stage 2 shape (HWT-T), 49-token shifted windows
    ("HSWA", 8, 8, 2, 24, 32, True),       # cfg5 stage 4 (7x7 padded to 8x8, 8x8 windows: N = 64 < one tile)
]


@pytest.mark.parametrize("case", RPB_CASES, ids=lambda c: "%s%d_d%d" % (c[0], c[1], c[5]))
def test_rpb_fwd_bwd_vs_oracle(case):
    """HWT's global relative position bias: O, LSE,
    dQ, dK, dV under the north_star bound; the table gradient (a sum over up to
    B*N pairs per offset) under a relative L2 bound (reading R20)."""
    kind, g, w, B, H, d, fused = case
    N = g * g
    shift = (w * w) // 2 if kind == "HSWA" else 0
    q, k, v, do = _inputs(B, N, H, d, seed=21)
    layer = hla.HilbertLocalAttention(kind, g, g, w, w, B, H, d, shift=shift, device=DEV, fused=fused, rpb=True)
    table = torch.rand(layer.rpb.shape, generator=torch.Generator().manual_seed(5), dtype=torch.float64)
    layer.rpb.copy_((2 * table - 1).float())            # U(-1, 1): the bias moves the softmax
    o = layer.forward(q, k, v)
    dq, dk, dv = layer.backward(do)
    torch.cuda.synchronize()
    spec = Spec(kind, g, g, w, w, shift=shift)
    s2c = hilbert.hilbert_order(g, g)[0] if spec.order == "hilbert" else np.arange(N)
    seq = lambda t: hilbert.to_sequence(to_np(t), s2c)   # noqa: E731  grid -> sequence order
    T = layer.rpb.double().cpu().numpy()
    O_ref, L_ref = oatt.attn_fwd(seq(q), seq(k), seq(v), spec, rpb=T)
    dQ_ref, dK_ref, dV_ref, dT_ref = oatt.attn_bwd(seq(q), seq(k), seq(v), seq(do), spec, rpb=T)
    assert_close("rpb O", seq(o), O_ref)
    assert np.abs(to_np(layer.lse) - L_ref).max() <= LSE_MAX_ABS
    for name, got, ref in (("dQ", dq, dQ_ref), ("dK", dk, dK_ref), ("dV", dv, dV_ref)):
        assert_close("rpb " + name, seq(got), ref)
    dT = layer.drpb.double().cpu().numpy()
    rel = np.linalg.norm(dT - dT_ref) / np.linalg.norm(dT_ref)
    assert rel <= 2e-2, rel
    assert abs(dT.sum()) <= 1e-3 * np.abs(dT_ref).sum() + 1e-3   # rows of dS sum to zero


def test_rpb_zero_table_matches_no_bias():
    """A zero table leaves O / gradients at the no-bias result (same tiles, same
    arithmetic up to the log2-domain reassociation of the score)."""
    g, w, B, H, d = 32, 8, 1, 2, 64
    q, k, v, do = _inputs(B, g * g, H, d, seed=22)
    a = hla.HilbertLocalAttention("HWA", g, g, w, w, B, H, d, device=DEV)
    b = hla.HilbertLocalAttention("HWA", g, g, w, w, B, H, d, device=DEV, rpb=True)
    ra = [t.clone() for t in (a.forward(q, k, v),) + a.backward(do)]
    rb = [t.clone() for t in (b.forward(q, k, v),) + b.backward(do)]
    torch.cuda.synchronize()
    for x, y in zip(ra, rb):
        assert (x.float() - y.float()).abs().max().item() <= 2e-2


@pytest.mark.parametrize("kind,g,w,B,H,d", [("HWA", 64, 16, 2, 4, 64), ("HSA", 64, 16, 2, 3, 64),
                                             ("HNA", 32, 5, 2, 2, 32), ("DENSE", 16, 1, 1, 2, 64),
                                             ("HWA", 56, 7, 2, 3, 32), ("HSWA", 32, 8, 2, 2, 64),
                                             ("WSA", 32, 8, 2, 2, 64)])
@pytest.mark.parametrize("fused", [True, False])
def test_dq_plan_matches_no_plan(kind, g, w, B, H, d, fused):
    """The backward's dQ plan (TMEM chaining, direct bf16 dQ for local q-blocks) changes
    only the summation of dQ partials: dK, dV bit-identical, dQ within fp32-order
    rounding of the same products, both against a mask without plan."""
    if not fused and kind.startswith("H") and g & (g - 1):
        pytest.skip("the explicit permutation kernel needs a 2^k grid")
    q, k, v, do = _inputs(B, g * g, H, d, seed=5)
    shift = (w * w) // 2 if kind == "HSWA" else 0
    a = hla.HilbertLocalAttention(kind, g, g, w, w, B, H, d, shift=shift, device=DEV, fused=fused)
    b = hla.HilbertLocalAttention(kind, g, g, w, w, B, H, d, shift=shift, device=DEV, fused=fused, dq_plan=False)
    assert a.mask.n_dq_nonlocal >= 0 and b.mask.n_dq_nonlocal == -1
    r1 = [t.clone() for t in (a.forward(q, k, v),) + a.backward(do)]
    r2 = [t.clone() for t in (b.forward(q, k, v),) + b.backward(do)]
    torch.cuda.synchronize()
    assert torch.equal(r1[0], r2[0])
    assert torch.equal(r1[3], r2[3])   # dV = P^T dO: the same products in the same order
    if a.fused_bwd:   # D formed in the kernel: fp32 summation order of rowsum(dO o O) differs
        assert (r1[2].float() - r2[2].float()).abs().max().item() <= 2e-3
    else:
        assert torch.equal(r1[2], r2[2])
    assert (r1[1].float() - r2[1].float()).abs().max().item() <= 2e-3


@pytest.mark.parametrize("g,w,B,H,d,blk", [(64, 16, 2, 4, 64, 128), (32, 16, 2, 3, 32, 128), (48, 16, 1, 2, 64, 128),
                                           (16, 16, 1, 2, 64, 128), (32, 8, 2, 3, 32, 128), (32, 8, 2, 3, 32, 64),
                                           (16, 8, 2, 2, 64, 64), (8, 8, 2, 3, 32, 64), (8, 8, 1, 2, 32, 128)])
@pytest.mark.parametrize("fused", [True, False])
def test_bwd_fused_preprocess_matches_staged(g, w, B, H, d, blk, fused):
    """hla_attn_bwd folds the preprocess into the main kernel when every q-block's dQ is local
    (HWA windows of whole 128-blocks, cfg2: full-tile schedule; 64-token windows, cfg5: half-tile
    schedule, block 128 or 64): D = rowsum(dO o O) and LSE log2(e) are formed
    in the kernel from the raw LSE and the O tile.  Against the staged calls (preprocess ->
    main -> finalize) on the same mask: dV bit-identical, dQ / dK within fp32 order of D; and
    one (b, h) slice against the fp64 oracle."""
    if not fused and g & (g - 1):
        pytest.skip("the explicit permutation kernel needs a 2^k grid")
    N = g * g
    q, k, v, do = _inputs(B, N, H, d, seed=31)
    lay = hla.HilbertLocalAttention("HWA", g, g, w, w, B, H, d, block=blk, device=DEV, fused=fused)
    assert lay.fused_bwd and lay.mask.n_dq_nonlocal == 0   # (windows of whole block pairs: never ragged)
    lay.forward(q, k, v)
    r1 = [t.clone() for t in lay.backward(do)]
    # the staged path on the same mask, in the layer's sequence order
    qq, kk, vv, oo = lay._saved
    dos = do
    if lay.hilbert and not lay.fused:
        dos = torch.empty_like(do)
        api.hla_hilbert_perm(g, g, api.TO_HILBERT, (do,), (dos,))
    ws = torch.empty_like(lay.workspace)
    dq2, dk2, dv2 = torch.empty_like(q), torch.empty_like(q), torch.empty_like(q)
    api.hla_attn_bwd_preprocess(oo, dos, lay.lse, ws, seq_to_cell=lay.s2c, mask=lay.mask)
    api.hla_attn_bwd_main(lay.desc, lay.mask, qq, kk, vv, dos, dq2, dk2, dv2, ws, seq_to_cell=lay.s2c)
    api.hla_attn_bwd_finalize(ws, dq2, seq_to_cell=lay.s2c, mask=lay.mask)
    r2 = [dq2, dk2, dv2]
    if lay.hilbert and not lay.fused:
        r2 = [torch.empty_like(q) for _ in range(3)]
        api.hla_hilbert_perm(g, g, api.FROM_HILBERT, (dq2, dk2, dv2), tuple(r2))
    torch.cuda.synchronize()
    assert torch.equal(r1[2], r2[2])
    for x, y in zip(r1[:2], r2[:2]):
        assert (x.float() - y.float()).abs().max().item() <= 2e-3
    # one slice against the fp64 oracle (grid order in, grid order out)
    spec = Spec("HWA", g, g, w, w)
    s2c = hilbert.hilbert_order(g, g)[0]
    b, h = B - 1, H - 1
    sl = lambda t: to_np(t[b, :, h, :])[s2c]   # grid order -> sequence order   # noqa: E731
    dq_r, dk_r, dv_r = oatt.attn_bwd_slice(sl(q), sl(k), sl(v), sl(do), spec)[:3]
    for name, got, ref in (("dq", r1[0], dq_r), ("dk", r1[1], dk_r), ("dv", r1[2], dv_r)):
        assert_close(name, sl(got), ref)


def test_rpb_gradient_small_upstream_gradient():
    """the table gradient sums dL/dscore over many pairs; with a mean-reduced loss
    dO is ~1e-6 and every per-pair term is tiny.  The per-tile power-of-two fixed-point scale
    keeps the relative accuracy independent of that magnitude (reading R20's bound)."""
    kind, g, w, B, H, d = "HWA", 32, 8, 2, 2, 64
    N = g * g
    q, k, v, do = _inputs(B, N, H, d, seed=23)
    do = (do.float() * 1e-6).to(torch.bfloat16)
    layer = hla.HilbertLocalAttention(kind, g, g, w, w, B, H, d, device=DEV, rpb=True)
    table = torch.rand(layer.rpb.shape, generator=torch.Generator().manual_seed(6), dtype=torch.float64)
    layer.rpb = (2 * table - 1).float()
    layer.forward(q, k, v)
    layer.backward(do)
    torch.cuda.synchronize()
    spec = Spec(kind, g, g, w, w)
    s2c = hilbert.hilbert_order(g, g)[0]
    seq = lambda t: hilbert.to_sequence(to_np(t), s2c)   # noqa: E731
    T = layer.rpb.double().cpu().numpy()
    _, _, _, dT_ref = oatt.attn_bwd(seq(q), seq(k), seq(v), seq(do), spec, rpb=T)
    dT = layer.drpb.double().cpu().numpy()
    assert np.abs(dT_ref).max() < 1e-4          # the regime of the finding
    rel = np.linalg.norm(dT - dT_ref) / np.linalg.norm(dT_ref)
    assert rel <= 2e-2, rel


def test_bwd_rejects_before_launching():
    """hla.h: on a non-OK status nothing has been launched -- hla_attn_bwd validates every
    stage (a missing O here) before it zeroes drpb or runs the preprocess."""
    g, w, B, H, d = 32, 8, 1, 2, 64
    q, k, v, do = _inputs(B, g * g, H, d, seed=24)
    layer = hla.HilbertLocalAttention("HWA", g, g, w, w, B, H, d, device=DEV, rpb=True)
    o, lse = layer.forward(q, k, v), layer.lse
    layer.drpb.fill_(7.0)
    ws = torch.full((hla.hla_attn_bwd_workspace(B, H, g * g, d),), 0x5A, dtype=torch.uint8, device=DEV)
    with pytest.raises(hla.HlaError):
        hla.hla_attn_bwd(layer.desc, layer.mask, q, k, v, None, lse, do, workspace=ws, seq_to_cell=layer.s2c,
                         mod=layer.mod)
    torch.cuda.synchronize()
    assert bool((layer.drpb == 7.0).all()) and bool((ws == 0x5A).all())


# the HWT-T stack bench.py times as cfg5-hwt (bench.py STACK): grid, heads, window side
CFG5_HWT = [(56, 3, 7), (28, 6, 7), (14, 12, 7), (8, 24, 8)]


@pytest.mark.parametrize("kind", ["HWA", "HSWA"])
@pytest.mark.parametrize("g,H,w", CFG5_HWT, ids=lambda v: str(v))
def test_cfg5_hwt_layer_as_timed(g, H, w, kind):
    """Every layer shape of the timed HWT stack (generalized Hilbert curve, ragged N, 49-token
    windows, HWA / HSWA with shift = half a window, global RPB, d32) at B = 2 through the layer
    API exactly as bench.py runs it: O, dQ, dK, dV of every (b, h) slice under the north_star
    bound, the RPB table gradient under reading R20's relative bound."""
    B, d = 2, 32
    N = g * g
    shift = (w * w) // 2 if kind == "HSWA" else 0
    q, k, v, do = _inputs(B, N, H, d, seed=31)
    layer = hla.HilbertLocalAttention(kind, g, g, w, w, B, H, d, shift=shift, device=DEV, rpb=True)
    table = torch.rand(layer.rpb.shape, generator=torch.Generator().manual_seed(g), dtype=torch.float64)
    layer.rpb = (2 * table - 1).float()
    o = layer.forward(q, k, v).clone()
    dq, dk, dv = (t.clone() for t in layer.backward(do))
    torch.cuda.synchronize()
    spec = Spec(kind, g, g, w, w, shift=shift)
    s2c = hilbert.hilbert_order(g, g)[0]
    T = layer.rpb.double().cpu().numpy()
    dT_ref = np.zeros_like(T)
    for b in range(B):
        for h in range(H):
            Q, K, V, DO = (to_np(t[b, :, h])[s2c] for t in (q, k, v, do))
            dQ, dK, dV, O, _, dTh = oatt.attn_bwd_slice(Q, K, V, DO, spec, rpb=T[h])
            dT_ref[h] += dTh
            for name, got, ref in (("O", o, O), ("dQ", dq, dQ), ("dK", dk, dK), ("dV", dv, dV)):
                assert_close("cfg5-hwt %s g%d b%d h%d %s" % (kind, g, b, h, name), to_np(got[b, :, h])[s2c], ref)
    dT = layer.drpb.double().cpu().numpy()
    assert np.linalg.norm(dT - dT_ref) / np.linalg.norm(dT_ref) <= 2e-2


# ------------------------------------------------------------------ block 64
def _windows_ref(km):
    """Reference window lists of a block-64 kind matrix (tests only): per 128-row tile the
    union of the two 64-blocks' non-empty columns, cut greedily into (u, u + 1) windows;
    kind 1 iff all four 64 x 64 sub-tiles are full (include/hla.h hla_build_tile_lists)."""
    from oracle import blocks
    M = km.shape[0]
    rp, cols, kinds = [0], [], []
    for t in range((M + 1) // 2):
        rows = [r for r in (2 * t, 2 * t + 1) if r < M]
        u = sorted({int(c) for r in rows for c in np.nonzero(km[r])[0]})
        covered = -1
        for c in u:
            if c <= covered:
                continue
            sub = [km[r, cc] if (r < M and cc < km.shape[1]) else 0 for r in (2 * t, 2 * t + 1) for cc in (c, c + 1)]
            cols.append(c)
            kinds.append(1 if all(k == blocks.FULL for k in sub) else 2)
            covered = c + 1
        rp.append(len(cols))
    return np.array(rp), np.array(cols), np.array(kinds)


B64_MASKS = [("HNA", 128, 128, 7, 7), ("HWA", 64, 64, 8, 8), ("HWA", 56, 56, 7, 7), ("HSA", 64, 64, 16, 16),
             ("NA2D", 56, 56, 7, 7), ("WSA", 64, 64, 8, 8), ("DENSE", 24, 20, 1, 1), ("HSWA", 32, 32, 8, 8)]


@pytest.mark.parametrize("kind,H,W,wh,ww", B64_MASKS)
def test_block64_window_lists(kind, H, W, wh, ww):
    from oracle import blocks
    shift = (wh * ww) // 2 if kind == "HSWA" else 0
    spec = Spec(kind, H, W, wh, ww, shift=shift)
    km = blocks.classify_spec(spec, 64, 64)
    m = hla.hla_build_block_mask(hla.pattern_desc(kind, H, W, wh, ww, block=64, shift=shift), DEV)
    for rows, (wrp, wcol, wkind) in (((m.w_row_ptr, m.w_col, m.w_kind), _windows_ref(km)),
                                     ((m.wt_row_ptr, m.wt_col, m.wt_kind), _windows_ref(km.T))):
        n = int(wrp[-1])
        assert np.array_equal(rows[0].cpu().numpy(), wrp)
        assert np.array_equal(rows[1].cpu().numpy()[:n], wcol)
        assert np.array_equal(rows[2].cpu().numpy()[:n], wkind)
    assert m.w_counts[0] == int(_windows_ref(km)[0][-1])


B64_CASES = [
    # kind, grid, window, B, heads, d
    ("HWA", 32, 32, 8, 8, 2, 2, 64),      # 64-token windows: one full 64 x 64 sub-tile per q-block
    ("HNA", 32, 32, 7, 7, 2, 2, 64),      # cfg4 family (49 tokens)
    ("HSA", 32, 32, 9, 9, 1, 2, 32),
    ("HSWA", 32, 32, 8, 8, 1, 2, 64),
    ("WSA", 32, 32, 8, 8, 1, 2, 64),
    ("NA2D", 24, 16, 5, 3, 1, 2, 32),      # 2D, non-power-of-two width
    ("HWA", 56, 56, 7, 7, 1, 2, 32),       # ragged: N = 3136 = 49 blocks of 64 (odd: last tile one block)
    ("DENSE", 10, 20, 1, 1, 1, 2, 64),     # N = 200
]


@pytest.mark.parametrize("case", B64_CASES, ids=lambda c: "%s_%dx%d_w%dx%d_d%d" % (c[0], c[1], c[2], c[3], c[4], c[7]))
def test_block64_fwd_bwd(case):
    kind, gh, gw, wh, ww, B, H, d = case
    shift = (wh * ww) // 2 if kind == "HSWA" else 0
    N = gh * gw
    q, k, v, do = _inputs(B, N, H, d, seed=41)
    layer = hla.HilbertLocalAttention(kind, gh, gw, wh, ww, B, H, d, block=64, shift=shift, device=DEV)
    visited = torch.zeros(1, dtype=torch.int64, device=DEV)
    hla.hla_attn_fwd(layer.desc, layer.mask, q, k, v, tiles_visited=visited, seq_to_cell=layer.s2c)
    layer.forward(q, k, v)
    dq, dk, dv = layer.backward(do)
    torch.cuda.synchronize()
    assert int(visited.item()) == B * H * layer.tiles
    spec = Spec(kind, gh, gw, wh, ww, shift=shift)
    s2c = hilbert.hilbert_order(gh, gw)[0] if layer.hilbert else np.arange(N)
    seq = lambda t: hilbert.to_sequence(to_np(t), s2c)   # noqa: E731
    O_ref, L_ref = oatt.attn_fwd(seq(q), seq(k), seq(v), spec)
    dQ, dK, dV = oatt.attn_bwd(seq(q), seq(k), seq(v), seq(do), spec)
    assert_close("b64 O", seq(layer.o), O_ref)
    assert np.abs(to_np(layer.lse) - L_ref).max() <= LSE_MAX_ABS
    for name, got, ref in (("dQ", dq, dQ), ("dK", dk, dK), ("dV", dv, dV)):
        assert_close("b64 " + name, seq(got), ref)


@pytest.mark.parametrize("case", B64_CASES, ids=lambda c: "%s_%dx%d_w%dx%d_d%d" % (c[0], c[1], c[2], c[3], c[4], c[7]))
def test_block64_dq_plan_matches_no_plan(case):
    """Block 64: the dQ plan runs over the window lists when every window starts on a 128-row
    boundary (HWA with 64-token windows: cfg5 at block 64) -- then every q tile's dQ is local and
    written directly; otherwise there is no plan.  Same contract as test_dq_plan_matches_no_plan."""
    kind, gh, gw, wh, ww, B, H, d = case
    shift = (wh * ww) // 2 if kind == "HSWA" else 0
    q, k, v, do = _inputs(B, gh * gw, H, d, seed=43)
    a = hla.HilbertLocalAttention(kind, gh, gw, wh, ww, B, H, d, block=64, shift=shift, device=DEV)
    b = hla.HilbertLocalAttention(kind, gh, gw, wh, ww, B, H, d, block=64, shift=shift, device=DEV, dq_plan=False)
    aligned = bool((a.mask.w_col[:a.mask.w_counts[0]] % 2 == 0).all()) and \
        bool((a.mask.wt_col[:a.mask.w_counts[2]] % 2 == 0).all())
    assert (a.mask.n_dq_nonlocal >= 0) == aligned and b.mask.n_dq_nonlocal == -1
    if kind == "HWA" and wh * ww == 64:
        assert a.mask.n_dq_nonlocal == 0        # every 64-token window inside one 128-row tile
    r1 = [t.clone() for t in (a.forward(q, k, v),) + a.backward(do)]
    r2 = [t.clone() for t in (b.forward(q, k, v),) + b.backward(do)]
    torch.cuda.synchronize()
    assert torch.equal(r1[0], r2[0])
    assert torch.equal(r1[3], r2[3])
    tol = 2e-3 if a.fused_bwd else 0.0
    assert (r1[2].float() - r2[2].float()).abs().max().item() <= tol
    assert (r1[1].float() - r2[1].float()).abs().max().item() <= 2e-3


def test_block64_cfg4_slice_and_rpb():
    """cfg4 at block 64 (the shape of the b = 64 bench line) on sampled slices, and the global
    RPB score_mod at block 64 (both backward schedules see window lists)."""
    B, H, d, g = 2, 12, 64, 128
    q, k, v, do = _inputs(B, g * g, H, d, seed=0)
    layer = hla.HilbertLocalAttention("HNA", g, g, 7, 7, B, H, d, block=64, device=DEV)
    o = layer.forward(q, k, v).clone()
    dq, dk, dv = (t.clone() for t in layer.backward(do))
    torch.cuda.synchronize()
    spec = Spec("HNA", g, g, 7, 7)
    s2c = hilbert.hilbert_order(g, g)[0]
    b, h = B - 1, 5
    Q, K, V, DO = (to_np(t[b, :, h])[s2c] for t in (q, k, v, do))
    dQ, dK, dV, O, _ = oatt.attn_bwd_slice(Q, K, V, DO, spec, chunk=512)
    for name, got, ref in (("O", o, O), ("dQ", dq, dQ), ("dK", dk, dK), ("dV", dv, dV)):
        assert_close("cfg4-b64 " + name, to_np(got[b, :, h])[s2c], ref)
    g2, w2 = 32, 8
    q, k, v, do = _inputs(1, g2 * g2, 2, 32, seed=42)
    lay = hla.HilbertLocalAttention("HWA", g2, g2, w2, w2, 1, 2, 32, block=64, device=DEV, rpb=True)
    table = torch.rand(lay.rpb.shape, generator=torch.Generator().manual_seed(7), dtype=torch.float64)
    lay.rpb = (2 * table - 1).float()
    lay.forward(q, k, v)
    lay.backward(do)
    torch.cuda.synchronize()
    spec = Spec("HWA", g2, g2, w2, w2)
    s2c = hilbert.hilbert_order(g2, g2)[0]
    seq = lambda t: hilbert.to_sequence(to_np(t), s2c)   # noqa: E731
    T = lay.rpb.double().cpu().numpy()
    O_ref, _ = oatt.attn_fwd(seq(q), seq(k), seq(v), spec, rpb=T)
    _, _, _, dT_ref = oatt.attn_bwd(seq(q), seq(k), seq(v), seq(do), spec, rpb=T)
    assert_close("b64 rpb O", seq(lay.o), O_ref)
    dT = lay.drpb.double().cpu().numpy()
    assert np.linalg.norm(dT - dT_ref) / np.linalg.norm(dT_ref) <= 2e-2
