"""Pins for oracle.attention (CPU only).

The attention oracle is the plain definition of masked softmax attention (P:L85,
P:L275).  It is pinned against things other than itself:
  * a library routine: torch.nn.functional.scaled_dot_product_attention in
    float64 with a boolean attn_mask (and torch.autograd through it for the
    backward);
  * closed forms: constant V -> O = V; a single
    allowed key -> O = v_k; Q = K = 0 -> mean of the allowed V rows;
  * scipy.special.logsumexp for the LSE;
  * central finite differences in fp64 at N=16, d=4 (rel <= 1e-6);
  * permutation equivariance and HWA(4^k) == WSA(2^k x 2^k) after
    un-permutation (the Hilbert quadrant property);
  * backward invariants sum_k dK[k] = 0 and sum_k dV[k] = sum_q dO[q].
"""

import numpy as np
import pytest
import torch
from scipy.special import logsumexp

from oracle import attention, hilbert, patterns
from oracle.patterns import Spec

SPECS = [
    Spec("HWA", 8, 8, 4, 4), Spec("HSA", 8, 8, 3, 3), Spec("HNA", 8, 8, 3, 3),
    Spec("HSWA", 8, 8, 4, 4, shift=8), Spec("WSA", 8, 8, 4, 4), Spec("SA", 8, 8, 3, 3),
    Spec("NA2D", 8, 8, 5, 5), Spec("DENSE", 8, 8), Spec("SA", 8, 8, 4, 4),
]


def _rand(shape, seed):
    return np.random.default_rng(seed).standard_normal(shape)


def _sdpa(Q, K, V, M, scale):
    t = lambda a: torch.from_numpy(np.ascontiguousarray(a))
    return torch.nn.functional.scaled_dot_product_attention(
        t(Q)[None, None], t(K)[None, None], t(V)[None, None],
        attn_mask=t(M)[None, None], scale=scale)[0, 0].numpy()


@pytest.mark.parametrize("spec", SPECS, ids=lambda s: s.kind + str(s.win_h))
def test_fwd_matches_sdpa_fp64(spec):
    N, d = spec.n_tokens, 16
    Q, K, V = _rand((N, d), 1), _rand((N, d), 2), _rand((N, d), 3)
    M = patterns.materialize(spec)
    O, LSE = attention.attn_fwd_slice(Q, K, V, spec, chunk=7)
    sc = 1 / np.sqrt(d)
    assert np.allclose(O, _sdpa(Q, K, V, M, sc), rtol=0, atol=1e-12)
    S = sc * Q @ K.T
    lse = np.array([logsumexp(S[i][M[i]]) for i in range(N)])
    assert np.allclose(LSE, lse, rtol=0, atol=1e-12)


def test_closed_forms():
    spec = Spec("HNA", 8, 8, 3, 3)
    N, d = 64, 8
    Q, K = _rand((N, d), 4), _rand((N, d), 5)
    c = _rand((d,), 6)
    O, _ = attention.attn_fwd_slice(Q, K, np.tile(c, (N, 1)), spec)
    assert np.allclose(O, np.tile(c, (N, 1)), atol=1e-14)
    Z = np.zeros((N, d))
    V = _rand((N, d), 7)
    O, _ = attention.attn_fwd_slice(Z, Z, V, spec)
    M = patterns.materialize(spec)
    assert np.allclose(O, (M @ V) / M.sum(1, keepdims=True), atol=1e-14)
    # single allowed key: HWA with window of one token -> O = v_q
    O, _ = attention.attn_fwd_slice(Q, K, V, Spec("HWA", 8, 8, 1, 1))
    assert np.allclose(O, V, atol=1e-14)


def test_permutation_equivariance():
    # f(Pq, Pk, Pv, P M P^T) = P f(q, k, v, M) -- here with P = the Hilbert
    # order: an HWA computed on the Hilbert sequence, mapped back to the grid,
    # equals attention on the grid with the conjugated mask.
    H = W = 8
    spec = Spec("HWA", H, W, 2, 4)          # windows of 8 tokens: irregular 2D shapes
    s2c, c2s = hilbert.hilbert_order(H, W)
    N, d = H * W, 8
    q, k, v = (_rand((1, N, 1, d), s) for s in (8, 9, 10))
    O_seq, _ = attention.attn_fwd(hilbert.to_sequence(q, s2c), hilbert.to_sequence(k, s2c),
                                  hilbert.to_sequence(v, s2c), spec)
    M_seq = patterns.materialize(spec)
    M_grid = M_seq[np.ix_(c2s, c2s)]        # allowed(cell a, cell b) in grid indices
    O_grid = _sdpa(q[0, :, 0], k[0, :, 0], v[0, :, 0], M_grid, 1 / np.sqrt(d))
    assert np.allclose(hilbert.to_grid(O_seq, s2c)[0, :, 0], O_grid, atol=1e-12)


@pytest.mark.parametrize("k", [1, 2, 3])
def test_hwa_equals_wsa_after_unpermutation(k):
    # SURVEY finding 4: aligned Hilbert runs of 4^k tokens are aligned 2^k squares,
    # so HWA(4^k) un-permuted == WSA(2^k x 2^k) on the grid.
    H = W = 16
    side = 1 << k
    s2c, _ = hilbert.hilbert_order(H, W)
    N, d = H * W, 4
    q, kk, v = (_rand((2, N, 3, d), s) for s in (11, 12, 13))
    O_h, L_h = attention.attn_fwd(*(hilbert.to_sequence(x, s2c) for x in (q, kk, v)),
                                  Spec("HWA", H, W, side, side))
    O_w, L_w = attention.attn_fwd(q, kk, v, Spec("WSA", H, W, side, side))
    assert np.allclose(hilbert.to_grid(O_h, s2c), O_w, atol=1e-12)
    assert np.allclose(L_h[:, :, np.argsort(s2c)], L_w, atol=1e-12)


@pytest.mark.parametrize("spec", SPECS, ids=lambda s: s.kind + str(s.win_h))
def test_bwd_matches_autograd_sdpa(spec):
    N, d = spec.n_tokens, 8
    Q, K, V, dO = (_rand((N, d), s) for s in (20, 21, 22, 23))
    dQ, dK, dV, O, _ = attention.attn_bwd_slice(Q, K, V, dO, spec, chunk=5)
    M = torch.from_numpy(patterns.materialize(spec))
    tq, tk, tv = (torch.from_numpy(a).requires_grad_(True) for a in (Q, K, V))
    out = torch.nn.functional.scaled_dot_product_attention(tq[None], tk[None], tv[None],
                                                           attn_mask=M[None], scale=1 / np.sqrt(d))[0]
    out.backward(torch.from_numpy(dO))
    assert np.allclose(O, out.detach().numpy(), atol=1e-12)
    for mine, ref in ((dQ, tq.grad), (dK, tk.grad), (dV, tv.grad)):
        assert np.allclose(mine, ref.numpy(), rtol=0, atol=1e-11)
    # invariants from sum_k Phat = 1 and sum_k dS = 0
    assert np.allclose(dK.sum(0), 0, atol=1e-11)
    assert np.allclose(dV.sum(0), dO.sum(0), atol=1e-11)


def test_bwd_finite_differences():
    # N=16, head_dim=4, fp64, central differences h=1e-5, rel err <= 1e-6
    spec = Spec("HSA", 4, 4, 3, 3)
    N, d, h = 16, 4, 1e-5
    Q, K, V, dO = (_rand((N, d), s) for s in (30, 31, 32, 33))
    dQ, dK, dV, _, _ = attention.attn_bwd_slice(Q, K, V, dO, spec)

    def loss(Q_, K_, V_):
        O, _ = attention.attn_fwd_slice(Q_, K_, V_, spec)
        return float((O * dO).sum())

    for which, grad in ((0, dQ), (1, dK), (2, dV)):
        num = np.zeros((N, d))
        for i in range(N):
            for j in range(d):
                args_p = [Q.copy(), K.copy(), V.copy()]
                args_m = [Q.copy(), K.copy(), V.copy()]
                args_p[which][i, j] += h
                args_m[which][i, j] -= h
                num[i, j] = (loss(*args_p) - loss(*args_m)) / (2 * h)
        rel = np.abs(num - grad).max() / np.abs(grad).max()
        assert rel <= 1e-6, (which, rel)


def test_zero_upstream_gradient():
    spec = Spec("NA2D", 4, 4, 3, 3)
    N, d = 16, 4
    Q, K, V = (_rand((N, d), s) for s in (40, 41, 42))
    dQ, dK, dV, _, _ = attention.attn_bwd_slice(Q, K, V, np.zeros((N, d)), spec)
    assert not dQ.any() and not dK.any() and not dV.any()


# ------------------------------------------------------------- global RPB (R19)
# bias = table[h, dr + H - 1, dc + W - 1] with (dr, dc)
# the 2D cell offset cell(q) - cell(k) recovered through the ordering's cell map.

def test_rpb_hand_example():
    # 2x2 grid.  Hilbert path (gilbert2d): seq 0..3 -> cells (0,0) (1,0) (1,1) (0,1);
    # row-major: (0,0) (0,1) (1,0) (1,1).  Table T[i][j] = 3i + j, i = dr + 1, j = dc + 1.
    T = np.arange(9.0).reshape(3, 3)
    hil = np.array([[4, 1, 0, 3], [7, 4, 3, 6], [8, 5, 4, 7], [5, 2, 1, 4]], dtype=float)
    rm = np.array([[4, 3, 1, 0], [5, 4, 2, 1], [7, 6, 4, 3], [8, 7, 5, 4]], dtype=float)
    assert np.array_equal(attention.rpb_bias(Spec("HWA", 2, 2, 2, 2), T, np.arange(4)), hil)
    assert np.array_equal(attention.rpb_bias(Spec("WSA", 2, 2, 2, 2), T, np.arange(4)), rm)


def test_rpb_depends_on_cells_not_order():
    # the same (q, k) cell pair under row-major and Hilbert order -> same bias
    H, W = 8, 12
    T = _rand((2 * H - 1, 2 * W - 1), 50)
    s2c, c2s = hilbert.hilbert_order(H, W)
    bh = attention.rpb_bias(Spec("HWA", H, W, 2, 2), T, np.arange(H * W))
    brm = attention.rpb_bias(Spec("WSA", H, W, 2, 2), T, np.arange(H * W))
    assert np.array_equal(bh[np.ix_(c2s, c2s)], brm)


def test_rpb_zero_table_is_identity():
    spec = Spec("HSWA", 8, 8, 4, 4, shift=8)
    N, d = 64, 8
    Q, K, V, dO = (_rand((N, d), s) for s in (51, 52, 53, 54))
    Z = np.zeros((15, 15))
    O0, L0 = attention.attn_fwd_slice(Q, K, V, spec)
    O1, L1 = attention.attn_fwd_slice(Q, K, V, spec, rpb=Z)
    assert np.array_equal(O0, O1) and np.array_equal(L0, L1)
    g0 = attention.attn_bwd_slice(Q, K, V, dO, spec)
    g1 = attention.attn_bwd_slice(Q, K, V, dO, spec, rpb=Z)
    for a, b in zip(g0[:3], g1[:3]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("spec", [Spec("HWA", 8, 8, 4, 4), Spec("HSWA", 8, 8, 4, 4, shift=8),
                                  Spec("HNA", 8, 8, 3, 3), Spec("WSA", 8, 8, 4, 4)],
                         ids=lambda s: s.kind)
def test_rpb_matches_autograd_sdpa(spec):
    # library pin: SDPA fp64 with an additive float mask (bias where allowed, -inf
    # elsewhere); the table gradient comes from torch autograd through a gather
    H, W = spec.grid_h, spec.grid_w
    N, d = H * W, 8
    Q, K, V, dO = (_rand((N, d), s) for s in (60, 61, 62, 63))
    T = _rand((2 * H - 1, 2 * W - 1), 64)
    dQ, dK, dV, O, LSE, dT = attention.attn_bwd_slice(Q, K, V, dO, spec, chunk=9, rpb=T)
    r, c = attention.seq_cells(spec)
    ir = torch.from_numpy(r[:, None] - r[None, :] + H - 1)
    ic = torch.from_numpy(c[:, None] - c[None, :] + W - 1)
    tT = torch.from_numpy(T).requires_grad_(True)
    tq, tk, tv = (torch.from_numpy(a).requires_grad_(True) for a in (Q, K, V))
    M = torch.from_numpy(patterns.materialize(spec))
    bias = torch.where(M, tT[ir, ic], torch.tensor(-np.inf, dtype=torch.float64))
    out = torch.nn.functional.scaled_dot_product_attention(tq[None], tk[None], tv[None], attn_mask=bias[None],
                                                           scale=1 / np.sqrt(d))[0]
    out.backward(torch.from_numpy(dO))
    assert np.allclose(O, out.detach().numpy(), atol=1e-12)
    for mine, ref in ((dQ, tq.grad), (dK, tk.grad), (dV, tv.grad), (dT, tT.grad)):
        assert np.allclose(mine, ref.numpy(), rtol=0, atol=1e-11)
    # sum over the table gradient = sum of dS = 0 (rows of dS sum to zero)
    assert abs(dT.sum()) < 1e-11


def test_rpb_finite_differences():
    # S:L279 extended to the table: fp64 central differences, h = 1e-5, rel <= 1e-6
    spec = Spec("HSA", 4, 4, 3, 3)
    N, d, h = 16, 4, 1e-5
    Q, K, V, dO = (_rand((N, d), s) for s in (70, 71, 72, 73))
    T = _rand((7, 7), 74)
    dT = attention.attn_bwd_slice(Q, K, V, dO, spec, rpb=T)[5]

    def loss(T_):
        O, _ = attention.attn_fwd_slice(Q, K, V, spec, rpb=T_)
        return float((O * dO).sum())

    num = np.zeros_like(T)
    for i in range(7):
        for j in range(7):
            Tp, Tm = T.copy(), T.copy()
            Tp[i, j] += h
            Tm[i, j] -= h
            num[i, j] = (loss(Tp) - loss(Tm)) / (2 * h)
    rel = np.abs(num - dT).max() / np.abs(dT).max()
    assert rel <= 1e-6, rel
