"""Pins for oracle.hilbert (CPU only).

What fixes the Hilbert ordering independently of the oracle's own code:
  * P:L91 (Fig. 3 text): on a 4x4 grid with a 2x2 window, tokens 1-4 (0-indexed
    0-3) form the first 2x2 window and tokens 5-8 the second;
  * mathematics of the curve: a bijection whose consecutive cells are
    4-neighbours, and (2^k grids) every aligned run of 4^j tokens is an aligned
    2^j x 2^j square (the locality property the method relies on);
  * a second, unrelated algorithm: the bit-twiddling d2xy/xy2d construction,
    written out below in this test, must give the same curve on 2^k grids.
"""

import numpy as np
import pytest

from oracle import hilbert


def _d2xy(n, d):
    # classic iterative Hilbert d -> (x, y) (bit loop), independent of gilbert2d
    t = d
    x = y = 0
    s = 1
    while s < n:
        rx = 1 & (t // 2)
        ry = 1 & (t ^ rx)
        if ry == 0:
            if rx == 1:
                x = s - 1 - x
                y = s - 1 - y
            x, y = y, x
        x += s * rx
        y += s * ry
        t //= 4
        s *= 2
    return x, y


@pytest.mark.parametrize("H,W", [(1, 1), (2, 2), (4, 4), (3, 3), (5, 7), (56, 56), (16, 32), (96, 96), (7, 2)])
def test_bijection_and_adjacency(H, W):
    s2c, c2s = hilbert.hilbert_order(H, W)
    N = H * W
    assert sorted(s2c.tolist()) == list(range(N))
    assert np.array_equal(c2s[s2c], np.arange(N))
    r, c = s2c // W, s2c % W
    cheb = np.maximum(np.abs(np.diff(r)), np.abs(np.diff(c)))
    manh = np.abs(np.diff(r)) + np.abs(np.diff(c))
    assert (cheb == 1).all()
    if H % 2 == 0 or W % 2 == 0:
        assert (manh == 1).all()
    else:
        assert (manh == 2).sum() <= 1      # one diagonal step at most


@pytest.mark.parametrize("k", range(0, 8))
def test_matches_bitloop_d2xy(k):
    n = 1 << k
    s2c, _ = hilbert.hilbert_order(n, n)
    expect = []
    for d in range(n * n):
        x, y = _d2xy(n, d)
        expect.append(y * n + x)
    assert s2c.tolist() == expect


@pytest.mark.parametrize("k", range(1, 8))
def test_quadrant_property(k):
    n = 1 << k
    s2c, _ = hilbert.hilbert_order(n, n)
    rows, cols = s2c // n, s2c % n
    for j in range(1, k + 1):
        side = 1 << j
        run = side * side
        for s0 in range(0, n * n, run):
            rr, cc = rows[s0:s0 + run], cols[s0:s0 + run]
            assert rr.max() - rr.min() == side - 1 and cc.max() - cc.min() == side - 1
            assert rr.min() % side == 0 and cc.min() % side == 0


def test_paper_fig3_statements():
    # "With 2x2 window size, the first window takes (1,2,3,4) tokens ...,
    # and the second takes (5,6,7,8) tokens" -- each a 2x2 square of the 4x4 map,
    # while row-major windows are (1,2,5,6) and (3,4,7,8).
    s2c, _ = hilbert.hilbert_order(4, 4)
    first = {(t // 4, t % 4) for t in s2c[0:4]}
    second = {(t // 4, t % 4) for t in s2c[4:8]}
    for win in (first, second):
        rs = {r for r, _ in win}
        cs = {c for _, c in win}
        assert len(rs) == 2 and len(cs) == 2 and min(rs) % 2 == 0 and min(cs) % 2 == 0
    assert first != second
    # the curve starts at (0,0) (reading R1)
    assert s2c[0] == 0


def test_to_sequence_roundtrip():
    rng = np.random.default_rng(0)
    x = rng.standard_normal((2, 64, 3, 4))
    s2c, _ = hilbert.hilbert_order(8, 8)
    y = hilbert.to_sequence(x, s2c)
    assert np.array_equal(y[:, 5], x[:, s2c[5]])
    assert np.array_equal(hilbert.to_grid(y, s2c), x)


# ---------------------------------------------------------------- tiled order (R23)
@pytest.mark.parametrize("k", [3, 4, 5, 6, 7])
def test_tiled_order_segments_are_squares(k):
    """The tiled order relabels inside aligned 64-token segments; it is well formed because
    every such segment of the curve is an aligned 8 x 8 square (the quadrant property at
    j = 3), so each aligned 8 positions of the tiled order are 8 consecutive cells of one row."""
    n = 2 ** k
    s2c, c2s = hilbert.hilbert_tiled_order(n, n)
    h2c, _ = hilbert.hilbert_order(n, n)
    assert sorted(s2c.tolist()) == list(range(n * n))
    assert np.array_equal(c2s[s2c], np.arange(n * n))
    for s0 in range(0, n * n, 64):
        rows, cols = s2c[s0:s0 + 64] // n, s2c[s0:s0 + 64] % n
        # the same cells as the Hilbert segment (a relabeling inside the segment only)
        assert set(s2c[s0:s0 + 64].tolist()) == set(h2c[s0:s0 + 64].tolist())
        assert rows.min() % 8 == 0 and cols.min() % 8 == 0
        assert np.array_equal(rows, rows.min() + np.repeat(np.arange(8), 8))
        assert np.array_equal(cols, cols.min() + np.tile(np.arange(8), 8))


@pytest.mark.parametrize("k,win", [(3, 8), (5, 8), (6, 16), (7, 8), (7, 32)])
def test_tiled_order_keeps_hwa_windows(k, win):
    """HWA with n = win^2 tokens (a multiple of 64): window(s) = s // n holds the same set of
    cells under both orders, so the attention of every cell is unchanged (reading R23)."""
    n = 2 ** k
    t2c, _ = hilbert.hilbert_tiled_order(n, n)
    h2c, _ = hilbert.hilbert_order(n, n)
    nt = win * win
    for w0 in range(0, n * n, nt):
        assert set(t2c[w0:w0 + nt].tolist()) == set(h2c[w0:w0 + nt].tolist())
