"""Grid orderings for the oracle (TEST INFRASTRUCTURE ONLY; see oracle/__init__.py).

Paper: "By reordering the token sequence according to the Hilbert curve, windows
or neighborhoods can be generated contiguously in the 1D sequence while
preserving 2D spatial locality.  With 2x2 window size, the first window takes
(1,2,3,4) tokens ..., and the second takes (5,6,7,8) tokens" (P:L90-91,
Sec. 3.1, Fig. 3).  "feature maps of the same size generate the same Hilbert
curve path, the path can be precomputed and cached".

The paper's figures are not available ([FIGURE]), so the curve
variant is a reading (reading R1): the generalized-Hilbert
("gilbert2d") recursion that SPEC recommends, starting at cell
(row 0, col 0).  On 2^k x 2^k grids this is the classic Hilbert curve; the GPU
path computes it with an unrelated bit-loop algorithm (d2xy/xy2d), so
agreement between the two is a real cross-check.

Coordinates: x = column, y = row; cell id t = row*W + col (row-major).
  seq_to_cell[s] = cell id of the s-th token of the sequence
  cell_to_seq[t] = position of cell t in the sequence
"""

import numpy as np


def _sgn(v):
    return (v > 0) - (v < 0)


def gilbert2d(width, height):
    """Return the list of (x, y) cells visited by the generalized Hilbert curve.

    Recursive rectangle splitting, written from the specification in SURVEY.md
    section 8(c) O2 (which restates the public gilbert2d construction): split
    the longer side in two (w > 1.5 h) or cut the rectangle into three parts
    (short side halved) so that consecutive cells stay 4-neighbours.
    """
    out = []

    def gen(x, y, ax, ay, bx, by):
        w = abs(ax + ay)
        h = abs(bx + by)
        dax, day = _sgn(ax), _sgn(ay)      # unit step along the major axis
        dbx, dby = _sgn(bx), _sgn(by)      # unit step along the minor axis
        if h == 1:                         # a single row: walk it
            for _ in range(w):
                out.append((x, y))
                x, y = x + dax, y + day
            return
        if w == 1:                         # a single column: walk it
            for _ in range(h):
                out.append((x, y))
                x, y = x + dbx, y + dby
            return
        ax2, ay2 = ax // 2, ay // 2
        bx2, by2 = bx // 2, by // 2
        w2 = abs(ax2 + ay2)
        h2 = abs(bx2 + by2)
        if 2 * w > 3 * h:
            # long rectangle: split along the major axis into two halves
            if (w2 % 2) and (w > 2):
                ax2, ay2 = ax2 + dax, ay2 + day
            gen(x, y, ax2, ay2, bx, by)
            gen(x + ax2, y + ay2, ax - ax2, ay - ay2, bx, by)
        else:
            # standard case: one step up, one long horizontal, one step down
            if (h2 % 2) and (h > 2):
                bx2, by2 = bx2 + dbx, by2 + dby
            gen(x, y, bx2, by2, ax2, ay2)
            gen(x + bx2, y + by2, ax, ay, bx - bx2, by - by2)
            gen(x + (ax - dax) + (bx2 - dbx), y + (ay - day) + (by2 - dby),
                -bx2, -by2, -(ax - ax2), -(ay - ay2))

    if width >= height:
        gen(0, 0, width, 0, 0, height)
    else:
        gen(0, 0, 0, height, width, 0)
    return out


def hilbert_order(grid_h, grid_w):
    """(seq_to_cell, cell_to_seq) int64 arrays for the Hilbert ordering."""
    cells = gilbert2d(grid_w, grid_h)
    n = grid_h * grid_w
    assert len(cells) == n
    seq_to_cell = np.array([y * grid_w + x for (x, y) in cells], dtype=np.int64)
    cell_to_seq = np.empty(n, dtype=np.int64)
    cell_to_seq[seq_to_cell] = np.arange(n, dtype=np.int64)
    return seq_to_cell, cell_to_seq


def hilbert_tiled_order(grid_h, grid_w, seg=64):
    """(seq_to_cell, cell_to_seq) of the implementation's tiled Hilbert order (include/hla.h
    HLA_ORDER_HILBERT_TILED; reading R23 -- NOT a curve of the paper): the Hilbert
    order with the cells of every aligned `seg`-token segment listed in row-major order
    (ascending cell id = (row, col) order).  Written from that definition: sort each segment."""
    s2c, _ = hilbert_order(grid_h, grid_w)
    n = grid_h * grid_w
    assert n % seg == 0
    seq_to_cell = np.sort(s2c.reshape(-1, seg), axis=1).reshape(-1)
    cell_to_seq = np.empty(n, dtype=np.int64)
    cell_to_seq[seq_to_cell] = np.arange(n, dtype=np.int64)
    return seq_to_cell, cell_to_seq


def row_major_order(grid_h, grid_w):
    """(seq_to_cell, cell_to_seq) of the conventional row-major order."""
    n = grid_h * grid_w
    ident = np.arange(n, dtype=np.int64)
    return ident, ident.copy()


def to_sequence(x, seq_to_cell):
    """Reorder token rows of x[B, N, ...] from grid order into sequence order.

    out[:, s] = x[:, seq_to_cell[s]]  ("reordered according to the Hilbert curve
    path").  Plain numpy fancy indexing.
    """
    return x[:, seq_to_cell]


def to_grid(x, seq_to_cell):
    """Inverse of to_sequence: out[:, seq_to_cell[s]] = x[:, s]."""
    out = np.empty_like(x)
    out[:, seq_to_cell] = x
    return out
