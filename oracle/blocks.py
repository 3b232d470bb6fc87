"""Block taxonomy, CSR lists and sparsity (TEST INFRASTRUCTURE ONLY).

Paper, Sec. 3.1: "Block-sparse attention ... tiles the N x N matrix into
fixed-size blocks, each with a shape of b_q x b_k.  If all elements within a
block participate in the computation, it is called a full block; if some
elements are masked, it is a partial block; and if all elements in the block are
masked, it is an empty block, which is skipped."

"The sparsity metric denotes the ratio of empty blocks".  Numerically
the paper's Sparsity column is FlexAttention's 1 - R*b_q*b_k/N^2 with the
unpadded N (reading R7; the only formula that reproduces the 56x56 rows
79.84/80.17/87.84).  Both that value and the plain
empty-tile ratio are reported.

Two independent classifiers, which tests require to agree:
  (i)  tile_counts_exhaustive - materialise the boolean mask a q-block at a time
       and count allowed pairs per tile;
  (ii) tile_counts_counter    - each query row's allowed key set is a union of
       intervals; count |interval intersect tile| in closed form.
Kinds: 0 = empty, 1 = full, 2 = partial.  A tile that contains padding rows or
columns (N % b != 0) can never be full ("no padding positions").
"""

import numpy as np

from . import patterns

EMPTY, FULL, PARTIAL = 0, 1, 2


def n_blocks(N, b):
    return (N + b - 1) // b


def tile_counts_exhaustive(spec, bq, bk):
    """int64 [Mq, Mk]: number of allowed (q, k) pairs inside each tile, by enumeration."""
    N = spec.n_tokens
    Mq, Mk = n_blocks(N, bq), n_blocks(N, bk)
    counts = np.zeros((Mq, Mk), dtype=np.int64)
    for i in range(Mq):
        rows = np.arange(i * bq, min((i + 1) * bq, N))
        m = patterns.mask_rows(spec, rows)                     # [nq, N] bool
        padded = np.zeros((len(rows), Mk * bk), dtype=bool)     # phantom columns never allowed
        padded[:, :N] = m
        counts[i] = padded.reshape(len(rows), Mk, bk).sum(axis=(0, 2))
    return counts


def allowed_intervals(spec, q):
    """Half-open key intervals [a, b) whose union is the allowed set of each query.

    Returns (a, b), int64 arrays of shape [len(q), n_int].  Empty intervals have a >= b.
    """
    q = np.asarray(q, dtype=np.int64)
    N, H, W = spec.n_tokens, spec.grid_h, spec.grid_w
    kind = spec.kind
    if kind == "DENSE":
        return np.zeros((len(q), 1), np.int64), np.full((len(q), 1), N, np.int64)
    if kind in patterns.HILBERT_KINDS:
        n = spec.win_h * spec.win_w
        r = n // 2
        if kind == "HWA":
            a = (q // n) * n
            b = np.minimum(a + n, N)
        elif kind == "HSA":
            a = np.maximum(q - r, 0)
            b = np.minimum(q + r + 1, N)
        elif kind == "HNA":
            L = 2 * r + 1
            a = np.clip(q - r, 0, N - L)
            b = a + L
        elif kind == "HSWA":
            s = spec.shift
            w = (q - s) // n
            a = np.maximum(w * n + s, 0)
            b = np.minimum(w * n + s + n, N)
        return a[:, None], b[:, None]
    kh, kw = spec.win_h, spec.win_w
    rq, cq = q // W, q % W
    if kind == "WSA":
        r0 = (rq // kh) * kh
        rows = r0[:, None] + np.arange(kh)[None, :]
        c0 = (cq // kw) * kw
        c1 = c0 + kw
    elif kind == "SA":
        rows = rq[:, None] + np.arange(-(kh // 2), kh // 2 + 1)[None, :]
        c0 = np.maximum(cq - kw // 2, 0)
        c1 = np.minimum(cq + kw // 2 + 1, W)
    elif kind == "NA2D":
        sr = np.clip(rq - kh // 2, 0, H - kh)
        rows = sr[:, None] + np.arange(kh)[None, :]
        c0 = np.clip(cq - kw // 2, 0, W - kw)
        c1 = c0 + kw
    else:
        raise ValueError(kind)
    valid = (rows >= 0) & (rows < H)
    a = rows * W + c0[:, None]
    b = rows * W + c1[:, None]
    b = np.where(valid, b, a)          # rows outside the grid contribute nothing
    return a, b


def tile_counts_counter(spec, bq, bk):
    """int64 [Mq, Mk]: allowed pairs per tile from interval arithmetic (no mask)."""
    N = spec.n_tokens
    Mq, Mk = n_blocks(N, bq), n_blocks(N, bk)
    lo = np.arange(Mk, dtype=np.int64) * bk
    hi = np.minimum(lo + bk, N)
    counts = np.zeros((Mq, Mk), dtype=np.int64)
    for i in range(Mq):
        q = np.arange(i * bq, min((i + 1) * bq, N))
        a, b = allowed_intervals(spec, q)                       # [nq, n_int]
        ov = np.minimum(b[..., None], hi) - np.maximum(a[..., None], lo)
        counts[i] = np.clip(ov, 0, None).sum(axis=(0, 1))
    return counts


def classify(counts, N, bq, bk):
    """uint8 [Mq, Mk] kinds from per-tile allowed-pair counts."""
    Mq, Mk = counts.shape
    real_rows = np.minimum(np.arange(Mq) * bq + bq, N) - np.arange(Mq) * bq
    real_cols = np.minimum(np.arange(Mk) * bk + bk, N) - np.arange(Mk) * bk
    no_pad = (real_rows[:, None] == bq) & (real_cols[None, :] == bk)
    kind = np.full(counts.shape, PARTIAL, dtype=np.uint8)
    kind[counts == 0] = EMPTY
    kind[(counts == bq * bk) & no_pad] = FULL
    return kind


def classify_spec(spec, bq, bk, method="counter"):
    counts = (tile_counts_counter if method == "counter" else tile_counts_exhaustive)(spec, bq, bk)
    return classify(counts, spec.n_tokens, bq, bk)


def csr(kind):
    """Per q-block ascending list of non-empty kv-blocks: (row_ptr, col_idx, kind_list)."""
    Mq, Mk = kind.shape
    row_ptr = np.zeros(Mq + 1, dtype=np.int32)
    cols, kinds = [], []
    for i in range(Mq):
        js = [j for j in range(Mk) if kind[i, j] != EMPTY]
        cols.extend(js)
        kinds.extend(int(kind[i, j]) for j in js)
        row_ptr[i + 1] = row_ptr[i] + len(js)
    return row_ptr, np.array(cols, dtype=np.int32), np.array(kinds, dtype=np.uint8)


def csr_transpose(kind):
    """Per kv-block ascending list of q-blocks (the backward pass walks these)."""
    return csr(np.ascontiguousarray(kind.T))


def stats(kind, N, bq, bk):
    """Integer counts first, then the two ratios as IEEE doubles."""
    n_full = int((kind == FULL).sum())
    n_partial = int((kind == PARTIAL).sum())
    n_total = int(kind.size)
    nnz = n_full + n_partial
    n_empty = n_total - nnz
    return {
        "nnz": nnz,
        "n_full": n_full,
        "n_partial": n_partial,
        "n_empty": n_empty,
        "empty_tile_ratio": n_empty / float(n_total),
        "sparsity": 1.0 - float(nnz * bq * bk) / (float(N) * float(N)),
    }
