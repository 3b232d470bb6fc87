"""Dense masked attention, forward and backward, in fp64 (TEST INFRASTRUCTURE ONLY).

What the method computes: softmax attention restricted to the pattern's allowed
pairs.  Block sparsity changes the cost, never the result: "they do not affect
model accuracy but primarily differ in computational efficiency";
"the same attention pattern has identical outputs for the FlexAttention
block-sparse kernel and for the dense implementation".  So the oracle
is the plain definition, block-free (reading R12):

    S      = scale * Q K^T                       (scale = 1/sqrt(d), reading R11)
    m_q    = max_{k allowed} S[q, k]
    P[q,k] = exp(S[q,k] - m_q) if allowed(q,k) else 0     (excluded, not -inf-added)
    l_q    = sum_k P[q, k]
    O      = P V / l,    LSE_q = m_q + ln l_q     (natural log)

Backward (standard softmax-attention differentiation; the paper measures it,
P:L148 "Backward" columns, without restating it):
    Phat = P / l,  D_q = sum_d dO[q,d] O[q,d]
    dV = Phat^T dO,  dP = dO V^T,  dS = Phat o (dP - D),
    dQ = scale dS K,  dK = scale dS^T Q.

Optional score modification, global relative position bias (global RPB; P:L120
"HWT enlarges the window to the full feature map, enabling a global relative
position bias"; reading R19):
    S[q, k] += table[h, dr + H - 1, dc + W - 1],  (dr, dc) = cell(q) - cell(k)
with cell() the pattern's sequence -> grid-cell map (Hilbert path or row-major)
and table of shape (heads, 2H - 1, 2W - 1).  The bias enters the score after the
scale and before the mask; its gradient is the scatter-add of dS over the pairs
sharing an offset:  dtable[h, idx(q, k)] += dS[q, k].

Tensors use the product layout [B, N, heads, d] (any float dtype; upcast to
fp64).  Rows are processed `chunk` query rows at a time purely to bound memory;
every sum is over the full key range of the definition (the dK/dV sums over
queries are accumulated chunk by chunk in fp64).
"""

import numpy as np

from . import hilbert, patterns


def _scale(d, scale):
    return 1.0 / np.sqrt(d) if (scale is None or scale <= 0) else float(scale)


def _softmax_rows(S, M):
    """(P, m, l) for score rows S with allowed mask M; disallowed entries excluded."""
    m = np.where(M, S, -np.inf).max(axis=1)
    P = np.zeros_like(S)
    P[M] = np.exp((S - m[:, None])[M])
    l = P.sum(axis=1)
    return P, m, l


def seq_cells(spec):
    """Grid cell (row, col) of every sequence position of the pattern's ordering."""
    order = hilbert.hilbert_order if spec.order == "hilbert" else hilbert.row_major_order
    s2c, _ = order(spec.grid_h, spec.grid_w)
    return s2c // spec.grid_w, s2c % spec.grid_w


def rpb_index(spec, rows):
    """(row index, column index) into a (2H-1, 2W-1) RPB table for the pairs
    (q in rows, every k): the 2D offset cell(q) - cell(k) shifted by (H-1, W-1)."""
    r, c = seq_cells(spec)
    rows = np.asarray(rows, dtype=np.int64)
    return (r[rows][:, None] - r[None, :] + spec.grid_h - 1,
            c[rows][:, None] - c[None, :] + spec.grid_w - 1)


def rpb_bias(spec, table_h, rows):
    """Bias rows [len(rows), N] of one head: table_h[idx(q, k)] (global RPB)."""
    ir, ic = rpb_index(spec, rows)
    return np.asarray(table_h, dtype=np.float64)[ir, ic]


def attn_fwd_slice(Q, K, V, spec, scale=None, rows=None, chunk=1024, rpb=None):
    """One (b, h) slice: Q, K, V are [N, d]; rpb = this head's (2H-1, 2W-1) table or
    None.  Returns (O[rows], LSE[rows]) in fp64."""
    Q = np.asarray(Q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    N, d = Q.shape
    sc = _scale(d, scale)
    rows = np.arange(N) if rows is None else np.asarray(rows, dtype=np.int64)
    O = np.empty((len(rows), V.shape[1]), dtype=np.float64)
    LSE = np.empty(len(rows), dtype=np.float64)
    for c0 in range(0, len(rows), chunk):
        r = rows[c0:c0 + chunk]
        S = sc * (Q[r] @ K.T)
        if rpb is not None:
            S = S + rpb_bias(spec, rpb, r)
        M = patterns.mask_rows(spec, r)
        P, m, l = _softmax_rows(S, M)
        O[c0:c0 + len(r)] = (P @ V) / l[:, None]
        LSE[c0:c0 + len(r)] = m + np.log(l)
    return O, LSE


def attn_fwd(q, k, v, spec, scale=None, chunk=1024, rpb=None):
    """Full tensors [B, N, H, d] -> (O [B, N, H, d] fp64, LSE [B, H, N] fp64);
    rpb: optional (heads, 2H-1, 2W-1) global-RPB table."""
    B, N, H, d = q.shape
    O = np.empty((B, N, H, v.shape[3]), dtype=np.float64)
    LSE = np.empty((B, H, N), dtype=np.float64)
    for b in range(B):
        for h in range(H):
            O[b, :, h], LSE[b, h] = attn_fwd_slice(q[b, :, h], k[b, :, h], v[b, :, h],
                                                   spec, scale, chunk=chunk,
                                                   rpb=None if rpb is None else rpb[h])
    return O, LSE


def attn_bwd_slice(Q, K, V, dO, spec, scale=None, chunk=1024, rpb=None):
    """One (b, h) slice.  Returns (dQ, dK, dV, O, LSE), all fp64; O is the oracle's own.
    With rpb (this head's table) returns (dQ, dK, dV, O, LSE, dRPB)."""
    Q = np.asarray(Q, dtype=np.float64)
    K = np.asarray(K, dtype=np.float64)
    V = np.asarray(V, dtype=np.float64)
    dO = np.asarray(dO, dtype=np.float64)
    N, d = Q.shape
    sc = _scale(d, scale)
    dQ = np.zeros_like(Q)
    dK = np.zeros_like(K)
    dV = np.zeros_like(V)
    O = np.empty_like(dO)
    LSE = np.empty(N)
    dT = None if rpb is None else np.zeros(np.shape(rpb), dtype=np.float64)
    for c0 in range(0, N, chunk):
        r = np.arange(c0, min(c0 + chunk, N))
        S = sc * (Q[r] @ K.T)
        if rpb is not None:
            S = S + rpb_bias(spec, rpb, r)
        M = patterns.mask_rows(spec, r)
        P, m, l = _softmax_rows(S, M)
        Phat = P / l[:, None]
        O[r] = Phat @ V
        LSE[r] = m + np.log(l)
        D = (dO[r] * O[r]).sum(axis=1)
        dV += Phat.T @ dO[r]
        dP = dO[r] @ V.T
        dS = Phat * (dP - D[:, None])
        dQ[r] = sc * (dS @ K)
        dK += sc * (dS.T @ Q[r])
        if dT is not None:
            ir, ic = rpb_index(spec, r)
            np.add.at(dT, (ir, ic), dS)        # scatter-add over pairs sharing an offset
    if dT is not None:
        return dQ, dK, dV, O, LSE, dT
    return dQ, dK, dV, O, LSE


def attn_bwd(q, k, v, dout, spec, scale=None, chunk=1024, rpb=None):
    """Full tensors [B, N, H, d] -> (dQ, dK, dV) [B, N, H, d] fp64; with an rpb table
    (heads, 2H-1, 2W-1) -> (dQ, dK, dV, dRPB), dRPB summed over the batch."""
    B, N, H, d = q.shape
    dQ = np.empty((B, N, H, d))
    dK = np.empty((B, N, H, d))
    dV = np.empty((B, N, H, v.shape[3]))
    dT = None if rpb is None else np.zeros(np.shape(rpb), dtype=np.float64)
    for b in range(B):
        for h in range(H):
            res = attn_bwd_slice(q[b, :, h], k[b, :, h], v[b, :, h], dout[b, :, h], spec, scale,
                                 chunk=chunk, rpb=None if rpb is None else rpb[h])
            dQ[b, :, h], dK[b, :, h], dV[b, :, h] = res[0], res[1], res[2]
            if dT is not None:
                dT[h] += res[5]
    if dT is not None:
        return dQ, dK, dV, dT
    return dQ, dK, dV
