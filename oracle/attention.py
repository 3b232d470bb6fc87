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

Tensors use the product layout [B, N, heads, d] (any float dtype; upcast to
fp64).  Rows are processed `chunk` query rows at a time purely to bound memory;
every sum is over the full key range of the definition (the dK/dV sums over
queries are accumulated chunk by chunk in fp64).
"""

import numpy as np

from . import patterns


def _scale(d, scale):
    return 1.0 / np.sqrt(d) if (scale is None or scale <= 0) else float(scale)


def _softmax_rows(S, M):
    """(P, m, l) for score rows S with allowed mask M; disallowed entries excluded."""
    m = np.where(M, S, -np.inf).max(axis=1)
    P = np.zeros_like(S)
    P[M] = np.exp((S - m[:, None])[M])
    l = P.sum(axis=1)
    return P, m, l


def attn_fwd_slice(Q, K, V, spec, scale=None, rows=None, chunk=1024):
    """One (b, h) slice: Q, K, V are [N, d].  Returns (O[rows], LSE[rows]) in fp64."""
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
        M = patterns.mask_rows(spec, r)
        P, m, l = _softmax_rows(S, M)
        O[c0:c0 + len(r)] = (P @ V) / l[:, None]
        LSE[c0:c0 + len(r)] = m + np.log(l)
    return O, LSE


def attn_fwd(q, k, v, spec, scale=None, chunk=1024):
    """Full tensors [B, N, H, d] -> (O [B, N, H, d] fp64, LSE [B, H, N] fp64)."""
    B, N, H, d = q.shape
    O = np.empty((B, N, H, v.shape[3]), dtype=np.float64)
    LSE = np.empty((B, H, N), dtype=np.float64)
    for b in range(B):
        for h in range(H):
            O[b, :, h], LSE[b, h] = attn_fwd_slice(q[b, :, h], k[b, :, h], v[b, :, h],
                                                   spec, scale, chunk=chunk)
    return O, LSE


def attn_bwd_slice(Q, K, V, dO, spec, scale=None, chunk=1024):
    """One (b, h) slice.  Returns (dQ, dK, dV, O, LSE), all fp64; O is the oracle's own."""
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
    for c0 in range(0, N, chunk):
        r = np.arange(c0, min(c0 + chunk, N))
        S = sc * (Q[r] @ K.T)
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
    return dQ, dK, dV, O, LSE


def attn_bwd(q, k, v, dout, spec, scale=None, chunk=1024):
    """Full tensors [B, N, H, d] -> (dQ, dK, dV) [B, N, H, d] fp64."""
    B, N, H, d = q.shape
    dQ = np.empty((B, N, H, d))
    dK = np.empty((B, N, H, d))
    dV = np.empty((B, N, H, v.shape[3]))
    for b in range(B):
        for h in range(H):
            dQ[b, :, h], dK[b, :, h], dV[b, :, h], _, _ = attn_bwd_slice(
                q[b, :, h], k[b, :, h], v[b, :, h], dout[b, :, h], spec, scale, chunk=chunk)
    return dQ, dK, dV
