"""Shared helpers of the GPU parity tests (test infrastructure)."""

import numpy as np

# north_star tolerances for attention outputs and gradients (bf16 in, fp32 accumulate)
MAX_ABS = 2e-2
MEAN_ABS = 2e-3
LSE_MAX_ABS = 1e-3     # proposed in SURVEY 8(c) O9 (LSE is fp32 end to end)


def to_np(t):
    return t.detach().float().cpu().numpy().astype(np.float64)


def assert_close(name, got, ref, max_abs=MAX_ABS, mean_abs=MEAN_ABS):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, (name, got.shape, ref.shape)
    assert np.isfinite(got).all(), "%s: non-finite values" % name
    err = np.abs(got - ref)
    assert err.max() <= max_abs and err.mean() <= mean_abs, \
        "%s: max-abs %.3g (tol %.1g), mean-abs %.3g (tol %.1g)" % (name, err.max(), max_abs, err.mean(), mean_abs)
    return float(err.max()), float(err.mean())


# --------------------------------------------------------------------------------------
# bf16 rounding model of the kernels (reading R16): fp64 attention with the
# values rounded to bf16 exactly where the CUDA path rounds them -- P before the PV and dV
# MMAs (the forward's P relative to its running, lazily rescaled max), dS before the dK /
# dQ MMAs, O / dQ / dK / dV on output (fp32 accumulation is modelled as exact).  It is a TOLERANCE MODEL for stress inputs, not the oracle: the
# parity claim stays "GPU vs the fp64 oracle"; this model says how far a correct bf16
# kernel can land from it.  Built from the oracle's mask and plain numpy only.

def bf16_round(x):
    """Round-to-nearest-even to bf16 (via fp32), returned as float64."""
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    bits = a.view(np.uint32).astype(np.uint64)
    r = (((bits + 0x7FFF + ((bits >> 16) & 1)) >> 16) << 16).astype(np.uint32)
    return r.view(np.float32).astype(np.float64)


def emulated_slice(Q, K, V, dO, spec, scale=None, block=128):
    """One (b, h) slice [N, d] -> (O, dQ, dK, dV) with the kernels' bf16 rounding points.

    Forward as the kernel runs it (attn_fwd.cu): kv tiles of `block` keys in ascending
    order, online softmax in the log2 domain with the lazy rescale (the reference max moves
    only when a tile's max exceeds it by more than 8, P = 2^(s - m_ref)), P rounded to bf16
    into the PV product, fp32 row sum of the unrounded P, O = bf16(O_acc / l)."""
    from oracle import patterns
    Q, K, V, dO = (np.asarray(t, dtype=np.float64) for t in (Q, K, V, dO))
    N, d = Q.shape
    sc = 1.0 / np.sqrt(d) if not scale else scale
    M = patterns.mask_rows(spec, np.arange(N))
    S = sc * (Q @ K.T)
    s2 = np.where(M, S * np.log2(np.e), -np.inf)
    m_ref = np.full(N, -np.inf)
    l = np.zeros(N)
    acc = np.zeros((N, V.shape[1]))
    for k0 in range(0, N, block):
        st = s2[:, k0:k0 + block]
        m_tile = st.max(axis=1)
        m_new = np.where(m_tile > m_ref + 8.0, m_tile, m_ref)
        with np.errstate(invalid="ignore"):   # -inf - -inf where a row has no key yet (alpha unused)
            alpha = np.where(m_new == m_ref, 1.0, np.exp2(m_ref - m_new))
        m_ref = m_new
        m_use = np.where(np.isinf(m_ref), 0.0, m_ref)
        p = np.exp2(st - m_use[:, None])
        l = l * alpha + p.sum(axis=1)
        acc = acc * alpha[:, None] + bf16_round(p) @ V[k0:k0 + block]
    O = bf16_round(acc / l[:, None])
    LSE = (m_ref + np.log2(l)) * np.log(2.0)
    Pb = np.where(M, np.exp(S - LSE[:, None]), 0.0)            # backward recompute (fp32 ~ exact)
    dV = bf16_round(bf16_round(Pb).T @ dO)
    D = (dO * O).sum(axis=1)                                     # uses the bf16 forward output
    dS = bf16_round(sc * Pb * (dO @ V.T - D[:, None]))           # bf16 dS into dK, dQ
    return O, bf16_round(dS @ K), bf16_round(dS.T @ Q), dV
