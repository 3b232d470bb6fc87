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
