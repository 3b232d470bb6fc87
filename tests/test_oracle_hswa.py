"""HSWA pinned against the construction the paper describes (CPU only).

P:L120: "HWT performs the window shift along the 1D sequence by moving each window forward
by a fixed offset ... window shift may introduce tokens at the beginning and end of the
sequence that are not adjacent in 2D space.  Even if they fall into the same window,
irrelevant attention connections must be masked out."  S:L139-140 realises it as Swin's
cyclic shift: roll the sequence by `shift`, cut windows of n tokens, and inside the one
wrapped window mask the head tokens (sequence start) apart from the tail tokens.

Built here step by step with a roll and segment ids -- a different construction from the
oracle's closed form floor((q - s) / n) == floor((k - s) / n) (oracle/patterns.py) and
from its interval form (oracle/blocks.py allowed_intervals), which it must equal.  Windows
divide the grid (enforced by both validators), so n | N; shift 0 degenerates to HWA.
"""

import numpy as np
import pytest

from oracle import blocks, patterns
from oracle.patterns import Spec


def roll_and_mask(N, n, s):
    """Boolean N x N mask of the cyclic-shift construction."""
    pos = np.arange(N)
    rolled = np.roll(pos, -s)               # rolled[r] = original token at rolled position r
    window_of = np.empty(N, dtype=np.int64)
    window_of[rolled] = np.arange(N) // n   # window of every original token
    head = pos < s                          # tokens that wrapped from the sequence start
    same_window = window_of[:, None] == window_of[None, :]
    same_segment = head[:, None] == head[None, :]
    return same_window & same_segment


CASES = [(4, 4, 2, 2, 2), (8, 8, 4, 4, 8), (8, 8, 2, 2, 1), (16, 16, 4, 4, 5), (8, 16, 4, 4, 15),
         (16, 8, 8, 4, 16), (12, 12, 3, 3, 4), (28, 28, 7, 7, 24), (16, 16, 4, 4, 0)]


@pytest.mark.parametrize("H,W,wh,ww,s", CASES)
def test_hswa_equals_roll_and_segment_mask(H, W, wh, ww, s):
    N, n = H * W, wh * ww
    ref = roll_and_mask(N, n, s)
    spec = Spec("HSWA", H, W, wh, ww, shift=s)
    assert (patterns.materialize(spec) == ref).all()
    # the interval form used by the interval classifier
    a, b = blocks.allowed_intervals(spec, np.arange(N))
    k = np.arange(N)
    via_int = np.zeros((N, N), dtype=bool)
    for j in range(a.shape[1]):
        via_int |= (k[None, :] >= a[:, j:j + 1]) & (k[None, :] < b[:, j:j + 1])
    assert (via_int == ref).all()
    if s == 0:   # no shift: the windows of HWA
        assert (ref == patterns.materialize(Spec("HWA", H, W, wh, ww))).all()
    else:
        patterns.validate(spec)


def test_hswa_wrapped_window_is_split():
    # the wrapped window holds the last n - s tail tokens and the s head tokens; they never mix
    N, n, s = 64, 16, 8
    m = roll_and_mask(N, n, s)
    tail = np.arange(N - (n - s), N)
    head = np.arange(s)
    assert not m[np.ix_(tail, head)].any() and m[np.ix_(tail, tail)].all() and m[np.ix_(head, head)].all()
    with pytest.raises(ValueError):
        patterns.validate(Spec("HSWA", 8, 8, 4, 4, shift=0))
    with pytest.raises(ValueError):
        patterns.validate(Spec("HSWA", 8, 8, 4, 4, shift=16))
