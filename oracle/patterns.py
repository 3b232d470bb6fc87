"""allowed(q, k) predicates of the local-attention patterns (TEST INFRASTRUCTURE ONLY).

q and k are 0-indexed positions in the sequence the tensors are stored in:
  * Hilbert patterns (HWA, HSA, HNA, HSWA) act on the Hilbert-ordered sequence
    ("windows and neighborhoods are then formed on the reordered 1D sequence",
    P:L7);
  * row-major patterns (WSA, SA, NA2D) act on row-major grid order, with cell
    t = (row, col) = (t // W, t % W);
  * DENSE allows every pair (FlashAttention baseline).

Window/kernel sizes are given in cells (win_h, win_w).  Hilbert patterns use
n = win_h * win_w tokens (reading R3: "2x2 window -> tokens 1,2,3,4") and
radius r = n // 2 (reading R4: token-count parity with the 2D kernel, S:L138;
reproduces every HSA/HNA sparsity value in the paper's tables).

Each predicate below is the plain definition, vectorised with numpy broadcasting.
"""

from dataclasses import dataclass

import numpy as np

HILBERT_KINDS = ("HWA", "HSA", "HNA", "HSWA")
ROWMAJOR_KINDS = ("WSA", "SA", "NA2D")
ALL_KINDS = HILBERT_KINDS + ROWMAJOR_KINDS + ("DENSE",)


@dataclass(frozen=True)
class Spec:
    kind: str          # one of ALL_KINDS
    grid_h: int
    grid_w: int
    win_h: int = 1     # window (WSA/HWA/HSWA) or kernel (SA/NA2D/HSA/HNA) height in cells
    win_w: int = 1
    shift: int = 0     # HSWA 1D shift in tokens ("a fixed offset"; reading R10)

    @property
    def n_tokens(self):
        return self.grid_h * self.grid_w

    @property
    def order(self):
        return "hilbert" if self.kind in HILBERT_KINDS else "row_major"


def allowed(spec, q, k):
    """Boolean array allowed(q, k) for broadcastable integer arrays q, k."""
    q = np.asarray(q, dtype=np.int64)
    k = np.asarray(k, dtype=np.int64)
    N = spec.n_tokens
    H, W = spec.grid_h, spec.grid_w
    kind = spec.kind

    if kind == "DENSE":
        return np.ones(np.broadcast(q, k).shape, dtype=bool)

    if kind in HILBERT_KINDS:
        n = spec.win_h * spec.win_w
        r = n // 2
        if kind == "HWA":
            # same window of n consecutive Hilbert tokens
            return (q // n) == (k // n)
        if kind == "HSA":
            # 1D slide band |q - k| <= r; sequence ends simply see fewer keys
            return np.abs(q - k) <= r
        if kind == "HNA":
            # 1D neighborhood of L = 2r+1 keys whose start is clamped into [0, N-L]
            # (NATTEN na1d semantics; "repeats the same window")
            L = 2 * r + 1
            s = np.clip(q - r, 0, N - L)
            return (k >= s) & (k < s + L)
        if kind == "HSWA":
            # windows moved forward along the 1D sequence by `shift`; tokens of the
            # head and tail that fall into one wrapped window are masked apart
            # (P:L120).  Floor division on (t - shift) realises exactly that.
            s = spec.shift
            return ((q - s) // n) == ((k - s) // n)

    rq, cq = q // W, q % W
    rk, ck = k // W, k % W
    kh, kw = spec.win_h, spec.win_w
    if kind == "WSA":
        # same regular kh x kw square window in row-major order
        return ((rq // kh) == (rk // kh)) & ((cq // kw) == (ck // kw))
    if kind == "SA":
        # 2D sliding window, zero-padding at the border
        return (np.abs(rq - rk) <= kh // 2) & (np.abs(cq - ck) <= kw // 2)
    if kind == "NA2D":
        # 2D neighborhood whose window is clamped into the grid
        sr = np.clip(rq - kh // 2, 0, H - kh)
        sc = np.clip(cq - kw // 2, 0, W - kw)
        return (rk >= sr) & (rk < sr + kh) & (ck >= sc) & (ck < sc + kw)
    raise ValueError("unknown pattern kind %r" % (kind,))


def validate(spec):
    """Argument checks of SPEC S:L98-100 (window divides grid, kernel fits)."""
    N = spec.n_tokens
    if spec.kind in ("WSA", "HWA", "HSWA"):
        if spec.grid_h % spec.win_h or spec.grid_w % spec.win_w:
            raise ValueError("window does not divide the grid")
    if spec.kind == "HSWA" and not 0 < spec.shift < spec.win_h * spec.win_w:
        raise ValueError("HSWA shift must lie in (0, n) (S:L139-140)")
    if spec.kind in ("SA", "NA2D"):
        if spec.win_h > spec.grid_h or spec.win_w > spec.grid_w:
            raise ValueError("kernel larger than grid")
    if spec.kind in ("HSA", "HNA"):
        n = spec.win_h * spec.win_w
        if n > N:
            raise ValueError("neighborhood longer than the sequence")
    return True


def mask_rows(spec, rows):
    """Materialised mask rows: bool [len(rows), N]."""
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.arange(spec.n_tokens, dtype=np.int64)
    return allowed(spec, rows[:, None], cols[None, :])


def materialize(spec):
    """Full N x N boolean mask (small N only)."""
    return mask_rows(spec, np.arange(spec.n_tokens))
