"""Pins for oracle.patterns and oracle.blocks (CPU only).

Pinned against:
  * every block-sparse "Sparsity" value the paper prints (tests/golden/paper_sparsity.csv,
    each row citing its PAPER.md line) -- 106 table cells;
  * the worked 4x4 example of Sec. 3.1 / Fig. 3;
  * SPEC's examples;
  * two independent classifiers (enumeration vs interval arithmetic) agreeing;
  * monotone blocking and pattern cardinalities.
"""

import csv
import os

import numpy as np
import pytest

from oracle import blocks, patterns
from oracle.patterns import Spec


def _golden_rows(golden_dir):
    with open(os.path.join(golden_dir, "paper_sparsity.csv")) as f:
        lines = [ln for ln in f if not ln.startswith("#")]
    return list(csv.reader(lines))


def test_paper_sparsity_values(golden_dir):
    rows = _golden_rows(golden_dir)
    assert len(rows) == 106
    for line, table, H, W, kind, wh, ww, b, pct in rows:
        spec = Spec(kind, int(H), int(W), int(wh), int(ww))
        kind_m = blocks.classify_spec(spec, int(b), int(b))
        st = blocks.stats(kind_m, spec.n_tokens, int(b), int(b))
        got = "%.2f" % (100.0 * st["sparsity"])
        assert got == pct, "P:L%s %s %s: got %s want %s" % (line, table, kind, got, pct)


def test_fig3_worked_example():
    # WSA "first eight tokens ... form four partial blocks, each of which is half full"
    wsa = Spec("WSA", 4, 4, 2, 2)
    c = blocks.tile_counts_exhaustive(wsa, 4, 4)
    k = blocks.classify(c, 16, 4, 4)
    assert (k[:2, :2] == blocks.PARTIAL).all() and (c[:2, :2] == 8).all()
    # HWA "forms two full blocks and two empty blocks" (0% -> 50% empty)
    hwa = Spec("HWA", 4, 4, 2, 2)
    k = blocks.classify_spec(hwa, 4, 4, method="exhaustive")
    assert k[0, 0] == k[1, 1] == blocks.FULL and k[0, 1] == k[1, 0] == blocks.EMPTY
    # slide "empty blocks ratio remains unchanged, partial ratio 100% -> 50%"
    sa = blocks.classify_spec(Spec("SA", 4, 4, 3, 3), 4, 4)[:2, :2]
    hsa = blocks.classify_spec(Spec("HSA", 4, 4, 3, 3), 4, 4)[:2, :2]
    assert (sa == blocks.EMPTY).sum() == (hsa == blocks.EMPTY).sum() == 0
    assert (sa == blocks.PARTIAL).mean() == 1.0 and (hsa == blocks.PARTIAL).mean() == 0.5


def test_spec_examples():
    # S:L115-119
    assert patterns.allowed(Spec("WSA", 4, 4, 2, 2), 0, 1) and not patterns.allowed(Spec("WSA", 4, 4, 2, 2), 0, 2)
    assert patterns.allowed(Spec("HWA", 4, 4, 2, 2), 0, 3) and not patterns.allowed(Spec("HWA", 4, 4, 2, 2), 0, 4)
    assert patterns.mask_rows(Spec("NA2D", 4, 4, 3, 3), [0]).sum() == 9
    assert patterns.mask_rows(Spec("SA", 4, 4, 3, 3), [0]).sum() == 4
    # S:L127-129
    assert patterns.materialize(Spec("WSA", 4, 4, 2, 2)).sum() == 64
    # WSA 4x4 w2 b4 -> 8 partial + 8 empty; HWA -> 4 full diagonal + 12 empty
    k = blocks.classify_spec(Spec("WSA", 4, 4, 2, 2), 4, 4)
    assert (k == blocks.PARTIAL).sum() == 8 and (k == blocks.EMPTY).sum() == 8
    k = blocks.classify_spec(Spec("HWA", 4, 4, 2, 2), 4, 4)
    assert (np.diag(k) == blocks.FULL).all() and (k == blocks.EMPTY).sum() == 12
    # HWA row i -> [i] full; WSA row 0 -> [0 partial, 1 partial]
    rp, ci, kd = blocks.csr(blocks.classify_spec(Spec("HWA", 4, 4, 2, 2), 4, 4))
    assert rp.tolist() == [0, 1, 2, 3, 4] and ci.tolist() == [0, 1, 2, 3] and (kd == 1).all()
    rp, ci, kd = blocks.csr(blocks.classify_spec(Spec("WSA", 4, 4, 2, 2), 4, 4))
    assert ci[rp[0]:rp[1]].tolist() == [0, 1] and kd[rp[0]:rp[1]].tolist() == [2, 2]


def test_hna_hsa_row_sums():
    # HNA N=16 radius 1 -> every row 3 keys; HSA -> 2 at the ends, 3 elsewhere
    hna = patterns.materialize(Spec("HNA", 4, 4, 1, 3))
    hsa = patterns.materialize(Spec("HSA", 4, 4, 1, 3))
    assert (hna.sum(1) == 3).all()
    assert hsa.sum(1).tolist() == [2] + [3] * 14 + [2]


SPECS_SMALL = [
    Spec("HWA", 16, 16, 8, 8), Spec("HSA", 16, 16, 5, 5), Spec("HNA", 16, 16, 7, 7),
    Spec("HSWA", 16, 16, 8, 8, shift=32), Spec("WSA", 16, 16, 4, 4), Spec("SA", 16, 16, 5, 5),
    Spec("NA2D", 16, 16, 7, 7), Spec("DENSE", 16, 16), Spec("SA", 16, 16, 16, 16),
    Spec("NA2D", 12, 20, 3, 5), Spec("WSA", 12, 20, 4, 5), Spec("HNA", 12, 20, 3, 3),
]


@pytest.mark.parametrize("spec", SPECS_SMALL, ids=lambda s: "%s%dx%d" % (s.kind, s.win_h, s.win_w))
@pytest.mark.parametrize("b", [1, 5, 16, 64, 128])
def test_counter_equals_enumeration(spec, b):
    assert np.array_equal(blocks.tile_counts_counter(spec, b, b), blocks.tile_counts_exhaustive(spec, b, b))


@pytest.mark.parametrize("spec", SPECS_SMALL, ids=lambda s: "%s%dx%d" % (s.kind, s.win_h, s.win_w))
def test_pattern_invariants(spec):
    M = patterns.materialize(spec)
    N = spec.n_tokens
    assert M[np.arange(N), np.arange(N)].all()                      # diagonal
    if spec.kind in ("WSA", "HWA", "SA", "HSA", "DENSE"):
        assert np.array_equal(M, M.T)                                # symmetry
    if spec.kind == "NA2D":
        assert (M.sum(1) == spec.win_h * spec.win_w).all()           # cardinality
    if spec.kind in ("WSA", "HWA"):
        assert (M.sum(1) == spec.win_h * spec.win_w).all()
    if spec.kind == "HNA":
        assert (M.sum(1) == 2 * ((spec.win_h * spec.win_w) // 2) + 1).all()


def test_monotone_blocking():
    # coarser tiles never have a larger empty ratio (tab:blocksize obeys it)
    for spec in SPECS_SMALL:
        prev = None
        for b in (4, 8, 16, 32, 64):
            st = blocks.stats(blocks.classify_spec(spec, b, b), spec.n_tokens, b, b)
            if prev is not None:
                assert st["empty_tile_ratio"] <= prev + 1e-15
            prev = st["empty_tile_ratio"]


def test_csr_transpose_roundtrip():
    spec = Spec("NA2D", 64, 64, 7, 7)
    kind = blocks.classify_spec(spec, 128, 128)
    rp, ci, kd = blocks.csr(kind)
    trp, tci, tkd = blocks.csr_transpose(kind)
    assert rp[-1] == trp[-1] == (kind != 0).sum()
    rebuilt = np.zeros_like(kind)
    for j in range(kind.shape[1]):
        for p in range(trp[j], trp[j + 1]):
            rebuilt[tci[p], j] = tkd[p]
    assert np.array_equal(rebuilt, kind)
    for i in range(kind.shape[0]):
        assert np.all(np.diff(ci[rp[i]:rp[i + 1]]) > 0)


def test_baseline_config_counts():
    # R per (b,h) for the BASELINE configs (these are our own
    # computations, cross-checked by the two classifiers above).
    def R(spec, b):
        st = blocks.stats(blocks.classify_spec(spec, b, b), spec.n_tokens, b, b)
        return st["nnz"], st["n_full"], st["n_partial"]
    assert R(Spec("HWA", 16, 16, 8, 8), 16) == (64, 64, 0)
    assert R(Spec("WSA", 16, 16, 8, 8), 16) == (128, 0, 128)
    assert R(Spec("HWA", 64, 64, 16, 16), 128) == (64, 64, 0)
    assert R(Spec("WSA", 64, 64, 16, 16), 128) == (256, 0, 256)
    assert R(Spec("HSA", 64, 64, 16, 16), 128) == (94, 32, 62)
    assert R(Spec("SA", 64, 64, 16, 16), 128) == (268, 0, 268)
