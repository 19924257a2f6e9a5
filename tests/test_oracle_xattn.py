"""Pins of oracle/xattn.py (reading R25) against facts fixed independently of
its formulas: the strided antidiagonal score equals the antidiagonal sum read off
the full Q K^T matrix (brute force); softmax rows make each block-score row sum to
B/st; threshold 1 keeps every causal block, threshold 0 only the diagonal; a
planted dominant block is selected first; the 64-token expansion covers exactly the
causal part of the 128-blocks kept."""
import numpy as np
import pytest

from oracle import xattn as X
from oracle.sparseformat import key_set

S, d = 1024, 128


def _qk(seed=0):
    r = np.random.default_rng(seed)
    return r.standard_normal((S, d)), r.standard_normal((S, d))


def test_antidiagonal_scores_match_full_matrix():
    q, k = _qk()
    A = X.antidiag_scores(q, k)
    full = q @ k.T / np.sqrt(d)
    for i, j in [(0, 0), (5, 3), (63, 0), (40, 40), (17, 60)]:
        ref = sum(full[i * 16 + 15 - s, j * 16 + s] for s in range(16)) / 16
        assert A[i, j] == pytest.approx(ref, rel=1e-12, abs=1e-12)


def test_block_score_rows_sum_to_block_over_stride():
    q, k = _qk(1)
    Bs = X.block_scores(q, k)
    assert np.allclose(Bs.sum(axis=1), 128 / 16, rtol=1e-12)
    assert np.all(np.triu(Bs, 1) == 0)


def test_threshold_extremes():
    q, k = _qk(2)
    Bs = X.block_scores(q, k)
    all_ = X.select_blocks(Bs, 1.0)
    assert all(np.array_equal(r, np.arange(I + 1)) for I, r in enumerate(all_))
    diag = X.select_blocks(Bs, 0.0)
    assert all(np.array_equal(r, [I]) for I, r in enumerate(diag))


def test_planted_block_selected():
    """k rows of key block 2 aligned with every query (large dot products): every
    later query block keeps block 2, and at a low threshold keeps little else."""
    q, k = _qk(3)
    u = np.zeros(d); u[0] = 1.0
    q = 0.1 * q + 6.0 * u
    k = 0.1 * k
    k[256:384] += 6.0 * u
    Bs = X.block_scores(q, k)
    sel = X.select_blocks(Bs, 0.5)
    for I in range(3, S // 128):
        assert 2 in sel[I] and len(sel[I]) <= 2, sel[I]


def test_block64_expansion_is_causal_cover():
    q, k = _qk(4)
    sel = X.select_blocks(X.block_scores(q, k), 0.9)
    rows = X.to_block64(sel)
    for g, r in enumerate(rows):
        assert np.all(np.diff(r) > 0) and r.max() <= g
        I = g // 2
        # every token of a kept 128-block at or before each query is a key
        for n in (g * 64, g * 64 + 63):
            ks = set(key_set(n, r, np.zeros(0, np.int64)).tolist())
            want = {m for J in sel[I] for m in range(J * 128, J * 128 + 128) if m <= n}
            assert ks == want


def test_sampled_rows_equal_full_computation():
    q, k = _qk(5)
    Bs = X.block_scores(q, k)
    rows = X.block_score_rows(q, k, [0, 3, 7])
    for I, r in rows.items():
        assert np.allclose(r, Bs[I, : I + 1], rtol=1e-12, atol=1e-14)
