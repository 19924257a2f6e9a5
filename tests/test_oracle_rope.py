"""Pins of oracle/rope.py against what the paper and the mathematics fix (not a
retyping of its formulas): RoPE is a rotation (norm-preserving, identity at n = 0,
inverse = transpose), and q.k after RoPE depends only on n - m (PAPER.md P:123-127,
Theorem 3.1's premise; P:611-619 expand exactly this dot product); YaRN keeps the
highest frequencies, divides the lowest by the factor, and scales by 0.1 ln s + 1."""
import numpy as np
import pytest

from oracle import rope as R


def _rand(T, H=3, d=128, seed=0):
    return np.random.default_rng(seed).standard_normal((T, H, d))


def test_identity_at_position_zero_and_norm_preserved():
    th, _ = R.inv_freq()
    x = _rand(5)
    y = R.rope(x, np.zeros(5), th)
    assert np.allclose(y, x, atol=0)
    z = R.rope(x, np.arange(5) * 1234.5, th)
    assert np.allclose(np.linalg.norm(z, axis=-1), np.linalg.norm(x, axis=-1), rtol=1e-13)


def test_inverse_is_transpose():
    th, _ = R.inv_freq()
    x = _rand(7, seed=1)
    pos = np.arange(7) * 77777
    assert np.allclose(R.rope(R.rope(x, pos, th), pos, th, inverse=True), x, atol=1e-12)


def test_dot_product_depends_only_on_relative_position():
    th, _ = R.inv_freq()
    q, k = _rand(1, 1, seed=2)[0, 0], _rand(1, 1, seed=3)[0, 0]
    def z(n, m):
        return float(R.rope(q[None, None], np.array([n]), th)[0, 0]
                     @ R.rope(k[None, None], np.array([m]), th)[0, 0])
    for n, m in [(10, 3), (500000, 499993), (7, 0)]:
        assert z(n, m) == pytest.approx(z(n - m, 0), rel=1e-9, abs=1e-9)


def test_half_split_pairing_matches_paper_expansion():
    """z = q_lo cos k_lo + q_hi cos k_hi + q_lo sin k_hi - q_hi sin k_lo
    with (n - m) theta per pair index (i mod d/2)."""
    th, _ = R.inv_freq(d=8, base=100.0)
    q, k = _rand(1, 1, d=8, seed=4)[0, 0], _rand(1, 1, d=8, seed=5)[0, 0]
    n, m = 9, 4
    zq = R.rope(q[None, None], np.array([n]), th)[0, 0]
    zk = R.rope(k[None, None], np.array([m]), th)[0, 0]
    c, s = np.cos((n - m) * th), np.sin((n - m) * th)
    exp = (q[:4] * c) @ k[:4] + (q[4:] * c) @ k[4:] + (q[:4] * s) @ k[4:] - (q[4:] * s) @ k[:4]
    assert float(zq @ zk) == pytest.approx(float(exp), rel=1e-12)


def test_yarn_reduces_and_interpolates():
    th, ms = R.inv_freq(yarn_factor=1.0)
    assert ms == 1.0
    ty, my = R.inv_freq(yarn_factor=32.0, original_max_position=32768)
    assert my == pytest.approx(0.1 * np.log(32.0) + 1.0)
    assert ty[0] == th[0]                           # fastest rotation: extrapolated
    assert ty[-1] == pytest.approx(th[-1] / 32.0)   # slowest: interpolated by s
    assert np.all(ty <= th) and np.all(ty >= th / 32.0 - 1e-30)
    assert np.all(np.diff(ty / th) <= 1e-15)        # monotone ramp from 1 down to 1/s
