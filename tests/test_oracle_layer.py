"""Pins of oracle/layer.py: its hand-derived backward against central finite
differences of its forward (index held fixed) on a tiny layer — a check the
chain rule cannot pass by construction (a dropped term, a wrong sign or a transposed
operand in any step moves a directional derivative); plus the residual structure:
with zero output projections the layer is the identity."""
import numpy as np
import pytest

from oracle import layer as L
from oracle import rope as R

S, D, HQ, HKV, d, I = 128, 24, 2, 1, 8, 40


def _setup(seed=0):
    rng = np.random.default_rng(seed)
    P = dict(w1=1 + 0.1 * rng.standard_normal(D), w2=1 + 0.1 * rng.standard_normal(D),
             Wqkv=0.3 * rng.standard_normal(((HQ + 2 * HKV) * d, D)),
             bqkv=0.1 * rng.standard_normal((HQ + 2 * HKV) * d),
             Wo=0.3 * rng.standard_normal((D, HQ * d)), Wg=0.3 * rng.standard_normal((I, D)),
             Wu=0.3 * rng.standard_normal((I, D)), Wd=0.3 * rng.standard_normal((D, I)))
    x = rng.standard_normal((S, D))
    i_v = [np.array([0, 5, 70, 100], dtype=np.int32), np.array([0, 3], dtype=np.int32)]
    i_s = [np.array([0], dtype=np.int32), np.array([0, 1], dtype=np.int32)]
    th, ms = R.inv_freq(d, base=100.0, yarn_factor=4.0, original_max_position=32)
    return rng, P, x, np.arange(S) * 7 + 3, th, ms, i_v, i_s


def test_backward_matches_finite_differences():
    rng, P, x, pos, th, ms, i_v, i_s = _setup()
    args = (pos, th, ms, i_v, i_s, HQ, HKV, d)
    dy = rng.standard_normal((S, D))
    y, c = L.forward(x, P, *args)
    dx, G = L.backward(dy, P, c, *args)
    f = lambda xx, PP: float(np.sum(L.forward(xx, PP, *args)[0] * dy))
    eps = 1e-5
    dirx = rng.standard_normal(x.shape)
    fd = (f(x + eps * dirx, P) - f(x - eps * dirx, P)) / (2 * eps)
    assert np.sum(dx * dirx) == pytest.approx(fd, rel=1e-6)
    for name in P:
        dirp = rng.standard_normal(P[name].shape)
        Pp = dict(P); Pp[name] = P[name] + eps * dirp
        Pm = dict(P); Pm[name] = P[name] - eps * dirp
        fd = (f(x, Pp) - f(x, Pm)) / (2 * eps)
        assert np.sum(G[name] * dirp) == pytest.approx(fd, rel=1e-6), name


def test_zero_output_projections_give_identity():
    _, P, x, pos, th, ms, i_v, i_s = _setup(1)
    P = dict(P, Wo=np.zeros_like(P["Wo"]), Wd=np.zeros_like(P["Wd"]))
    y, _ = L.forward(x, P, pos, th, ms, i_v, i_s, HQ, HKV, d)
    assert np.array_equal(y, x)
