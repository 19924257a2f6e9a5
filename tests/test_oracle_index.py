"""Pins for the VS-IDX v1 index oracle (oracle/vsidx.py, oracle/_vsidx_ref.c).

Each test pins the oracle to something other than itself: the math library,
float64 textbook softmax, Python big-int / Fraction recomputation, SPEC worked
examples (tests/golden), planted inputs, and closed-form special cases.
"""
import json
import math
from fractions import Fraction
from pathlib import Path

import numpy as np
import pytest

from oracle import vsidx
from synth.generator import bf16_bits_to_f32, f32_to_bf16_bits, make_qkv

GOLD = json.loads((Path(__file__).parent / "golden" / "spec_examples.json").read_text())
F32 = np.float32


def test_constants_rederived():
    # C_d = RN(log2(e)/sqrt(d)) and c_k = RN(ln2^k/k!) from the math library.
    assert vsidx.c_d(128) == F32(math.log2(math.e) / math.sqrt(128))
    for kk, c in enumerate(vsidx.EXP2_COEF):
        assert c == F32(math.log(2) ** kk / math.factorial(kk))


def test_exp2s_close_to_libm():
    y = np.concatenate([np.linspace(-125, 0, 200001, dtype=np.float64),
                        -np.random.default_rng(0).random(100000) * 125]).astype(F32)
    e = vsidx.exp2s(y).astype(np.float64)
    ref = np.exp2(y.astype(np.float64))
    ulp = np.spacing(ref.astype(F32)).astype(np.float64)
    assert np.max(np.abs(e - ref) / ulp) <= 4.0
    assert vsidx.exp2s(np.array([0.0], F32))[0] == 1.0
    assert vsidx.exp2s(np.array([-125.5, -200.0], F32)).tolist() == [0.0, 0.0]


@pytest.mark.parametrize("case", GOLD["topp"])
def test_topp_golden(case):
    assert vsidx.topp_budget(np.array(case["scores"], np.uint64), case["p"]) == case["k"]


@pytest.mark.parametrize("case", GOLD["argtopk"])
def test_argtopk_golden(case):
    assert vsidx.argtopk(np.array(case["scores"], np.uint64), case["k"]).tolist() == case["idx"]


def test_topp_minimality_random():
    # Exact rational check: sum(top k-1) < p*T <= sum(top k), with p the float32 value.
    rng = np.random.default_rng(1)
    for _ in range(1000):
        n = int(rng.integers(1, 40))
        s = rng.integers(0, 1 << 20, n).astype(np.uint64)
        s[rng.integers(0, n)] += 1  # never all zero
        p = float(F32(rng.uniform(0.05, 1.0)))
        k = vsidx.topp_budget(s, p)
        top = sorted(s.tolist(), reverse=True)
        T = sum(top)
        target = Fraction(p) * T
        assert sum(top[:k]) >= target
        assert k == 1 or sum(top[:k - 1]) < target


def test_topp_monotone_in_p():
    rng = np.random.default_rng(2)
    s = rng.integers(0, 1000, 300).astype(np.uint64)
    ks = [vsidx.topp_budget(s, p) for p in np.linspace(0.05, 1.0, 40)]
    assert all(a <= b for a, b in zip(ks, ks[1:]))
    assert ks[-1] == s.size


def _window(S, seed=3, a=8.0):
    q, k, _ = make_qkv(S, 1, 1, seed=seed, a=a)
    qf, kf = bf16_bits_to_f32(q), bf16_bits_to_f32(k)
    return np.ascontiguousarray(qf[S - 64:, 0]), np.ascontiguousarray(kf[:, 0])


def test_window_scores_are_fp32_dot_products():
    qw, k = _window(256)
    t = vsidx.window_scores(qw, k)
    exact = qw.astype(np.float64) @ k.astype(np.float64).T
    bound = 128 * 2.0 ** -24 * (np.abs(qw).astype(np.float64) @ np.abs(k).astype(np.float64).T)
    n = 256 - 64 + np.arange(64)
    causal = np.arange(256)[None, :] <= n[:, None]
    assert np.all(np.abs(t[causal] - exact[causal]) <= bound[causal] + 1e-30)
    assert np.all(np.isneginf(t[~causal]))
    # small-integer inputs: every partial sum is exact -> t equals the exact dot product
    qi = np.random.default_rng(4).integers(-8, 8, (64, 128)).astype(F32)
    ki = np.random.default_rng(5).integers(-8, 8, (128, 128)).astype(F32)
    ti = vsidx.window_scores(qi, ki)
    ei = qi.astype(np.float64) @ ki.astype(np.float64).T
    c = np.arange(128)[None, :] <= (64 + np.arange(64))[:, None]
    assert np.array_equal(ti[c], ei[c])


def test_window_probabilities_match_float64_softmax():
    # I3-I5 approximate softmax(q k^T / sqrt(d)) to fixed-point precision.
    qw, k = _window(512)
    t = vsidx.window_scores(qw, k)
    _, E, w = vsidx.window_stats(t, 128)
    s = np.where(np.isfinite(t), t.astype(np.float64) / math.sqrt(128), -np.inf)
    ref = np.exp(s - s.max(axis=1, keepdims=True))
    ref /= ref.sum(axis=1, keepdims=True)
    got = w.astype(np.float64) / 2.0 ** 32
    assert np.max(np.abs(got - ref)) < 2e-6
    rows = w.sum(axis=1, dtype=np.uint64).astype(np.float64) / 2.0 ** 32
    assert np.all(np.abs(rows - 1.0) < 1e-5)


def test_fixed_point_bruteforce_python_ints():
    # I4-I6 recomputed with Python big ints and exact float decoding.
    qw, k = _window(192, seed=6)
    t = vsidx.window_scores(qw, k)
    M, E, w = vsidx.window_stats(t, 128)
    V, sigma = vsidx.column_and_slash_scores(w)
    cd = vsidx.c_d(128)
    for i in range(0, 64, 7):
        fin = np.isfinite(t[i])
        assert M[i] == t[i][fin].max()
        y = ((t[i][fin] - M[i]).astype(F32) * cd).astype(F32)
        e = vsidx.exp2s(y)
        Ei = sum(math.floor(Fraction(float(x)) * 2 ** 31) for x in e)
        assert Ei == int(E[i])
        l = F32(float(Ei)) * F32(2.0 ** -31)
        for m_idx, x in zip(np.nonzero(fin)[0][::17], e[::17]):
            p = F32(x) / l
            assert math.floor(Fraction(float(p)) * 2 ** 32) == int(w[i, m_idx])
    assert [int(x) for x in V] == [sum(int(w[i, m]) for i in range(64)) for m in range(192)]
    P = [sum(int(V[m]) for m in range(b * 64, b * 64 + 64)) for b in range(3)]
    assert [int(x) for x in sigma] == P[::-1]


def test_planted_vertical_and_forced_members():
    # All window mass on column 7: verticals contain 7, slashes contain 0.
    S, d = 512, 128
    qw = np.zeros((64, d), F32)
    qw[:, 0] = 16.0
    k = np.zeros((S, d), F32)
    k[7, 0] = 16.0
    iv, is_ = vsidx.vs_index_head(qw, k, 0.9, 0.9, use_c=False)
    assert 7 in iv and 0 in iv and 0 in is_
    assert iv.tolist() == [0, 7]
    # slash: block of column 7 is block 0 -> offset nb-1 carries the mass
    assert (S // 64 - 1) in is_


def test_full_budget_selects_everything():
    qw, k = _window(256, seed=7)
    iv, is_ = vsidx.vs_index_head(qw, k, 1.0, 1.0, use_c=False)
    assert iv.tolist() == list(range(256))
    assert is_.tolist() == list(range(4))


def _libm_fmaf():
    import ctypes
    import ctypes.util
    m = ctypes.CDLL(ctypes.util.find_library("m") or "libm.so.6")
    m.fmaf.restype = ctypes.c_float
    m.fmaf.argtypes = [ctypes.c_float] * 3
    return m.fmaf


def _extreme_bf16(shape, rng):
    """bf16 values spanning the whole exponent range: normals from 2^-126 to
    2^100, subnormal bf16s, signed zeros.  Products of two such values underflow
    below 2^-149 or land in fp32's subnormal range (the cases where a rounded
    product and a fused multiply-add differ)."""
    mant = rng.integers(0, 128, shape)
    sign = rng.integers(0, 2, shape)
    expo = rng.choice(np.r_[np.arange(1, 40), np.arange(100, 140), np.arange(200, 228)], shape)
    expo[rng.random(shape) < 0.05] = 0  # bf16 subnormals and zeros
    bits = (sign << 15) | (expo << 7) | mant
    return bf16_bits_to_f32(bits.astype(np.uint16))


def test_window_scores_fold_is_libm_fmaf():
    # I1 = sequential fold of IEEE fusedMultiplyAdd (the C library's fmaf), pinned
    # on ordinary and on extreme bf16 inputs (products below 2^-149, subnormal
    # partial sums, partial sums near 2^100) where a separately rounded product
    # would give other bits.
    fmaf = _libm_fmaf()
    rng = np.random.default_rng(21)
    d, S = 16, 96
    with np.errstate(over="ignore", invalid="ignore"):
        _fmaf_cases(fmaf, rng, d, S)


def _fmaf_cases(fmaf, rng, d, S):
    for qw, k in [(_extreme_bf16((64, d), rng), _extreme_bf16((S, d), rng)),
                  (rng.standard_normal((64, d)).astype(F32) * F32(2.0 ** -70),
                   rng.standard_normal((S, d)).astype(F32) * F32(2.0 ** -70))]:
        qw = bf16_bits_to_f32(f32_to_bf16_bits(qw))
        k = bf16_bits_to_f32(f32_to_bf16_bits(k))
        t = vsidx.window_scores(qw, k)
        n = S - 64 + np.arange(64)
        diff_from_rounded_product = 0
        for i in range(64):
            for m in range(0, int(n[i]) + 1):
                acc = 0.0
                rp = F32(0.0)
                for c in range(d):
                    acc = fmaf(float(qw[i, c]), float(k[m, c]), acc)
                    rp = F32(rp + F32(qw[i, c] * k[m, c]))
                assert np.array_equal(np.array([acc], F32).view(np.uint32),
                                      np.array([t[i, m]], F32).view(np.uint32)), (i, m)
                diff_from_rounded_product += int(F32(acc) != rp)
        # the extreme inputs really exercise the difference
        assert diff_from_rounded_product > 0


def test_c_fast_path_matches_numpy_bitwise():
    # S >= 4096 spans several 1024-key OpenMP chunks of the C helper; the last case
    # adds planted tiny values (products underflowing fp32) to the generator's keys.
    rng = np.random.default_rng(22)
    for S, seed, tiny in [(256, 8, False), (1024, 9, False), (4096, 10, False), (5120, 11, True)]:
        qw, k = _window(S, seed=seed, a=12.0)
        if tiny:
            sel = rng.random(k.shape) < 0.2
            k = np.where(sel, k * F32(2.0 ** -120), k).astype(F32)
            k = bf16_bits_to_f32(f32_to_bf16_bits(k))
            qw = np.where(rng.random(qw.shape) < 0.2, qw * F32(2.0 ** -40), qw).astype(F32)
            qw = bf16_bits_to_f32(f32_to_bf16_bits(qw))
        assert np.array_equal(vsidx.column_scores(qw, k, use_c=True),
                              vsidx.column_scores(qw, k, use_c=False))


def test_bf16_rounding_helper():
    x = np.array([1.0, 1.00390625, 1.0039062500001, -2.5, 3e-19, 1e-30], F32)
    b = f32_to_bf16_bits(x)
    assert bf16_bits_to_f32(b)[0] == 1.0
    assert bf16_bits_to_f32(b)[1] == 1.0          # tie -> even
    assert bf16_bits_to_f32(b)[3] == -2.5
    assert b[5] != 0 and abs(bf16_bits_to_f32(b)[5] / F32(1e-30) - 1) < 2 ** -8  # no flushing
