"""Pins for the fp64 attention oracle (oracle/attention.py, oracle/sparseformat.py)."""
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import attention as A
from oracle import sparseformat as SF

GOLD = json.loads((Path(__file__).parent / "golden" / "spec_examples.json").read_text())


def _rand(S, Hq, Hkv, d, seed):
    r = np.random.default_rng(seed)
    return (r.standard_normal((S, Hq, d)), r.standard_normal((S, Hkv, d)),
            r.standard_normal((S, Hkv, d)))


def _rand_index(S, Hq, seed, n_off=3, n_col=10):
    r = np.random.default_rng(seed)
    nb = S // 64
    iv = [np.unique(np.r_[0, r.choice(S, n_col, replace=False)]) for _ in range(Hq)]
    is_ = [np.unique(np.r_[0, r.choice(nb, min(n_off, nb), replace=False)]) for _ in range(Hq)]
    return iv, is_


@pytest.mark.parametrize("case", GOLD["dense_forward"])
def test_dense_golden(case):
    O, L = A.dense_attention_forward(np.array(case["q"], float), np.array(case["k"], float),
                                     np.array(case["v"], float))
    assert np.allclose(O, case["O"]) and np.allclose(L, case["LSE"])


def test_dense_uniform_rows_average_values():
    # uniform scores, full mask -> every row is the mean of V.
    v = np.eye(4)
    O, L = A.dense_attention_forward(np.zeros((4, 4)), np.zeros((4, 4)), v, mask=np.ones((4, 4), bool))
    assert np.allclose(O, 0.25) and np.allclose(L, np.log(4))


def test_dense_matches_rowwise_textbook():
    q, k, v = (np.random.default_rng(0).standard_normal((64, 16)) for _ in range(3))
    O, L = A.dense_attention_forward(q, k, v)
    for n in range(64):
        s = np.array([q[n] @ k[m] / 4.0 for m in range(n + 1)])
        p = np.exp(s) / np.exp(s).sum()
        assert np.allclose(O[n], p @ v[: n + 1], atol=1e-12)
        assert abs(L[n] - np.log(np.exp(s).sum())) < 1e-12


def test_full_budget_sparse_equals_dense_causal():
    S, Hq, Hkv, d = 256, 2, 1, 32
    q, k, v = _rand(S, Hq, Hkv, d, 1)
    iv = [np.arange(S)] * Hq
    is_ = [np.arange(S // 64)] * Hq
    O, L = A.sparse_attention_forward(q, k, v, iv, is_)
    for h in range(Hq):
        Od, Ld = A.dense_attention_forward(q[:, h], k[:, 0], v[:, 0])
        assert np.max(np.abs(O[:, h] - Od)) < 1e-12 and np.max(np.abs(L[h] - Ld)) < 1e-12


def test_sparse_equals_masked_dense_bruteforce():
    S, Hq, Hkv, d = 256, 2, 1, 16
    q, k, v = _rand(S, Hq, Hkv, d, 2)
    iv, is_ = _rand_index(S, Hq, 3)
    O, L = A.sparse_attention_forward(q, k, v, iv, is_)
    for h in range(Hq):
        mask = SF.union_mask(iv[h], is_[h], S)
        Od, Ld = A.dense_attention_forward(q[:, h], k[:, 0], v[:, 0], mask=mask)
        assert np.max(np.abs(O[:, h] - Od)) < 1e-12 and np.max(np.abs(L[h] - Ld)) < 1e-12


def test_diagonal_only_is_blockwise_causal():
    S, d = 192, 8
    q, k, v = _rand(S, 1, 1, d, 4)
    O, L = A.sparse_attention_forward(q, k, v, [np.array([0])], [np.array([0])])
    for g in range(3):
        r = slice(64 * g, 64 * g + 64)
        Od, _ = A.dense_attention_forward(q[r, 0], k[r, 0], v[r, 0])
        if g == 0:
            assert np.allclose(O[r, 0], Od, atol=1e-12)
    # block 1 row 0 attends column 0 (vertical) plus itself
    n = 64
    s = np.array([q[n, 0] @ k[0, 0], q[n, 0] @ k[n, 0]]) / np.sqrt(d)
    p = np.exp(s - s.max()); p /= p.sum()
    assert np.allclose(O[n, 0], p[0] * v[0, 0] + p[1] * v[n, 0], atol=1e-12)


def test_merge_identities():
    r = np.random.default_rng(5)
    Oa, La = r.standard_normal((8, 4)), r.standard_normal(8)
    O, L = A.merge_out_and_lse(Oa, La, np.zeros((8, 4)), np.full(8, -np.inf))
    assert np.allclose(O, Oa) and np.allclose(L, La)
    O, L = A.merge_out_and_lse(Oa, La, Oa, La)
    assert np.allclose(O, Oa) and np.allclose(L, La + np.log(2))
    q, k, v = (r.standard_normal((16, 8)) for _ in range(3))
    full = A.dense_attention_forward(q, k, v, mask=np.ones((16, 16), bool))
    a = A.dense_attention_forward(q, k[:7], v[:7], mask=np.ones((16, 7), bool))
    b = A.dense_attention_forward(q, k[7:], v[7:], mask=np.ones((16, 9), bool))
    O, L = A.merge_out_and_lse(a[0], a[1], b[0], b[1])
    assert np.max(np.abs(O - full[0])) < 1e-12 and np.max(np.abs(L - full[1])) < 1e-12


def test_backward_zero_cotangent_and_single_token():
    q, k, v = _rand(128, 2, 1, 8, 6)
    iv, is_ = _rand_index(128, 2, 7)
    O, L = A.sparse_attention_forward(q, k, v, iv, is_)
    dq, dk, dv = A.sparse_attention_backward(q, k, v, O, L, np.zeros_like(q), iv, is_)
    assert not dq.any() and not dk.any() and not dv.any()
    # a single key: dV = dO, dQ = dK = 0
    dQ, dK, dV = A.dense_attention_backward(np.ones((1, 4)), np.ones((1, 4)), np.ones((1, 4)),
                                            np.arange(4.0)[None])
    assert np.allclose(dV, np.arange(4.0)) and np.allclose(dQ, 0) and np.allclose(dK, 0)


def test_backward_finite_differences():
    # S:59 / S:219 — central differences of <dO, O> with the index held fixed.
    S, Hq, Hkv, d = 128, 2, 1, 16
    q, k, v = _rand(S, Hq, Hkv, d, 8)
    dO = np.random.default_rng(9).standard_normal((S, Hq, d))
    iv, is_ = _rand_index(S, Hq, 10, n_off=1, n_col=6)
    O, L = A.sparse_attention_forward(q, k, v, iv, is_)
    dq, dk, dv = A.sparse_attention_backward(q, k, v, O, L, dO, iv, is_)
    f = lambda q_, k_, v_: float((A.sparse_attention_forward(q_, k_, v_, iv, is_)[0] * dO).sum())
    r = np.random.default_rng(11)
    h = 1e-5
    for name, X, G in (("q", q, dq), ("k", k, dk), ("v", v, dv)):
        for _ in range(6):
            idx = tuple(int(r.integers(0, n)) for n in X.shape)
            Xp, Xm = X.copy(), X.copy()
            Xp[idx] += h
            Xm[idx] -= h
            args_p = {"q": (Xp, k, v), "k": (q, Xp, v), "v": (q, k, Xp)}[name]
            args_m = {"q": (Xm, k, v), "k": (q, Xm, v), "v": (q, k, Xm)}[name]
            fd = (f(*args_p) - f(*args_m)) / (2 * h)
            assert abs(fd - G[idx]) <= 1e-5 * max(1.0, abs(fd)), (name, idx, fd, G[idx])


def test_backward_full_budget_equals_dense_eq1():
    S, d = 128, 16
    q, k, v = _rand(S, 1, 1, d, 12)
    dO = np.random.default_rng(13).standard_normal((S, 1, d))
    iv, is_ = [np.arange(S)], [np.arange(2)]
    O, L = A.sparse_attention_forward(q, k, v, iv, is_)
    dq, dk, dv = A.sparse_attention_backward(q, k, v, O, L, dO, iv, is_)
    Dq, Dk, Dv = A.dense_attention_backward(q[:, 0], k[:, 0], v[:, 0], dO[:, 0])
    for a, b in ((dq[:, 0], Dq), (dk[:, 0], Dk), (dv[:, 0], Dv)):
        assert np.max(np.abs(a - b)) < 1e-11


def test_count_pairs_matches_mask():
    S = 256
    iv, is_ = _rand_index(S, 2, 14)
    cnt = A.count_pairs(iv, is_, S)
    for h in range(2):
        assert cnt[h] == SF.union_mask(iv[h], is_[h], S).sum()
    # restricted to some query blocks: the mask rows of those blocks
    blocks = [0, 2, 3]
    sub = A.count_pairs(iv, is_, S, rows=blocks)
    for h in range(2):
        m = SF.union_mask(iv[h], is_[h], S)
        assert sub[h] == sum(m[g * 64:(g + 1) * 64].sum() for g in blocks)


def test_gqa_mapping_equals_repeat_interleaved_mha():
    # Reading R10 ("per head", GQA of Qwen2.5): q head h reads kv head
    # h // (Hq/Hkv).  Pinned against the plain multi-head computation on K/V repeated
    # per q head (repeat-interleave: q heads 0..grp-1 -> kv head 0, ...): the GQA
    # outputs and dQ must equal the MHA ones, and the GQA dK/dV of a kv head must
    # equal the sum of the MHA dK/dV of its q heads.  Hkv = 2 and 4 with Hq = 8, and
    # a different index per q head, so a wrong head -> kv-head map fails.
    rng = np.random.default_rng(31)
    S, Hq, d = 256, 8, 16
    for Hkv in (2, 4):
        grp = Hq // Hkv
        q = rng.standard_normal((S, Hq, d))
        k = rng.standard_normal((S, Hkv, d))
        v = rng.standard_normal((S, Hkv, d))
        dO = rng.standard_normal((S, Hq, d))
        iv, is_ = [], []
        for h in range(Hq):
            iv.append(np.unique(np.r_[0, rng.choice(S, 12, replace=False)]).astype(np.int32))
            is_.append(np.unique(np.r_[0, rng.choice(S // 64, 2, replace=False)]).astype(np.int32))
        k_mha = np.repeat(k, grp, axis=1)   # [S][Hq][d], q head h -> kv head h // grp
        v_mha = np.repeat(v, grp, axis=1)
        O, L = A.sparse_attention_forward(q, k, v, iv, is_)
        Om, Lm = A.sparse_attention_forward(q, k_mha, v_mha, iv, is_)
        assert np.allclose(O, Om, atol=1e-12) and np.allclose(L, Lm, atol=1e-12)
        dq, dk, dv = A.sparse_attention_backward(q, k, v, O, L, dO, iv, is_)
        dqm, dkm, dvm = A.sparse_attention_backward(q, k_mha, v_mha, Om, Lm, dO, iv, is_)
        assert np.allclose(dq, dqm, atol=1e-12)
        assert np.allclose(dk, dkm.reshape(S, Hkv, grp, d).sum(axis=2), atol=1e-12)
        assert np.allclose(dv, dvm.reshape(S, Hkv, grp, d).sum(axis=2), atol=1e-12)
        # and the map is not the trivial one: a different kv head gives other outputs
        O_wrong, _ = A.sparse_attention_forward(q, np.roll(k_mha, grp, axis=1),
                                                 np.roll(v_mha, grp, axis=1), iv, is_)
        assert not np.allclose(O, O_wrong)
