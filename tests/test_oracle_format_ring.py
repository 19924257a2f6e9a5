"""Pins for sparseformat / convert_index / striping and the ring simulation."""
import json
from pathlib import Path

import numpy as np
import pytest

from oracle import attention as A
from oracle import ring as R
from oracle import sparseformat as SF

GOLD = json.loads((Path(__file__).parent / "golden" / "spec_examples.json").read_text())


@pytest.mark.parametrize("case", GOLD["sparseformat"])
def test_sparseformat_golden(case):
    B, C = SF.sparseformat(case["i_v"], case["i_s"], case["S"])
    assert [b.tolist() for b in B] == case["B"]
    assert [c.tolist() for c in C] == case["C"]


@pytest.mark.parametrize("case", GOLD["layout"])
def test_layout_golden(case):
    perm = SF.stripe_perm(case["S"], case["W"])
    blocks = [sorted(set((perm[r] // 64).tolist())) for r in range(case["W"])]
    assert blocks == case["rank_blocks"]


def test_stripe_is_bijection_and_identity_at_w1():
    S = 1024
    for W in (1, 2, 4, 8):
        p = SF.stripe_perm(S, W)
        assert sorted(p.ravel().tolist()) == list(range(S))
    assert SF.stripe_perm(S, 1)[0].tolist() == list(range(S))
    with pytest.raises(ValueError):
        SF.stripe_perm(1000, 2)


def test_mask_union_oracle():
    S = 320
    r = np.random.default_rng(0)
    for trial in range(6):
        iv = np.unique(np.r_[0, r.choice(S, 12, replace=False)])
        is_ = np.unique(np.r_[0, r.choice(S // 64, 2, replace=False)])
        B, C = SF.sparseformat(iv, is_, S)
        assert np.array_equal(SF.index_to_mask(B, C, S), SF.union_mask(iv, is_, S))
        # no double counting: bars never inside a selected slash block
        for g in range(S // 64):
            assert not set((C[g] // 64).tolist()) & set(B[g].tolist())


@pytest.mark.parametrize("W", [2, 4])
def test_convert_index_coverage(W):
    S = 512
    r = np.random.default_rng(W)
    iv = np.unique(np.r_[0, r.choice(S, 20, replace=False)])
    is_ = np.unique(np.r_[0, r.choice(S // 64, 3, replace=False)])
    B, C = SF.sparseformat(iv, is_, S)
    perm = SF.stripe_perm(S, W)
    got = np.zeros((S, S), bool)
    for rank in range(W):
        plan = SF.convert_index(B, C, S, W, rank)
        for s in range(W):
            for j, (lb, lc) in enumerate(plan[s]):
                keys = np.concatenate([np.arange(b * 64, b * 64 + 64) for b in lb] + [lc]).astype(int)
                rows = perm[rank][j * 64:(j + 1) * 64]
                for n in rows:
                    gk = perm[s][keys]
                    got[n, gk[gk <= n]] = True
    assert np.array_equal(got, SF.index_to_mask(B, C, S))


@pytest.mark.parametrize("case", GOLD["convert_index"])
def test_convert_index_golden_diagonal(case):
    S, W = case["S"], case["W"]
    B, C = SF.sparseformat([], case["i_s"], S)
    for rank in range(W):
        plan = SF.convert_index(B, C, S, W, rank)
        assert sum(len(lb) for lb, _ in plan[rank]) == case["step0_blocks_per_rank"]
        assert all(len(lb) == 0 for s in range(W) if s != rank for lb, _ in plan[s])


def test_dense_causal_balanced_across_ranks():
    # P:64 "Under causal full attention, both variants maintain balanced workload".
    # Block striping: rank r owns query blocks g = jW + r, each needing g + 1 key
    # blocks, so total_r = W n(n-1)/2 + n(r+1) with n = nb/W: balanced up to
    # (W-1)/(W n / 2), vanishing with sequence length.
    for S, W in ((1024, 4), (2048, 8)):
        B, C = SF.sparseformat(np.arange(S), np.arange(S // 64), S)
        n = S // 64 // W
        tot = []
        for rank in range(W):
            plan = SF.convert_index(B, C, S, W, rank)
            tot.append(sum(len(lb) for s in range(W) for lb, _ in plan[s]))
        assert tot == [W * n * (n - 1) // 2 + n * (rank + 1) for rank in range(W)]
        assert max(tot) / np.mean(tot) < 1 + 2.0 / n


@pytest.mark.parametrize("W,inner", [(4, None), (4, 2), (8, 4), (8, 2), (6, 3)])
def test_schedule_visits_each_origin_once(W, inner):
    sched = R.schedule(W, inner)
    assert len(sched) == W
    for r in range(W):
        assert sorted(step[r] for step in sched) == list(range(W))
    G = W if inner is None else inner
    for t, step in enumerate(sched):
        i, j = divmod(t, G)
        for r in range(W):
            n, l = divmod(r, G)
            assert step[r] == ((n - i) % (W // G)) * G + (l - j) % G


def _problem(S=512, Hq=2, Hkv=1, d=16, seed=0):
    rng = np.random.default_rng(seed)
    q, k, v = (rng.standard_normal((S, h, d)) for h in (Hq, Hkv, Hkv))
    iv = [np.unique(np.r_[0, rng.choice(S, 15, replace=False)]) for _ in range(Hq)]
    is_ = [np.unique(np.r_[0, 1, rng.choice(S // 64, 2, replace=False)]) for _ in range(Hq)]
    return q, k, v, iv, is_


@pytest.mark.parametrize("W,inner", [(1, None), (2, None), (4, None), (4, 2), (8, 4)])
def test_ring_forward_equals_single_device(W, inner):
    q, k, v, iv, is_ = _problem(seed=W)
    O, L = A.sparse_attention_forward(q, k, v, iv, is_)
    Or, Lr, _ = R.ring_forward(q, k, v, iv, is_, W, inner)
    assert np.max(np.abs(Or - O)) < 1e-12 and np.max(np.abs(Lr - L)) < 1e-12


@pytest.mark.parametrize("W,inner", [(2, None), (4, None), (4, 2)])
def test_ring_backward_equals_single_device(W, inner):
    q, k, v, iv, is_ = _problem(seed=10 + W)
    dO = np.random.default_rng(99).standard_normal(q.shape)
    O, L = A.sparse_attention_forward(q, k, v, iv, is_)
    ref = A.sparse_attention_backward(q, k, v, O, L, dO, iv, is_)
    got = R.ring_backward(q, k, v, O, L, dO, iv, is_, W, inner)
    for a, b in zip(got, ref):
        assert np.max(np.abs(a - b)) < 1e-11


def test_hierarchical_equals_flat_both_factorizations():
    q, k, v, iv, is_ = _problem(seed=21)
    flat = R.ring_forward(q, k, v, iv, is_, 8, None)[0]
    for inner in (4, 2):
        assert np.max(np.abs(R.ring_forward(q, k, v, iv, is_, 8, inner)[0] - flat)) < 1e-12


# ------------------------------------------------------------------ zigzag layout (f1)
@pytest.mark.parametrize("case", GOLD["layout_zigzag"])
def test_zigzag_golden(case):
    perm = SF.zigzag_perm(case["S"], case["W"])
    assert [sorted(p.tolist()) for p in perm] == case["rank_tokens"]


def test_zigzag_bijection_two_runs_identity_at_w1():
    for S, W in ((1024, 2), (1024, 4), (2048, 8)):
        p = SF.zigzag_perm(S, W)
        assert sorted(p.ravel().tolist()) == list(range(S))
        for r in range(W):  # exactly two contiguous ascending runs of S / 2W tokens
            d = np.diff(p[r])
            assert (d > 0).all() and int((d != 1).sum()) == (1 if r < W - 1 else 0)
    assert SF.zigzag_perm(256, 1)[0].tolist() == list(range(256))
    with pytest.raises(ValueError):
        SF.layout_perm(64 * 6, 2, "zigzag")   # chunks must be whole 64-token blocks


def test_zigzag_causal_balance_exact():
    # P:64 "Under causal full attention, both variants maintain balanced workload";
    # per-rank planned work is EXACTLY equal for zigzag (chunk w and its
    # mirror 2W-1-w together hold (2W-1)c^2 + c(c+1) causal pairs, independent of w),
    # unlike block striping (test_dense_causal_balanced_across_ranks).
    for S, W in ((1024, 2), (1024, 4), (2048, 8)):
        B, C = SF.sparseformat(np.arange(S), np.arange(S // 64), S)
        tot = []
        for rank in range(W):
            plan = SF.convert_index(B, C, S, W, rank, layout="zigzag")
            tot.append(sum(len(lb) for s in range(W) for lb, _ in plan[s]))
        assert len(set(tot)) == 1, tot
        c = S // 64 // (2 * W)
        assert tot[0] == (2 * W - 1) * c * c + c * (c + 1)


@pytest.mark.parametrize("W", [2, 4])
def test_convert_index_coverage_zigzag(W):
    # the union over (rank, origin) of the local plans, mapped back through
    # the layout, is exactly the global index mask (no gaps, no duplicates)
    S = 1024
    r = np.random.default_rng(30 + W)
    iv = np.unique(np.r_[0, r.choice(S, 25, replace=False)])
    is_ = np.unique(np.r_[0, r.choice(S // 64, 4, replace=False)])
    B, C = SF.sparseformat(iv, is_, S)
    perm = SF.zigzag_perm(S, W)
    got = np.zeros((S, S), np.int64)
    for rank in range(W):
        plan = SF.convert_index(B, C, S, W, rank, layout="zigzag")
        for s in range(W):
            for j, (lb, lc) in enumerate(plan[s]):
                keys = np.concatenate([np.arange(b * 64, b * 64 + 64) for b in lb] + [lc]).astype(int)
                for n in perm[rank][j * 64:(j + 1) * 64]:
                    gk = perm[s][keys]
                    got[n, gk[gk <= n]] += 1
    assert np.array_equal(got, SF.union_mask(iv, is_, S).astype(np.int64))


@pytest.mark.parametrize("W,inner", [(2, None), (4, None), (4, 2)])
def test_ring_zigzag_equals_single_device(W, inner):
    q, k, v, iv, is_ = _problem(S=1024, seed=50 + W)
    dO = np.random.default_rng(7).standard_normal(q.shape)
    O, L = A.sparse_attention_forward(q, k, v, iv, is_)
    Or, Lr, _ = R.ring_forward(q, k, v, iv, is_, W, inner, layout="zigzag")
    assert np.max(np.abs(Or - O)) < 1e-12 and np.max(np.abs(Lr - L)) < 1e-12
    ref = A.sparse_attention_backward(q, k, v, O, L, dO, iv, is_)
    got = R.ring_backward(q, k, v, O, L, dO, iv, is_, W, inner, layout="zigzag")
    for a, b in zip(got, ref):
        assert np.max(np.abs(a - b)) < 1e-11
