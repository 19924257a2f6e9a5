"""Workload-balance analysis (paper_2510_18830_b200/balance.py).

Pinned against a brute-force count over the materialised mask of the oracle
(`union_mask`: verticals U slash blocks, causal) and against properties the
paper states: under full causal attention both ZigZag and Striped are balanced
across workers."""
import numpy as np
import pytest

from oracle.sparseformat import union_mask
from paper_2510_18830_b200 import balance
from tests.gpu_util import random_index


def _owner_tokens(S, W, layout):
    """Token -> rank, written out independently of balance.block_owner."""
    tok = np.arange(S)
    b = tok // 64
    nb = S // 64
    if layout == "striped":
        return b % W
    if layout == "contiguous":
        return tok // (S // W)
    chunks = [list(range(c * S // (2 * W), (c + 1) * S // (2 * W))) for c in range(2 * W)]
    own = np.empty(S, dtype=np.int64)
    for r in range(W):
        own[chunks[r]] = r
        own[chunks[2 * W - 1 - r]] = r
    return own


@pytest.mark.parametrize("layout", balance.LAYOUTS)
@pytest.mark.parametrize("W", [2, 4])
def test_pairs_by_origin_matches_bruteforce_mask(layout, W):
    S, Hq = 1024, 3
    iv, is_ = random_index(S, Hq, 7 + W, n_off=5, n_col=40)
    M = balance.pairs_by_origin(iv, is_, S, W, layout)
    own = _owner_tokens(S, W, layout)
    ref = np.zeros((W, W), dtype=np.int64)
    for h in range(Hq):
        mask = union_mask(iv[h], is_[h], S)
        for r in range(W):
            for s in range(W):
                ref[r, s] += mask[np.ix_(own == r, own == s)].sum()
    assert np.array_equal(M, ref)


def test_flat_schedule_visits_every_origin_once():
    for W in (1, 2, 4, 8):
        held = balance.flat_schedule(W)
        for r in range(W):
            assert sorted(held[:, r]) == list(range(W))
        assert all(held[0, r] == r for r in range(W))  # step 0: own chunk


def test_dense_causal_is_worker_balanced_for_striped_and_zigzag():
    """Full budget (every offset) = dense causal attention: both layouts balance
    the per-worker totals, contiguous does not (rank W-1 has ~2W-1 x rank 0)."""
    S, W = 8192, 4
    nb = S // 64
    iv = [np.array([0], np.int32)]
    is_ = [np.arange(nb, dtype=np.int32)]
    tot = {}
    for layout in balance.LAYOUTS:
        P = balance.pairs_by_step(balance.pairs_by_origin(iv, is_, S, W, layout),
                                  balance.flat_schedule(W))
        assert P.sum() == S * (S + 1) // 2  # all causal pairs
        tot[layout] = balance.imbalance(P).total_id
    # striping leaves rank W-1 one block row ahead per stripe: 1 + O(W / nb) (1.023 here)
    assert tot["striped"] < 1.03 and tot["zigzag"] < 1.001
    assert tot["contiguous"] > 1.5


def test_imbalance_metrics_closed_forms():
    P = np.array([[4, 1], [2, 3]])  # ranks x steps
    m = balance.imbalance(P)
    # steps: max/mean = 4/3, 3/2 -> worker ID mean 17/12; ranks: 4/2.5, 3/2.5 -> 1.4
    assert m.worker_id == pytest.approx(17 / 12)
    assert m.step_id == pytest.approx(1.4)
    assert m.comp_ratio == pytest.approx((3 + 2) / (4 + 3))
    assert m.total_id == pytest.approx(1.0)


@pytest.mark.parametrize("layout", balance.LAYOUTS)
def test_block_index_pairs_match_bruteforce_mask(layout):
    """Explicit block rows (the XAttention / block-CSR form): brute-force count over
    the materialised causal block mask."""
    S, W = 1024, 4
    nb = S // 64
    rng = np.random.default_rng(3)
    B = [[np.unique(np.r_[rng.choice(g + 1, min(g + 1, 3), replace=False), g]).astype(np.int32)
          for g in range(nb)] for _ in range(2)]
    M = balance.pairs_by_origin_blocks(B, S, W, layout)
    own = _owner_tokens(S, W, layout)
    ref = np.zeros((W, W), dtype=np.int64)
    tok = np.arange(S)
    for rows in B:
        mask = np.zeros((S, S), bool)
        for g, r in enumerate(rows):
            for kb in r:
                mask[g * 64:(g + 1) * 64, kb * 64:(kb + 1) * 64] = True
        mask &= tok[:, None] >= tok[None, :]
        for a in range(W):
            for b in range(W):
                ref[a, b] += mask[np.ix_(own == a, own == b)].sum()
    assert np.array_equal(M, ref)


def test_bwd_slot_occupancy_matches_enumeration():
    """Brute force over the tiles (k, k + 1), k even, and query blocks g."""
    rng = np.random.default_rng(11)
    for nb in (17, 32):
        i_s = [np.unique(np.r_[0, rng.choice(nb, 6, replace=False)]) for _ in range(3)]
        chunks = live = 0
        for O in i_s:
            Os = set(int(x) for x in O)
            for k in range(0, nb, 2):
                for g in range(nb):
                    a = (g - k) in Os
                    b = k + 1 < nb and (g - k - 1) in Os
                    if a or b:
                        chunks += 1
                        live += int(a) + int(b)
        occ = balance.bwd_slot_occupancy(i_s, nb)
        assert (occ["chunks"], occ["live_slots"]) == (chunks, live)
