"""Host-side logic of the product package checked on CPU (no GPU needed)."""
import numpy as np

from oracle import attention as OA
from paper_2510_18830_b200 import stats
from tests.gpu_util import random_index


def test_pair_accounting_matches_oracle_mask_count():
    for S, seed in ((512, 1), (2048, 2), (4096, 3)):
        iv, is_ = random_index(S, 3, seed, n_off=7, n_col=60)
        assert np.array_equal(stats.pairs_per_head(iv, is_, S), OA.count_pairs(iv, is_, S))
    S = 1024
    full = stats.pairs_per_head([np.arange(S)], [np.arange(S // 64)], S)
    assert full[0] == stats.causal_pairs(S)


def test_block_index_lists_roundtrip_host():
    """BlockIndex (the block-CSR argument of mt_block_sparse_attn_* / mt_xattn_index):
    global row pointers [Hq][nb + 1], empty rows, round trip through the lists."""
    from paper_2510_18830_b200.ops import BlockIndex
    B = [[np.array([0], np.int32), np.zeros(0, np.int32), np.array([0, 2], np.int32)],
         [np.array([0], np.int32), np.array([0, 1], np.int32), np.zeros(0, np.int32)]]
    bi = BlockIndex.from_lists(B, device="cpu")
    assert bi.n == 6
    assert bi.ptr.tolist() == [[0, 1, 1, 3], [3, 4, 6, 6]]
    back = bi.to_lists()
    assert all(np.array_equal(a, b) for ra, rb in zip(back, B) for a, b in zip(ra, rb))
