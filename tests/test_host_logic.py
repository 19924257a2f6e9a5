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
