"""GPU per-query-block key lists (mt_vs_format_count / fill, the sparseformat step,
PAPER.md P:231-232, reading I9) vs the oracle's sparseformat: integer work, bit-exact."""
import numpy as np
import pytest
import torch

from oracle.sparseformat import sparseformat
from oracle import vsidx
from paper_2510_18830_b200 import ops
from synth.generator import bf16_bits_to_f32, make_qkv
from tests.gpu_util import random_index

pytestmark = pytest.mark.gpu


def _check(iv, is_, S):
    idx = ops.VSIndex.from_lists(iv, is_, S)
    bp, bi, cp, ci = ops.vs_format(idx, S)
    torch.cuda.synchronize()
    bp, bi, cp, ci = (t.cpu().numpy() for t in (bp, bi, cp, ci))
    nb = S // 64
    for h in range(len(iv)):
        B, C = sparseformat(iv[h], is_[h], S)
        for g in range(nb):
            assert np.array_equal(bi[bp[h, g]:bp[h, g + 1]], B[g]), (h, g)
            assert np.array_equal(ci[cp[h, g]:cp[h, g + 1]], C[g]), (h, g)
    # rows of consecutive heads are contiguous
    assert all(bp[h, nb] == bp[h + 1, 0] and cp[h, nb] == cp[h + 1, 0] for h in range(len(iv) - 1))


@pytest.mark.parametrize("S,n_off,n_col", [(64, 1, 1), (4096, 5, 300), (8192, 40, 900)])
def test_format_matches_oracle_random(cuda_lib, S, n_off, n_col):
    iv, is_ = random_index(S, 4, S + n_off, n_off=n_off, n_col=n_col)
    _check(iv, is_, S)


def test_format_matches_oracle_generator_index(cuda_lib):
    S = 4096
    q, k, _ = make_qkv(S, 4, 1, seed=31)
    iv, is_ = vsidx.build_vs_index(bf16_bits_to_f32(q), bf16_bits_to_f32(k), 0.9, 0.9)
    _check(iv, is_, S)


def test_format_dense_causal(cuda_lib):
    S = 2048
    nb = S // 64
    iv = [np.arange(S, dtype=np.int32)] * 2          # every column: all covered by offsets
    is_ = [np.arange(nb, dtype=np.int32)] * 2        # every offset: dense causal blocks
    _check(iv, is_, S)
