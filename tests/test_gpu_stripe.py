"""GPU layouts (mt_stripe / mt_unstripe, mt_layout_to_local / _to_global) vs the oracle's
layout_perm: block-striped and zigzag.  Byte copies: bit-exact."""
import numpy as np
import pytest
import torch

from oracle.sparseformat import layout_perm
from paper_2510_18830_b200 import _lib, ops

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("layout", ["striped", "zigzag"])
@pytest.mark.parametrize("S,W", [(4096, 1), (4096, 2), (8192, 4), (131072, 8)])
def test_stripe_roundtrip_matches_oracle_perm(cuda_lib, S, W, layout):
    g = torch.Generator().manual_seed(S + W)
    x = torch.randint(-30000, 30000, (S, 3, 128), generator=g, dtype=torch.int16).cuda()
    perm = layout_perm(S, W, layout)
    back = torch.zeros_like(x)
    for r in range(W):
        loc = ops.stripe(x, W, r, layout)
        ref = x.cpu().numpy()[perm[r]]
        assert np.array_equal(loc.cpu().numpy(), ref)
        ops.unstripe(loc, W, r, back, layout)
    torch.cuda.synchronize()
    assert torch.equal(back, x)


def test_stripe_errors(cuda_lib):
    x = torch.zeros(4096, 1, 8, dtype=torch.int16, device="cuda")  # 16-byte rows
    lib = _lib.lib()
    y = torch.zeros(1024, 1, 8, dtype=torch.int16, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    assert lib.mt_stripe(4096, 16, 4, 0, x.data_ptr(), y.data_ptr(), s) == 0
    assert lib.mt_stripe(4096, 12, 4, 0, x.data_ptr(), y.data_ptr(), s) == 1   # MT_ESHAPE
    assert lib.mt_stripe(4096, 16, 4, 4, x.data_ptr(), y.data_ptr(), s) == 1   # rank out of range
    assert lib.mt_stripe(4000, 16, 1, 0, x.data_ptr(), y.data_ptr(), s) == 2   # MT_EWINDOW
    assert lib.mt_stripe(4096 + 64, 16, 2, 0, x.data_ptr(), y.data_ptr(), s) == 4  # MT_ELAYOUT


def test_zigzag_layout_errors(cuda_lib):
    x = torch.zeros(4096, 1, 8, dtype=torch.int16, device="cuda")
    y = torch.zeros(2048, 1, 8, dtype=torch.int16, device="cuda")
    lib = _lib.lib()
    s = torch.cuda.current_stream().cuda_stream
    assert lib.mt_layout_to_local(1, 4096, 16, 2, 1, x.data_ptr(), y.data_ptr(), s) == 0
    assert lib.mt_layout_to_local(1, 64 * 6, 16, 2, 0, x.data_ptr(), y.data_ptr(), s) == 4  # MT_ELAYOUT
    assert lib.mt_layout_to_local(7, 4096, 16, 2, 0, x.data_ptr(), y.data_ptr(), s) == 1    # MT_ESHAPE
