"""The library's host-side frequency table (mt_rope_inv_freq) against the oracle's
inv_freq (Appendix A; P:339 YaRN factor 32; reading R-rope).
Host code only: runs without a GPU."""
import ctypes

import numpy as np
import pytest

from oracle import rope as R
from paper_2510_18830_b200 import _lib, ops


@pytest.mark.parametrize("base,factor,L", [(1e6, 1.0, 32768), (1e6, 32.0, 32768),
                                           (1e4, 4.0, 4096), (5e5, 8.0, 8192)])
def test_inv_freq_matches_oracle(base, factor, L):
    th, ms = ops.rope_freqs(base, factor, L)
    ref, ms_ref = R.inv_freq(128, base, factor, L)
    assert np.allclose(np.asarray(th[:]), ref, rtol=1e-14, atol=0)
    assert ms == pytest.approx(ms_ref, rel=1e-7)


def test_inv_freq_errors():
    th = (ctypes.c_double * 64)()
    ms = ctypes.c_float()
    lib = _lib.lib()
    assert lib.mt_rope_inv_freq(64, 1e6, 1.0, 32768, th, ctypes.byref(ms)) != 0
    assert lib.mt_rope_inv_freq(128, 1e6, 0.5, 32768, th, ctypes.byref(ms)) != 0
    assert lib.mt_rope_inv_freq(128, 1e6, 2.0, 0, th, ctypes.byref(ms)) != 0
