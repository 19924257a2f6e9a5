"""GPU RoPE (mt_rope) vs the fp64 oracle (oracle/rope.py; Appendix A
P:603-625, P:339 YaRN): block-striped global positions up to 512K, forward and
inverse, with and without YaRN.  Tolerance: the output is one bf16 rounding of a
value computed in fp32 from an fp64-reduced angle, so per element
|got - ref| <= 2^-8 |ref| + 2^-12 max|row| (the second term covers the fp32 sin/cos
error on near-cancelling pairs)."""
import numpy as np
import pytest
import torch

from oracle import rope as R
from oracle.sparseformat import stripe_perm
from paper_2510_18830_b200 import ops
from synth.generator import bf16_bits_to_f32
from tests.gpu_util import to_dev_bf16

pytestmark = pytest.mark.gpu


def _check(got, ref):
    rowmax = np.max(np.abs(ref), axis=-1, keepdims=True)
    bound = 2.0 ** -8 * np.abs(ref) + 2.0 ** -12 * rowmax
    assert np.all(np.abs(got - ref) <= bound), float(np.max(np.abs(got - ref) - bound))


@pytest.mark.parametrize("S,W,r,factor,inverse", [
    (4096, 1, 0, 1.0, False), (4096, 1, 0, 32.0, False), (8192, 4, 3, 32.0, True),
    (524288, 64, 63, 32.0, False), (524288, 64, 17, 1.0, True)])
def test_rope_matches_oracle(cuda_lib, S, W, r, factor, inverse):
    H = 3
    rng = np.random.default_rng(S + W + r)
    x32 = rng.standard_normal((S // W, H, 128)).astype(np.float32)
    bits = (x32.view(np.uint32) >> 16).astype(np.uint16)  # truncate to bf16 bit patterns
    xd = to_dev_bf16(bits)
    fr = ops.rope_freqs(1e6, factor, 32768)
    ops.rope_(xd, fr, seq_len=S, world=W, rank=r, inverse=inverse)
    torch.cuda.synchronize()
    got = xd.float().cpu().numpy().astype(np.float64)
    th, ms = R.inv_freq(128, 1e6, factor, 32768)
    pos = stripe_perm(S, W)[r]
    ref = R.rope(bf16_bits_to_f32(bits).astype(np.float64), pos, th, ms, inverse=inverse)
    _check(got, ref)


def test_rope_roundtrip_within_two_roundings(cuda_lib):
    x = torch.randn(2048, 2, 128, device="cuda").bfloat16()
    y = x.clone()
    fr = ops.rope_freqs()
    ops.rope_(y, fr, seq_len=2048 * 8, world=8, rank=5)
    ops.rope_(y, fr, seq_len=2048 * 8, world=8, rank=5, inverse=True)
    torch.cuda.synchronize()
    # each rounding lands ~2^-9 |pair| on either component of the rotated pair
    xf, yf = x.float(), y.float()
    rowmax = xf.abs().amax(dim=-1, keepdim=True)
    assert ((yf - xf).abs() <= 2 ** -7 * xf.abs() + 2 ** -7 * rowmax).all()
