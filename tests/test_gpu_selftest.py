"""tcgen05 / TMEM / TMA building blocks on one CTA vs a plain fp32 matmul."""
import pytest
import torch

from paper_2510_18830_b200 import _lib

pytestmark = pytest.mark.gpu


def _run(variant, A, B, N):
    D = torch.zeros(128, N, dtype=torch.float32, device="cuda")
    _lib.check(_lib.lib().mt_selftest_mma(variant, A.data_ptr(), B.data_ptr(), D.data_ptr(),
                                          torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    return D


@pytest.mark.parametrize("variant", [0, 1, 2, 3, 4])
def test_mma_variant(cuda_lib, variant):
    g = torch.Generator(device="cpu").manual_seed(100 + variant)
    rnd = lambda *s: torch.randn(*s, generator=g).to(torch.bfloat16).cuda()
    if variant == 0:
        A, B = rnd(128, 128), rnd(64, 128)
        ref = A.float() @ B.float().T
    elif variant in (1, 3):
        A, B = rnd(128, 64), rnd(64, 128)
        ref = A.float() @ B.float()
    elif variant == 2:
        A, B = rnd(128, 128), rnd(128, 64)
        ref = A.float().T @ B.float()
    else:
        A, B = rnd(256, 2, 128), rnd(256, 2, 128)
        ref = A[128:256, 1].float() @ B[64:128, 0].float().T
    D = _run(variant, A, B, ref.shape[1])
    err = (D - ref).abs().max().item() / ref.abs().max().item()
    assert err < 1e-5, f"variant {variant}: rel err {err}"
