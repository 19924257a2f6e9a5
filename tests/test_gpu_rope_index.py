"""f3 upstream fusion (P:339 RoPE/YaRN, Appendix A): the RoPE-fused
index builder mt_rope_vs_index against the unfused composition mt_rope + mt_build_vs_index.

Contract (include/mtsa.h): from PRE-RoPE q / k it returns RoPE(q), RoPE(k) with the same
bf16 bits as mt_rope and exactly the lists mt_build_vs_index gives for them.  Both sides
are pinned to the oracle separately: mt_rope by tests/test_gpu_rope.py (vs oracle/rope.py),
mt_build_vs_index bit-exact by tests/test_gpu_index.py (vs oracle/vsidx.py); this test
closes the chain with bit equality (bytes and lists), so no oracle input comes from the
CUDA path."""
import numpy as np
import pytest
import torch

from paper_2510_18830_b200 import _lib, ops
from synth.generator import make_qkv
from tests.gpu_util import to_dev_bf16

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("S,Hq,Hkv,factor", [(4096, 8, 1, 32.0), (8192, 4, 2, 1.0), (65536, 16, 2, 32.0)])
def test_rope_index_equals_rope_then_index(cuda_lib, S, Hq, Hkv, factor):
    q, k, _ = make_qkv(S, Hq, Hkv, seed=S + 3, a=8.0)
    qd, kd = to_dev_bf16(q), to_dev_bf16(k)
    fr = ops.rope_freqs(1e6, factor, 32768)
    idx_f, q_rot, k_rot = ops.rope_vs_index(qd, kd, fr, 0.9, 0.9)
    qr, kr = qd.clone(), kd.clone()
    ops.rope_(qr, fr)
    ops.rope_(kr, fr)
    idx_u = ops.build_vs_index(qr, kr, 0.9, 0.9)
    torch.cuda.synchronize()
    assert torch.equal(q_rot.view(torch.int16), qr.view(torch.int16))
    assert torch.equal(k_rot.view(torch.int16), kr.view(torch.int16))
    a, b = idx_f.to_lists(), idx_u.to_lists()
    for h in range(Hq):
        assert np.array_equal(a[0][h], b[0][h]) and np.array_equal(a[1][h], b[1][h]), h
    # inputs untouched (out of place)
    assert torch.equal(qd.view(torch.int16), to_dev_bf16(q).view(torch.int16))


def test_rope_index_rejects_aliased_k(cuda_lib):
    S, Hq, Hkv = 2048, 2, 1
    q, k, _ = make_qkv(S, Hq, Hkv, seed=5)
    qd, kd = to_dev_bf16(q), to_dev_bf16(k)
    th, ms = ops.rope_freqs()
    sh = ops.shape(S, Hq, Hkv)
    L = _lib.lib()
    ws = ops.workspace(L.mt_build_vs_index_workspace_bytes(ops.ctypes.byref(sh), 1))
    idx = ops.VSIndex.uninit(S, Hq)
    ci = idx.c_struct()
    prm = ops.VSParams(0.9, 0.9)
    st = L.mt_rope_vs_index(None, ops.ctypes.byref(sh), ops.ctypes.byref(prm), th, ms, qd.data_ptr(),
                            kd.data_ptr(), qd.data_ptr(), kd.data_ptr(), ops.ctypes.byref(ci),
                            ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream)
    assert st == 1  # MT_ESHAPE
