"""GPU Alg. 1 index (mt_build_vs_index) vs the VS-IDX v1 oracle: bit-exact."""
import numpy as np
import pytest
import torch

from oracle import vsidx
from paper_2510_18830_b200 import ops
from synth.generator import bf16_bits_to_f32, make_qkv
from tests.gpu_util import to_dev_bf16

pytestmark = pytest.mark.gpu


def _oracle_scores(q, k):
    S, Hq, _ = q.shape
    grp = Hq // k.shape[1]
    qf, kf = bf16_bits_to_f32(q), bf16_bits_to_f32(k)
    cols, sl = [], []
    for h in range(Hq):
        V = vsidx.column_scores(np.ascontiguousarray(qf[S - 64:, h]), np.ascontiguousarray(kf[:, h // grp]))
        cols.append(V)
        sl.append(V.reshape(-1, 64).sum(axis=1, dtype=np.uint64)[::-1])
    return np.stack(cols), np.stack(sl)


@pytest.mark.parametrize("S,Hq,Hkv,seed", [(4096, 8, 1, 11), (8192, 4, 2, 12)])
def test_column_scores_bitexact(cuda_lib, S, Hq, Hkv, seed):
    q, k, _ = make_qkv(S, Hq, Hkv, seed=seed)
    col, sl = ops.vs_column_scores(to_dev_bf16(q), to_dev_bf16(k))
    torch.cuda.synchronize()
    ref_c, ref_s = _oracle_scores(q, k)
    assert np.array_equal(col.cpu().numpy().view(np.uint64), ref_c)
    assert np.array_equal(sl.cpu().numpy().view(np.uint64), ref_s)


@pytest.mark.parametrize("S,Hq,Hkv,p", [(4096, 8, 1, 0.9), (4096, 8, 1, 0.97), (65536, 16, 2, 0.9),
                                        (2048, 2, 1, 1.0), (8192, 4, 1, 0.9), (8192, 2, 1, 0.5)])
def test_index_lists_bitexact(cuda_lib, S, Hq, Hkv, p):
    q, k, _ = make_qkv(S, Hq, Hkv, seed=S + Hq)
    idx = ops.build_vs_index(to_dev_bf16(q), to_dev_bf16(k), p, p)
    torch.cuda.synchronize()
    iv, is_ = idx.to_lists()
    riv, ris = vsidx.build_vs_index(bf16_bits_to_f32(q), bf16_bits_to_f32(k), p, p)
    for h in range(Hq):
        assert np.array_equal(iv[h], riv[h]), (h, len(iv[h]), len(riv[h]))
        assert np.array_equal(is_[h], ris[h]), (h, len(is_[h]), len(ris[h]))
    if p == 1.0:
        assert all(len(x) == S for x in iv) and all(len(x) == S // 64 for x in is_)


def test_index_deterministic_and_forced(cuda_lib):
    S, Hq, Hkv = 8192, 4, 1
    q, k, _ = make_qkv(S, Hq, Hkv, seed=3)
    qd, kd = to_dev_bf16(q), to_dev_bf16(k)
    a = ops.build_vs_index(qd, kd, 0.9, 0.9).to_lists()
    b = ops.build_vs_index(qd, kd, 0.9, 0.9).to_lists()
    for x, y in zip(a[0] + a[1], b[0] + b[1]):
        assert np.array_equal(x, y)
    assert all(x[0] == 0 for x in a[0]) and all(x[0] == 0 for x in a[1])


def test_index_rejects_bad_p(cuda_lib):
    from paper_2510_18830_b200 import _lib
    q = torch.zeros(128, 2, 128, dtype=torch.bfloat16, device="cuda")
    with pytest.raises(_lib.MTError) as e:
        ops.build_vs_index(q, q[:, :1].contiguous(), 0.0, 0.5)
    assert e.value.name == "MT_ECONFIG"


_PER_HEAD_SCRIPT = r"""
import sys, numpy as np, torch
from paper_2510_18830_b200 import ops
from synth.generator import make_qkv
from tests.gpu_util import to_dev_bf16
S, Hq, Hkv, out = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4]
q, k, _ = make_qkv(S, Hq, Hkv, seed=S + 7)
iv, is_ = ops.build_vs_index(to_dev_bf16(q), to_dev_bf16(k), 0.9, 0.9).to_lists()
np.savez(out, *(list(iv) + list(is_)))
"""


@pytest.mark.parametrize("S,Hq,Hkv,env", [
    (65536, 16, 2, {"MT_VS_SORT_PER_HEAD": "1"}),
    (4096, 8, 1, {"MT_VS_SORT_PER_HEAD": "1", "MT_VS_SELECT_SMALL": "0"}),
    (8192, 4, 1, {"MT_VS_SELECT_SMALL": "0"})])
def test_index_sort_paths_agree(cuda_lib, tmp_path, S, Hq, Hkv, env):
    """The select paths give the same lists: the one-sort path (head id in the key's top
    bits), the per-head sorts (forced by MT_VS_SORT_PER_HEAD=1, the layout used when the
    head bits do not fit) and, for S <= 8192, the one-launch shared-memory select
    (MT_VS_SELECT_SMALL=0 forces the radix-sort path there)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = str(tmp_path / "per_head.npz")
    env = dict(os.environ, PYTHONPATH=root, **env)
    subprocess.run([sys.executable, "-c", _PER_HEAD_SCRIPT, str(S), str(Hq), str(Hkv), out],
                   check=True, env=env, cwd=root, timeout=600)
    ref = np.load(out)
    q, k, _ = make_qkv(S, Hq, Hkv, seed=S + 7)
    iv, is_ = ops.build_vs_index(to_dev_bf16(q), to_dev_bf16(k), 0.9, 0.9).to_lists()
    got = list(iv) + list(is_)
    assert len(got) == len(ref.files)
    for i, x in enumerate(got):
        assert np.array_equal(x, ref[f"arr_{i}"]), i


def test_column_scores_bitexact_extreme_values(cuda_lib):
    # VS-IDX I1 is a fused multiply-add fold (reading R11): the GPU's __fmaf_rn and the
    # oracle's exact sums must agree on EVERY bf16 input, including products below fp32's
    # subnormal range (2^-149) and subnormal partial sums, where a separately rounded
    # product would differ.  Planted: 20% of the keys scaled by 2^-120, 20% of the window
    # queries by 2^-40 (products ~2^-160), plus bf16 subnormals.
    from synth.generator import f32_to_bf16_bits
    S, Hq, Hkv = 4096, 4, 2
    q, k, _ = make_qkv(S, Hq, Hkv, seed=17)
    r = np.random.default_rng(18)
    qf, kf = bf16_bits_to_f32(q).copy(), bf16_bits_to_f32(k).copy()
    kf[r.random(kf.shape) < 0.2] *= np.float32(2.0 ** -120)
    qf[r.random(qf.shape) < 0.2] *= np.float32(2.0 ** -40)
    kf[r.random(kf.shape) < 0.01] = np.float32(2.0 ** -130)   # bf16 subnormal
    q, k = f32_to_bf16_bits(qf), f32_to_bf16_bits(kf)
    col, sl = ops.vs_column_scores(to_dev_bf16(q), to_dev_bf16(k))
    torch.cuda.synchronize()
    ref_c, ref_s = _oracle_scores(q, k)
    assert np.array_equal(col.cpu().numpy().view(np.uint64), ref_c)
    assert np.array_equal(sl.cpu().numpy().view(np.uint64), ref_s)
    idx = ops.build_vs_index(to_dev_bf16(q), to_dev_bf16(k), 0.9, 0.9)
    torch.cuda.synchronize()
    iv, is_ = idx.to_lists()
    riv, ris = vsidx.build_vs_index(bf16_bits_to_f32(q), bf16_bits_to_f32(k), 0.9, 0.9)
    for h in range(Hq):
        assert np.array_equal(iv[h], riv[h]) and np.array_equal(is_[h], ris[h]), h
