"""GPU XAttention block index (mt_xattn_index_count/fill, reading R25;
SURVEY §8(f) f2) vs the fp64 oracle (oracle/xattn.py).

* block scores: element-wise within 2e-4 (bf16 inputs are exact; the GPU sums in
  fp32: a 2048-term GEMM, a softmax over <= S/16 terms, 64-term block sums);
* selection (a floating-point decision, taken in fp32 on the GPU and fp64 in the
  oracle): compared where it is unique — >= 99% of rows identical — and checked
  valid everywhere against the ORACLE's scores within eps = 1e-3: diagonal kept,
  threshold mass reached, greedy order, minimality;
* the 64-token CSR equals the expansion (step 5) of the GPU's own kept sets, bit
  for bit, and drives the block-sparse attention to finite outputs;
* 2944 tokens: a partial last 128-row tile of the fused score kernel (xattn_score.cu);
* at 512K (the bench shape; head batches of the fused kernel), sampled rows of four heads.
"""
import numpy as np
import pytest
import torch

from oracle import xattn as X
from paper_2510_18830_b200 import ops
from synth.generator import make_grad_out, make_qkv
from tests.gpu_util import f64, to_dev_bf16

pytestmark = pytest.mark.gpu
TAU, EPS = 0.9, 1e-3


def _kept_from_csr(rows64, nI):
    """128-granularity kept sets from the 64-token rows (row 2I + 1 holds 2J, 2J + 1)."""
    return [np.unique(np.asarray(rows64[2 * I + 1]) // 2).astype(np.int32) for I in range(nI)]


def _valid(kept, bs, I):
    tot = bs.sum()
    K = list(kept)
    assert I in K
    assert bs[K].sum() >= TAU * tot - EPS
    rest = [J for J in K if J != I]
    if rest:
        lo = min(bs[J] for J in rest)
        out = [J for J in range(I + 1) if J not in K]
        assert all(bs[J] <= lo + EPS for J in out)
        ok_min = bs[K].sum() - min(bs[J] for J in K) < TAU * tot + EPS or \
            bs[rest].sum() - lo < TAU * tot + EPS
        assert ok_min


def _tri_row(scores_h, I):
    b = I * (I + 1) // 2
    return scores_h[b: b + I + 1]


@pytest.mark.parametrize("S,Hq,Hkv,a", [(4096, 4, 2, 6.0), (2048, 2, 1, 16.0), (2944, 3, 1, 6.0)])
def test_xattn_index_matches_oracle(cuda_lib, S, Hq, Hkv, a):
    q, k, v = make_qkv(S, Hq, Hkv, seed=S + 3, a=a)
    qd, kd = to_dev_bf16(q), to_dev_bf16(k)
    bi, scores = ops.xattn_index(qd, kd, TAU, with_scores=True)
    torch.cuda.synchronize()
    B64_ref, BS_ref, SEL_ref = X.xattn_index(f64(q), f64(k), TAU)
    sc = scores.cpu().numpy().astype(np.float64)
    rows64 = bi.to_lists()
    nI = S // 128
    same = total = 0
    for h in range(Hq):
        for I in range(nI):
            assert np.max(np.abs(_tri_row(sc[h], I) - BS_ref[h][I, : I + 1])) <= 2e-4
        kept = _kept_from_csr(rows64[h], nI)
        assert all(np.array_equal(a_, b_) for a_, b_ in zip(rows64[h], X.to_block64(kept)))
        for I in range(nI):
            _valid(kept[I], BS_ref[h][I, : I + 1], I)
            same += np.array_equal(kept[I], SEL_ref[h][I])
            total += 1
    assert same >= 0.99 * total, (same, total)
    # the index drives the block-sparse attention
    vd, dOd = to_dev_bf16(v), to_dev_bf16(make_grad_out(S, Hq, seed=1))
    o, lse = ops.block_sparse_attn_fwd(qd, kd, vd, bi)
    dq, dk, dv = ops.block_sparse_attn_bwd(qd, kd, vd, o, lse, dOd, bi)
    torch.cuda.synchronize()
    for t in (o, lse, dq, dk, dv):
        assert torch.isfinite(t.float()).all()


def test_xattn_index_at_512k_sampled_rows(cuda_lib):
    S, Hq, Hkv = 524288, 16, 2
    q, k, _ = make_qkv(S, Hq, Hkv, seed=0)
    qd, kd = to_dev_bf16(q), to_dev_bf16(k)
    bi, scores = ops.xattn_index(qd, kd, TAU, with_scores=True)
    torch.cuda.synchronize()
    nI = S // 128
    ptr = bi.ptr.cpu().numpy()
    idx = bi.idx.cpu().numpy()
    sc = scores.cpu().numpy()
    for h in (0, 7, 8, 15):
        qh = f64(q[:, h, :])
        kh = f64(k[:, h // 8, :])
        for I in (0, 1, 1000, 2047, 2048, nI - 1):
            ref = X.block_score_rows(qh, kh, [I])[I]
            assert np.max(np.abs(_tri_row(sc[h], I).astype(np.float64) - ref)) <= 2e-4
            r64 = idx[ptr[h, 2 * I + 1]: ptr[h, 2 * I + 2]]
            kept = np.unique(r64 // 2)
            _valid(kept, ref, I)
    dens = idx.size / (Hq * (S // 64) * (S // 64 + 1) / 2)
    assert 0 < dens < 1
