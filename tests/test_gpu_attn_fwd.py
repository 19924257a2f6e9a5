"""GPU sparse forward (tcgen05 kernel through the C ABI) vs the fp64 oracle.

Tolerance (BASELINE.json north_star; reading R20): per-head normwise
max|O - O_ref| / max|O_ref| <= 2e-2 for the bf16 output; LSE absolute <= 1e-3.
"""
import numpy as np
import pytest
import torch

from oracle import attention as OA
from oracle import ring as OR
from oracle import vsidx
from oracle.sparseformat import layout_perm
from paper_2510_18830_b200 import ops
from synth.generator import bf16_bits_to_f32, make_qkv
from tests.gpu_util import f64, normwise_err, random_index, to_dev_bf16

pytestmark = pytest.mark.gpu

TOL_O = 2e-2
TOL_LSE = 1e-3


def _check(q, k, v, iv, is_):
    O_ref, L_ref = OA.sparse_attention_forward(f64(q), f64(k), f64(v), iv, is_)
    idx = ops.VSIndex.from_lists(iv, is_, q.shape[0])
    o, lse = ops.sparse_attn_fwd(to_dev_bf16(q), to_dev_bf16(k), to_dev_bf16(v), idx)
    torch.cuda.synchronize()
    o = o.float().cpu().numpy().astype(np.float64)
    lse = lse.cpu().numpy().astype(np.float64)
    assert np.isfinite(o).all() and np.isfinite(lse).all()
    e_o = normwise_err(o, O_ref, 1)
    e_l = np.max(np.abs(lse - L_ref))
    assert e_o <= TOL_O and e_l <= TOL_LSE, (e_o, e_l)
    return e_o, e_l


def test_fwd_c1_generator_index(cuda_lib):
    # BASELINE config 1: 8 q heads, 1 kv head, d = 128, S = 4096; index from Alg. 1 oracle
    S, Hq, Hkv = 4096, 8, 1
    q, k, v = make_qkv(S, Hq, Hkv, seed=1)
    iv, is_ = vsidx.build_vs_index(bf16_bits_to_f32(q), bf16_bits_to_f32(k), 0.9, 0.9)
    _check(q, k, v, iv, is_)


def test_fwd_full_budget_dense_causal(cuda_lib):
    S, Hq, Hkv = 1024, 2, 1
    q, k, v = make_qkv(S, Hq, Hkv, seed=2, a=4.0)
    _check(q, k, v, [np.arange(S, dtype=np.int32)] * Hq, [np.arange(S // 64, dtype=np.int32)] * Hq)


def test_fwd_diagonal_only(cuda_lib):
    S, Hq, Hkv = 512, 2, 2
    q, k, v = make_qkv(S, Hq, Hkv, seed=3, a=4.0)
    _check(q, k, v, [np.array([0], np.int32)] * Hq, [np.array([0], np.int32)] * Hq)


@pytest.mark.parametrize("S", [2112, 4096])
def test_fwd_random_index_many_bars_gqa(cuda_lib, S):
    # odd local block count (2112 = 33 x 64) exercises the half-empty last tile;
    # many verticals exercise multi-chunk bar gathers; Hq/Hkv = 2 exercises GQA.
    Hq, Hkv = 4, 2
    q, k, v = make_qkv(S, Hq, Hkv, seed=4, a=6.0)
    iv, is_ = random_index(S, Hq, 5, n_off=5, n_col=300)
    _check(q, k, v, iv, is_)


@pytest.mark.parametrize("layout", ["striped", "zigzag"])
@pytest.mark.parametrize("W", [2, 4, 8])
def test_fwd_ring_steps_emulated(cuda_lib, W, layout):
    """Every (rank, step) of a W-rank ring on one GPU vs the oracle ring, in the method's
    block-striped layout and in the zigzag layout of the f1 ablation."""
    S, Hq, Hkv = 2048, 4, 2
    q, k, v = make_qkv(S, Hq, Hkv, seed=6, a=6.0)
    iv, is_ = random_index(S, Hq, 7, n_off=6, n_col=80)
    O_ref, L_ref, sched = OR.ring_forward(f64(q), f64(k), f64(v), iv, is_, W, layout=layout)
    idx = ops.VSIndex.from_lists(iv, is_, S)
    perm = layout_perm(S, W, layout)
    Lq = S // W
    qd = [to_dev_bf16(q[perm[r]]) for r in range(W)]
    kd = [to_dev_bf16(k[perm[r]]) for r in range(W)]
    vd = [to_dev_bf16(v[perm[r]]) for r in range(W)]
    o = [torch.empty(Lq, Hq, 128, dtype=torch.bfloat16, device="cuda") for _ in range(W)]
    oacc = [torch.empty(Lq, Hq, 128, dtype=torch.float32, device="cuda") for _ in range(W)]
    lse = [torch.empty(Hq, Lq, dtype=torch.float32, device="cuda") for _ in range(W)]
    for t, held in enumerate(sched):
        for r in range(W):
            s = held[r]
            ops.attn_fwd_step(S, W, r, s, t == 0, t == W - 1, qd[r], kd[s], vd[s], idx,
                              o[r], oacc[r], lse[r], layout=layout)
    torch.cuda.synchronize()
    Og = np.zeros((S, Hq, 128))
    Lg = np.zeros((Hq, S))
    for r in range(W):
        Og[perm[r]] = o[r].float().cpu().numpy()
        Lg[:, perm[r]] = lse[r].cpu().numpy()
    assert normwise_err(Og, O_ref, 1) <= TOL_O
    assert np.max(np.abs(Lg - L_ref)) <= TOL_LSE


def test_fwd_rejects_bad_shapes(cuda_lib):
    from paper_2510_18830_b200 import _lib
    q = torch.zeros(100, 2, 128, dtype=torch.bfloat16, device="cuda")
    idx = ops.VSIndex.empty(128, 2)
    with pytest.raises(_lib.MTError) as e:
        ops.sparse_attn_fwd(q, q[:, :1].contiguous(), q[:, :1].contiguous(), idx)
    assert e.value.name == "MT_EWINDOW"


def test_fwd_stabiliser_overflow_fixup(cuda_lib):
    # The forward fixes each query column's stabiliser from the tile's first chunk (the
    # diagonal + next offset) and routes tiles whose later scores exceed it by more than
    # 2^64 to the exact two-pass attn_fwd_fixup kernel.  Plant such scores: queries of
    # blocks 6 and 10 (dimension 0 = 40) against vertical columns 5 and 200 (dimension
    # 0 = 40), which sit in bar chunks after the slash chunk, 1600 / sqrt(128) = 141 nats
    # (204 log2 units) above anything in chunk 0.  P:879's merge and LSE must still match.
    S, Hq, Hkv = 1024, 2, 1
    q, k, v = make_qkv(S, Hq, Hkv, seed=5, a=4.0)
    from synth.generator import f32_to_bf16_bits
    qf, kf = bf16_bits_to_f32(q).copy(), bf16_bits_to_f32(k).copy()
    for g in (6, 10):
        qf[g * 64:(g + 1) * 64, :, 0] = 40.0
    kf[[5, 200], :, 0] = 40.0
    q, k = f32_to_bf16_bits(qf), f32_to_bf16_bits(kf)
    iv = [np.array([0, 5, 200, 333], np.int32)] * Hq
    is_ = [np.array([0, 1], np.int32)] * Hq
    _check(q, k, v, iv, is_)
    # the backward recomputes P from the fixed-up LSE
    from synth.generator import make_grad_out
    dO = make_grad_out(S, Hq, seed=5)
    O, L = OA.sparse_attention_forward(f64(q), f64(k), f64(v), iv, is_)
    ref = OA.sparse_attention_backward(f64(q), f64(k), f64(v), O, L, f64(dO), iv, is_)
    idx = ops.VSIndex.from_lists(iv, is_, S)
    qd, kd, vd = to_dev_bf16(q), to_dev_bf16(k), to_dev_bf16(v)
    o, lse = ops.sparse_attn_fwd(qd, kd, vd, idx)
    g = ops.sparse_attn_bwd(qd, kd, vd, o, lse, to_dev_bf16(dO), idx)
    torch.cuda.synchronize()
    for got, r in zip(g, ref):
        assert normwise_err(got.float().cpu().numpy().astype(np.float64), r, 1) <= TOL_O
