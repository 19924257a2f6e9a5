"""GPU sparse backward (tcgen05 kernels through the C ABI) vs the fp64 oracle.

Tolerance (north_star; reading R20): per-head normwise error <= 2e-2 for the bf16
dQ, dK, dV.  The oracle backward is fed the oracle forward's O/LSE; the GPU
backward is fed the GPU forward's bf16 O and fp32 LSE (the path as used).
"""
import numpy as np
import pytest
import torch

from oracle import attention as OA
from oracle import ring as OR
from oracle import vsidx
from oracle.sparseformat import layout_perm
from paper_2510_18830_b200 import ops
from synth.generator import bf16_bits_to_f32, make_grad_out, make_qkv
from tests.gpu_util import f64, normwise_err, random_index, to_dev_bf16

pytestmark = pytest.mark.gpu
TOL = 2e-2


def _check(q, k, v, dO, iv, is_):
    qf, kf, vf, dOf = f64(q), f64(k), f64(v), f64(dO)
    O_ref, L_ref = OA.sparse_attention_forward(qf, kf, vf, iv, is_)
    dq_r, dk_r, dv_r = OA.sparse_attention_backward(qf, kf, vf, O_ref, L_ref, dOf, iv, is_)
    idx = ops.VSIndex.from_lists(iv, is_, q.shape[0])
    qd, kd, vd, dOd = (to_dev_bf16(x) for x in (q, k, v, dO))
    o, lse = ops.sparse_attn_fwd(qd, kd, vd, idx)
    dq, dk, dv = ops.sparse_attn_bwd(qd, kd, vd, o, lse, dOd, idx)
    torch.cuda.synchronize()
    errs = []
    for got, ref in ((dq, dq_r), (dk, dk_r), (dv, dv_r)):
        g = got.float().cpu().numpy().astype(np.float64)
        assert np.isfinite(g).all()
        errs.append(normwise_err(g, ref, 1))
    assert max(errs) <= TOL, errs
    return errs


def test_bwd_c1_generator_index(cuda_lib):
    S, Hq, Hkv = 4096, 8, 1
    q, k, v = make_qkv(S, Hq, Hkv, seed=21)
    dO = make_grad_out(S, Hq, seed=21)
    iv, is_ = vsidx.build_vs_index(bf16_bits_to_f32(q), bf16_bits_to_f32(k), 0.9, 0.9)
    _check(q, k, v, dO, iv, is_)


def test_bwd_full_budget_dense_causal(cuda_lib):
    S, Hq, Hkv = 1024, 2, 1
    q, k, v = make_qkv(S, Hq, Hkv, seed=22, a=4.0)
    dO = make_grad_out(S, Hq, seed=22)
    _check(q, k, v, dO, [np.arange(S, dtype=np.int32)] * Hq, [np.arange(S // 64, dtype=np.int32)] * Hq)


@pytest.mark.parametrize("S", [2112, 4096])
def test_bwd_random_index_many_bars_gqa(cuda_lib, S):
    Hq, Hkv = 4, 2
    q, k, v = make_qkv(S, Hq, Hkv, seed=23, a=6.0)
    dO = make_grad_out(S, Hq, seed=23)
    iv, is_ = random_index(S, Hq, 24, n_off=5, n_col=300)
    _check(q, k, v, dO, iv, is_)


@pytest.mark.parametrize("layout", ["striped", "zigzag"])
@pytest.mark.parametrize("W", [2, 4, 8])
def test_bwd_ring_steps_emulated(cuda_lib, W, layout):
    """Every (rank, step) of the backward ring on one GPU vs the oracle ring backward
    (block-striped, and the zigzag layout of the f1 ablation)."""
    S, Hq, Hkv = 2048, 4, 2
    q, k, v = make_qkv(S, Hq, Hkv, seed=25, a=6.0)
    dO = make_grad_out(S, Hq, seed=25)
    iv, is_ = random_index(S, Hq, 26, n_off=6, n_col=80)
    qf, kf, vf, dOf = f64(q), f64(k), f64(v), f64(dO)
    O_ref, L_ref = OA.sparse_attention_forward(qf, kf, vf, iv, is_)
    ref = OR.ring_backward(qf, kf, vf, O_ref, L_ref, dOf, iv, is_, W, layout=layout)
    idx = ops.VSIndex.from_lists(iv, is_, S)
    # forward on one GPU (global order), then stripe O/LSE to ranks
    o, lse = ops.sparse_attn_fwd(to_dev_bf16(q), to_dev_bf16(k), to_dev_bf16(v), idx)
    perm = layout_perm(S, W, layout)
    pt = [torch.from_numpy(perm[r]).cuda() for r in range(W)]
    Lq = S // W
    loc = lambda x, r: x[pt[r]].contiguous()
    qd, kd, vd, dOd = (to_dev_bf16(x) for x in (q, k, v, dO))
    D = [torch.empty(Hq, Lq, dtype=torch.float32, device="cuda") for _ in range(W)]
    dq = [torch.zeros(Lq, Hq, 128, dtype=torch.float32, device="cuda") for _ in range(W)]
    dk = [torch.zeros(Lq, Hkv, 128, dtype=torch.float32, device="cuda") for _ in range(W)]
    dv = [torch.zeros(Lq, Hkv, 128, dtype=torch.float32, device="cuda") for _ in range(W)]
    for r in range(W):
        ops.attn_bwd_preprocess(S, W, loc(o, r), loc(dOd, r), D[r], layout=layout)
    sched = OR.schedule(W)
    for held in sched:
        for r in range(W):
            s = held[r]
            # the chunk's dK/dV accumulate directly at its owner (same sums as travelling)
            ops.attn_bwd_step(S, W, r, s, loc(qd, r), loc(kd, s), loc(vd, s), loc(dOd, r),
                              lse[:, pt[r]].contiguous(), D[r], idx, dq[r], dk[s], dv[s],
                              layout=layout)
    torch.cuda.synchronize()
    out = [np.zeros((S, Hq, 128)), np.zeros((S, Hkv, 128)), np.zeros((S, Hkv, 128))]
    for r in range(W):
        out[0][perm[r]] = dq[r].cpu().numpy()
        out[1][perm[r]] = dk[r].cpu().numpy()
        out[2][perm[r]] = dv[r].cpu().numpy()
    for got, rf in zip(out, ref):
        assert normwise_err(got, rf, 1) <= TOL
