"""Degenerate shapes and indexes through the C ABI vs the fp64 oracle (③: the empty, the
smallest and the degenerate cases of the method).

* one 64-token block (S = 64): a single query block, a single key pair slot, the window is
  the whole sequence;
* the minimal index (column 0 and offset 0 only, reading R7) at several lengths;
* index budgets at the extremes: p -> 0 (only the forced members plus the first top item)
  and p = 1 (dense causal, reading R22), built by the GPU and compared with the oracle's lists;
* a 2-rank ring with one local block per rank, every (rank, step) on one GPU.
Tolerances as everywhere (reading R20): normwise 2e-2 per (tensor, head), LSE 1e-3.
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
from tests.gpu_util import f64, normwise_err, to_dev_bf16

pytestmark = pytest.mark.gpu
TOL, TOL_LSE = 2e-2, 1e-3


def _fwd_bwd(q, k, v, dO, iv, is_):
    S = q.shape[0]
    O, L = OA.sparse_attention_forward(f64(q), f64(k), f64(v), iv, is_)
    ref = OA.sparse_attention_backward(f64(q), f64(k), f64(v), O, L, f64(dO), iv, is_)
    idx = ops.VSIndex.from_lists(iv, is_, S)
    qd, kd, vd, dd = (to_dev_bf16(x) for x in (q, k, v, dO))
    o, lse = ops.sparse_attn_fwd(qd, kd, vd, idx)
    g = ops.sparse_attn_bwd(qd, kd, vd, o, lse, dd, idx)
    torch.cuda.synchronize()
    cpu = lambda t: t.float().cpu().numpy().astype(np.float64)
    assert normwise_err(cpu(o), O, 1) <= TOL
    assert np.max(np.abs(lse.cpu().numpy() - L)) <= TOL_LSE
    for got, want in zip(g, ref):
        assert np.isfinite(cpu(got)).all()
        assert normwise_err(cpu(got), want, 1) <= TOL


def test_single_block_sequence(cuda_lib):
    S, Hq, Hkv = 64, 2, 1
    q, k, v = make_qkv(S, Hq, Hkv, seed=91, a=6.0)
    dO = make_grad_out(S, Hq, seed=91)
    # the GPU index of a one-block sequence is the forced members plus what top-p keeps
    idx = ops.build_vs_index(to_dev_bf16(q), to_dev_bf16(k), 0.9, 0.9)
    torch.cuda.synchronize()
    iv, is_ = idx.to_lists()
    riv, ris = vsidx.build_vs_index(bf16_bits_to_f32(q), bf16_bits_to_f32(k), 0.9, 0.9)
    for h in range(Hq):
        assert np.array_equal(iv[h], riv[h]) and np.array_equal(is_[h], ris[h])
        assert list(is_[h]) == [0]
    _fwd_bwd(q, k, v, dO, riv, ris)


@pytest.mark.parametrize("S", [128, 1088, 4096])
def test_minimal_index(cuda_lib, S):
    Hq, Hkv = 4, 2
    q, k, v = make_qkv(S, Hq, Hkv, seed=S + 92, a=6.0)
    dO = make_grad_out(S, Hq, seed=S + 92)
    _fwd_bwd(q, k, v, dO, [np.array([0], np.int32)] * Hq, [np.array([0], np.int32)] * Hq)


@pytest.mark.parametrize("p", [1e-6, 1.0])
def test_budget_extremes_index_bitexact(cuda_lib, p):
    S, Hq, Hkv = 2048, 4, 1
    q, k, _ = make_qkv(S, Hq, Hkv, seed=93)
    idx = ops.build_vs_index(to_dev_bf16(q), to_dev_bf16(k), p, p)
    torch.cuda.synchronize()
    iv, is_ = idx.to_lists()
    riv, ris = vsidx.build_vs_index(bf16_bits_to_f32(q), bf16_bits_to_f32(k), p, p)
    for h in range(Hq):
        assert np.array_equal(iv[h], riv[h]) and np.array_equal(is_[h], ris[h])
        if p == 1.0:
            assert len(iv[h]) == S and len(is_[h]) == S // 64
        else:  # forced members and the single top item of each list at most
            assert 1 <= len(iv[h]) <= 2 and 1 <= len(is_[h]) <= 2 and iv[h][0] == 0 and is_[h][0] == 0


@pytest.mark.parametrize("layout", ["striped", "zigzag"])
def test_ring_one_block_per_rank(cuda_lib, layout):
    # W = 2 and S = 128 (striped) / 256 (zigzag: two 64-token chunks per rank): nloc = 1 / 2
    W, Hq, Hkv = 2, 2, 1
    S = 128 if layout == "striped" else 256
    q, k, v = make_qkv(S, Hq, Hkv, seed=94, a=6.0)
    iv = [np.array([0, 5, 70], np.int32), np.array([0, 33], np.int32)]
    is_ = [np.arange(S // 64, dtype=np.int32), np.array([0], np.int32)]
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
            ops.attn_fwd_step(S, W, r, s, t == 0, t == W - 1, qd[r], kd[s], vd[s], idx, o[r], oacc[r],
                              lse[r], layout=layout)
    torch.cuda.synchronize()
    Og = np.zeros((S, Hq, 128))
    Lg = np.zeros((Hq, S))
    for r in range(W):
        Og[perm[r]] = o[r].float().cpu().numpy()
        Lg[:, perm[r]] = lse[r].cpu().numpy()
    assert normwise_err(Og, O_ref, 1) <= TOL
    assert np.max(np.abs(Lg - L_ref)) <= TOL_LSE
