"""Full-size parity (512K tokens, 16 q / 2 kv heads, p = 0.9: BASELINE config C4 at W = 1),
in the launch configuration `bench.py` times (single GPU, C ABI via ops), on outputs the
fp64 oracle can compute one by one:

* index lists of all 16 q heads, bit-exact (VS-IDX v1); the ORACLE's lists
  then drive both the GPU attention (uploaded through the C ABI) and the fp64 oracle, so
  no oracle input comes from the GPU;
* O and LSE of sampled query blocks (first, window = last, random);
* dQ of the same blocks;
* dK / dV of late key blocks, whose attending query blocks are few enough for the
  oracle to enumerate (all q heads of the group, the oracle's own O/LSE).

Tolerance: north_star's 2e-2, normwise per (tensor, head) over the sampled rows (R20).
No expected value comes from the GPU: the oracle recomputes everything it compares.
"""
import numpy as np
import pytest
import torch

from oracle import attention as OA
from oracle import vsidx
from oracle.sparseformat import sparseformat_block
from paper_2510_18830_b200 import ops
from synth.generator import bf16_bits_to_f32, make_grad_out, make_qkv
from tests.gpu_util import to_dev_bf16

pytestmark = pytest.mark.gpu
TOL = 2e-2
S, HQ, HKV, P = 524288, 16, 2, 0.9
NB = S // 64
GRP = HQ // HKV


def nerr(got, ref):
    """R20 normwise error of one (tensor, head) sample: max|x - ref| / max|ref|."""
    return float(np.max(np.abs(got - ref)) / np.max(np.abs(ref)))


class Lazy64:
    """bf16 bit array read as exact fp64 slice by slice (the oracle indexes
    q[rows, h, :] and k[keys, g, :]; a dense fp64 copy of 512K x 16 x 128 is 8.6 GB)."""

    def __init__(self, bits):
        self.bits, self.shape = bits, bits.shape

    def __getitem__(self, key):
        return bf16_bits_to_f32(self.bits[key]).astype(np.float64)


class Rows:
    """Stand-in for the oracle's O [S][Hq][d] / LSE [Hq][S] holding only the query
    blocks the test computed (indexed by (block slice, head) or (head, block slice))."""

    def __init__(self, lse=False):
        self.lse, self.d = lse, {}

    def _k(self, key):
        h, rows = (key[0], key[1]) if self.lse else (key[1], key[0])
        return rows.start, h

    def __getitem__(self, key):
        return self.d[self._k(key)]

    def __setitem__(self, key, val):
        self.d[self._k(key)] = np.array(val)


@pytest.fixture(scope="module")
def run(cuda_lib):
    q, k, v = make_qkv(S, HQ, HKV, seed=0)       # the bench's inputs
    dO = make_grad_out(S, HQ, seed=0)
    qd, kd, vd, dd = (to_dev_bf16(x) for x in (q, k, v, dO))
    gpu_iv, gpu_is = ops.build_vs_index(qd, kd, P, P).to_lists()
    iv, is_ = vsidx.build_vs_index(bf16_bits_to_f32(q), bf16_bits_to_f32(k), P, P)
    idx = ops.VSIndex.from_lists(iv, is_, S)
    o, lse = ops.sparse_attn_fwd(qd, kd, vd, idx)
    dq, dk, dv = ops.sparse_attn_bwd(qd, kd, vd, o, lse, dd, idx)
    torch.cuda.synchronize()
    qf, kf, vf, dOf = (Lazy64(x) for x in (q, k, v, dO))
    return dict(q=q, k=k, qf=qf, kf=kf, vf=vf, dOf=dOf, iv=iv, is_=is_, gpu_iv=gpu_iv, gpu_is=gpu_is,
                o=o.float().cpu().numpy(), lse=lse.cpu().numpy(),
                dq=dq.float().cpu().numpy(), dk=dk.float().cpu().numpy(),
                dv=dv.float().cpu().numpy())


def test_index_lists_bitexact_at_512k(run):
    for h in range(HQ):  # every q head: GPU Alg. 1 == oracle Alg. 1, bitwise
        assert np.array_equal(np.asarray(run["gpu_iv"][h]), np.asarray(run["iv"][h])), h
        assert np.array_equal(np.asarray(run["gpu_is"][h]), np.asarray(run["is_"][h])), h


def _blocks():
    rng = np.random.default_rng(1)
    return sorted({0, 1, NB // 2, NB - 1, *rng.choice(NB, 4, replace=False).tolist()})


@pytest.mark.parametrize("h", [0, 5, GRP, HQ - 1])
def test_forward_and_dq_sampled_query_blocks(run, h):
    r = run
    O_ref, L_ref = Rows(), Rows(lse=True)
    got_o, ref_o, got_l, ref_l, got_dq, ref_dq = [], [], [], [], [], []
    for g in _blocks():
        B, C = sparseformat_block(r["iv"][h], r["is_"][h], g)
        rows = slice(g * 64, g * 64 + 64)
        O_ref[rows, h], L_ref[h, rows] = OA.forward_block(r["qf"], r["kf"], r["vf"], h, g, B, C)
        dq, _, _, _ = OA.backward_block(r["qf"], r["kf"], r["vf"], O_ref, L_ref, r["dOf"], h, g, B, C)
        got_o.append(r["o"][rows, h]); ref_o.append(O_ref[rows, h])
        got_l.append(r["lse"][h, rows]); ref_l.append(L_ref[h, rows])
        got_dq.append(r["dq"][rows, h]); ref_dq.append(dq)
    assert nerr(np.concatenate(got_o), np.concatenate(ref_o)) <= TOL
    assert np.max(np.abs(np.concatenate(got_l) - np.concatenate(ref_l))) <= 1e-3
    assert nerr(np.concatenate(got_dq), np.concatenate(ref_dq)) <= TOL


@pytest.mark.parametrize("g_kv", [0, 1])
def test_dk_dv_late_key_blocks(run, g_kv):
    """dK/dV of the last key blocks: attended only by query blocks kb + o < nb (few
    offsets) and by nothing else when the block holds no selected vertical column."""
    r = run
    heads = range(g_kv * GRP, (g_kv + 1) * GRP)
    cand = [kb for kb in range(NB - 24, NB)
            if not any(((np.asarray(r["iv"][h]) // 64) == kb).any() for h in heads)][:3]
    assert cand, "no vertical-free late key block to sample"
    got_k, ref_k, got_v, ref_v = [], [], [], []
    for kb in cand:
        dk = np.zeros((64, 128))
        dv = np.zeros((64, 128))
        for h in heads:
            offs = np.asarray(r["is_"][h])
            O_ref, L_ref = Rows(), Rows(lse=True)
            for o in offs[(offs >= 0) & (kb + offs < NB)]:
                g = kb + int(o)
                B, C = sparseformat_block(r["iv"][h], r["is_"][h], g)
                rows = slice(g * 64, g * 64 + 64)
                O_ref[rows, h], L_ref[h, rows] = OA.forward_block(r["qf"], r["kf"], r["vf"], h, g, B, C)
                _, keys, dkb, dvb = OA.backward_block(r["qf"], r["kf"], r["vf"], O_ref, L_ref,
                                                      r["dOf"], h, g, B, C)
                sel = (keys >= kb * 64) & (keys < kb * 64 + 64)
                dk[keys[sel] - kb * 64] += dkb[sel]
                dv[keys[sel] - kb * 64] += dvb[sel]
        got_k.append(r["dk"][kb * 64: kb * 64 + 64, g_kv]); ref_k.append(dk)
        got_v.append(r["dv"][kb * 64: kb * 64 + 64, g_kv]); ref_v.append(dv)
    assert nerr(np.concatenate(got_k), np.concatenate(ref_k)) <= TOL
    assert nerr(np.concatenate(got_v), np.concatenate(ref_v)) <= TOL
