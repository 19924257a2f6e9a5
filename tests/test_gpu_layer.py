"""The decoder layer (paper_2510_18830_b200/layer.py) forward and
backward on the GPU vs the fp64 oracle composite oracle/layer.py (itself pinned by
finite differences in test_oracle_layer.py), same bf16 weights / inputs and the
same explicit index (held fixed).

Tolerance: the GPU rounds to bf16 at every stage boundary (~2^-9 each, about ten
stages) — normwise per tensor (reading R20's form) <= 2e-2, the north_star bound;
the output is compared as the layer's increment y - x, so the residual does not
hide errors."""
import numpy as np
import pytest
import torch

from oracle import layer as OL
from oracle import rope as R
from paper_2510_18830_b200.layer import VSDecoderLayer
from synth.generator import bf16_bits_to_f32, f32_to_bf16_bits
from tests.gpu_util import random_index

pytestmark = pytest.mark.gpu
TOL = 2e-2
S, D, HQ, HKV, I = 2048, 256, 4, 2, 512


def _bf(a):
    """fp32 array -> (exact fp64 of its bf16 rounding, bf16 torch tensor on cuda)."""
    bits = f32_to_bf16_bits(a)
    t = torch.from_numpy(bits.view(np.int16)).view(torch.bfloat16).cuda()
    return bf16_bits_to_f32(bits).astype(np.float64), t


def _nerr(got, ref):
    return float(np.max(np.abs(got - ref)) / np.max(np.abs(ref)))


@pytest.mark.parametrize("yarn", [1.0, 32.0])
def test_layer_forward_backward_matches_oracle(cuda_lib, yarn):
    rng = np.random.default_rng(7)
    layer = VSDecoderLayer(hidden=D, n_q_heads=HQ, n_kv_heads=HKV, intermediate=I,
                           yarn_factor=yarn)
    shapes = dict(w1=(D,), Wqkv=((HQ + 2 * HKV) * 128, D), bqkv=((HQ + 2 * HKV) * 128,),
                  Wo=(D, HQ * 128), w2=(D,), Wg=(I, D), Wu=(I, D), Wd=(D, I))
    mods = dict(w1=layer.ln1.weight, Wqkv=layer.qkv.weight, bqkv=layer.qkv.bias,
                Wo=layer.o_proj.weight, w2=layer.ln2.weight, Wg=layer.gate.weight,
                Wu=layer.up.weight, Wd=layer.down.weight)
    P = {}
    for n, shp in shapes.items():
        if n in ("w1", "w2"):
            a = 1.0 + 0.1 * rng.standard_normal(shp)
        elif n == "bqkv":
            a = 0.1 * rng.standard_normal(shp)
        else:
            a = rng.standard_normal(shp) / np.sqrt(shp[1])
        P[n], t = _bf(a.astype(np.float32))
        with torch.no_grad():
            mods[n].copy_(t)
    x64, x = _bf(rng.standard_normal((S, D)).astype(np.float32))
    dy64, dy = _bf(rng.standard_normal((S, D)).astype(np.float32))
    iv, is_ = random_index(S, HQ, seed=3, n_off=6, n_col=150)
    from paper_2510_18830_b200 import ops
    idx = ops.VSIndex.from_lists(iv, is_, S)

    x.requires_grad_(True)
    y = layer(x, index=idx)
    y.backward(dy)
    torch.cuda.synchronize()

    th, ms = R.inv_freq(128, 1e6, yarn, 32768)
    args = (np.arange(S), th, ms, iv, is_, HQ, HKV, 128)
    y_ref, cache = OL.forward(x64, P, *args)
    dx_ref, G = OL.backward(dy64, P, cache, *args)

    errs = {"y-x": _nerr(y.detach().double().cpu().numpy() - x64, y_ref - x64),
            "dx": _nerr(x.grad.double().cpu().numpy(), dx_ref)}
    for n, p in mods.items():
        errs[n] = _nerr(p.grad.double().cpu().numpy(), G[n])
    assert max(errs.values()) <= TOL, errs


def test_layer_builds_its_own_index(cuda_lib):
    """Without an explicit index the layer runs Alg. 1 on its post-RoPE q/k
    and the result is a valid index: forced members present, lists sorted, unique."""
    layer = VSDecoderLayer(hidden=D, n_q_heads=HQ, n_kv_heads=HKV, intermediate=I)
    x = torch.randn(S, D, device="cuda", dtype=torch.bfloat16, requires_grad=True)
    y = layer(x)
    y.float().square().sum().backward()
    torch.cuda.synchronize()
    assert torch.isfinite(y).all() and torch.isfinite(x.grad).all()
    iv, is_ = layer.last_index.to_lists()
    for h in range(HQ):
        assert iv[h][0] == 0 and is_[h][0] == 0
        assert np.all(np.diff(iv[h]) > 0) and np.all(np.diff(is_[h]) > 0)
        assert iv[h][-1] < S and is_[h][-1] < S // 64
