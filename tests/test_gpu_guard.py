"""Out-of-bounds and uninitialised-read checks for the C ABI calls (index, forward, backward).

compute-sanitizer is closed on the GPU pool, so this is the substitute: every device buffer a call
touches (inputs, outputs, index arrays, workspace) is a view into a larger allocation whose guard
regions before and after are filled with 0xFF bytes, and outputs and workspace start as 0xFF too
(NaN in bf16 / fp32). After the call:
- every guard byte is still 0xFF (no write outside the buffer the header declares, include/mtsa.h);
- the inputs are unchanged (const pointers are not written);
- the outputs hold no NaN (every element written, and nothing read from unwritten workspace or output);
- the results equal the same call on ordinary buffers (the index bit for bit; attention to 1e-2 of the
  tensor's max, since the dQ reduce-add and the dynamic tile order do not fix the fp32 summation order).
Sizes: an odd block count (S = 37 x 64) and the C1 shape, with GQA.
"""
import ctypes

import numpy as np
import pytest
import torch

from paper_2510_18830_b200 import _lib, ops
from synth.generator import make_grad_out, make_qkv
from tests.gpu_util import random_index, to_dev_bf16

pytestmark = pytest.mark.gpu

G = 1 << 16  # guard bytes on each side (keeps the 1 KiB / 16 B alignment TMA and the kernels expect)


class Guarded:
    """A tensor view at byte offset G inside a 0xFF-filled allocation of nbytes + 2 G."""

    def __init__(self, shape, dtype, src: torch.Tensor | None = None):
        n = int(np.prod(shape)) * torch.empty((), dtype=dtype).element_size()
        self.n = n
        self.base = torch.full((n + 2 * G,), 0xFF, dtype=torch.uint8, device="cuda")
        self.t = self.base[G:G + n].view(dtype).view(*shape)
        if src is not None:
            self.t.copy_(src)
        self.before = src.clone() if src is not None else None

    def guards_intact(self) -> bool:
        return bool((self.base[:G] == 0xFF).all()) and bool((self.base[G + self.n:] == 0xFF).all())


def _case(S, Hq, Hkv, seed):
    q, k, v = make_qkv(S, Hq, Hkv, seed=seed)
    dO = make_grad_out(S, Hq, seed=seed + 1)
    return tuple(to_dev_bf16(x) for x in (q, k, v, dO))


def _guarded_index(S, Hq, src: ops.VSIndex | None = None):
    nb = S // ops.BLOCK
    parts = [Guarded((Hq,), torch.int32, None if src is None else src.v_cnt),
             Guarded((Hq, S), torch.int32, None if src is None else src.v_idx),
             Guarded((Hq,), torch.int32, None if src is None else src.s_cnt),
             Guarded((Hq, nb), torch.int32, None if src is None else src.s_off)]
    return parts, ops.VSIndex(*(p.t for p in parts))


def _close(name, got, want):
    err = (got.float() - want.float()).abs().max().item()
    assert err <= 1e-2 * want.float().abs().max().item(), (name, err)


def _check_all(bufs):
    for name, b in bufs.items():
        assert b.guards_intact(), f"write outside {name}"
        if b.before is not None:
            same = torch.equal(b.t.reshape(-1).view(torch.uint8), b.before.reshape(-1).view(torch.uint8))
            assert same, f"input {name} modified"  # bytewise: random bf16 bit patterns include NaN


@pytest.mark.parametrize("S,Hq,Hkv", [(37 * 64, 8, 1), (4096, 16, 2)])
def test_guarded_index(cuda_lib, S, Hq, Hkv):
    q, k, _, _ = _case(S, Hq, Hkv, seed=3)
    ref = ops.build_vs_index(q, k, 0.9, 0.9)
    sh = ops.shape(S, Hq, Hkv)
    L = _lib.lib()
    nws = L.mt_build_vs_index_workspace_bytes(ctypes.byref(sh), 1)
    bufs = {"q": Guarded(q.shape, q.dtype, q), "k": Guarded(k.shape, k.dtype, k),
            "ws": Guarded((nws,), torch.uint8)}
    parts, idx = _guarded_index(S, Hq)
    bufs.update({f"idx{i}": p for i, p in enumerate(parts)})
    prm = ops.VSParams(0.9, 0.9)
    ci = idx.c_struct()
    _lib.check(L.mt_build_vs_index(None, ctypes.byref(sh), ctypes.byref(prm), bufs["q"].t.data_ptr(),
                                   bufs["k"].t.data_ptr(), ctypes.byref(ci), bufs["ws"].t.data_ptr(), nws,
                                   ops._stream()))
    torch.cuda.synchronize()
    _check_all(bufs)
    a, b = idx.to_lists(), ref.to_lists()
    for h in range(Hq):
        assert np.array_equal(a[0][h], b[0][h]) and np.array_equal(a[1][h], b[1][h]), h


@pytest.mark.parametrize("S,Hq,Hkv,gen", [(37 * 64, 8, 1, True), (4096, 16, 2, False)])
def test_guarded_fwd_bwd(cuda_lib, S, Hq, Hkv, gen):
    q, k, v, dO = _case(S, Hq, Hkv, seed=5)
    if gen:
        ref_idx = ops.build_vs_index(q, k, 0.9, 0.9)
    else:  # many bars and offsets, GQA
        ref_idx = ops.VSIndex.from_lists(*random_index(S, Hq, seed=9, n_off=12, n_col=300), S)
    o_ref, lse_ref = ops.sparse_attn_fwd(q, k, v, ref_idx)
    g_ref = ops.sparse_attn_bwd(q, k, v, o_ref, lse_ref, dO, ref_idx)
    torch.cuda.synchronize()

    sh = ops.shape(S, Hq, Hkv)
    L = _lib.lib()
    parts, idx = _guarded_index(S, Hq, ref_idx)
    ci = idx.c_struct()
    ins = {n: Guarded(x.shape, x.dtype, x) for n, x in (("q", q), ("k", k), ("v", v), ("dO", dO))}
    nf = L.mt_sparse_attn_fwd_workspace_bytes(ctypes.byref(sh), 1)
    fw = {"o": Guarded(q.shape, q.dtype), "lse": Guarded((Hq, S), torch.float32),
          "ws_fwd": Guarded((nf,), torch.uint8)}
    p = lambda b: b.t.data_ptr()
    _lib.check(L.mt_sparse_attn_fwd(ctypes.byref(sh), p(ins["q"]), p(ins["k"]), p(ins["v"]), ctypes.byref(ci),
                                    p(fw["o"]), p(fw["lse"]), p(fw["ws_fwd"]), nf, ops._stream()))
    torch.cuda.synchronize()
    assert not torch.isnan(fw["o"].t.float()).any() and not torch.isnan(fw["lse"].t).any()
    _close("o", fw["o"].t, o_ref)
    assert (fw["lse"].t - lse_ref).abs().max().item() <= 1e-4

    # the backward reads O / LSE from guarded buffers of their own
    o_in, lse_in = Guarded(q.shape, q.dtype, fw["o"].t), Guarded((Hq, S), torch.float32, fw["lse"].t)
    nb_ = L.mt_sparse_attn_bwd_workspace_bytes(ctypes.byref(sh))
    bw = {"dq": Guarded(q.shape, q.dtype), "dk": Guarded(k.shape, k.dtype), "dv": Guarded(v.shape, v.dtype),
          "ws_bwd": Guarded((nb_,), torch.uint8)}
    _lib.check(L.mt_sparse_attn_bwd(ctypes.byref(sh), p(ins["q"]), p(ins["k"]), p(ins["v"]), p(o_in), p(lse_in),
                                    p(ins["dO"]), ctypes.byref(ci), p(bw["dq"]), p(bw["dk"]), p(bw["dv"]),
                                    p(bw["ws_bwd"]), nb_, ops._stream()))
    torch.cuda.synchronize()
    _check_all({**ins, **fw, **bw, "o_in": o_in, "lse_in": lse_in,
                **{f"idx{i}": b for i, b in enumerate(parts)}})
    for name, got, want in zip(("dq", "dk", "dv"), (bw["dq"].t, bw["dk"].t, bw["dv"].t), g_ref):
        assert not torch.isnan(got.float()).any(), name
        _close(name, got, want)


def test_guarded_ring_steps(cuda_lib, monkeypatch):
    """Every (rank, step) of a W = 4 ring emulated on one GPU (mt_attn_fwd_step, mt_attn_bwd_preprocess,
    mt_attn_bwd_step), 9 local blocks per rank, with every buffer and each call's workspace guarded."""
    from oracle.ring import schedule
    from oracle.sparseformat import stripe_perm

    W, S, Hq, Hkv = 4, 4 * 9 * 64, 4, 2
    Lq = S // W
    q, k, v, dO = _case(S, Hq, Hkv, seed=11)
    idx = ops.VSIndex.from_lists(*random_index(S, Hq, seed=12, n_off=6, n_col=80), S)
    wss = []

    def guarded_ws(nbytes, device=None):
        wss.append(Guarded((max(nbytes, 1),), torch.uint8))
        return wss[-1].t

    perm = stripe_perm(S, W)
    pt = [torch.from_numpy(perm[r]).cuda() for r in range(W)]
    sched = schedule(W)

    def run(guard):
        mk = (lambda shape, dt, src=None: Guarded(shape, dt, src)) if guard else \
             (lambda shape, dt, src=None: type("T", (), {"t": src.clone() if src is not None else
                                                       torch.empty(shape, dtype=dt, device="cuda")})())
        loc = lambda x, r: mk(x[pt[r]].shape, x.dtype, x[pt[r]].contiguous())
        bufs = {}
        for n, x in (("q", q), ("k", k), ("v", v), ("dO", dO)):
            for r in range(W):
                bufs[f"{n}{r}"] = loc(x, r)
        for r in range(W):
            bufs[f"o{r}"] = mk((Lq, Hq, 128), torch.bfloat16)
            bufs[f"oacc{r}"] = mk((Lq, Hq, 128), torch.float32)
            bufs[f"lse{r}"] = mk((Hq, Lq), torch.float32)
            bufs[f"D{r}"] = mk((Hq, Lq), torch.float32)
            for n, h in (("dq", Hq), ("dk", Hkv), ("dv", Hkv)):
                bufs[f"{n}{r}"] = mk((Lq, h, 128), torch.float32, torch.zeros(Lq, h, 128, device="cuda"))
        B = lambda n: bufs[n].t
        for t, held in enumerate(sched):
            for r in range(W):
                s = held[r]
                ops.attn_fwd_step(S, W, r, s, t == 0, t == W - 1, B(f"q{r}"), B(f"k{s}"), B(f"v{s}"), idx,
                                  B(f"o{r}"), B(f"oacc{r}"), B(f"lse{r}"))
        for r in range(W):
            ops.attn_bwd_preprocess(S, W, B(f"o{r}"), B(f"dO{r}"), B(f"D{r}"))
        for held in sched:
            for r in range(W):
                s = held[r]
                ops.attn_bwd_step(S, W, r, s, B(f"q{r}"), B(f"k{s}"), B(f"v{s}"), B(f"dO{r}"), B(f"lse{r}"),
                                  B(f"D{r}"), idx, B(f"dq{r}"), B(f"dk{s}"), B(f"dv{s}"))
        torch.cuda.synchronize()
        return bufs

    ref = run(False)
    monkeypatch.setattr(ops, "workspace", guarded_ws)
    got = run(True)
    assert wss
    for i, w in enumerate(wss):
        assert w.guards_intact(), f"write outside workspace {i}"
    for n, b in got.items():
        assert b.guards_intact(), f"write outside {n}"
        if n[:1] in "qkv" or n.startswith("dO"):
            if b.before is not None and not n.startswith(("dq", "dk", "dv")):
                assert torch.equal(b.t, b.before), f"input {n} modified"
        if n.startswith(("o", "lse", "D", "dq", "dk", "dv")) and not n.startswith("oacc"):
            assert not torch.isnan(b.t.float()).any(), n
            _close(n, b.t, ref[n].t)


def test_guarded_stripe_unstripe(cuda_lib):
    """a1: mt_stripe / mt_unstripe of every rank's share at W = 4, odd local block count."""
    W, S = 4, 4 * 9 * 64
    L = _lib.lib()
    x = torch.randint(-2 ** 15, 2 ** 15, (S, 2, 128), dtype=torch.int16, device="cuda").view(torch.bfloat16)
    row = x[0].numel() * x.element_size()
    src = Guarded(x.shape, x.dtype, x)
    back = Guarded(x.shape, x.dtype)
    locs = []
    for r in range(W):
        loc = Guarded((S // W, 2, 128), x.dtype)
        _lib.check(L.mt_stripe(S, row, W, r, src.t.data_ptr(), loc.t.data_ptr(), ops._stream()))
        locs.append(loc)
    for r in range(W):
        _lib.check(L.mt_unstripe(S, row, W, r, locs[r].t.data_ptr(), back.t.data_ptr(), ops._stream()))
    torch.cuda.synchronize()
    _check_all({"src": src, "back": back, **{f"loc{r}": b for r, b in enumerate(locs)}})
    assert torch.equal(back.t.view(torch.int16), x.view(torch.int16))


def test_guarded_vs_format(cuda_lib):
    """a6: mt_vs_format_count / fill with the CSR arrays sized exactly to the counts."""
    S, Hq = 37 * 64, 8
    nb = S // 64
    idx = ops.VSIndex.from_lists(*random_index(S, Hq, seed=14, n_off=7, n_col=120), S)
    ref = ops.vs_format(idx, S)
    torch.cuda.synchronize()
    sh = ops.shape(S, Hq, 1)
    L = _lib.lib()
    nws = L.mt_vs_format_workspace_bytes(ctypes.byref(sh))
    parts, gidx = _guarded_index(S, Hq, idx)
    ci = gidx.c_struct()
    bp, cp, ws = Guarded((Hq, nb + 1), torch.int64), Guarded((Hq, nb + 1), torch.int64), Guarded((nws,), torch.uint8)
    nbk, ncl = ctypes.c_int64(), ctypes.c_int64()
    _lib.check(L.mt_vs_format_count(ctypes.byref(sh), ctypes.byref(ci), bp.t.data_ptr(), cp.t.data_ptr(),
                                    ctypes.byref(nbk), ctypes.byref(ncl), ws.t.data_ptr(), nws, ops._stream()))
    assert nbk.value == ref[1].numel() and ncl.value == ref[3].numel()
    bi, cl = Guarded((nbk.value,), torch.int32), Guarded((ncl.value,), torch.int32)
    _lib.check(L.mt_vs_format_fill(ctypes.byref(sh), ctypes.byref(ci), bp.t.data_ptr(), cp.t.data_ptr(),
                                   bi.t.data_ptr(), nbk.value, cl.t.data_ptr(), ncl.value, nbk.value, ncl.value,
                                   ws.t.data_ptr(), nws, ops._stream()))
    torch.cuda.synchronize()
    _check_all({"bp": bp, "cp": cp, "ws": ws, "bi": bi, "cl": cl, **{f"idx{i}": b for i, b in enumerate(parts)}})
    for got, want in zip((bp.t, bi.t, cp.t, cl.t), ref):
        assert torch.equal(got, want)


@pytest.mark.parametrize("S", [524288, 1048576])
def test_guarded_fullsize(cuda_lib, S):
    """The bench configuration (C4 512K, and C5's 1M on one GPU): index, forward and backward with every
    buffer and workspace guarded, against the same calls on ordinary buffers (large-offset arithmetic)."""
    Hq, Hkv = 16, 2
    q, k, v, dO = _case(S, Hq, Hkv, seed=0)
    idx_ref = ops.build_vs_index(q, k, 0.9, 0.9)
    o_ref, lse_ref = ops.sparse_attn_fwd(q, k, v, idx_ref)
    g_ref = ops.sparse_attn_bwd(q, k, v, o_ref, lse_ref, dO, idx_ref)
    torch.cuda.synchronize()
    ins = {n: Guarded(x.shape, x.dtype, x) for n, x in (("q", q), ("k", k), ("v", v), ("dO", dO))}
    del q, k, v, dO
    wss = []
    ws_plain = ops.workspace

    def guarded_ws(nbytes, device=None):
        wss.append(Guarded((max(nbytes, 1),), torch.uint8))
        return wss[-1].t

    ops.workspace = guarded_ws
    try:
        idx = ops.build_vs_index(ins["q"].t, ins["k"].t, 0.9, 0.9)
        o, lse = ops.sparse_attn_fwd(ins["q"].t, ins["k"].t, ins["v"].t, idx)
        g = ops.sparse_attn_bwd(ins["q"].t, ins["k"].t, ins["v"].t, o, lse, ins["dO"].t, idx)
        torch.cuda.synchronize()
    finally:
        ops.workspace = ws_plain
    _check_all({**ins, **{f"ws{i}": w for i, w in enumerate(wss)}})
    # entries past each count are unspecified (VSIndex.uninit): compare the lists
    for a, b in zip(idx.to_lists(), idx_ref.to_lists()):
        assert len(a) == len(b) and all(np.array_equal(x, y) for x, y in zip(a, b))
    _close("o", o, o_ref)
    assert (lse - lse_ref).abs().max().item() <= 1e-4
    for name, got, want in zip(("dq", "dk", "dv"), g, g_ref):
        assert not torch.isnan(got.float()).any(), name
        _close(name, got, want)
