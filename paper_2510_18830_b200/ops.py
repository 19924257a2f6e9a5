"""Torch-facing wrappers over the C ABI (include/mtsa.h).

Argument marshalling only (pointers, sizes, the current CUDA stream); every
step of the hot path runs inside libmtsa.so.  Tensors must already live on the
GPU in the documented layouts; nothing here falls back to CPU code.
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib

BLOCK = 64
HEAD_DIM = 128


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("tensor must be on the GPU")
    if not t.is_contiguous():
        raise ValueError("tensor must be contiguous")
    return t.data_ptr()


LAYOUTS = {"striped": 0, "zigzag": 1}  # MT_LAYOUT_STRIPED / MT_LAYOUT_ZIGZAG (include/mtsa.h)


def shape(seq_len: int, n_q_heads: int, n_kv_heads: int, layout: str = "striped") -> _lib.Shape:
    return _lib.Shape(seq_len, n_q_heads, n_kv_heads, HEAD_DIM, BLOCK, BLOCK, LAYOUTS[layout])


@dataclass
class VSIndex:
    """Device-resident vertical-slash index (mt_vs_index)."""
    v_cnt: torch.Tensor   # [Hq] int32
    v_idx: torch.Tensor   # [Hq][v_stride] int32
    s_cnt: torch.Tensor   # [Hq] int32
    s_off: torch.Tensor   # [Hq][s_stride] int32

    @staticmethod
    def empty(seq_len: int, n_q_heads: int, device="cuda") -> "VSIndex":
        nb = seq_len // BLOCK
        z = lambda *s: torch.zeros(*s, dtype=torch.int32, device=device)
        return VSIndex(z(n_q_heads), z(n_q_heads, seq_len), z(n_q_heads), z(n_q_heads, nb))

    @staticmethod
    def uninit(seq_len: int, n_q_heads: int, device="cuda") -> "VSIndex":
        """Output buffers for mt_build_vs_index, which writes the counts and every entry
        below them (entries past a count are never read): no fill kernels."""
        nb = seq_len // BLOCK
        e = lambda *s: torch.empty(*s, dtype=torch.int32, device=device)
        return VSIndex(e(n_q_heads), e(n_q_heads, seq_len), e(n_q_heads), e(n_q_heads, nb))

    @staticmethod
    def from_lists(i_v, i_s, seq_len: int, device="cuda") -> "VSIndex":
        """Upload explicit per-head lists (e.g. a controlled-density pattern).

        The lists must be what Alg. 1 produces (include/mtsa.h, mt_vs_index): strictly
        ascending, columns in [0, seq_len), offsets in [0, seq_len/64), offset 0 present
        (reading R7: every query keeps its diagonal).  Violations raise ValueError here
        instead of producing unspecified attention results.
        """
        Hq = len(i_v)
        nb = seq_len // BLOCK
        for h in range(Hq):
            for name, x, hi in (("i_v", i_v[h], seq_len), ("i_s", i_s[h], nb)):
                x = [int(t) for t in x]
                if any(b <= a for a, b in zip(x, x[1:])):
                    raise ValueError(f"{name}[{h}] is not strictly ascending")
                if x and (x[0] < 0 or x[-1] >= hi):
                    raise ValueError(f"{name}[{h}] has entries outside [0, {hi})")
            if len(i_s[h]) == 0 or int(i_s[h][0]) != 0:
                raise ValueError(f"i_s[{h}] must contain offset 0 (the diagonal)")
        idx = VSIndex.empty(seq_len, Hq, device="cpu")
        for h in range(Hq):
            a, b = torch.as_tensor(i_v[h], dtype=torch.int32), torch.as_tensor(i_s[h], dtype=torch.int32)
            idx.v_cnt[h], idx.s_cnt[h] = a.numel(), b.numel()
            idx.v_idx[h, : a.numel()] = a
            idx.s_off[h, : b.numel()] = b
        return VSIndex(*(t.to(device) for t in (idx.v_cnt, idx.v_idx, idx.s_cnt, idx.s_off)))

    def to_lists(self):
        vc, vi, sc, so = (t.cpu() for t in (self.v_cnt, self.v_idx, self.s_cnt, self.s_off))
        iv = [vi[h, : int(vc[h])].numpy().copy() for h in range(vc.numel())]
        is_ = [so[h, : int(sc[h])].numpy().copy() for h in range(sc.numel())]
        return iv, is_

    def c_struct(self) -> "MTIndex":
        return MTIndex(_ptr(self.v_cnt), _ptr(self.v_idx), self.v_idx.shape[1],
                       _ptr(self.s_cnt), _ptr(self.s_off), self.s_off.shape[1])


class MTIndex(ctypes.Structure):
    _fields_ = [("v_cnt", ctypes.c_void_p), ("v_idx", ctypes.c_void_p), ("v_stride", ctypes.c_int64),
                ("s_cnt", ctypes.c_void_p), ("s_off", ctypes.c_void_p), ("s_stride", ctypes.c_int64)]


_WS: dict = {}


def workspace(nbytes: int, device=None) -> torch.Tensor:
    """Cached byte workspace on the current device (grown on demand)."""
    dev = torch.device("cuda", torch.cuda.current_device()) if device is None else torch.device(device)
    buf = _WS.get(dev)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=dev)
        _WS[dev] = buf
    return buf


def sparse_attn_fwd(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, idx: VSIndex):
    """Single-GPU VS sparse attention forward -> (o bf16 [S][Hq][128], lse f32 [Hq][S])."""
    S, Hq, _ = q.shape
    sh = shape(S, Hq, k.shape[1])
    L = _lib.lib()
    nbytes = L.mt_sparse_attn_fwd_workspace_bytes(ctypes.byref(sh), 1)
    ws = workspace(nbytes)
    o = torch.empty_like(q)
    lse = torch.empty(Hq, S, dtype=torch.float32, device=q.device)
    ci = idx.c_struct()
    _lib.check(L.mt_sparse_attn_fwd(ctypes.byref(sh), _ptr(q), _ptr(k), _ptr(v), ctypes.byref(ci),
                                    _ptr(o), _ptr(lse), _ptr(ws), ws.numel(), _stream()))
    return o, lse


def attn_fwd_step(seq_len: int, world: int, rank: int, origin: int, first: bool, last: bool,
                  q_loc, k_chunk, v_chunk, idx: VSIndex, o, o_acc, lse, layout: str = "striped"):
    """One ring step (mt_attn_fwd_step); tensors are rank-local (in `layout`)."""
    sh = shape(seq_len, q_loc.shape[1], k_chunk.shape[1], layout)
    L = _lib.lib()
    nbytes = L.mt_sparse_attn_fwd_workspace_bytes(ctypes.byref(sh), world)
    ws = workspace(nbytes)
    ci = idx.c_struct()
    _lib.check(L.mt_attn_fwd_step(ctypes.byref(sh), world, rank, origin, int(first), int(last),
                                  _ptr(q_loc), _ptr(k_chunk), _ptr(v_chunk), ctypes.byref(ci),
                                  _ptr(o), _ptr(o_acc), _ptr(lse), _ptr(ws), ws.numel(), _stream()))


class VSParams(ctypes.Structure):
    _fields_ = [("p_v", ctypes.c_float), ("p_s", ctypes.c_float)]


def build_vs_index(q: torch.Tensor, k: torch.Tensor, p_v: float, p_s: float, comm=None,
                   seq_len: int | None = None, layout: str = "striped") -> VSIndex:
    """Alg. 1 index on the GPU (mt_build_vs_index).  With `comm`, q/k are the
    rank-local slices in `layout` and `seq_len` is the global length."""
    S = q.shape[0] if seq_len is None else seq_len
    Hq = q.shape[1]
    world = 1 if comm is None else comm.world
    sh = shape(S, Hq, k.shape[1], layout)
    L = _lib.lib()
    ws = workspace(L.mt_build_vs_index_workspace_bytes(ctypes.byref(sh), world))
    idx = VSIndex.uninit(S, Hq, device=q.device)
    ci = idx.c_struct()
    prm = VSParams(p_v, p_s)
    _lib.check(L.mt_build_vs_index(None if comm is None else comm.handle, ctypes.byref(sh),
                                   ctypes.byref(prm), _ptr(q), _ptr(k), ctypes.byref(ci),
                                   _ptr(ws), ws.numel(), _stream()))
    return idx


def rope_vs_index(q: torch.Tensor, k: torch.Tensor, freqs, p_v: float, p_s: float, comm=None,
                  seq_len: int | None = None, layout: str = "striped"):
    """f3 fusion (mt_rope_vs_index): from PRE-RoPE q / k, returns (index, RoPE(q), RoPE(k)),
    the index equal to build_vs_index(RoPE(q), RoPE(k)).  freqs = rope_freqs(...)."""
    th, ms = freqs
    S = q.shape[0] if seq_len is None else seq_len
    Hq = q.shape[1]
    world = 1 if comm is None else comm.world
    sh = shape(S, Hq, k.shape[1], layout)
    L = _lib.lib()
    ws = workspace(L.mt_build_vs_index_workspace_bytes(ctypes.byref(sh), world))
    idx = VSIndex.uninit(S, Hq, device=q.device)
    ci = idx.c_struct()
    prm = VSParams(p_v, p_s)
    q_out, k_out = torch.empty_like(q), torch.empty_like(k)
    _lib.check(L.mt_rope_vs_index(None if comm is None else comm.handle, ctypes.byref(sh),
                                  ctypes.byref(prm), th, ms, _ptr(q), _ptr(k), _ptr(q_out),
                                  _ptr(k_out), ctypes.byref(ci), _ptr(ws), ws.numel(), _stream()))
    return idx, q_out, k_out


def vs_column_scores(q: torch.Tensor, k: torch.Tensor):
    """Test hook: exact Alg. 1 intermediate scores (uint64 as int64 tensors)."""
    S, Hq, _ = q.shape
    sh = shape(S, Hq, k.shape[1])
    L = _lib.lib()
    ws = workspace(L.mt_build_vs_index_workspace_bytes(ctypes.byref(sh), 1))
    col = torch.zeros(Hq, S, dtype=torch.int64, device=q.device)
    sl = torch.zeros(Hq, S // BLOCK, dtype=torch.int64, device=q.device)
    _lib.check(L.mt_vs_column_scores(ctypes.byref(sh), _ptr(q), _ptr(k), _ptr(col), _ptr(sl),
                                     _ptr(ws), ws.numel(), _stream()))
    return col, sl


def sparse_attn_bwd(q, k, v, o, lse, dO, idx: VSIndex):
    """Single-GPU backward -> (dq, dk, dv) bf16."""
    S, Hq, _ = q.shape
    sh = shape(S, Hq, k.shape[1])
    L = _lib.lib()
    ws = workspace(L.mt_sparse_attn_bwd_workspace_bytes(ctypes.byref(sh)))
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    ci = idx.c_struct()
    _lib.check(L.mt_sparse_attn_bwd(ctypes.byref(sh), _ptr(q), _ptr(k), _ptr(v), _ptr(o), _ptr(lse),
                                    _ptr(dO), ctypes.byref(ci), _ptr(dq), _ptr(dk), _ptr(dv),
                                    _ptr(ws), ws.numel(), _stream()))
    return dq, dk, dv


def attn_bwd_preprocess(seq_len: int, world: int, o_loc, dO_loc, D_loc, layout: str = "striped"):
    sh = shape(seq_len, o_loc.shape[1], 1, layout)
    _lib.check(_lib.lib().mt_attn_bwd_preprocess(ctypes.byref(sh), world, _ptr(o_loc), _ptr(dO_loc),
                                                 _ptr(D_loc), _stream()))


def attn_bwd_step(seq_len: int, world: int, rank: int, origin: int, q_loc, k_chunk, v_chunk,
                  dO_loc, lse_loc, D_loc, idx: VSIndex, dq_acc, dk_acc, dv_acc,
                  layout: str = "striped"):
    sh = shape(seq_len, q_loc.shape[1], k_chunk.shape[1], layout)
    L = _lib.lib()
    ws = workspace(L.mt_attn_step_workspace_bytes(ctypes.byref(sh), world))
    ci = idx.c_struct()
    _lib.check(L.mt_attn_bwd_step(ctypes.byref(sh), world, rank, origin, _ptr(q_loc), _ptr(k_chunk),
                                  _ptr(v_chunk), _ptr(dO_loc), _ptr(lse_loc), _ptr(D_loc),
                                  ctypes.byref(ci), _ptr(dq_acc), _ptr(dk_acc), _ptr(dv_acc),
                                  _ptr(ws), ws.numel(), _stream()))


class Comm:
    """mt_comm over a torch.distributed process group (one process per GPU)."""

    def __init__(self, handle, world: int, rank: int, inner: int):
        self.handle, self.world, self.rank, self.inner = handle, world, rank, inner
        self.ring_ws = None  # the ring calls' own workspace (registered for the copy engines)

    def ring_workspace(self, nbytes: int) -> torch.Tensor:
        """The ring calls' workspace: at least `nbytes` plus the reserved flag words at its
        end (mt_ring_flags_bytes).  Grown collectively (every rank asks for the same size
        at the same call), and (re)registered with mt_comm_register_workspace so the flat
        forward ring moves KV chunks with the copy engines (MT_RING_CE=0 keeps NCCL)."""
        import os
        L = _lib.lib()
        need = nbytes + int(L.mt_ring_flags_bytes())
        if self.ring_ws is None or self.ring_ws.numel() < need:
            self.ring_ws = torch.empty(max(need, 1 << 20), dtype=torch.uint8, device="cuda")
            if os.environ.get("MT_RING_CE", "1") != "0":
                _lib.check(L.mt_comm_register_workspace(self.handle, _ptr(self.ring_ws),
                                                        self.ring_ws.numel(), _stream()))
        return self.ring_ws

    def copy_engine(self) -> bool:
        return bool(_lib.lib().mt_comm_copy_engine(self.handle))

    @staticmethod
    def create(world: int, rank: int, inner: int | None = None, group=None) -> "Comm":
        import torch.distributed as dist
        L = _lib.lib()
        buf = (ctypes.c_uint8 * 128)()
        if rank == 0:
            _lib.check(L.mt_comm_unique_id(buf))
        ids = [bytes(buf)] if rank == 0 else [None]
        # `rank` is the ring rank (rank within `group`): the id travels from the group's
        # rank 0, whose global rank is not 0 when a sub-group is passed
        src = 0 if group is None else dist.get_global_rank(group, 0)
        dist.broadcast_object_list(ids, src=src, group=group)
        uid = (ctypes.c_uint8 * 128).from_buffer_copy(ids[0])
        h = ctypes.c_void_p()
        inner = world if not inner else inner
        _lib.check(L.mt_comm_create(uid, world, rank, inner, ctypes.byref(h)))
        return Comm(h, world, rank, inner)

    def destroy(self):
        if self.handle:
            _lib.check(_lib.lib().mt_comm_destroy(self.handle))
            self.handle = None

    def check(self):
        """Raise if the communicator saw an asynchronous NCCL/CUDA failure (mt_comm_check)."""
        _lib.check(_lib.lib().mt_comm_check(self.handle))

    def profile(self, enable: bool = True):
        """Record per-step CUDA events in later ring calls (mt_comm_profile)."""
        _lib.check(_lib.lib().mt_comm_profile(self.handle, int(enable)))

    def step_times(self, backward: bool):
        """[(compute, inner KV, outer KV, dK/dV partial) ms per step] of the last
        profiled ring call (-1 where a step had no such transfer)."""
        n = ctypes.c_int()
        out = (ctypes.c_float * (4 * 64))()
        _lib.check(_lib.lib().mt_comm_step_times(self.handle, int(backward), 64, out,
                                                 ctypes.byref(n)))
        return [tuple(out[4 * t + k] for k in range(4)) for t in range(n.value)]


def vs_format(idx: VSIndex, seq_len: int, n_kv_heads: int = 1):
    """Per-query-block key lists (mt_vs_format_count/fill): (blk_ptr, blk_idx, col_ptr,
    col_idx) device tensors, pointers int64 [Hq][nb + 1] with global offsets."""
    Hq, nb = idx.v_cnt.numel(), seq_len // BLOCK
    sh = shape(seq_len, Hq, n_kv_heads)
    L = _lib.lib()
    ws = workspace(L.mt_vs_format_workspace_bytes(ctypes.byref(sh)))
    bp = torch.empty(Hq, nb + 1, dtype=torch.int64, device=idx.v_cnt.device)
    cp = torch.empty_like(bp)
    nbk, ncl = ctypes.c_int64(), ctypes.c_int64()
    ci = idx.c_struct()
    _lib.check(L.mt_vs_format_count(ctypes.byref(sh), ctypes.byref(ci), _ptr(bp), _ptr(cp),
                                    ctypes.byref(nbk), ctypes.byref(ncl), _ptr(ws), ws.numel(),
                                    _stream()))
    bi = torch.empty(max(nbk.value, 1), dtype=torch.int32, device=bp.device)
    cl = torch.empty(max(ncl.value, 1), dtype=torch.int32, device=bp.device)
    _lib.check(L.mt_vs_format_fill(ctypes.byref(sh), ctypes.byref(ci), _ptr(bp), _ptr(cp), _ptr(bi),
                                   bi.numel(), _ptr(cl), cl.numel(), nbk.value, ncl.value, _ptr(ws),
                                   ws.numel(), _stream()))
    return bp, bi[: nbk.value], cp, cl[: ncl.value]


@dataclass
class BlockIndex:
    """Explicit block index (the CSR of mt_vs_format / mt_xattn_index): key blocks of
    query block g of head h are idx[ptr[h, g] : ptr[h, g + 1]] (global offsets)."""
    ptr: torch.Tensor   # int64 [Hq][nb + 1]
    idx: torch.Tensor   # int32 [n]

    @property
    def n(self) -> int:
        return int(self.idx.numel())

    @staticmethod
    def from_lists(B, device="cuda") -> "BlockIndex":
        """B[h][g]: ascending key blocks (<= g) of query block g of head h."""
        Hq, nb = len(B), len(B[0])
        ptr = torch.zeros(Hq, nb + 1, dtype=torch.int64)
        flat, run = [], 0
        for h in range(Hq):
            for g in range(nb):
                ptr[h, g] = run
                flat.extend(int(x) for x in B[h][g])
                run += len(B[h][g])
            ptr[h, nb] = run
        idx = torch.tensor(flat if flat else [0], dtype=torch.int32)[: run]
        return BlockIndex(ptr.to(device), idx.to(device))

    def to_lists(self):
        p, x = self.ptr.cpu().numpy(), self.idx.cpu().numpy()
        return [[x[p[h, g]: p[h, g + 1]].copy() for g in range(p.shape[1] - 1)]
                for h in range(p.shape[0])]


class XAttnParams(ctypes.Structure):
    _fields_ = [("block", ctypes.c_int), ("stride", ctypes.c_int), ("threshold", ctypes.c_float)]


def xattn_index(q: torch.Tensor, k: torch.Tensor, threshold: float = 0.9,
                with_scores: bool = False):
    """XAttention block index on the GPU (mt_xattn_index_count/fill) -> BlockIndex
    (and the fp32 block scores [Hq][nI (nI + 1) / 2] when with_scores)."""
    S, Hq, _ = q.shape
    sh = shape(S, Hq, k.shape[1])
    L = _lib.lib()
    prm = XAttnParams(128, 16, threshold)
    ws = workspace(L.mt_xattn_index_workspace_bytes(ctypes.byref(sh)))
    nI = S // 128
    ptr = torch.empty(Hq, S // 64 + 1, dtype=torch.int64, device=q.device)
    scores = (torch.empty(Hq, nI * (nI + 1) // 2, dtype=torch.float32, device=q.device)
              if with_scores else None)
    n = ctypes.c_int64()
    _lib.check(L.mt_xattn_index_count(ctypes.byref(sh), ctypes.byref(prm), _ptr(q), _ptr(k),
                                      _ptr(ptr), ctypes.byref(n), _ptr(scores), _ptr(ws),
                                      ws.numel(), _stream()))
    idx = torch.empty(max(n.value, 1), dtype=torch.int32, device=q.device)
    _lib.check(L.mt_xattn_index_fill(ctypes.byref(sh), ctypes.byref(prm), _ptr(ptr), _ptr(idx),
                                     idx.numel(), n.value, _ptr(ws), ws.numel(), _stream()))
    bi = BlockIndex(ptr, idx[: n.value])
    return (bi, scores) if with_scores else bi


def block_sparse_attn_fwd(q, k, v, bidx: BlockIndex):
    """mt_block_sparse_attn_fwd -> (o bf16 [S][Hq][128], lse f32 [Hq][S])."""
    S, Hq, _ = q.shape
    sh = shape(S, Hq, k.shape[1])
    L = _lib.lib()
    ws = workspace(L.mt_block_sparse_attn_fwd_workspace_bytes(ctypes.byref(sh)))
    o = torch.empty_like(q)
    lse = torch.empty(Hq, S, dtype=torch.float32, device=q.device)
    _lib.check(L.mt_block_sparse_attn_fwd(ctypes.byref(sh), _ptr(q), _ptr(k), _ptr(v),
                                          _ptr(bidx.ptr), _ptr(bidx.idx), bidx.n, _ptr(o),
                                          _ptr(lse), _ptr(ws), ws.numel(), _stream()))
    return o, lse


def block_sparse_attn_bwd(q, k, v, o, lse, dO, bidx: BlockIndex):
    """mt_block_sparse_attn_bwd -> (dq, dk, dv) bf16."""
    S, Hq, _ = q.shape
    sh = shape(S, Hq, k.shape[1])
    L = _lib.lib()
    ws = workspace(L.mt_block_sparse_attn_bwd_workspace_bytes(ctypes.byref(sh), bidx.n))
    dq, dk, dv = torch.empty_like(q), torch.empty_like(k), torch.empty_like(v)
    _lib.check(L.mt_block_sparse_attn_bwd(ctypes.byref(sh), _ptr(q), _ptr(k), _ptr(v), _ptr(o),
                                          _ptr(lse), _ptr(dO), _ptr(bidx.ptr), _ptr(bidx.idx),
                                          bidx.n, _ptr(dq), _ptr(dk), _ptr(dv), _ptr(ws),
                                          ws.numel(), _stream()))
    return dq, dk, dv


def rope_freqs(base: float = 1e6, yarn_factor: float = 1.0, original_max_position: int = 32768):
    """(theta[64] as ctypes doubles, mscale) from the library (mt_rope_inv_freq)."""
    th = (ctypes.c_double * 64)()
    ms = ctypes.c_float()
    _lib.check(_lib.lib().mt_rope_inv_freq(128, base, yarn_factor, original_max_position, th,
                                           ctypes.byref(ms)))
    return th, ms.value


def rope_(x: torch.Tensor, freqs, seq_len: int | None = None, world: int = 1, rank: int = 0,
          inverse: bool = False) -> torch.Tensor:
    """In-place RoPE on a token-major bf16 [S/W][H][128] tensor (mt_rope)."""
    th, ms = freqs
    S = seq_len or x.shape[0] * world
    _lib.check(_lib.lib().mt_rope(S, world, rank, x.shape[1], th, ms, int(inverse), _ptr(x),
                                  _stream()))
    return x


def stripe(x_global: torch.Tensor, world: int, rank: int, layout: str = "striped") -> torch.Tensor:
    """Rank `rank`'s share of a token-major tensor in `layout` (mt_stripe /
    mt_layout_to_local)."""
    S = x_global.shape[0]
    out = torch.empty((S // world,) + tuple(x_global.shape[1:]), dtype=x_global.dtype,
                      device=x_global.device)
    row = x_global[0].numel() * x_global.element_size()
    if layout == "striped":
        _lib.check(_lib.lib().mt_stripe(S, row, world, rank, _ptr(x_global), _ptr(out), _stream()))
    else:
        _lib.check(_lib.lib().mt_layout_to_local(LAYOUTS[layout], S, row, world, rank, _ptr(x_global),
                                                 _ptr(out), _stream()))
    return out


def unstripe(x_local: torch.Tensor, world: int, rank: int, out: torch.Tensor,
             layout: str = "striped") -> torch.Tensor:
    """Scatter rank `rank`'s local rows back into the global tensor `out` (mt_unstripe /
    mt_layout_to_global)."""
    S = out.shape[0]
    row = out[0].numel() * out.element_size()
    if layout == "striped":
        _lib.check(_lib.lib().mt_unstripe(S, row, world, rank, _ptr(x_local), _ptr(out), _stream()))
    else:
        _lib.check(_lib.lib().mt_layout_to_global(LAYOUTS[layout], S, row, world, rank, _ptr(x_local),
                                                  _ptr(out), _stream()))
    return out


def ring_schedule(world: int, inner: int | None = None):
    """Host-side schedule from the library: held[t][x] = origin at rank x, step t."""
    out = (ctypes.c_int32 * (world * world))()
    _lib.check(_lib.lib().mt_ring_schedule(world, inner or world, out))
    return [[out[t * world + x] for x in range(world)] for t in range(world)]


def ring_attn_fwd(comm: Comm, seq_len: int, q_loc, k_loc, v_loc, idx: VSIndex,
                  layout: str = "striped"):
    sh = shape(seq_len, q_loc.shape[1], k_loc.shape[1], layout)
    L = _lib.lib()
    ws = comm.ring_workspace(max(L.mt_ring_attn_workspace_bytes(ctypes.byref(sh), comm.world, 0),
                                 L.mt_ring_attn_workspace_bytes(ctypes.byref(sh), comm.world, 1)))
    o = torch.empty_like(q_loc)
    lse = torch.empty(q_loc.shape[1], q_loc.shape[0], dtype=torch.float32, device=q_loc.device)
    ci = idx.c_struct()
    _lib.check(L.mt_ring_attn_fwd(comm.handle, ctypes.byref(sh), _ptr(q_loc), _ptr(k_loc), _ptr(v_loc),
                                  ctypes.byref(ci), _ptr(o), _ptr(lse), _ptr(ws), ws.numel(), _stream()))
    return o, lse


def ring_attn_bwd(comm: Comm, seq_len: int, q_loc, k_loc, v_loc, o_loc, lse_loc, dO_loc, idx: VSIndex,
                  layout: str = "striped"):
    sh = shape(seq_len, q_loc.shape[1], k_loc.shape[1], layout)
    L = _lib.lib()
    ws = comm.ring_workspace(max(L.mt_ring_attn_workspace_bytes(ctypes.byref(sh), comm.world, 0),
                                 L.mt_ring_attn_workspace_bytes(ctypes.byref(sh), comm.world, 1)))
    dq, dk, dv = torch.empty_like(q_loc), torch.empty_like(k_loc), torch.empty_like(v_loc)
    ci = idx.c_struct()
    _lib.check(L.mt_ring_attn_bwd(comm.handle, ctypes.byref(sh), _ptr(q_loc), _ptr(k_loc), _ptr(v_loc),
                                  _ptr(o_loc), _ptr(lse_loc), _ptr(dO_loc), ctypes.byref(ci),
                                  _ptr(dq), _ptr(dk), _ptr(dv), _ptr(ws), ws.numel(), _stream()))
    return dq, dk, dv
