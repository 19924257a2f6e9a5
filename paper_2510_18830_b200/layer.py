"""A Qwen2.5-3B-shaped decoder layer around the VS sparse attention.

The paper trains Qwen2.5-3B with every attention replaced by vertical-slash sparse
attention (Alg. 1).  This module is that layer with random
weights (reading R-layer in DESIGN.md):

  RMSNorm -> QKV projection (+bias) -> RoPE/YaRN (mt_rope) -> VS index
  (mt_build_vs_index, no gradient) -> sparse attention (mt_sparse_attn_fwd /
  _bwd, or the ring over a Comm) -> O projection -> residual -> RMSNorm -> SwiGLU
  MLP -> residual.

The path's steps (RoPE, index, attention, ring) run in this package's CUDA library;
the dense projections are cuBLAS GEMMs through torch (library GEMMs), the norms and
the SwiGLU product torch elementwise ops.  Under a Comm, `x` is the rank's
block-striped slice (mt_stripe) and the weight gradients are rank-local partials
(their data-parallel all-reduce belongs to the training framework, out of scope).
"""
from __future__ import annotations

import torch
import torch.nn.functional as F
from torch import nn

from . import ops


class _Rope(torch.autograd.Function):
    """y = mscale R(n) x; backward dx = mscale R(-n) dy (the transpose rotation)."""

    @staticmethod
    def forward(ctx, x, freqs, seq_len, world, rank):
        y = x.contiguous().clone()
        ops.rope_(y, freqs, seq_len=seq_len, world=world, rank=rank)
        ctx.args = (freqs, seq_len, world, rank)
        return y

    @staticmethod
    def backward(ctx, dy):
        freqs, seq_len, world, rank = ctx.args
        dx = dy.contiguous().clone()
        ops.rope_(dx, freqs, seq_len=seq_len, world=world, rank=rank, inverse=True)
        return dx, None, None, None, None


# When a list, _SparseAttn appends (tag, start event, end event) around its library
# calls (tools/layer_bench.py reads it to split the layer step).
EVENTS: list | None = None


def _mark():
    if EVENTS is None:
        return None
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


class _SparseAttn(torch.autograd.Function):
    """O = sparse(softmax(QK^T/sqrt d) V, i_vs) with the index held fixed."""

    @staticmethod
    def forward(ctx, q, k, v, idx, comm, seq_len):
        e0 = _mark()
        if comm is None:
            o, lse = ops.sparse_attn_fwd(q, k, v, idx)
        else:
            o, lse = ops.ring_attn_fwd(comm, seq_len, q, k, v, idx)
        if e0 is not None:
            EVENTS.append(("attn_fwd", e0, _mark()))
        ctx.save_for_backward(q, k, v, o, lse)
        ctx.idx, ctx.comm, ctx.seq_len = idx, comm, seq_len
        return o

    @staticmethod
    def backward(ctx, do):
        q, k, v, o, lse = ctx.saved_tensors
        do = do.contiguous()
        e0 = _mark()
        if ctx.comm is None:
            dq, dk, dv = ops.sparse_attn_bwd(q, k, v, o, lse, do, ctx.idx)
        else:
            dq, dk, dv = ops.ring_attn_bwd(ctx.comm, ctx.seq_len, q, k, v, o, lse, do, ctx.idx)
        if e0 is not None:
            EVENTS.append(("attn_bwd", e0, _mark()))
        return dq, dk, dv, None, None, None


class RMSNorm(nn.Module):
    def __init__(self, dim: int, eps: float = 1e-6, **kw):
        super().__init__()
        self.eps = eps
        self.weight = nn.Parameter(torch.ones(dim, **kw))

    def forward(self, x):
        xf = x.float()
        y = xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + self.eps)
        return (y * self.weight.float()).to(x.dtype)


class VSDecoderLayer(nn.Module):
    """Qwen2.5-3B decoder layer shape by default: hidden 2048, 16 q / 2 kv heads of
    128, SwiGLU intermediate 11008, RoPE base 1e6 with YaRN x32 from 32K."""

    def __init__(self, hidden: int = 2048, n_q_heads: int = 16, n_kv_heads: int = 2,
                 intermediate: int = 11008, p_v: float = 0.9, p_s: float = 0.9,
                 rope_base: float = 1e6, yarn_factor: float = 32.0,
                 original_max_position: int = 32768, device="cuda", dtype=torch.bfloat16):
        super().__init__()
        kw = dict(device=device, dtype=dtype)
        self.Hq, self.Hkv, self.d = n_q_heads, n_kv_heads, 128
        self.p_v, self.p_s = p_v, p_s
        self.ln1 = RMSNorm(hidden, **kw)
        self.qkv = nn.Linear(hidden, (n_q_heads + 2 * n_kv_heads) * 128, bias=True, **kw)
        self.o_proj = nn.Linear(n_q_heads * 128, hidden, bias=False, **kw)
        self.ln2 = RMSNorm(hidden, **kw)
        self.gate = nn.Linear(hidden, intermediate, bias=False, **kw)
        self.up = nn.Linear(hidden, intermediate, bias=False, **kw)
        self.down = nn.Linear(intermediate, hidden, bias=False, **kw)
        self.freqs = ops.rope_freqs(rope_base, yarn_factor, original_max_position)
        self.last_index: ops.VSIndex | None = None

    def attention(self, x, comm=None, seq_len=None, index=None):
        """x: [S_loc][hidden] -> (attention output before o_proj [S_loc][Hq * 128])."""
        S_loc = x.shape[0]
        world, rank = (1, 0) if comm is None else (comm.world, comm.rank)
        S = S_loc * world if seq_len is None else seq_len
        Hq, Hkv, d = self.Hq, self.Hkv, self.d
        qkv = self.qkv(self.ln1(x))
        q = qkv[:, : Hq * d].reshape(S_loc, Hq, d)
        k = qkv[:, Hq * d: (Hq + Hkv) * d].reshape(S_loc, Hkv, d)
        v = qkv[:, (Hq + Hkv) * d:].reshape(S_loc, Hkv, d).contiguous()
        q = _Rope.apply(q, self.freqs, S, world, rank)
        k = _Rope.apply(k, self.freqs, S, world, rank)
        if index is None:
            index = ops.build_vs_index(q.detach(), k.detach(), self.p_v, self.p_s, comm=comm,
                                       seq_len=S)
        self.last_index = index
        o = _SparseAttn.apply(q, k, v, index, comm, S)
        return o.reshape(S_loc, Hq * d)

    def forward(self, x, comm=None, seq_len=None, index=None):
        x2 = x + self.o_proj(self.attention(x, comm, seq_len, index))
        h2 = self.ln2(x2)
        return x2 + self.down(F.silu(self.gate(h2)) * self.up(h2))
