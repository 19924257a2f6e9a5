"""Ring-step latency model of Appendix C.

With per-step compute T_comp, intra-node transfer T_intra and inter-node transfer
T_inter, a flat (naive) sparse ring whose every hop may cross nodes runs W-1
communicating steps at max(T_comp, T_intra, T_inter) plus a last compute-only
step; the hierarchical ring overlaps the inter-node transfer with a
whole inner ring, so each of its W steps costs max(T_comp, T_inner).
Both add the once-per-pass costs: the index (or, backward, the vertical-line
pass) and the paper's "CPU operations" (zero in this build, whose
kernels derive the per-origin lists on the fly).  Times in ms.
"""
from __future__ import annotations


def flat_ring_total(t_pre: float, t_cpu: float, t_comp: float, t_intra: float, t_inter: float,
                    world: int) -> float:
    """T = T_pre + T_cpu + (W - 1) max(T_comp, T_intra, T_inter) + T_comp."""
    return t_pre + t_cpu + (world - 1) * max(t_comp, t_intra, t_inter) + t_comp


def hier_ring_total(t_pre: float, t_cpu: float, t_comp: float, t_inner: float,
                    world: int) -> float:
    """T = T_pre + T_cpu + W max(T_comp, T_inner)."""
    return t_pre + t_cpu + world * max(t_comp, t_inner)


def transfer_ms(nbytes: float, gbps: float) -> float:
    """Wire time of one step's message at a sustained link rate (GB/s)."""
    return nbytes / (gbps * 1e9) * 1e3


def step_bytes(seq_len: int, world: int, n_kv_heads: int, head_dim: int = 128,
               backward: bool = False) -> int:
    """Bytes one rank sends per ring step: the bf16 K and V chunk,
    plus (backward) the fp32 dK/dV partial of the chunk it held."""
    kv = 2 * (seq_len // world) * n_kv_heads * head_dim * 2
    return kv + (2 * (seq_len // world) * n_kv_heads * head_dim * 4 if backward else 0)
