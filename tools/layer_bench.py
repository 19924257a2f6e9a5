"""Tokens/s of one Qwen2.5-3B-shaped decoder layer with the VS
sparse attention at 512K on one GPU, and the attention's share of the layer step.

Step = Alg. 1 index on the workload's q/k (the bench's synthetic RoPE vertical-slash
generator, paper density) + layer forward + layer backward (all weight and input
gradients) with that index.  Random-init weights act on N(0,1) hidden states: their
own post-RoPE q/k carry no vertical-slash structure (a top-p index of noise is
near-dense), so the index comes from the workload generator, as in bench.py.
Prints one JSON line.  CUDA events on the current stream; max over nothing (1 GPU).
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_18830_b200 import layer as LY  # noqa: E402
from paper_2510_18830_b200 import ops  # noqa: E402
from synth.generator import make_qkv  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq", type=int, default=524288)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--p", type=float, default=0.9)
    a = ap.parse_args()
    S = a.seq
    torch.manual_seed(0)
    layer = LY.VSDecoderLayer()
    for m in (layer.qkv, layer.o_proj, layer.gate, layer.up, layer.down):
        torch.nn.init.normal_(m.weight, std=m.weight.shape[1] ** -0.5)
    q, k, _ = make_qkv(S, 16, 2, seed=0)
    qd = torch.from_numpy(q.view(np.int16)).view(torch.bfloat16).cuda()
    kd = torch.from_numpy(k.view(np.int16)).view(torch.bfloat16).cuda()
    x = torch.randn(S, 2048, device="cuda", dtype=torch.bfloat16, requires_grad=True)
    dy = torch.randn(S, 2048, device="cuda", dtype=torch.bfloat16)
    ev = lambda: torch.cuda.Event(enable_timing=True)

    def step(rec):
        LY.EVENTS = [] if rec else None
        e = [ev() for _ in range(4)]
        e[0].record()
        idx = ops.build_vs_index(qd, kd, a.p, a.p)
        e[1].record()
        y = layer(x, index=idx)
        e[2].record()
        y.backward(dy)
        e[3].record()
        out = (e, LY.EVENTS)
        LY.EVENTS = None
        layer.zero_grad(set_to_none=True)
        x.grad = None
        return out

    for _ in range(a.warmup):
        step(False)
    torch.cuda.synchronize()
    recs = [step(True) for _ in range(a.steps)]
    torch.cuda.synchronize()
    idx_ms = np.median([r[0][0].elapsed_time(r[0][1]) for r in recs])
    fwd_ms = np.median([r[0][1].elapsed_time(r[0][2]) for r in recs])
    bwd_ms = np.median([r[0][2].elapsed_time(r[0][3]) for r in recs])
    af = np.median([sum(s.elapsed_time(t) for g, s, t in r[1] if g == "attn_fwd") for r in recs])
    ab = np.median([sum(s.elapsed_time(t) for g, s, t in r[1] if g == "attn_bwd") for r in recs])
    total = idx_ms + fwd_ms + bwd_ms
    print(json.dumps({
        "metric": "layer_tokens_per_s", "value": S / (total / 1e3), "unit": "tokens/s",
        "config": {"workload": f"Qwen2.5-3B-shaped decoder layer, {S} tokens, 1 GPU",
                   "hidden": 2048, "heads": "16q/2kv x 128", "intermediate": 11008,
                   "rope": "base 1e6, YaRN x32 from 32K", "index": "synthetic workload, p=0.9"},
        "ms": {"index": idx_ms, "layer_fwd": fwd_ms, "layer_bwd": bwd_ms, "total": total,
               "attn_fwd": af, "attn_bwd": ab},
        "attention_share": (idx_ms + af + ab) / total,
        "peak_mem_gb": torch.cuda.max_memory_allocated() / 2 ** 30,
    }))


if __name__ == "__main__":
    main()
