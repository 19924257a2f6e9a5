"""f1: dense causal vs vertical-slash sparse attention through the SAME
kernels and ring, at 512K tokens (Qwen2.5-3B-shaped: 16 q / 2 kv heads, d = 128).

Dense = the full budget (reading R22): every slash offset selected (plus the forced
column 0), i.e. exact causal attention.  The sparse run uses Alg. 1's index (p = 0.9).
Prints one JSON line per mode with fwd / bwd ms (CUDA events, max over ranks), tokens/s
and activated TFLOP/s.  Single GPU or under torchrun (flat striped ring).

  python tools/dense_bench.py [--seq 524288] [--steps 2]
  python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 tools/dense_bench.py
"""
import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2510_18830_b200 import ops, stats  # noqa: E402
from synth.generator import make_grad_out, make_qkv  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--seq", type=int, default=524288)
ap.add_argument("--steps", type=int, default=2)
ap.add_argument("--warmup", type=int, default=1)
a = ap.parse_args()
W = int(os.environ.get("WORLD_SIZE", "1"))
rank = int(os.environ.get("RANK", "0"))
local = int(os.environ.get("LOCAL_RANK", "0"))
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
comm = None
if W > 1:
    dist.init_process_group("nccl", device_id=dev)
    comm = ops.Comm.create(W, rank, W)
S, Hq, Hkv = a.seq, 16, 2
q, k, v = make_qkv(S, Hq, Hkv, seed=0)
dO = make_grad_out(S, Hq, seed=0)
j = np.arange(S // W)
rows = ((j // 64) * W + rank) * 64 + j % 64
t = lambda x: torch.from_numpy(np.ascontiguousarray(x[rows]).view(np.int16)).view(torch.bfloat16).to(dev)
qd, kd, vd, dd = t(q), t(k), t(v), t(dO)
sparse_idx = ops.build_vs_index(qd, kd, 0.9, 0.9, comm=comm, seq_len=S)
nb = S // 64
dense_idx = ops.VSIndex.from_lists([np.array([0], np.int32)] * Hq, [np.arange(nb, dtype=np.int32)] * Hq, S,
                                   device=dev)
stream = torch.cuda.current_stream()
for name, idx in (("sparse p=0.9", sparse_idx), ("dense causal (full budget)", dense_idx)):
    iv, is_ = idx.to_lists()
    pairs = int(stats.pairs_per_head(iv, is_, S).sum())
    ev = lambda: torch.cuda.Event(enable_timing=True)
    tf, tb = [], []
    for it in range(a.warmup + a.steps):
        e0, e1, e2 = ev(), ev(), ev()
        if W > 1:
            dist.barrier(device_ids=[local])
        e0.record(stream)
        if comm is None:
            o, lse = ops.sparse_attn_fwd(qd, kd, vd, idx)
            e1.record(stream)
            ops.sparse_attn_bwd(qd, kd, vd, o, lse, dd, idx)
        else:
            o, lse = ops.ring_attn_fwd(comm, S, qd, kd, vd, idx)
            e1.record(stream)
            ops.ring_attn_bwd(comm, S, qd, kd, vd, o, lse, dd, idx)
        e2.record(stream)
        torch.cuda.synchronize()
        if it >= a.warmup:
            tf.append(e0.elapsed_time(e1))
            tb.append(e1.elapsed_time(e2))
    x = torch.tensor([np.mean(tf), np.mean(tb)], device=dev)
    if W > 1:
        dist.all_reduce(x, op=dist.ReduceOp.MAX)
    fms, bms = (float(y) for y in x.cpu())
    if rank == 0:
        print(json.dumps({"mode": name, "world": W, "seq_len": S, "activated_pairs": pairs,
                          "density": round(pairs / (Hq * stats.causal_pairs(S)), 4),
                          "fwd_ms": round(fms, 2), "bwd_ms": round(bms, 2),
                          "tokens_per_s_attn": S / ((fms + bms) / 1e3),
                          "fwd_tflops_per_gpu": round(4 * 128 * pairs / W / (fms / 1e3) / 1e12, 1),
                          "bwd_tflops_per_gpu": round(10 * 128 * pairs / W / (bms / 1e3) / 1e12, 1)}),
              flush=True)
if comm is not None:
    comm.destroy()
    dist.destroy_process_group()
