"""Worker for test_gpu_layer_ring.py (launched by torchrun, one process per GPU).

The decoder layer (paper_2510_18830_b200/layer.py) over W GPUs
- block-striped hidden states (mt_stripe), RoPE at striped global positions, the
distributed Alg. 1 index, the NCCL ring forward/backward - against the same layer
on one GPU (rank 0): outputs, input gradients and all-reduced weight gradients
must agree within bf16 reduction-order noise (the index is W-invariant, bit-exact).
Prints one JSON line on rank 0; exits non-zero on a mismatch."""
import argparse
import copy
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_18830_b200 import ops  # noqa: E402
from paper_2510_18830_b200.layer import VSDecoderLayer  # noqa: E402


def nerr(a, b):
    a, b = a.double(), b.double()
    return float((a - b).abs().max() / b.abs().max().clamp_min(1e-30))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seq", type=int, default=8192)
    ap.add_argument("--inner", type=int, default=0)
    a = ap.parse_args()
    W, rank, local = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    comm = ops.Comm.create(W, rank, a.inner or W)
    S, D = a.seq, 256
    torch.manual_seed(0)
    layer = VSDecoderLayer(hidden=D, n_q_heads=4, n_kv_heads=2, intermediate=512, device=dev)
    for m in (layer.qkv, layer.o_proj, layer.gate, layer.up, layer.down):
        torch.nn.init.normal_(m.weight, std=m.weight.shape[1] ** -0.5)
    ref_layer = copy.deepcopy(layer)
    g = torch.Generator().manual_seed(1)
    x = torch.randn(S, D, generator=g).to(dev, torch.bfloat16)
    dy = torch.randn(S, D, generator=g).to(dev, torch.bfloat16)

    xl = ops.stripe(x, W, rank).requires_grad_(True)
    yl = layer(xl, comm=comm, seq_len=S)
    yl.backward(ops.stripe(dy, W, rank))
    for p in layer.parameters():
        dist.all_reduce(p.grad)
    parts_y = [torch.empty_like(yl) for _ in range(W)]
    parts_dx = [torch.empty_like(yl) for _ in range(W)]
    dist.all_gather(parts_y, yl.detach().contiguous())
    dist.all_gather(parts_dx, xl.grad.contiguous())
    torch.cuda.synchronize()
    comm.check()
    bad = 0
    if rank == 0:
        y = torch.empty_like(x)
        dx = torch.empty_like(x)
        for r in range(W):
            ops.unstripe(parts_y[r], W, r, y)
            ops.unstripe(parts_dx[r], W, r, dx)
        xr = x.clone().requires_grad_(True)
        y_ref = ref_layer(xr)
        y_ref.backward(dy)
        torch.cuda.synchronize()
        errs = {"y-x": nerr(y.float() - x.float(), y_ref.detach().float() - x.float()),
                "dx": nerr(dx, xr.grad)}
        for (n, p), (_, q) in zip(layer.named_parameters(), ref_layer.named_parameters()):
            errs[n] = nerr(p.grad, q.grad)
        ok = max(errs.values()) <= 1e-2
        bad = 0 if ok else 1
        print(json.dumps({"world": W, "inner": a.inner or W, "seq": S, "ok": ok,
                          "max_err": max(errs.values()), "errs": errs}))
    flag = torch.tensor([bad], device=dev)
    dist.broadcast(flag, 0)
    comm.destroy()
    dist.destroy_process_group()
    sys.exit(int(flag.item()))


if __name__ == "__main__":
    main()
