"""Multi-process host logic on CPU (gloo, world size 2): schedule agreement,
unique-id style broadcast, block striping / un-striping round trip, zigzag row map."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ring as OR
from paper_2510_18830_b200 import ops


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # 1. every rank derives the same schedule from the library (host code)
    sched = torch.tensor(ops.ring_schedule(4, 2)).flatten()
    gathered = [torch.empty_like(sched) for _ in range(world)]
    dist.all_gather(gathered, sched)
    same = all(torch.equal(g, gathered[0]) for g in gathered)
    # 2. opaque 128-byte id broadcast (as Comm.create does for the NCCL id)
    ids = [bytes(range(128))] if rank == 0 else [None]
    dist.broadcast_object_list(ids, src=0)
    # 3. stripe -> all_gather -> un-stripe round trip (P:277 layout)
    S = 1024
    x = torch.arange(S, dtype=torch.float32)
    j = np.arange(S // world)
    rows = torch.from_numpy(((j // 64) * world + rank) * 64 + j % 64)
    parts = [torch.empty(S // world) for _ in range(world)]
    dist.all_gather(parts, x[rows].contiguous())
    y = torch.empty(S)
    for r in range(world):
        rr = torch.from_numpy(((j // 64) * world + r) * 64 + j % 64)
        y[rr] = parts[r]
    # 4. the zigzag layout's host row map (bench.zigzag_rows, the rows each rank feeds the
    # kernels) round-trips the same way and equals the oracle's permutation
    import bench
    from oracle.sparseformat import zigzag_perm
    zr = [torch.from_numpy(bench.zigzag_rows(S, world, r)) for r in range(world)]
    dist.all_gather(parts, x[zr[rank]].contiguous())
    z = torch.empty(S)
    for r in range(world):
        z[zr[r]] = parts[r]
    zz_ok = torch.equal(x, z) and all(np.array_equal(zr[r].numpy(), zigzag_perm(S, world)[r]) for r in range(world))
    out[rank] = int(same and ids[0] == bytes(range(128)) and torch.equal(x, y) and zz_ok)
    dist.destroy_process_group()


def test_gloo_world2_host_logic():
    world = 2
    out = mp.Manager().dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert dict(out) == {0: 1, 1: 1}


def test_library_schedule_matches_oracle():
    for W, G in [(1, None), (2, None), (4, None), (4, 2), (8, 4), (8, 2), (6, 3)]:
        assert ops.ring_schedule(W, G) == OR.schedule(W, G)


def test_bench_layout_rows_match_oracle():
    import bench
    from oracle.sparseformat import layout_perm
    for S, W in ((4096, 1), (4096, 2), (8192, 4), (131072, 8)):
        for r in range(W):
            assert np.array_equal(bench.stripe_rows(S, W, r), layout_perm(S, W, "striped")[r])
            assert np.array_equal(bench.zigzag_rows(S, W, r), layout_perm(S, W, "zigzag")[r])
