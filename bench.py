#!/usr/bin/env python
"""bench.py — MTraining hot path on B200 (arXiv 2510.18830, BASELINE.json metric).

One step = one pass of the whole hot path over one synthetic 512K-token
Qwen2.5-3B-shaped attention layer (16 q heads, 2 kv heads, d = 128):
  1. Alg. 1 vertical-slash index (mt_build_vs_index, bit-exact VS-IDX v1),
  2. block-sparse attention forward (ring over N GPUs, or one GPU),
  3. block-sparse attention backward (dQ, dK, dV).
Metric: sparse attention fwd+bwd tokens/s at 512K (whole job, max over ranks),
with the kernel-level roofline of the dominant kernel and the CPU oracle as a
reported baseline.  Usage:
  python bench.py [--gpus N --steps K --warmup W]            (N > 1 under torchrun)
  python bench.py --impl reference ...                        (CPU oracle arm)
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
# stdout carries exactly one JSON line: NCCL's log (its version banner is printed at
# WARN level too) goes to stderr
os.environ["NCCL_DEBUG"] = os.environ.get("MT_NCCL_DEBUG", "WARN")
os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")

METRIC = "sparse attn fwd+bwd tokens/s at 512K, 1/2/4/8 B200; % of bf16 tensor peak"
UNIT = "tokens/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seq", type=int, default=524288)
    ap.add_argument("--hq", type=int, default=16)
    ap.add_argument("--hkv", type=int, default=2)
    ap.add_argument("--p", type=float, default=0.9)
    ap.add_argument("--inner", type=int, default=0, help="hierarchical inner ring size (0 = flat)")
    ap.add_argument("--layout", default="striped", choices=["striped", "zigzag"],
                    help="sequence layout of the ranks: the method's 64-token block striping, or "
                         "the zigzag layout of the 'Ours w/ ZigZag' ablation (P:345)")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="replay the step as one CUDA graph (auto: single GPU and S <= 128K, where "
                         "the step is launch-bound)")
    return ap.parse_args()


def peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text()), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


# ------------------------------------------------------------------ clocks
class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md)."""

    def __init__(self, gpu_index: int):
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={gpu_index}", f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None

    def stop(self) -> dict:
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        self.p.wait()
        self.f.flush()
        rows = [r.split(",") for r in Path(self.f.name).read_text().splitlines() if r.strip()]
        sm = [float(r[1]) for r in rows if len(r) > 2 and r[1].strip().replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if len(r) > 2 and r[2].strip().replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows if len(r) >= 9 for i in range(4)
                          if r[5 + i].strip().lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(rows)}


def workload_name(args, W: int) -> str:
    cfg = {4096: "C1", 65536: "C2", 131072: "C3", 524288: "C4", 1048576: "C5"}.get(args.seq, "custom")
    ring = "flat" if not args.inner or args.inner == W else f"{W // args.inner}x{args.inner}"
    lay = "" if args.layout == "striped" else f", {args.layout} layout"
    return (f"{cfg}-shape layer at W={W}: S={args.seq}, Hq={args.hq}, Hkv={args.hkv}, d=128, "
            f"p_v=p_s={args.p}, {ring} ring{lay}")


# ------------------------------------------------------------------ layout helpers
def stripe_rows(S: int, W: int, r: int) -> np.ndarray:
    """Global token of each local row of rank r (64-token block striping)."""
    j = np.arange(S // W)
    return ((j // 64) * W + r) * 64 + j % 64


def zigzag_rows(S: int, W: int, r: int) -> np.ndarray:
    """Global token of each local row of rank r in the zigzag layout (Fig. 1):
    2W chunks, rank r holds chunk r then chunk 2W-1-r."""
    c = S // (2 * W)
    return np.r_[np.arange(r * c, r * c + c), np.arange((2 * W - 1 - r) * c, (2 * W - r) * c)]


def bits_to_torch(bits: np.ndarray, dev):
    import torch
    return torch.from_numpy(np.ascontiguousarray(bits).view(np.int16)).view(torch.bfloat16).to(dev)


# ------------------------------------------------------------------ CPU oracle leg
def blas_threads() -> int | None:
    try:
        from threadpoolctl import threadpool_info
        np.ones((64, 64)) @ np.ones((64, 64))  # load the BLAS so it is reported
        n = [x["num_threads"] for x in threadpool_info() if x.get("user_api") == "blas"]
        return int(max(n)) if n else None
    except Exception:
        return None


class OracleSampler:
    """The CPU oracle (oracle/, test infrastructure) timed on a bounded sample of the
    workload -- the `cpu_baseline` of our arm and every step of `--impl reference`
    (identical code and sample size, so the two legs agree within noise).

    Setup (untimed): the oracle's own Alg. 1 index of every q head (C helper, VS-IDX v1)
    and the true activated-pair total, counted by oracle.attention.count_pairs.
    One sampled step (timed): the full Alg. 1 index of ONE q head (head i mod Hq on step
    i) and the fp64 forward + backward of `n_blocks` query blocks of that head spread over
    the sequence.  Extrapolation to the whole job: index time x Hq, attention time x
    (total activated pairs / sampled pairs).  So `value` is a projection of tokens/s for
    the full workload; `sample_seconds` is what a step really took.
    """

    def __init__(self, q, k, v, dO, p: float, S: int, Hq: int, Hkv: int, n_blocks: int = 48):
        from oracle import attention as OA
        from oracle import vsidx
        from synth.generator import bf16_bits_to_f32
        self.q, self.k, self.v, self.dO = q, k, v, dO
        self.p, self.S, self.Hq, self.Hkv, self.nb_sample = p, S, Hq, Hkv, n_blocks
        self.grp = Hq // Hkv
        t0 = time.perf_counter()
        self.iv, self.is_ = vsidx.build_vs_index(bf16_bits_to_f32(q), bf16_bits_to_f32(k), p, p)
        self.setup_index_s = time.perf_counter() - t0
        self.pairs = OA.count_pairs(self.iv, self.is_, S)
        self.total_pairs = int(self.pairs.sum())
        self.step_i = 0

    def step(self) -> dict:
        from oracle import attention as OA
        from oracle import sparseformat as SF
        from oracle import vsidx
        from synth.generator import bf16_bits_to_f32
        S, h = self.S, self.step_i % self.Hq
        self.step_i += 1
        g_kv = h // self.grp
        f64 = lambda x: bf16_bits_to_f32(x).astype(np.float64)
        t_start = time.perf_counter()
        q_win = np.ascontiguousarray(bf16_bits_to_f32(self.q[S - 64:, h]))
        kk = np.ascontiguousarray(bf16_bits_to_f32(self.k[:, g_kv]))
        t0 = time.perf_counter()
        iv, is_ = vsidx.vs_index_head(q_win, kk, self.p, self.p)
        t_idx = time.perf_counter() - t0
        assert np.array_equal(iv, self.iv[h]) and np.array_equal(is_, self.is_[h])
        nb = S // 64
        gs = np.unique(np.linspace(0, nb - 1, self.nb_sample).astype(int))
        qh, kh, vh, dh = (f64(x[:, c:c + 1]) for x, c in
                          ((self.q, h), (self.k, g_kv), (self.v, g_kv), (self.dO, h)))
        O = np.zeros_like(qh)
        L = np.zeros((1, S))
        pairs = 0
        t0 = time.perf_counter()
        for g in gs:
            B, C = SF.sparseformat_block(iv, is_, int(g))
            rows = slice(g * 64, g * 64 + 64)
            O[rows, 0], L[0, rows] = OA.forward_block(qh, kh, vh, 0, int(g), B, C)
            OA.backward_block(qh, kh, vh, O, L, dh, 0, int(g), B, C)
            pairs += int(OA.count_pairs([iv], [is_], S, rows=[int(g)])[0])
        t_attn = time.perf_counter() - t0
        t_job = t_idx * self.Hq + t_attn * self.total_pairs / max(pairs, 1)
        return {"value": S / t_job, "unit": UNIT, "kind": "oracle",
                "cores": len(os.sched_getaffinity(0)), "blas_threads": blas_threads(),
                "sample": (f"q head {h}: Alg. 1 index in full ({t_idx:.2f} s, x{self.Hq} heads) + "
                           f"fp64 fwd+bwd of {len(gs)} of {nb} query blocks ({t_attn:.2f} s, "
                           f"{pairs} of {self.total_pairs} activated pairs, all heads counted); "
                           f"projected to the whole {S}-token job"),
                "sample_seconds": time.perf_counter() - t_start,
                "projected_seconds_per_step": t_job}


def oracle_c1_full() -> dict:
    """The oracle on BASELINE config C1 (4K tokens, 8 q / 1 kv heads) IN FULL: Alg. 1 index
    of every head, fp64 sparse forward and backward of every row."""
    from oracle import attention as OA
    from oracle import vsidx
    from synth.generator import bf16_bits_to_f32, make_grad_out, make_qkv
    S, Hq, Hkv = 4096, 8, 1
    q, k, v = make_qkv(S, Hq, Hkv, seed=0)
    dO = make_grad_out(S, Hq, seed=0)
    f64 = lambda x: bf16_bits_to_f32(x).astype(np.float64)
    t0 = time.perf_counter()
    iv, is_ = vsidx.build_vs_index(bf16_bits_to_f32(q), bf16_bits_to_f32(k), 0.9, 0.9)
    O, L = OA.sparse_attention_forward(f64(q), f64(k), f64(v), iv, is_)
    OA.sparse_attention_backward(f64(q), f64(k), f64(v), O, L, f64(dO), iv, is_)
    t = time.perf_counter() - t0
    return {"workload": "C1: S=4096, Hq=8, Hkv=1, p=0.9, index + fwd + bwd in full",
            "seconds": round(t, 3), "tokens_per_s": S / t}


# ------------------------------------------------------------------ our arm
def run_ours(args):
    import torch
    import torch.distributed as dist
    from paper_2510_18830_b200 import _lib, ops, stats
    from synth.generator import make_grad_out, make_qkv

    W = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if W != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={W}: launch with torchrun for N > 1")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = None
    if W > 1:
        dist.init_process_group("nccl", device_id=dev)
        comm = ops.Comm.create(W, rank, args.inner or W)
    S, Hq, Hkv, p = args.seq, args.hq, args.hkv, args.p
    q, k, v = make_qkv(S, Hq, Hkv, seed=args.seed)
    dO = make_grad_out(S, Hq, seed=args.seed)
    lay = args.layout
    rows = (stripe_rows if lay == "striped" else zigzag_rows)(S, W, rank) if W > 1 else np.arange(S)
    hq_, hk_, hv_, hdo = (np.ascontiguousarray(x[rows]) for x in (q, k, v, dO))
    qd, kd, vd, dOd = (bits_to_torch(x, dev) for x in (hq_, hk_, hv_, hdo))
    stream = torch.cuda.current_stream()

    ev = lambda: torch.cuda.Event(enable_timing=True)

    def step(qx, kx, vx, dox, marks=None, mid=None):
        """index + forward + backward; mid() (if given) runs between the forward and the
        backward (the e2e loop queues its host copies there)."""
        e = [ev() for _ in range(4)] if marks is not None else None
        if e: e[0].record(stream)
        idx = ops.build_vs_index(qx, kx, p, p, comm=comm, seq_len=S, layout=lay)
        if e: e[1].record(stream)
        if comm is None:
            o, lse = ops.sparse_attn_fwd(qx, kx, vx, idx)
        else:
            o, lse = ops.ring_attn_fwd(comm, S, qx, kx, vx, idx, layout=lay)
        if e: e[2].record(stream)
        if mid is not None:
            mid()
        if comm is None:
            g = ops.sparse_attn_bwd(qx, kx, vx, o, lse, dox, idx)
        else:
            g = ops.ring_attn_bwd(comm, S, qx, kx, vx, o, lse, dox, idx, layout=lay)
        if e:
            e[3].record(stream)
            marks.append(e)
        return idx, g

    def barrier():
        if W > 1:
            dist.barrier(device_ids=[local])

    for _ in range(args.warmup):
        idx, _ = step(qd, kd, vd, dOd)
    torch.cuda.synchronize()
    iv, is_ = idx.to_lists()
    pairs = int(stats.pairs_per_head(iv, is_, S).sum())
    dens = pairs / (Hq * stats.causal_pairs(S))

    # L2 rule (B200_PROFILING.md): inputs larger than L2 between timed steps, else an L2
    # flush between steps (outside the per-step CUDA-event windows)
    L2_BYTES = 126 * 2 ** 20
    in_bytes = sum(x.numel() * x.element_size() for x in (qd, kd, vd, dOd))
    flush = None if in_bytes > 2 * L2_BYTES else torch.empty(4 * L2_BYTES, dtype=torch.uint8, device=dev)
    lib = _lib.lib()
    clocks = Clocks(local)
    barrier()
    torch.cuda.synchronize()
    n_launch0, n_lib0 = lib.mt_launch_count(), lib.mt_library_call_count()
    t0, t1 = ev(), ev()
    marks = []
    t0.record(stream)
    for _ in range(args.steps):
        if flush is not None:
            flush.fill_(1)
        step(qd, kd, vd, dOd, marks)
    t1.record(stream)
    torch.cuda.synchronize()
    barrier()
    n_launch = lib.mt_launch_count() - n_launch0
    n_lib = lib.mt_library_call_count() - n_lib0
    clk = clocks.stop()
    if flush is None:
        ms = t0.elapsed_time(t1)
    else:  # sum of the steps' own windows (index start -> backward end), flushes excluded
        ms = float(sum(m[0].elapsed_time(m[3]) for m in marks))
    eager_ms = ms
    # ---- CUDA-graph replay of the whole step (index + fwd + bwd: ~17 own kernels and the
    # CUB sorts, launch-bound at small S).  Captured once after the eager warm-up; each
    # timed replay recomputes everything from the same device inputs.
    graph_info = None
    use_graph = args.graph == "on" or (args.graph == "auto" and W == 1 and S <= 131072)
    if use_graph and W == 1:
        g_stream = torch.cuda.Stream(device=dev)
        g_stream.wait_stream(stream)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.stream(g_stream):
            step(qd, kd, vd, dOd)  # allocations of the step's outputs happen before capture
            with torch.cuda.graph(graph, stream=g_stream):
                step(qd, kd, vd, dOd)
        stream.wait_stream(g_stream)
        for _ in range(args.warmup):
            graph.replay()
        torch.cuda.synchronize()
        n_launch0 = lib.mt_launch_count()
        gms = []
        for _ in range(args.steps):
            if flush is not None:
                flush.fill_(1)
            a_, b_ = ev(), ev()
            a_.record(stream)
            graph.replay()
            b_.record(stream)
            gms.append((a_, b_))
        torch.cuda.synchronize()
        ms = float(sum(a_.elapsed_time(b_) for a_, b_ in gms))
        graph_info = {"replayed_ms_per_step": ms / args.steps, "eager_ms_per_step": eager_ms / args.steps,
                      "note": "value = CUDA-graph replay of the step; phase_ms and roofline from the eager "
                              "pass (per-phase CUDA events)"}
    ph = np.array([[m[0].elapsed_time(m[1]), m[1].elapsed_time(m[2]), m[2].elapsed_time(m[3])]
                   for m in marks]).mean(axis=0)
    t_max = torch.tensor([ms], device=dev)  # eager or graph-replay total
    if W > 1:
        dist.all_reduce(t_max, op=dist.ReduceOp.MAX)
    ms = float(t_max.item())

    # ---- end to end through the public API with host buffers.  Every step's inputs
    # are copied host->device from pinned memory and its dQ/dK/dV device->host inside
    # the timed region; copies run on their own streams, double-buffered.  They are queued
    # behind each step's forward, so they run during its backward: step i+1's upload and
    # step i-1's download overlap step i's backward, and the copy engines stay free for
    # the forward ring's KV transfers (a 600 MB host copy queued ahead of a ring transfer
    # on the same engine stalls the ring).  MT_BENCH_E2E_EARLY=1 (the default on one GPU):
    # uploads queued at the start of the step, downloads at its end.
    e2e = None
    if not args.no_e2e:
        # one GPU (no ring): the upload of step i+1 starts with step i (at C1's 0.22 ms steps a
        # copy queued behind the forward delays the next step: e2e 6.2 vs 2.8 M tokens/s)
        early = os.environ.get("MT_BENCH_E2E_EARLY", "1" if W == 1 else "0") == "1"
        pin = [torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).pin_memory()
               for x in (hq_, hk_, hv_, hdo)]
        h2d = sum(x.numel() * 2 for x in pin)
        dbuf = [[torch.empty(x.shape, dtype=x.dtype, device=dev) for x in pin] for _ in range(2)]
        out_shapes = [(S // W, Hq, 128), (S // W, Hkv, 128), (S // W, Hkv, 128)]  # dQ, dK, dV bf16
        host_out = [[torch.empty(sh_, dtype=torch.bfloat16, pin_memory=True) for sh_ in out_shapes]
                    for _ in range(2)]  # pinned before the timed region (cudaHostAlloc syncs)
        cin, cout = torch.cuda.Stream(device=dev), torch.cuda.Stream(device=dev)
        ev_in = [torch.cuda.Event() for _ in range(2)]
        ev_done = [torch.cuda.Event() for _ in range(2)]
        keep = [None, None]
        barrier()
        torch.cuda.synchronize()
        a, b = ev(), ev()
        a.record(stream)

        def upload(i, after):
            bb = i % 2
            cin.wait_event(after)
            if i >= 2:
                cin.wait_event(ev_done[bb])  # step i-2 finished reading this buffer
            with torch.cuda.stream(cin):
                for d_, h_ in zip(dbuf[bb], pin):
                    d_.copy_(h_, non_blocking=True)
            ev_in[bb].record(cin)

        def download(i, after):
            bb = i % 2
            cout.wait_event(after)
            with torch.cuda.stream(cout):
                for hy, y in zip(host_out[bb], keep[bb]):
                    hy.copy_(y, non_blocking=True)
                    y.record_stream(cout)

        upload(0, a)
        d2h = 0
        for i in range(args.steps):
            bb = i % 2
            if early and i + 1 < args.steps:
                upload(i + 1, a)
            stream.wait_event(ev_in[bb])

            def mid(i=i):
                if early:
                    return
                fwd_done = torch.cuda.Event()
                fwd_done.record(stream)
                if i + 1 < args.steps:
                    upload(i + 1, fwd_done)
                if i >= 1:
                    download(i - 1, fwd_done)

            _, g = step(*dbuf[bb], mid=mid)
            ev_done[bb].record(stream)
            keep[bb] = g
            if early or i == args.steps - 1:
                download(i, ev_done[bb])
            d2h = sum(y.numel() * y.element_size() for y in g)
        stream.wait_stream(cout)
        b.record(stream)
        torch.cuda.synchronize()
        barrier()
        et = torch.tensor([a.elapsed_time(b)], device=dev)
        if W > 1:
            dist.all_reduce(et, op=dist.ReduceOp.MAX)
        e2e = {"value": S * args.steps / (float(et.item()) / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "copies": ("pinned host <-> device on two copy streams, double-buffered; queued at the start / end "
                             "of each step" if early else
                             "pinned host <-> device on two copy streams, double-buffered; step i+1's "
                             "upload and step i-1's download run during step i's backward")}

    # ---- ring step profile: one extra, untimed step with CUDA events
    # around each step's kernels and transfers (rank 0's view)
    ring = None
    if comm is not None:
        comm.profile(True)
        barrier()
        step(qd, kd, vd, dOd)
        torch.cuda.synchronize()
        ring = {"profiled": "one untimed step after the timed region, rank 0", "passes": {}}
        for name, bwd in (("fwd", False), ("bwd", True)):
            tt = np.array(comm.step_times(bwd))  # [steps][compute, inner, outer, dkv]
            kv = np.where(tt[:, 1] >= 0, tt[:, 1], tt[:, 2])
            kvb = 2 * (S // W) * Hkv * 128 * 2
            d = {"compute_ms_median": round(float(np.median(tt[:, 0])), 3),
                 "compute_ms_per_step": [round(float(x), 3) for x in tt[:, 0]],
                 "kv_bytes_per_step": kvb}
            # transfer events include waiting for the peer to post its receive: the
            # fastest step is the closest to wire time
            kvs = kv[kv > 0]
            if len(kvs):
                d["kv_ms_median"] = round(float(np.median(kvs)), 3)
                d["kv_ms_min"] = round(float(kvs.min()), 3)
                d["kv_gbps_best"] = round(kvb / (float(kvs.min()) / 1e3) / 1e9, 1)
            if bwd:
                dk = tt[:, 3][tt[:, 3] > 0]
                if len(dk):
                    dkb = 2 * (S // W) * Hkv * 128 * 4
                    d["dkv_bytes_per_step"] = dkb
                    d["dkv_ms_median"] = round(float(np.median(dk)), 3)
                    d["dkv_ms_min"] = round(float(dk.min()), 3)
                    d["dkv_gbps_best"] = round(dkb / (float(dk.min()) / 1e3) / 1e9, 1)
            ring["passes"][name] = d
        comm.profile(False)

    pk, pk_src = peaks()
    fl_bwd = 10 * 128 * pairs / W
    fl_fwd = 4 * 128 * pairs / W
    t_bwd, t_fwd = ph[2] / 1e3, ph[1] / 1e3
    ach = fl_bwd / t_bwd / 1e12
    roof = {"bound": "tensor", "kernel": ("attn_bwd per rank and ring step: slash-block launch + vertical-bar launch "
                                          "when nloc > 2048 blocks, else one mixed launch"),
            "achieved": round(ach, 1), "peak": pk["bf16_tflops_sustained"], "unit": "TFLOP/s",
            "frac": round(ach / pk["bf16_tflops_sustained"], 4),
            "peak_source": f"{pk_src} bf16 cuBLAS sustained (burst {pk['bf16_tflops']})",
            "traffic": None,
            "fwd_tflops": round(fl_fwd / t_fwd / 1e12, 1),
            "phase_ms": {"index": round(ph[0], 3), "fwd": round(ph[1], 3), "bwd": round(ph[2], 3)}}
    if W == 1:
        # live share of the backward block pass's 128-key MMA rows:
        # "achieved" counts algorithmic FLOPs; the block pass executes 1/occupancy of them
        from paper_2510_18830_b200 import balance
        occ = balance.bwd_slot_occupancy(is_, S // 64)
        roof["bwd_block_slot_occupancy"] = round(occ["occupancy"], 4)
    tr = ROOT / "profiles" / "traffic.json"
    if tr.exists():
        try:
            t = json.loads(tr.read_text())
            if t.get("seq_len") == S and t.get("world") == W:  # measured on this config only
                roof["traffic"] = t.get("attn_bwd_bytes_per_launch")
        except Exception:
            pass

    line = {"metric": METRIC, "value": S * args.steps / (ms / 1e3), "unit": UNIT, "n_gpus": W,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic (seeded RoPE vertical-slash generator, DESIGN.md §3)",
            "config": {"workload": workload_name(args, W),
                       "seq_len": S, "global_batch": 1, "parallelism": f"cp{W}",
                       "density": round(dens, 4), "activated_pairs": pairs,
                       "l2": (f"inputs larger than L2: Q/K/V/dO {in_bytes / 2 ** 30:.2f} GiB per rank "
                              f"vs 126 MB L2" if flush is None else
                              f"L2 flushed between steps (inputs {in_bytes / 2 ** 20:.1f} MiB per rank "
                              f"fit the 126 MB L2); per-step CUDA-event windows summed"),
                       **({"emulated_inter_node": {"gbps": float(os.environ["MT_EMU_INTER_GBPS"]),
                                                   "ranks_per_node": int(os.environ.get("MT_EMU_NODE", args.inner or W))}}
                          if os.environ.get("MT_EMU_INTER_GBPS") else {})},
            "roofline": roof, "e2e": e2e, "clocks": clk,
            **({"cuda_graph": graph_info} if graph_info else {}),
            **({"ring": ring} if ring else {}),
            # counted by libmtsa.so over the timed region (max over ranks is not needed: every
            # rank launches the same kernels); CUB sorts are library calls, counted apart
            "gpu_launches": int(n_launch),
            "gpu_launches_detail": {"own_kernels_per_step": n_launch / args.steps,
                                    "cub_radix_sort_calls_per_step": n_lib / args.steps}}
    if rank == 0 and W == 1 and not args.no_cpu_baseline:
        smp = OracleSampler(q, k, v, dO, p, S, Hq, Hkv)
        runs = [smp.step() for _ in range(3)]
        cb = dict(runs[-1])
        cb["value"] = float(np.median([r["value"] for r in runs]))
        cb["sample"] = (f"median of 3 sampled steps (q heads 0-2), each: " + runs[-1]["sample"])
        cb["c1_full"] = oracle_c1_full()
        line["cpu_baseline"] = cb
    if rank == 0:
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.destroy()
        dist.destroy_process_group()


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    """The CPU oracle as the reference arm (tier framing): each of the W + K steps is one
    OracleSampler step (the same code and sample size as our arm's cpu_baseline) of the
    same workload; rank 0 only."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from synth.generator import make_grad_out, make_qkv
    S, Hq, Hkv, p = args.seq, args.hq, args.hkv, args.p
    q, k, v = make_qkv(S, Hq, Hkv, seed=args.seed)
    dO = make_grad_out(S, Hq, seed=args.seed)
    smp = OracleSampler(q, k, v, dO, p, S, Hq, Hkv)
    runs = [smp.step() for _ in range(args.warmup + args.steps)][args.warmup:]
    val = float(np.median([r["value"] for r in runs]))
    wall = [r["sample_seconds"] for r in runs]
    line = {"metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup,
            # each step really took sample_seconds; the projected time of a full step is
            # reported beside it (value is the projection's tokens/s)
            "ms_per_step": float(np.mean(wall)) * 1e3,
            "projected_ms_per_full_step": S / val * 1e3,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f64 (attention), f32/u64 (index)",
            "data": "synthetic (seeded RoPE vertical-slash generator, DESIGN.md §3)",
            "config": {"workload": workload_name(args, args.gpus), "seq_len": S, "global_batch": 1,
                       "parallelism": f"cp{args.gpus} (the oracle runs on rank 0's host cores)"},
            "impl": "reference",
            "cpu_baseline": {"value": val, "unit": UNIT, "cores": runs[-1]["cores"],
                             "blas_threads": runs[-1]["blas_threads"], "kind": "oracle",
                             "sample": f"median of {len(runs)} sampled steps, each: " + runs[-1]["sample"],
                             "setup_index_seconds": round(smp.setup_index_s, 2)},
            "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    a = parse()
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)
