#!/usr/bin/env python
"""Benchmark of the sketch hot path (BASELINE.json metric) -- one JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--no-configs] [--no-cpu] [--share-gpu] [--c5-n N5]

Headline (BASELINE.json configs[1], "C2"): A = n x n Gaussian-kernel matrix,
n = 16384, x_i ~ U[0,1]^8 (seed = rank), h = 0.5, +1e-2 on the diagonal,
generated in HBM (2.15 GB, far larger than the 126 MB L2, so no flush is
needed between steps).  One STEP = the SJLT sketch S = A R^T with d = 512,
alpha = 4 (block construction, R drawn by the reference's generator with
SeedSequence((0, 0))), i.e. one full pass over A.  `value` is the A-streamed
GB/s of the whole job (sum over ranks / max-over-ranks time).  Beside it:
S' on the same A, the Gaussian d = 512 product (FP64 TFLOP/s, next to cuBLAS
DGEMM on the same operands), a sustained (>= 400 launch) figure, and the end
to end numbers through the public API from pinned and from pageable host
arrays.

Sub-records under "configs" (the other BASELINE.json configs, N = 1 only
unless noted): c1 (n = 4096 S and S', graph R, L2 flushed between launches),
c3_adaptive (the whole 16-increment S + S' schedule of configs[2]),
c4_srht (configs[3]) and c5 (configs[4], at EVERY N: strong-scaled
n = 131072 row-sharded over the ranks, S local + S' summed through the p2p
peer-store exchange, SJLT d = 2048 alpha = 8 and Gaussian d = 512).  Each
carries ms, its roofline fraction (MEASURED_PEAKS.json) and the CPU-port
baseline on a bounded slab of the same workload.

Multi-GPU: `--gpus N` without torchrun re-launches itself under
torch.distributed.run with N ranks (one per GPU; fails if fewer are
visible); under torchrun WORLD_SIZE must equal --gpus.  `--share-gpu` puts
every rank on GPU 0 with a gloo group (exercises the multi-rank path on a
one-GPU box; its timings are not scaling numbers).

--impl reference times the reference algorithm on the host CPU: the C
restatement in oracle/ (bit-exact with hsskit's SjltBlock.apply_right; the
reference itself is pure Python/numpy and is not shipped to the GPU box),
on all host cores, one bounded row slab of the same workload per step.
"""

from __future__ import annotations

import argparse
import contextlib
import gc
import json
import os
import socket
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N = 16384
D = 512
ALPHA = 4
DIM = 8
H = 0.5
METRIC = "sketch S=A·R^T: A-streamed GB/s (SJLT) and FP64 TFLOP/s (Gaussian) vs roofline"


def _peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback"


def _traffic_from_profiles(kernel_key: str):
    """Per-launch DRAM bytes of the kernel from the committed ncu summary."""
    path = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        with open(path) as f:
            prof = json.load(f)
        ent = prof["kernels"][kernel_key]
        return ent["dram_bytes_per_launch"]
    except Exception:  # noqa: BLE001
        return None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled in the background."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int, period_ms: int = 50):
        self.samples = []
        self.proc = None
        self.gpu = gpu_index
        self.period = period_ms
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", f"-lms={self.period}"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:  # noqa: BLE001
            self.proc = None
            return self
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.samples.append((time.perf_counter(), parts))

    def stop(self):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:  # noqa: BLE001
                self.proc.kill()

    def summary(self, t0: float, t1: float):
        win = [p for t, p in self.samples if t0 <= t <= t1]
        src = "timed_region"
        if not win:  # timed region shorter than the sampling period
            near = sorted(self.samples, key=lambda s: min(abs(s[0] - t0), abs(s[0] - t1)))[:3]
            win = [p for _, p in near]
            src = "nearest_samples"
        if not win:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0,
                    "source": "unavailable"}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(p[1]) for p in win if num(p[1]) is not None]
        pw = [num(p[3]) for p in win if num(p[3]) is not None]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for p in win:
            for name, v in zip(names, p[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": num(win[0][2]), "reasons": sorted(reasons),
                "power_w_max": max(pw) if pw else None,
                "samples": len(win), "source": src}


# --------------------------------------------------------------- reference

def host_kernel_slab(rows: int, seed: int = 0) -> np.ndarray:
    """Rows [0, rows) of the C2 Gaussian-kernel matrix computed on the host."""
    x = np.random.default_rng(seed).uniform(0.0, 1.0, (N, DIM))
    out = np.empty((rows, N), order="F")
    sq = np.sum(x * x, axis=1)
    for c0 in range(0, N, 2048):
        c1 = min(N, c0 + 2048)
        g = x[:rows] @ x[c0:c1].T
        d2 = np.maximum(sq[:rows, None] + sq[None, c0:c1] - 2.0 * g, 0.0)
        out[:, c0:c1] = np.exp(-d2 / (2 * H * H))
    idx = np.arange(rows)
    out[idx, idx] += 1e-2
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle as O
    from paper_2302_01977_b200 import draws
    threads = os.cpu_count() or 1
    pos, sg = draws.sjlt_draw(N, D, np.random.SeedSequence((0, 0)), ALPHA, "block")
    scale = 1.0 / np.sqrt(ALPHA)
    rows = int(os.environ.get("HSK_REF_ROWS", "2048"))
    slab = host_kernel_slab(rows)
    for _ in range(max(args.warmup, 1)):
        O.sjlt_right(slab, pos, sg, D, scale, nthreads=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        O.sjlt_right(slab, pos, sg, D, scale, nthreads=threads)
        times.append(time.perf_counter() - t0)
    t = statistics.median(times)
    gbs = slab.nbytes / t / 1e9
    sample = f"row slab {rows} x {N} of the C2 matrix per step (S rows are independent)"
    line = {
        "impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "c2_sjlt_S", "n": N, "d": D, "alpha": ALPHA,
                   "construction": "block", "rows_per_step": rows},
        "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": threads, "kind": "port",
                         "sample": sample},
        "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------- rank setup

class Ctx:
    """Rank, world, device and process group of this bench process."""

    def __init__(self, args):
        import torch
        import torch.distributed as dist
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        if self.world != args.gpus:
            raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={self.world}")
        if not torch.cuda.is_available():
            raise SystemExit("bench.py: no CUDA device visible")
        self.share = args.share_gpu
        self.dev_index = 0 if self.share else self.local
        if not self.share and torch.cuda.device_count() <= self.local:
            raise SystemExit(f"bench.py: rank {self.rank} needs GPU {self.local}, "
                             f"{torch.cuda.device_count()} visible")
        torch.cuda.set_device(self.dev_index)
        self.group = None
        if self.world > 1:
            if self.share:
                dist.init_process_group("gloo")
            else:
                dist.init_process_group("nccl", device_id=torch.device("cuda", self.local))
        self.dist = dist if self.world > 1 else None

    def barrier(self):
        if self.dist is not None:
            self.dist.barrier()

    def max_over_ranks(self, values):
        """Element-wise max of a list of floats over all ranks."""
        import torch
        if self.dist is None:
            return list(values)
        t = torch.tensor(list(values), dtype=torch.float64,
                         device="cpu" if self.share else "cuda")
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return [float(v) for v in t.tolist()]

    def close(self):
        if self.dist is not None:
            self.dist.barrier()
            self.dist.destroy_process_group()


def _free():
    import torch
    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()


def _events(n):
    import torch
    return [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            for _ in range(n)]


def time_launches(fn, reps: int, warmup: int, stream, flush=None):
    """Average device ms per call of fn over `reps` calls, each bracketed by
    CUDA events on `stream` (an optional L2 flush runs between calls, outside
    the events)."""
    import torch
    for _ in range(warmup):
        fn()
        if flush is not None:
            flush()
    torch.cuda.synchronize()
    evs = _events(reps)
    for e0, e1 in evs:
        e0.record(stream)
        fn()
        e1.record(stream)
        if flush is not None:
            flush()
    torch.cuda.synchronize()
    return statistics.mean(a.elapsed_time(b) for a, b in evs)


def fp64_tensor_peak(stream) -> float:
    """FP64 tensor-pipe TFLOP/s of this GPU, measured live (MEASURED_PEAKS.json
    has no FP64 entry): hsk_dmma_probe, best of 3."""
    import torch
    from paper_2302_01977_b200 import _lib
    L = _lib.load()
    x = torch.zeros(1, dtype=torch.float64, device="cuda")
    iters = 20000
    best = 0.0
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _lib.call("hsk_dmma_probe", iters, x.data_ptr(), stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize()
        best = max(best, L.hsk_dmma_probe_flops(iters) / (e0.elapsed_time(e1) * 1e-3) / 1e12)
    return best


def roofline(bytes_per_launch: float, ms: float, peak: float):
    ach = bytes_per_launch / (ms * 1e-3) / 1e9
    return {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
            "algorithmic_bytes_per_launch": int(bytes_per_launch), "avg_launch_ms": ms}


def cpu_rate(fn, nbytes: int, budget_s: float = 6.0, min_reps: int = 2):
    """Host GB/s of fn() streaming nbytes of A per call (median)."""
    fn()
    ts = []
    t_start = time.perf_counter()
    while len(ts) < min_reps or (time.perf_counter() - t_start < budget_s and len(ts) < 30):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    t = statistics.median(ts)
    return nbytes / t / 1e9, t, len(ts)


# --------------------------------------------------------------- headline

def run_headline(args, ctx, out):
    import torch
    from paper_2302_01977_b200 import device, matgen
    from paper_2302_01977_b200 import sketching as sk

    world, rank = ctx.world, ctx.rank
    stream = torch.cuda.current_stream()
    sptr = stream.cuda_stream
    op = sk.new_operator(sk.SJLT, N, D, np.random.SeedSequence((0, 0)), alpha=ALPHA,
                         construction=sk.BLOCK)
    blk = op.blocks[0]
    A = matgen.gaussian_kernel(N, DIM, H, 1e-2, seed=rank)
    S = device.DeviceMatrix.empty(N, D)
    device.block_state(blk)
    torch.cuda.synchronize()

    def sjlt(trans=False, o=S):
        device.apply_block(blk, A, trans, o, 0, sptr)

    for _ in range(args.warmup):
        sjlt()
    torch.cuda.synchronize()

    sampler = ClockSampler(torch.cuda.current_device()).start()
    time.sleep(0.3)
    evs = _events(args.steps)
    ctx.barrier()
    torch.cuda.synchronize()
    t_wall0 = time.perf_counter()
    g0 = torch.cuda.Event(enable_timing=True)
    g1 = torch.cuda.Event(enable_timing=True)
    g0.record(stream)
    for e0, e1 in evs:
        e0.record(stream)
        sjlt()
        e1.record(stream)
    g1.record(stream)
    torch.cuda.synchronize()
    t_wall1 = time.perf_counter()
    ctx.barrier()
    total_ms = g0.elapsed_time(g1)
    launch_ms = [a.elapsed_time(b) for a, b in evs]
    total_ms, = ctx.max_over_ranks([total_ms])

    # sustained: >= 400 back-to-back launches (the board's 1 kW cap engages
    # within ~100 ms of this kernel; the K-step region above is a burst when K
    # is small)
    sus_n = 400
    sus_evs = _events(sus_n)
    t_sus0 = time.perf_counter()
    for e0, e1 in sus_evs:
        e0.record(stream)
        sjlt()
        e1.record(stream)
    torch.cuda.synchronize()
    t_sus1 = time.perf_counter()
    sus_ms = statistics.mean(a.elapsed_time(b) for a, b in sus_evs)
    time.sleep(0.25)
    sampler.stop()
    clocks = sampler.summary(t_wall0, t_wall1)
    clocks_sus = sampler.summary(t_sus0, t_sus1)

    ms_per_step = total_ms / args.steps
    a_bytes = N * N * 8
    s_bytes = N * D * 8
    value = world * a_bytes / (ms_per_step * 1e-3) / 1e9
    avg_launch = statistics.mean(launch_ms)
    peak, peak_src = _peaks()
    roof = roofline(a_bytes + s_bytes, avg_launch, peak)
    roof["peak_source"] = peak_src
    roof["traffic"] = _traffic_from_profiles("sjlt_apply_S")

    # S' = A^T R^T on the same A (same algorithmic bytes)
    St = device.DeviceMatrix.empty(N, D)
    st_ms = time_launches(lambda: sjlt(True, St), max(20, min(args.steps, 100)), 3, stream)

    # Gaussian d=512 on the same A (the config's comparison) + cuBLAS DGEMM
    gop = sk.new_operator(sk.GAUSSIAN, N, D, np.random.SeedSequence((0, 0)))
    gblk = gop.blocks[0]
    gst = device.block_state(gblk)
    SG = device.DeviceMatrix.empty(N, D)
    g_ms = time_launches(lambda: device.apply_block(gblk, A, False, SG, 0, sptr), 5, 2, stream)
    gt_ms = time_launches(lambda: device.apply_block(gblk, A, True, SG, 0, sptr), 5, 2, stream)
    flops = 2.0 * N * N * D
    At = A.t[:, :N]               # (cols, rows) = A^T as a row-major tensor
    holder = {}

    def cublas():
        holder["c"] = torch.matmul(gst.R, At)   # R A^T = (A R^T)^T, cuBLAS DGEMM
    cublas_ms = time_launches(cublas, 5, 2, stream)
    holder.clear()
    del SG, St
    fp64_peak = fp64_tensor_peak(stream)

    # end to end through the public API: host A -> H2D -> kernel -> D2H S
    e2e = e2e_pageable = None
    host = torch.empty((N, N), dtype=torch.float64, pin_memory=True)
    host.copy_(A.t[:, :N])
    A_host = host.numpy().T           # F-ordered view of the pinned buffer
    e2e_steps = max(3, min(args.steps, 10))
    # warm-up as steady state looks: each call returns a fresh caller-owned
    # pinned array while the caller still holds the previous one, so the
    # second call is the one that grows the pinned pool (a one-time
    # cudaHostAlloc, ~27 ms measured)
    for _ in range(max(3, args.warmup)):
        S_host = sk.apply_right(A_host, op)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ctx.barrier()
    e0.record(stream)
    for _ in range(e2e_steps):
        S_host = sk.apply_right(A_host, op)
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms, = ctx.max_over_ranks([e0.elapsed_time(e1) / e2e_steps])
    e2e = {"value": world * a_bytes / (e2e_ms * 1e-3) / 1e9, "unit": "GB/s",
           "h2d_bytes_per_step": a_bytes, "d2h_bytes_per_step": int(S_host.nbytes),
           "ms_per_step": e2e_ms, "path": "sketching.apply_right(pinned host array)"}
    # the same call on a plain (pageable) numpy array -- what hsskit hands over
    page = np.empty((N, N), order="F")
    page[...] = A_host
    del host, A_host
    for _ in range(max(3, args.warmup)):   # staging + result buffers into the pinned pool
        S_host = sk.apply_right(page, op)
    torch.cuda.synchronize()
    ctx.barrier()
    t0 = time.perf_counter()
    e0.record(stream)
    for _ in range(e2e_steps):
        S_host = sk.apply_right(page, op)
    e1.record(stream)
    torch.cuda.synchronize()
    pg_ms, = ctx.max_over_ranks([e0.elapsed_time(e1) / e2e_steps])
    e2e_pageable = {"value": world * a_bytes / (pg_ms * 1e-3) / 1e9, "unit": "GB/s",
                    "h2d_bytes_per_step": a_bytes, "d2h_bytes_per_step": int(S_host.nbytes),
                    "ms_per_step": pg_ms, "path": "sketching.apply_right(pageable numpy array)"}
    del page, S_host

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        from oracle import oracle as O
        threads = os.cpu_count() or 1
        rows = 2048
        slab = np.asfortranarray(A.row_view(0, rows).to_host())
        gbs, t, reps = cpu_rate(lambda: O.sjlt_right(slab, blk._pos, blk._signs, D, blk._scale,
                                                     nthreads=threads), slab.nbytes, 10.0, 3)
        cpu = {"value": gbs, "unit": "GB/s", "cores": threads, "kind": "port",
               "sample": f"oracle SjltBlock.apply_right restatement on a {rows} x {N} row slab "
                         f"of the same A, median of {reps}"}
        # Gaussian: the reference's GaussianBlock.apply_right is numpy's
        # `buf @ matrix.T` (OpenBLAS dgemm, sketching.py:134-135) -- timed as is on
        # the same slab, at every host core and at one thread
        gflop = 2.0 * rows * N * D / 1e9
        Rh = gblk.matrix
        rates = {}
        try:
            from threadpoolctl import threadpool_limits
        except ImportError:  # pragma: no cover
            threadpool_limits = None
        for nth in (threads, 1):
            if threadpool_limits is None and nth == 1:
                continue
            ctxm = threadpool_limits(limits=nth) if threadpool_limits else contextlib.nullcontext()
            with ctxm:
                _, tg, rg = cpu_rate(lambda: slab @ Rh.T, slab.nbytes, 6.0, 2)
            rates[nth] = (gflop / tg / 1e3, rg)
        cpu["gaussian"] = {"value": rates[threads][0], "unit": "TFLOP/s", "cores": threads,
                           "value_1_thread": rates.get(1, (None,))[0], "kind": "reference",
                           "sample": f"numpy (OpenBLAS) slab @ R^T on the {rows} x {N} slab, "
                                     f"d={D}: the reference GaussianBlock.apply_right itself"}
    del A, S
    _free()

    out.update({
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": "c2_sjlt_S", "n": N, "d": D, "alpha": ALPHA,
                   "construction": "block", "matrix": "gaussian kernel 8-D h=0.5",
                   "parallelism": f"rowshard{world}" + ("-shared-gpu" if ctx.share else ""),
                   "l2": "inputs larger than L2 (2.15 GB A)"},
        "roofline": roof,
        "gpu_launches": args.steps,
        "clocks": clocks,
        "sustained": {"launches": sus_n, "avg_launch_ms": sus_ms,
                      "frac": (a_bytes + s_bytes) / (sus_ms * 1e-3) / 1e9 / peak,
                      "clocks": clocks_sus},
        "e2e": e2e,
        "e2e_pageable": e2e_pageable,
        "cpu_baseline": cpu,
        "transposed": {"metric": "S'=A^T R^T A-streamed GB/s", "ms": st_ms,
                       "value": a_bytes / (st_ms * 1e-3) / 1e9,
                       "frac": (a_bytes + s_bytes) / (st_ms * 1e-3) / 1e9 / peak},
        "gaussian": {"metric": "FP64 TFLOP/s, S=A R^T d=512 (DMMA)", "ms": g_ms,
                     "value": flops / (g_ms * 1e-3) / 1e12, "unit": "TFLOP/s",
                     "transposed_ms": gt_ms,
                     "transposed_value": flops / (gt_ms * 1e-3) / 1e12,
                     "cublas_dgemm_ms": cublas_ms,
                     "cublas_dgemm_tflops": flops / (cublas_ms * 1e-3) / 1e12,
                     "vs_cublas": cublas_ms / g_ms,
                     "roofline": {"bound": "tensor", "achieved": flops / (g_ms * 1e-3) / 1e12,
                                  "peak": fp64_peak, "unit": "TFLOP/s",
                                  "frac": flops / (g_ms * 1e-3) / 1e12 / fp64_peak,
                                  "cublas_frac": flops / (cublas_ms * 1e-3) / 1e12 / fp64_peak,
                                  "peak_source": "measured live: hsk_dmma_probe (independent "
                                                 "DMMA.8x8x4 chains on every SM)"}},
    })


# ------------------------------------------------------------ sub-records

def cfg_c1(args, peak):
    """configs[0]: n = 4096, SJLT d = 256, alpha = 4, graph construction; S and
    S' per launch with the 126 MB L2 flushed between launches (A is 134 MB)."""
    import torch
    from paper_2302_01977_b200 import _lib, device, matgen
    from paper_2302_01977_b200 import sketching as sk
    n, d = 4096, 256
    stream = torch.cuda.current_stream()
    A = matgen.gaussian_kernel(n, 8, 0.5)
    op = sk.new_operator(sk.SJLT, n, d, np.random.SeedSequence((0, 0)), alpha=4,
                         construction=sk.GRAPH)
    blk = op.blocks[0]
    device.block_state(blk)
    S = device.DeviceMatrix.empty(n, d)
    scratch = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def flush():
        _lib.call("hsk_l2_flush", scratch.data_ptr(), scratch.numel(), stream.cuda_stream)
    bytes_ = n * n * 8 + n * d * 8
    s_ms = time_launches(lambda: device.apply_block(blk, A, False, S, 0), 200, 5, stream, flush)
    t_ms = time_launches(lambda: device.apply_block(blk, A, True, S, 0), 200, 5, stream, flush)
    rec = {"workload": "c1: n=4096 gaussian kernel, SJLT d=256 alpha=4 graph, S and S'",
           "l2": "flushed between launches", "S_ms": s_ms, "St_ms": t_ms,
           "roofline_S": roofline(bytes_, s_ms, peak), "roofline_St": roofline(bytes_, t_ms, peak),
           "gpu_launches": 400}
    if not args.no_cpu:
        from oracle import oracle as O
        Ah = A.to_host()
        th = os.cpu_count() or 1
        gbs, t, reps = cpu_rate(lambda: O.sjlt_right(Ah, blk._pos, blk._signs, d, blk._scale,
                                                     nthreads=th), Ah.nbytes, 4.0)
        gbs_t, t_t, _ = cpu_rate(lambda: O.sjlt_right_t(Ah, blk._pos, blk._signs, d, blk._scale,
                                                        nthreads=th), Ah.nbytes, 4.0)
        rec["cpu_baseline"] = {"value": gbs, "unit": "GB/s", "St_value": gbs_t, "cores": th,
                               "kind": "port", "sample": f"full C1 S and S' (median of {reps})",
                               "S_ms": t * 1e3, "St_ms": t_t * 1e3}
    del A, S, scratch
    _free()
    return rec


def cfg_c3(args, peak):
    """configs[2]: the adaptive schedule (16 increments of 64 columns, alpha = 8,
    S and S' extended in place per increment) on the n = 65536 Toeplitz-sine A."""
    import torch
    from paper_2302_01977_b200 import adaptive, device, matgen
    from paper_2302_01977_b200 import sketching as sk
    n, dd, incs, alpha = 65536, 64, 16, 8
    stream = torch.cuda.current_stream()
    A = matgen.toeplitz_sin(n)
    ops = [sk.new_operator(sk.SJLT, n, dd, np.random.SeedSequence((0, 0)), alpha=alpha,
                           construction=sk.BLOCK)]
    for i in range(1, incs):
        ops.append(sk.append_columns(ops[-1], dd, np.random.SeedSequence((0, i))))
    for b in ops[-1].blocks:
        device.block_state(b)
    ds = adaptive.DeviceSketch(A, dd * incs)

    def step():
        ds.start(ops[0])
        for o in ops[1:]:
            ds.extend(o)
    ms = time_launches(step, 5, 3, stream)
    a_bytes = 8 * n * n
    per = a_bytes + 8 * n * dd
    rec = {"workload": "c3_adaptive: n=65536 toeplitz-sine, 16 x 64-column SJLT increments "
                       "alpha=8, S and S' per increment",
           "ms_per_schedule": ms, "products": ds.products_per_schedule(incs),
           "A_passes": ds.passes_per_schedule(incs),
           "value": ds.passes_per_schedule(incs) * a_bytes / (ms * 1e-3) / 1e9, "unit": "GB/s",
           "fused": ds.fused,
           "roofline": roofline(ds.passes_per_schedule(incs) * per, ms, peak),
           "gpu_launches": 5 * ds.launches_per_schedule(incs)}
    rec["roofline"]["note"] = ("achieved = algorithmic bytes of the schedule's passes over A "
                               "(A + the increment's S and S' columns per pass) / schedule time; "
                               "from the fifth extension on S' runs as A^T R^T on a transposed "
                               "copy made once per schedule (its 2 x bytes(A) and time included)")
    rec["kept_transpose"] = ds.At is not None
    if not args.no_cpu:
        from oracle import oracle as O
        blk = ops[0].blocks[0]
        rows = np.asfortranarray(A.row_view(0, 256).to_host())
        cols = np.asfortranarray(A.to_host(0, 256))
        th = os.cpu_count() or 1
        gbs, _, _ = cpu_rate(lambda: O.sjlt_right(rows, blk._pos, blk._signs, dd, blk._scale,
                                                  nthreads=th), rows.nbytes, 3.0)
        gbs_t, _, _ = cpu_rate(lambda: O.sjlt_right_t(cols, blk._pos, blk._signs, dd, blk._scale,
                                                      nthreads=th), cols.nbytes, 3.0)
        sched_s = incs * (a_bytes / (gbs * 1e9) + a_bytes / (gbs_t * 1e9))
        rec["cpu_baseline"] = {"value": 2 * incs * a_bytes / sched_s / 1e9, "unit": "GB/s",
                               "cores": th, "kind": "port",
                               "sample": "one 64-column block on a 256-row slab (S) and a "
                                         "256-column slab (S'), extrapolated to the schedule",
                               "schedule_s_extrapolated": sched_s}
    del A, ds
    _free()
    return rec


def cfg_c4(args, peak):
    """configs[3]: SRHT d = 512 on the n = 2^16 Gaussian kernel (h = 0.25)."""
    import torch
    from paper_2302_01977_b200 import device, matgen
    from paper_2302_01977_b200 import sketching as sk
    n, d = 65536, 512
    stream = torch.cuda.current_stream()
    A = matgen.gaussian_kernel(n, 8, 0.25)
    op = sk.new_operator(sk.SRHT, n, d, np.random.SeedSequence((0, 0)))
    blk = op.blocks[0]
    device.block_state(blk)
    S = device.DeviceMatrix.empty(n, d)
    s_ms = time_launches(lambda: device.apply_block(blk, A, False, S, 0), 10, 2, stream)
    t_ms = time_launches(lambda: device.apply_block(blk, A, True, S, 0), 10, 2, stream)
    bytes_ = 8 * n * n + 8 * n * d
    rec = {"workload": "c4_srht: n=65536 gaussian kernel h=0.25, SRHT d=512, S and S'",
           "S_ms": s_ms, "St_ms": t_ms, "roofline_S": roofline(bytes_, s_ms, peak),
           "roofline_St": roofline(bytes_, t_ms, peak), "gpu_launches": 20}
    if not args.no_cpu:
        from oracle import oracle as O
        rows = np.asfortranarray(A.row_view(0, 64).to_host())
        th = os.cpu_count() or 1
        gbs, _, _ = cpu_rate(lambda: O.srht(rows, blk.signs, blk.sample, d, blk.scale, False,
                                            nthreads=th), rows.nbytes, 4.0)
        rec["cpu_baseline"] = {"value": gbs, "unit": "GB/s", "cores": th, "kind": "port",
                               "sample": "SrhtBlock._transform restatement on a 64-row slab"}
    del A, S
    _free()
    return rec


def cfg_c5(args, ctx, peak):
    """configs[4] at this world size, strong-scaled: n = n5 (131072) rows
    sharded over the ranks; per rank S = A_g R^T (local) and S' through the
    p2p exchange (distributed.sketch_row_sharded), SJLT d = 2048 alpha = 8 and
    Gaussian d = 512.  Device times, max over ranks."""
    import torch
    from paper_2302_01977_b200 import device, matgen
    from paper_2302_01977_b200 import distributed as hd
    from paper_2302_01977_b200 import sketching as sk
    n = args.c5_n
    world, rank = ctx.world, ctx.rank
    stream = torch.cuda.current_stream()
    r0, r1 = hd.shard_bounds(n, world)[rank]
    pts = matgen.kernel_points(n, 16, 0)
    A = matgen.gaussian_kernel(n, 16, 1.0, 1e-2, row0=r0, nrows=r1 - r0, points=pts)
    rec = {"workload": f"c5: n={n} gaussian kernel 16-D h=1.0 row-sharded over {world} rank(s); "
                       "S local, S' via p2p peer stores + rank-ordered sum",
           "n": n, "rows_per_rank": r1 - r0, "scaling": "strong", "transport": "p2p"}
    a_bytes = 8 * n * n
    res = {}
    for kind, d, kw in (("sjlt", 2048, dict(alpha=8, construction=sk.BLOCK)),
                        ("gaussian", 512, {})):
        op = sk.new_operator(kind, n, d, np.random.SeedSequence((0, 0)), **kw)
        sub = hd._restricted_cached(op, r0, r1)
        for b in op.blocks + sub.blocks:
            device.block_state(b)
        S = device.DeviceMatrix.empty(r1 - r0, d)
        reps, warm = (5, 3) if kind == "sjlt" else (2, 1)

        def fS():
            sk.apply_right_device(A, op, out=S)

        def fSt():
            try:
                hd.sketch_row_sharded(A, op, rank=rank, world=world, n_rows=n,
                                      transport=rec["transport"], local_right=lambda *_: None)
            except hd.PeerMappingError:   # raised on every rank together: all fall back
                rec["transport"] = "nccl"
                rec["workload"] = rec["workload"].replace("p2p peer stores + rank-ordered sum",
                                                          "NCCL reduce-scatter")
                fSt()
        ctx.barrier()
        s_ms = time_launches(fS, reps, warm, stream)
        ctx.barrier()
        t_ms = time_launches(fSt, reps, warm, stream)
        s_ms, t_ms = ctx.max_over_ranks([s_ms, t_ms])
        ent = {"S_ms": s_ms, "St_ms": t_ms, "step_ms": s_ms + t_ms}
        if kind == "sjlt":
            per = a_bytes / world + 8 * (r1 - r0) * d
            ent["value"] = 2 * a_bytes / ((s_ms + t_ms) * 1e-3) / 1e9
            ent["unit"] = "GB/s (A-streamed, S and S', whole job)"
            ent["roofline_S"] = roofline(per, s_ms, peak)
            ent["roofline_St"] = roofline(per, t_ms, peak)
            ent["roofline_St"]["note"] = "S' time includes the peer-store exchange and the slot sum"
        else:
            fl = 2.0 * n * n * d
            ent["value"] = 2 * fl / ((s_ms + t_ms) * 1e-3) / 1e12
            ent["unit"] = "TFLOP/s (FP64, S and S', whole job)"
            ent["S_tflops"] = fl / (s_ms * 1e-3) / 1e12
        res[kind] = ent
        del S
        _free()
    rec.update(res)
    if rank == 0 and world == 1 and not args.no_cpu:
        from oracle import oracle as O
        th = os.cpu_count() or 1
        op = sk.new_operator(sk.SJLT, n, 2048, np.random.SeedSequence((0, 0)), alpha=8,
                             construction=sk.BLOCK)
        blk = op.blocks[0]
        rows = np.asfortranarray(A.row_view(0, 64).to_host())
        gbs, _, _ = cpu_rate(lambda: O.sjlt_right(rows, blk._pos, blk._signs, 2048, blk._scale,
                                                  nthreads=th), rows.nbytes, 4.0)
        rec["cpu_baseline"] = {"value": gbs, "unit": "GB/s", "cores": th, "kind": "port",
                               "sample": "SJLT d=2048 S on a 64-row slab of the C5 matrix"}
    hd.release_peer_slots()
    del A
    _free()
    return rec


# --------------------------------------------------------------------- main

def _relaunch(args) -> int:
    """--gpus N > 1 without torchrun: run this script under
    torch.distributed.run with N ranks on this node."""
    import torch
    if not args.share_gpu and torch.cuda.device_count() < args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but {torch.cuda.device_count()} GPU(s) "
                                   "visible"}), flush=True)
        return 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline legs")
    ap.add_argument("--no-configs", action="store_true",
                    help="headline only (skip the c1/c3/c4/c5 sub-records)")
    ap.add_argument("--configs", default="c1,c3,c4,c5",
                    help="comma list of sub-records to run (N = 1: c1,c3,c4,c5; N > 1: c5)")
    ap.add_argument("--share-gpu", action="store_true",
                    help="all ranks on GPU 0 (gloo group): exercises the multi-rank path")
    ap.add_argument("--c5-n", type=int, default=131072)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(_relaunch(args))

    ctx = Ctx(args)
    from paper_2302_01977_b200 import _lib
    _lib.load()
    out = {}
    run_headline(args, ctx, out)
    peak, _ = _peaks()
    configs = {}
    want = [] if args.no_configs else [c for c in args.configs.split(",") if c]
    single = ctx.world == 1
    for name, fn in (("c1", cfg_c1), ("c3_adaptive", cfg_c3), ("c4_srht", cfg_c4)):
        if single and name.split("_")[0] in want:
            configs[name] = fn(args, peak)
    if "c5" in want:
        configs["c5"] = cfg_c5(args, ctx, peak)
    if configs:
        out["configs"] = configs
    if ctx.rank == 0:
        print(json.dumps(out), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
