#!/usr/bin/env python
"""Kernel micro-benchmark: CUDA-event time per launch for the sketch kernels
on BASELINE.json shapes (tuning aid; bench.py is the official measurement).

    python tools/kbench.py [--cases c1,c2s,c2g,c3] [--reps 20]
Env overrides HSK_SJLT_CFG / HSK_GAUSS_CFG select kernel variants.
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_01977_b200 import device, matgen  # noqa: E402
from paper_2302_01977_b200 import sketching as sk  # noqa: E402

def _peak():
    """HBM copy GB/s from MEASURED_PEAKS.json (driver-written), else the
    profiling recipe's fallback."""
    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"])
    except Exception:  # noqa: BLE001
        return 6455.9


PEAK = _peak()


def timeit(fn, reps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--cases", default="c1,c2s,c2g,c3,c4")
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    cases = args.cases.split(",")
    out = {}
    mats = {}

    def mat(n, dim=8, h=0.5, kind="gauss"):
        key = (n, dim, h, kind)
        if key not in mats:
            mats.clear()
            torch.cuda.empty_cache()
            mats[key] = (matgen.toeplitz_sin(n) if kind == "toep" else
                         matgen.gaussian_kernel(n, dim, h))
        return mats[key]

    for c in cases:
        if c in ("c1", "c2s", "c5s"):
            n, d, a, cons = {"c1": (4096, 256, 4, "graph"), "c2s": (16384, 512, 4, "block"),
                             "c5s": (32768, 2048, 8, "block")}[c]
            A = mat(n)
            op = sk.new_operator(sk.SJLT, n, d, np.random.SeedSequence((0, 0)), alpha=a,
                                 construction=cons)
            blk = op.blocks[0]
            S = device.DeviceMatrix.empty(n, d)
            flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if n <= 4096 else None

            def run(tr, S=S, blk=blk, A=A, flush=flush):
                if flush is not None:
                    flush.zero_()
                device.apply_block(blk, A, tr, S, 0)
            for tr in (False, True):
                if flush is not None:
                    t_fl = timeit(lambda: flush.zero_(), args.reps)
                else:
                    t_fl = 0.0
                ms = timeit(lambda: run(tr), args.reps) - t_fl
                byt = n * n * 8 + n * d * 8
                out[f"{c}_{'St' if tr else 'S'}"] = {"ms": ms, "GBs": byt / ms / 1e6,
                                                     "frac": byt / ms / 1e6 / PEAK}
        elif c.startswith("sj-"):  # sj-<n>-<d>-<alpha>: square Gaussian-kernel A, block construction
            n, d, a = (int(x) for x in c.split("-")[1:4])
            A = mat(n)
            op = sk.new_operator(sk.SJLT, n, d, np.random.SeedSequence((0, 0)), alpha=a,
                                 construction="block")
            blk = op.blocks[0]
            S = device.DeviceMatrix.empty(n, d)
            for tr in (False, True):
                ms = timeit(lambda: device.apply_block(blk, A, tr, S, 0), args.reps)
                byt = n * n * 8 + n * d * 8
                out[f"{c}_{'St' if tr else 'S'}"] = {"ms": ms, "GBs": byt / ms / 1e6,
                                                     "frac": byt / ms / 1e6 / PEAK}
        elif c in ("c5shard", "c5shard_t"):
            # BASELINE configs[4] at 8 GPUs: the 16384 x 131072 row shard of the
            # n = 131072 kernel matrix; S = A_g R^T (d = 2048, alpha = 8) and the
            # shard's S' partial A_g^T R_g^T (16384 input indices, 131072 output rows)
            n, rows, d = 131072, 16384, 2048
            key = ("c5shard",)
            if key not in mats:
                mats.clear()
                torch.cuda.empty_cache()
                pts = matgen.kernel_points(n, 16, 0)
                mats[key] = matgen.gaussian_kernel(n, 16, 1.0, 1e-2, row0=0, nrows=rows, points=pts)
            A = mats[key]
            op = sk.new_operator(sk.SJLT, n, d, np.random.SeedSequence((0, 0)), alpha=8,
                                 construction="block")
            if c == "c5shard":
                blk = op.blocks[0]
                S = device.DeviceMatrix.empty(rows, d)
                ms = timeit(lambda: device.apply_block(blk, A, False, S, 0), max(3, args.reps // 4))
                byt = rows * n * 8 + rows * d * 8
                out["c5shard_S"] = {"ms": ms, "GBs": byt / ms / 1e6, "frac": byt / ms / 1e6 / PEAK}
            else:
                from paper_2302_01977_b200 import distributed as hd
                sub = hd.restrict_operator(op, 0, rows).blocks[0]
                S = device.DeviceMatrix.empty(n, d)
                ms = timeit(lambda: device.apply_block(sub, A, True, S, 0), max(3, args.reps // 4))
                byt = rows * n * 8 + n * d * 8
                out["c5shard_St"] = {"ms": ms, "GBs": byt / ms / 1e6, "frac": byt / ms / 1e6 / PEAK}
        elif c == "c2g":
            n, d = 16384, 512
            A = mat(n)
            op = sk.new_operator(sk.GAUSSIAN, n, d, np.random.SeedSequence((0, 0)))
            blk = op.blocks[0]
            S = device.DeviceMatrix.empty(n, d)
            for tr in (False, True):
                ms = timeit(lambda: device.apply_block(blk, A, tr, S, 0), max(3, args.reps // 4))
                out[f"c2g_{'St' if tr else 'S'}"] = {"ms": ms, "TFs": 2 * n * n * d / ms / 1e9}
            st = device.block_state(blk)
            At = A.t[:, :n]
            ms = timeit(lambda: torch.matmul(st.R, At), max(3, args.reps // 4))
            out["c2g_cublas"] = {"ms": ms, "TFs": 2 * n * n * d / ms / 1e9}
        elif c == "c3":
            n = 65536
            A = mat(n, kind="toep")
            op = sk.new_operator(sk.SJLT, n, 64, np.random.SeedSequence((0, 5)), alpha=8,
                                 construction="block")
            blk = op.blocks[0]
            S = device.DeviceMatrix.empty(n, 64)
            for tr in (False, True):
                ms = timeit(lambda: device.apply_block(blk, A, tr, S, 0), max(3, args.reps // 4))
                byt = n * n * 8 + n * 64 * 8
                out[f"c3_{'St' if tr else 'S'}"] = {"ms": ms, "GBs": byt / ms / 1e6,
                                                    "frac": byt / ms / 1e6 / PEAK}
        elif c == "c3a4":  # C3's matrix with the paper's default alpha = 4 increments of 64
            n = 65536
            A = mat(n, kind="toep")
            op = sk.new_operator(sk.SJLT, n, 64, np.random.SeedSequence((0, 5)), alpha=4,
                                 construction="block")
            blk = op.blocks[0]
            S = device.DeviceMatrix.empty(n, 64)
            for tr in (False, True):
                ms = timeit(lambda: device.apply_block(blk, A, tr, S, 0), max(3, args.reps // 4))
                byt = n * n * 8 + n * 64 * 8
                out[f"c3a4_{'St' if tr else 'S'}"] = {"ms": ms, "GBs": byt / ms / 1e6,
                                                      "frac": byt / ms / 1e6 / PEAK}
        elif c == "c4":
            n = 65536
            A = mat(n, 8, 0.25)
            op = sk.new_operator(sk.SRHT, n, 512, np.random.SeedSequence((0, 0)))
            blk = op.blocks[0]
            S = device.DeviceMatrix.empty(n, 512)
            ms = timeit(lambda: device.apply_block(blk, A, False, S, 0), max(3, args.reps // 4))
            byt = n * n * 8 + n * 512 * 8
            out["c4_S"] = {"ms": ms, "GBs": byt / ms / 1e6, "frac": byt / ms / 1e6 / PEAK}
            ms = timeit(lambda: device.apply_block(blk, A, True, S, 0), max(3, args.reps // 4))
            out["c4_St"] = {"ms": ms, "GBs": byt / ms / 1e6, "frac": byt / ms / 1e6 / PEAK}
        print(json.dumps({k: v for k, v in out.items() if k.startswith(c)}), flush=True)
    print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("HSK_")},
                      "results": out}))


if __name__ == "__main__":
    main()
