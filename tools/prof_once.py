#!/usr/bin/env python
"""Launch each requested kernel case exactly twice (warm-up + profiled) for
ncu captures:  ncu -k regex:<kernel> -s 1 -c 1 python tools/prof_once.py c2s_S"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_01977_b200 import device, matgen  # noqa: E402
from paper_2302_01977_b200 import sketching as sk  # noqa: E402

CASES = {
    "c1": ("sjlt", 4096, 256, 4, "graph", "gauss"),
    "c2s": ("sjlt", 16384, 512, 4, "block", "gauss"),
    "c2g": ("gaussian", 16384, 512, None, None, "gauss"),
    "c3": ("sjlt", 65536, 64, 8, "block", "toep"),
    "c4": ("srht", 65536, 512, None, None, "gauss4"),
    # S' on tiles transposed in shared memory (modes 5): a = 8 / a = 4 entries per element and slab
    "xp8": ("sjlt", 16384, 256, 8, "block", "gauss"),
    "xp4": ("sjlt", 16384, 128, 4, "block", "gauss"),
    "c3a4": ("sjlt", 65536, 64, 4, "block", "toep"),
}


def c5shard(direction):
    """BASELINE configs[4] row shard at 8 GPUs: 16384 x 131072 of the n = 131072
    kernel matrix, SJLT d = 2048 alpha = 8 (S, or the shard's S' partial)."""
    from paper_2302_01977_b200 import distributed as hd
    n, rows, d = 131072, 16384, 2048
    A = matgen.gaussian_kernel(n, 16, 1.0, 1e-2, row0=0, nrows=rows,
                               points=matgen.kernel_points(n, 16, 0))
    op = sk.new_operator(sk.SJLT, n, d, np.random.SeedSequence((0, 0)), alpha=8,
                         construction="block")
    if direction == "S":
        blk, S = op.blocks[0], device.DeviceMatrix.empty(rows, d)
    else:
        blk, S = hd.restrict_operator(op, 0, rows).blocks[0], device.DeviceMatrix.empty(n, d)
    for _ in range(2):
        device.apply_block(blk, A, direction == "St", S, 0)
    torch.cuda.synchronize()


def pqr():
    """The C1 compression's largest interpolative decomposition shape: a
    2000 x 2048 sample (rank ~1990) through hsk_pqr."""
    from paper_2302_01977_b200 import hss_device
    rng = np.random.default_rng(0)
    rows, width = 2000, 2048
    sv = np.logspace(0, -9, rows)
    U0, _ = np.linalg.qr(rng.standard_normal((rows, rows)))
    V0, _ = np.linalg.qr(rng.standard_normal((width, rows)))
    S = torch.as_tensor((U0 * sv) @ V0.T, device="cuda")
    for _ in range(2):
        hss_device.row_interpolative_decomposition(S, 1e-12, 1e-300)
    torch.cuda.synchronize()


def main():
    for arg in sys.argv[1:]:
        if arg.startswith("c5shard_"):
            c5shard(arg.split("_")[1])
            continue
        if arg == "pqr":
            pqr()
            continue
        case, direction = arg.split("_")
        kind, n, d, alpha, cons, mat = CASES[case]
        A = (matgen.toeplitz_sin(n) if mat == "toep" else
             matgen.gaussian_kernel(n, 8, 0.25 if mat == "gauss4" else 0.5))
        kw = dict(alpha=alpha, construction=cons) if kind == "sjlt" else {}
        op = sk.new_operator(kind, n, d, np.random.SeedSequence((0, 0)), **kw)
        S = device.DeviceMatrix.empty(n, d)
        for _ in range(2):
            device.apply_block(op.blocks[0], A, direction == "St", S, 0)
        torch.cuda.synchronize()
        del A, S
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
