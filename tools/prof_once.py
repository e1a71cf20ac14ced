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
}


def main():
    for arg in sys.argv[1:]:
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
