#!/usr/bin/env python
"""Load-balance experiment: C2 shape with a random vs perfectly balanced
SJLT pattern (every bucket exactly once per 128-chunk)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_01977_b200 import device, matgen, operators  # noqa: E402
from paper_2302_01977_b200 import sketching as sk  # noqa: E402


def timeit(fn, reps=20):
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


n, d, a = 16384, 512, 4
A = matgen.gaussian_kernel(n, 8, 0.5)
S = device.DeviceMatrix.empty(n, d)
rng = np.random.default_rng(0)
op = sk.new_operator(sk.SJLT, n, d, np.random.SeedSequence((0, 0)), alpha=a, construction="block")
k = np.arange(n)
blk = d // a
perm = [rng.permutation(blk) for _ in range(a)]
pos_bal = np.stack([b * blk + perm[b][k % blk] for b in range(a)], axis=1)
signs = np.where(rng.random((n, a)) < 0.5, -1, 1).astype(np.int8)
bal = operators.SjltBlock.from_pattern(n, d, a, pos_bal, signs)
for name, b in (("random", op.blocks[0]), ("balanced", bal)):
    for tr in (False, True):
        ms = timeit(lambda: device.apply_block(b, A, tr, S, 0))
        print(name, "St" if tr else "S", round(ms, 4), "ms", round((n * n * 8 + n * d * 8) / ms / 1e6), "GB/s")
