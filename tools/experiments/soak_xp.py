"""Soak of the transposed-tile S' kernels (modes 5 / 6): thousands of launches,
every result compared bit for bit with the first (a race between the staging
ring, the copying warps and the consumers would show up as a differing sum)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2302_01977_b200 import device
from paper_2302_01977_b200 import sketching as sk

torch.manual_seed(0)
bad = 0
for n, m, d, a, ld_odd, reps in ((16384, 16384, 128, 4, 0, 1500), (16384, 16384, 256, 8, 0, 800),
                                 (16384, 16384, 64, 4, 0, 1500), (16384, 16384, 32, 2, 0, 1000),
                                 (8192, 5000, 64, 4, 1, 300), (8192, 5000, 256, 8, 1, 300),
                                 (4096, 4096, 256, 4, 0, 3000), (3000, 300, 200, 5, 0, 3000)):
    A = device.DeviceMatrix(n, m, ld=n + (n & 1) + ld_odd)
    A.t.normal_()
    op = sk.new_operator(sk.SJLT, n, d, np.random.SeedSequence((1, d)), alpha=a, construction="block")
    ref = device.DeviceMatrix.empty(m, d)
    device.apply_block(op.blocks[0], A, True, ref, 0)
    out = device.DeviceMatrix.empty(m, d)
    diff = 0
    for i in range(reps):
        out.t.zero_()
        device.apply_block(op.blocks[0], A, True, out, 0)
        if i % 10 == 9 or i == reps - 1:
            diff += int(not torch.equal(out.t[:, :m], ref.t[:, :m]))
    torch.cuda.synchronize()
    bad += diff
    print(f"n={n} m={m} d={d} alpha={a} odd_ld={ld_odd} launches={reps} differing_checks={diff}", flush=True)
print("soak", "FAILED" if bad else "ok")
sys.exit(1 if bad else 0)
