"""S' on an operand with an odd leading dimension (8-byte cp.async producers):
natural / XOR layouts (HSK_SJLT_XP=0: mode 1) vs the dense S layout (mode 6)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2302_01977_b200 import device
from paper_2302_01977_b200 import sketching as sk

def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

n = 16384
for ld in (n, n + 1):
    A = device.DeviceMatrix(n, n, ld=ld)
    A.t.normal_()
    for d, a in ((64, 4), (128, 4), (256, 8), (512, 4)):
        op = sk.new_operator(sk.SJLT, n, d, np.random.SeedSequence((0, 0)), alpha=a, construction="block")
        S = device.DeviceMatrix.empty(n, d)
        print("ld", ld, "d", d, "alpha", a, "S' ms", round(t(lambda: device.apply_block(op.blocks[0], A, True, S, 0)), 4), flush=True)
