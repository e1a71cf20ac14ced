"""C3 (n = 65536 Toeplitz-sine, d = 64, alpha = 8 paired): time of the A^T
copy, S' on A, and S on the kept A^T (the adaptive sketch's S' increments)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2302_01977_b200 import device, matgen
from paper_2302_01977_b200 import sketching as sk

def t(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

n = int(os.environ.get("N", "65536"))
A = matgen.toeplitz_sin(n)
op = sk.new_operator(sk.SJLT, n, 64, np.random.SeedSequence((0, 5)), alpha=8, construction="block")
blk = op.blocks[0]
S = device.DeviceMatrix.empty(n, 64)
hold = {}
ms_t = t(lambda: hold.__setitem__("At", A.transposed()), 3)
At = hold["At"]
print("transpose ms", round(ms_t, 3), "GB/s", round(2 * 8 * n * n / ms_t / 1e6, 1))
print("S on A ms", round(t(lambda: device.apply_block(blk, A, False, S, 0)), 3))
print("S' on A ms", round(t(lambda: device.apply_block(blk, A, True, S, 0)), 3))
print("S on A^T ms", round(t(lambda: device.apply_block(blk, At, False, S, 0)), 3))
ms_tt = t(lambda: hold.__setitem__("Bt", A.t[:, :n].T.contiguous()), 3)
print("torch transpose ms", round(ms_tt, 3), "GB/s", round(2 * 8 * n * n / ms_tt / 1e6, 1),
      "equal", bool(torch.equal(hold["Bt"], At.t[:, :n])))
