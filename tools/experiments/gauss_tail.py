"""Wave-quantisation check for the Gaussian DMMA GEMM: time vs row count."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2302_01977_b200 import device, matgen
from paper_2302_01977_b200 import sketching as sk
n, d = 16384, 512
A = matgen.gaussian_kernel(n, 8, 0.5)
op = sk.new_operator(sk.GAUSSIAN, n, d, np.random.SeedSequence((0, 0)))
blk = op.blocks[0]
def t(f, reps=5):
    for _ in range(2): f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): f()
    e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1) / reps
for m in (16384, 14208, 12800, 11392, 8576):
    Av = A.row_view(0, m)
    S = device.DeviceMatrix.empty(m, d)
    ms = t(lambda: device.apply_block(blk, Av, False, S, 0))
    print(m, "rows", round(ms, 3), "ms", round(2 * m * n * d / ms / 1e9, 2), "TF/s", "ratio", round(ms / 8.30, 3), "rows ratio", round(m / 16384, 3), flush=True)
