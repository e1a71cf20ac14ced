"""C3 increment S = A R^T on A, on a clone of A and on A^T: is the second 34 GB
buffer slower because of where it lies, or because of its contents?"""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2302_01977_b200 import device, matgen
from paper_2302_01977_b200 import sketching as sk

def t(fn, reps=8):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

n = 65536
A = matgen.toeplitz_sin(n)
op = sk.new_operator(sk.SJLT, n, 64, np.random.SeedSequence((0, 5)), alpha=8, construction="block")
blk = op.blocks[0]
S = device.DeviceMatrix.empty(n, 64)
print("S on A      ", round(t(lambda: device.apply_block(blk, A, False, S, 0)), 3))
B = device.DeviceMatrix(n, n, ld=A.ld)
B.t.copy_(A.t)
print("S on clone  ", round(t(lambda: device.apply_block(blk, B, False, S, 0)), 3))
print("S on A again", round(t(lambda: device.apply_block(blk, A, False, S, 0)), 3))
del B
torch.cuda.empty_cache()
At = A.transposed()
print("S on A^T    ", round(t(lambda: device.apply_block(blk, At, False, S, 0)), 3))
print("S on A again", round(t(lambda: device.apply_block(blk, A, False, S, 0)), 3))
# contents: A^T's values in A's buffer
A.t.copy_(At.t)
print("S on A holding A^T's values", round(t(lambda: device.apply_block(blk, A, False, S, 0)), 3))
print("ptrs", hex(A.ptr), hex(At.ptr))
