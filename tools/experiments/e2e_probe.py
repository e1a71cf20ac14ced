"""Break the e2e path (sketching.apply_right on a pinned host array) into parts."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2302_01977_b200 import device, matgen
from paper_2302_01977_b200 import sketching as sk

N, D = 16384, 512
op = sk.new_operator(sk.SJLT, N, D, np.random.SeedSequence((0, 0)), alpha=4, construction="block")
A = matgen.gaussian_kernel(N, 8, 0.5)
host = torch.empty((N, N), dtype=torch.float64, pin_memory=True)
host.copy_(A.t[:, :N])
A_host = host.numpy().T
sk.apply_right(A_host, op); torch.cuda.synchronize()
def t(f, reps=10):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): r = f()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps * 1e3, r
ms, _ = t(lambda: sk.apply_right(A_host, op)); print("apply_right e2e ms", ms)
ms, dA = t(lambda: sk.device_matrix_of(A_host)); print("device_matrix_of ms", ms)
ms, S = t(lambda: sk.apply_right_device(dA, op)); print("kernel ms", ms)
ms, _ = t(lambda: S.to_host()); print("to_host ms", ms)
ms, _ = t(lambda: sk._buffer_of(A_host)); print("_buffer_of ms", ms)
ms, _ = t(lambda: device.DeviceMatrix(N, N)); print("alloc ms", ms)
