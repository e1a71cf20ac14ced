"""e2e apply_right on a pinned host array: streamed slab counts vs one-shot."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2302_01977_b200 import matgen
from paper_2302_01977_b200 import sketching as sk
N, D = 16384, 512
op = sk.new_operator(sk.SJLT, N, D, np.random.SeedSequence((0, 0)), alpha=4, construction="block")
A = matgen.gaussian_kernel(N, 8, 0.5)
host = torch.empty((N, N), dtype=torch.float64, pin_memory=True)
host.copy_(A.t[:, :N])
Ah = host.numpy().T
def t(f, reps=5):
    f(); torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(reps): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / reps * 1e3
for slabs in (1, 2, 4, 8, 16):
    sk.STREAM_SLABS = slabs
    print("slabs", slabs, "S ms", round(t(lambda: sk.apply_right(Ah, op)), 2),
          "S' ms", round(t(lambda: sk.apply_right_transposed(Ah, op)), 2), flush=True)
sk.STREAM_MIN_BYTES = 1 << 62
print("one-shot S ms", round(t(lambda: sk.apply_right(Ah, op)), 2),
      "S' ms", round(t(lambda: sk.apply_right_transposed(Ah, op)), 2))
