"""e2e timing variants of bench.py's end-to-end leg (debug aid)."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_01977_b200 import matgen
from paper_2302_01977_b200 import sketching as sk
N, D = 16384, 512
op = sk.new_operator(sk.SJLT, N, D, np.random.SeedSequence((0, 0)), alpha=4, construction="block")
A = matgen.gaussian_kernel(N, 8, 0.5)
host = torch.empty((N, N), dtype=torch.float64, pin_memory=True)
host.copy_(A.t[:, :N])
Ah = host.numpy().T
stream = torch.cuda.current_stream()
for keep in (True, False):
    for use_ev in (True, False):
        S_host = sk.apply_right(Ah, op)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(stream)
        for _ in range(10):
            if keep:
                S_host = sk.apply_right(Ah, op)
            else:
                sk.apply_right(Ah, op)
        e1.record(stream)
        torch.cuda.synchronize()
        wall = (time.perf_counter() - t0) / 10 * 1e3
        print("keep", keep, "events", round(e0.elapsed_time(e1) / 10, 2), "wall", round(wall, 2), flush=True)
