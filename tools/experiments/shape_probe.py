"""S (and S') time for SJLT block construction over an (n, d) grid on the
8-D Gaussian kernel matrix, for the consumer-warp shape selected by
HSK_SJLT_W32 (16 / 20 / 24; unset = the default rule)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2302_01977_b200 import device, matgen, _lib
from paper_2302_01977_b200 import sketching as sk

def t(fn, reps=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

for n in (16384,):
    A = matgen.gaussian_kernel(n, 8, 0.5)
    for d in (300, 320, 384, 448, 600, 700, 900):
        row = []
        for ws in ("", "8", "16", "20", "24"):
            os.environ["HSK_SJLT_W32"] = ws
            _lib.load().hsk_tuning_reload()
            op = sk.new_operator(sk.SJLT, n, d, np.random.SeedSequence((0, 0)), alpha=4, construction="block")
            S = device.DeviceMatrix.empty(n, d)
            blk = op.blocks[0]
            row.append(f"W{ws or 'def'}={t(lambda: device.apply_block(blk, A, False, S, 0)):.4f}")
            if ws in ("", "16"):
                St = device.DeviceMatrix.empty(n, d)
                row.append(f"T{ws or 'def'}={t(lambda: device.apply_block(blk, A, True, St, 0)):.4f}")
        print(f"n={n} d={d}", " ".join(row), flush=True)
    del A
    torch.cuda.empty_cache()
