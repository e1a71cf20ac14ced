#!/usr/bin/env python
"""Per-shape timings of the sweep's dense kernels: hsk_pqr (row ID) and the
gate QR (torch.linalg.qr = cuSOLVER), CUDA events, after warm-up."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2302_01977_b200 import hss_device  # noqa: E402


def tm(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


rng = np.random.default_rng(0)
for rows, width, rank in [(128, 2048, 120), (256, 2048, 250), (1000, 2048, 990), (2000, 2048, 1990),
                          (2000, 2048, 600)]:
    sv = np.logspace(0, -9, min(rows, width))
    sv[rank:] = 0
    U0, _ = np.linalg.qr(rng.standard_normal((rows, min(rows, width))))
    V0, _ = np.linalg.qr(rng.standard_normal((width, min(rows, width))))
    S = torch.as_tensor((U0 * sv) @ V0.T, device="cuda")
    ms = tm(lambda: hss_device.row_interpolative_decomposition(S, 1e-12, 1e-300))
    r = hss_device.row_interpolative_decomposition(S, 1e-12, 1e-300)[1].size
    print(f"row ID {rows} x {width} (rank {r}): {ms:.3f} ms", flush=True)
for m, n in [(128, 128), (128, 64), (256, 64), (1000, 64), (2000, 64), (1000, 1000), (2000, 1984)]:
    X = torch.randn(m, n, dtype=torch.float64, device="cuda")
    print(f"torch.linalg.qr {m} x {n}: {tm(lambda: torch.linalg.qr(X, mode='reduced')):.3f} ms",
          flush=True)
    Xs = X[:, :n]
