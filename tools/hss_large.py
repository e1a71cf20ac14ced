#!/usr/bin/env python
"""Whole HSS compressions at BASELINE.json sizes through the device driver
(hss_device: the reference's _Driver with sketch, samples, gates and IDs in
HBM) -- sizes the reference compressor cannot reach on the host in any
reasonable time (its sketch alone is ~35 min per pass at n = 65536).

    python tools/hss_large.py [c3|c2] [eps]

c3: BASELINE configs[2]'s nonsymmetric Toeplitz-sine matrix, n = 65536 (34 GB in HBM),
    SJLT alpha = 8 block construction, d0 = 128, dd = 64, leaf 256.
c2: configs[1]'s Gaussian kernel, n = 16384.
Error: ||A x - H x|| / ||A x|| over four random x (hss_ops.matvec on the host)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.append(os.path.join(ROOT, "baseline", "_ref"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
from hsskit import build_uniform, matvec, stats  # noqa: E402
from hsskit.hss_compress import CompressOptions  # noqa: E402

from paper_2302_01977_b200 import hss_device, matgen  # noqa: E402
from paper_2302_01977_b200 import sketching as sk  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "c3"
eps = float(sys.argv[2]) if len(sys.argv) > 2 else 1e-6
if case == "c3":
    n = 65536
    A = matgen.toeplitz_sin(n)
    opts = CompressOptions(d0=128, dd=64, eps_rel=eps, eps_abs=1e-8, leaf_size=256, kind="sjlt",
                           alpha=8, construction="block", seed=0)
else:
    n = 16384
    A = matgen.gaussian_kernel(n, 8, 0.5)
    opts = CompressOptions(d0=128, dd=64, eps_rel=eps, eps_abs=1e-8, leaf_size=256, kind="sjlt",
                           alpha=4, construction="block", seed=0)
torch.cuda.synchronize()
acc = sk.DeviceAccessor(A)
tree = build_uniform(n, 256)
t0 = time.perf_counter()
H = hss_device.compress(acc, tree, opts)
torch.cuda.synchronize()
t = time.perf_counter() - t0
rng = np.random.default_rng(1)
X = rng.standard_normal((n, 4))
AX = (A.t[:, :n].T @ torch.as_tensor(X, device="cuda")).cpu().numpy()
HX = np.column_stack([matvec(H, X[:, j]) for j in range(4)])
st = stats(H)
print(json.dumps({"case": case, "n": n, "eps_rel": eps, "total_s": t, "sketch_s": H.sketch_seconds,
                  "rel_err_matvec": float(np.linalg.norm(AX - HX) / np.linalg.norm(AX)),
                  "final_d": H.final_d, "rounds": st.adaptation_rounds, "max_rank": st.max_rank,
                  "memory_pct": st.memory_fraction, "nodes": len(tree.nodes)}))
