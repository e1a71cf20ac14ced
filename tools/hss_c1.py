#!/usr/bin/env python
"""C1 end to end: the reference's own HSS compressor (hsskit, installed in
baseline/_ref) on the n=4096 Gaussian-kernel matrix, with its CPU sketch and
with the GPU drop-in (plugin.install).  Prints error, total time and the
compressor's own sketch timer (H.sketch_seconds) for both."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.append(os.path.join(ROOT, "baseline", "_ref"))
import hsskit.sketching as hs  # noqa: E402
from hsskit import build_uniform, compress, relative_error, stats  # noqa: E402
from hsskit.hss_compress import CompressOptions  # noqa: E402
from hsskit.sketching import DenseAccessor  # noqa: E402

from paper_2302_01977_b200 import matgen, plugin  # noqa: E402

n = 4096
Ah = matgen.gaussian_kernel(n, 8, 0.5).to_host()
opts = CompressOptions(d0=192, dd=64, eps_rel=1e-6, eps_abs=1e-8, leaf_size=128, kind="sjlt",
                       alpha=4, construction="graph", seed=0)
tree = build_uniform(n, 128)
res = {}
import torch  # noqa: E402
if os.environ.get("HSS_TORCH_THREADS"):
    torch.set_num_threads(int(os.environ["HSS_TORCH_THREADS"]))
labels = ["reference CPU sketch", "GPU sketch (plugin)"]
if os.environ.get("HSS_ONLY_GPU"):
    labels = labels[1:]
for label in labels:
    if label.startswith("GPU"):
        plugin.install(hs)
        compress(DenseAccessor(Ah[:512, :512]), build_uniform(512, 128), opts)  # warm-up
    try:
        t0 = time.perf_counter()
        H = compress(DenseAccessor(Ah), tree, opts)
        total = time.perf_counter() - t0
    finally:
        if label.startswith("GPU"):
            plugin.uninstall(hs)
    res[label] = (relative_error(Ah, H), total, H.sketch_seconds, stats(H).final_d)
    print(f"{label:22s} rel_error {res[label][0]:.6e}  total {total:7.2f} s  "
          f"sketch {H.sketch_seconds:7.3f} s  final_d {res[label][3]}", flush=True)
