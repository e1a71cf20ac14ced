#!/usr/bin/env python
"""Where the device driver's C1 compression time goes (host cProfile after a
warm-up run; syncs show up in .item()/.tolist()/cpu()).

    python tools/hss_profile.py [c1|qchem]
"""
import cProfile
import os
import pstats
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.append(os.path.join(ROOT, "baseline", "_ref"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
from hsskit import build_uniform, relative_error  # noqa: E402
from hsskit.hss_compress import CompressOptions  # noqa: E402
from hsskit.sketching import DenseAccessor  # noqa: E402

from paper_2302_01977_b200 import hss_device, matgen  # noqa: E402

case = sys.argv[1] if len(sys.argv) > 1 else "c1"
if case == "qchem":   # Table 7.1's QChem Toeplitz, n = 10000, eps 1e-2, S(1)
    from hsskit.matgen import qchem_toeplitz
    n, leaf = 10000, 256
    Ah = np.asfortranarray(qchem_toeplitz(n, 0.1).dense())
    opts = CompressOptions(d0=128, dd=64, eps_rel=1e-2, eps_abs=1e-8, leaf_size=leaf,
                           kind="sjlt", alpha=1, construction="block", seed=0)
else:                 # BASELINE configs[0] (C1)
    n, leaf = 4096, 128
    Ah = matgen.gaussian_kernel(n, 8, 0.5).to_host()
    opts = CompressOptions(d0=192, dd=64, eps_rel=1e-6, eps_abs=1e-8, leaf_size=leaf,
                           kind="sjlt", alpha=4, construction="graph", seed=0)
acc = DenseAccessor(Ah)
tree = build_uniform(n, leaf)
hss_device.compress(acc, tree, opts)
torch.cuda.synchronize()
t0 = time.perf_counter()
H = hss_device.compress(acc, tree, opts)
torch.cuda.synchronize()
print(f"device compress {time.perf_counter() - t0:.3f} s, sketch {H.sketch_seconds:.3f} s, "
      f"final_d {H.final_d}, rounds {H.adaptation_rounds}, nodes {len(tree.nodes)}")
pr = cProfile.Profile()
pr.enable()
hss_device.compress(acc, tree, opts)
torch.cuda.synchronize()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(22)
st.sort_stats("cumulative").print_stats(30)

# device-side kernel time by kernel name (CUPTI through torch.profiler)
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
    hss_device.compress(acc, tree, opts)
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=70))
