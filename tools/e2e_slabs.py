"""e2e A/B of the host-array slab pipeline: HSK_STAGE_THREADS / HSK_STREAM_SLABS
on a pageable and a pinned C2 matrix (wall clock per sketching.apply_right)."""
import os, sys, time, json
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2302_01977_b200 import matgen, sketching as sk
N=16384
A = matgen.gaussian_kernel(N, 8, 0.5)
op = sk.new_operator(sk.SJLT, N, 512, np.random.SeedSequence((0, 0)), alpha=4, construction=sk.BLOCK)
page = np.array(A.to_host(), order='F', copy=True)   # a plain pageable copy
host = torch.empty((N, N), dtype=torch.float64, pin_memory=True); host.copy_(A.t[:, :N]); pin = host.numpy().T
res = {}
for name, arr in (("pageable", page), ("pinned", pin)):
    for _ in range(2): sk.apply_right(arr, op)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(4): S = sk.apply_right(arr, op)
    torch.cuda.synchronize(); res[name] = (time.perf_counter() - t0) / 4 * 1e3
print(json.dumps({"threads": os.environ.get("HSK_STAGE_THREADS"), "slabs": os.environ.get("HSK_STREAM_SLABS"), "ms": res, "GBs": {k: N*N*8/v/1e6 for k, v in res.items()}, "cpus": os.cpu_count()}))
