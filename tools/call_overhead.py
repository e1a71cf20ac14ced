"""Per-call wall time of the drop-in products on a C1-sized accessor (the
compressor's call pattern: fresh 64-column SJLT blocks, host result)."""
import cProfile
import os
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_01977_b200 import sketching as sk  # noqa: E402

n = 4096
rng = np.random.default_rng(0)
A = sk.DenseAccessor(np.asfortranarray(rng.standard_normal((n, n))))
ops = [sk.new_operator(sk.SJLT, n, 64, np.random.SeedSequence((0, i)), alpha=4, construction="graph")
       for i in range(60)]
sk.apply_right(A, ops[0]); sk.apply_right_transposed(A, ops[0])
torch.cuda.synchronize()


def run():
    for op in ops[1:]:
        sk.apply_right(A, op)
        sk.apply_right_transposed(A, op)


t0 = time.perf_counter(); run(); t1 = time.perf_counter()
print("per call ms", (t1 - t0) / 118 * 1e3)
pr = cProfile.Profile(); pr.enable(); run(); pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
