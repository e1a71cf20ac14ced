"""One SJLT product on the GPU checked against the CPU oracle (debug aid; run
each case in its own process so a device fault does not hide the others):
    python tools/repro_one.py m n d alpha [t] [lda_pad]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402  (checker only)
from paper_2302_01977_b200 import sketching as sk  # noqa: E402

m, n, d, alpha = (int(x) for x in sys.argv[1:5])
tr = len(sys.argv) > 5 and sys.argv[5] == "t"
pad = int(sys.argv[6]) if len(sys.argv) > 6 else 0
op = sk.new_operator(sk.SJLT, n, d, seed=(m, n, d), alpha=alpha, construction="block")
rng = np.random.default_rng(0)
shape = (n, m) if tr else (m, n)
X = np.asfortranarray(rng.standard_normal((shape[0] + pad, shape[1])))[: shape[0]]
got = (sk.apply_right_transposed if tr else sk.apply_right)(X, op)
ref = (O.apply_right_transposed if tr else O.apply_right)(np.asfortranarray(X), op)
print("case", sys.argv[1:], "rel", O.rel_frobenius(got, ref))
