import sys, os, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_01977_b200 import sketching as sk
m, n, d, alpha = (int(x) for x in sys.argv[1:5])
tr = len(sys.argv) > 5 and sys.argv[5] == "t"
op = sk.new_operator(sk.SJLT, n, d, seed=(m, n, d), alpha=alpha, construction="block")
rng = np.random.default_rng(0)
if tr:
    B = rng.standard_normal((n, m)); print(sk.apply_right_transposed(B, op).sum())
else:
    A = rng.standard_normal((m, n)); print(sk.apply_right(A, op).sum())
