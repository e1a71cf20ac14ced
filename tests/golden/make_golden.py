"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container, where the reference is importable read-only:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

It imports hsskit (never hsskit.cli/plots: matplotlib is absent) and records,
for a list of small cases, the reference's own random operator draws
(`_pos`/`_signs`, `matrix`, `signs`/`sample`) and the reference's own
`apply_right` / `apply_right_transposed` outputs on seeded inputs.  Input
matrices are NOT stored: they are `np.random.default_rng(seed)
.standard_normal(shape)`, which is bit-reproducible, and a SHA-256 of their
bytes is stored to detect drift.  Large operator draws (config sizes) are
pinned by SHA-256 only.

Outputs: golden.npz (arrays) + golden.json (case manifest).  The reference
tree does not exist on the GPU box; tests read only these files there.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from hsskit import sketching as ref  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def seed_tuple(s):
    return list(s) if isinstance(s, tuple) else s


def mk_seed(s):
    return tuple(s) if isinstance(s, list) else s


def block_arrays(prefix: str, block, arrays: dict):
    if block.kind == ref.SJLT:
        arrays[prefix + "pos"] = np.asarray(block._pos, dtype=np.int64)
        arrays[prefix + "signs"] = np.asarray(block._signs, dtype=np.int8)
    elif block.kind == ref.GAUSSIAN:
        arrays[prefix + "matrix"] = block.matrix
    else:
        arrays[prefix + "signs"] = block.signs
        arrays[prefix + "sample"] = np.asarray(block.sample, dtype=np.int64)


def main():
    arrays: dict[str, np.ndarray] = {}
    cases = []

    # ---- operator cases: (name, kind, n, blocks=[(rows, seed)], alpha, construction,
    #                       m_right, m_left, data_seed)
    specs = [
        ("sjlt_block_a3", "sjlt", 12, [(6, 9)], 3, "block", 16, 16, 5),
        ("sjlt_graph_a3", "sjlt", 12, [(6, 9)], 3, "graph", 16, 16, 5),
        ("sjlt_graph_a2_T", "sjlt", 16, [(6, 10)], 2, "graph", 12, 12, 6),
        ("sjlt_block_a1", "sjlt", 33, [(5, 3)], 1, "block", 9, 7, 7),
        ("sjlt_block_a4", "sjlt", 40, [(8, 11)], 4, "block", 21, 19, 8),
        ("sjlt_graph_a4", "sjlt", 97, [(24, 12)], 4, "graph", 37, 41, 9),
        ("sjlt_block_a8_d64", "sjlt", 300, [(64, 13)], 8, "block", 70, 65, 10),
        ("sjlt_graph_a5", "sjlt", 200, [(10, 14)], 5, "graph", 33, 3, 11),
        ("sjlt_graph_a8_d200", "sjlt", 513, [(200, 15)], 8, "graph", 45, 29, 12),
        ("sjlt_block_append", "sjlt", 150, [(16, 20), (8, 21), (8, 22)], 4, "block", 40, 35, 13),
        ("sjlt_graph_medium", "sjlt", 1024, [(128, [0, 0])], 4, "graph", 128, 96, 14),
        ("sjlt_block_tuple_seed", "sjlt", 64, [(8, [16, 3])], 4, "block", 10, 10, 15),
        ("gauss_small", "gaussian", 20, [(7, 5)], None, None, 9, 9, 2),
        ("gauss_T", "gaussian", 9, [(7, 6)], None, None, 20, 20, 2),
        ("gauss_mid", "gaussian", 96, [(40, 7)], None, None, 50, 33, 16),
        ("gauss_append", "gaussian", 64, [(16, [17, 1]), (8, [18, 1])], None, None, 30, 31, 17),
        ("srht_pow2", "srht", 16, [(5, 1)], None, None, 8, 8, 3),
        ("srht_pad21", "srht", 21, [(5, 1)], None, None, 8, 8, 3),
        ("srht_T", "srht", 8, [(6, 2)], None, None, 21, 21, 3),
        ("srht_pad100", "srht", 100, [(24, 4)], None, None, 17, 13, 18),
        ("srht_1024", "srht", 1024, [(64, 5)], None, None, 33, 20, 19),
        ("srht_append", "srht", 32, [(6, 21), (5, 99)], None, None, 11, 12, 20),
        ("srht_n1", "srht", 1, [(1, 0)], None, None, 4, 4, 21),
    ]
    for name, kind, n, blocks, alpha, cons, m_r, m_l, dseed in specs:
        rows0, seed0 = blocks[0]
        kw = {}
        if kind == "sjlt":
            kw = dict(alpha=alpha, construction=cons)
        op = ref.new_operator(kind, n, rows0, mk_seed(seed0), **kw)
        for rows, s in blocks[1:]:
            op = ref.append_columns(op, rows, mk_seed(s))
        rng = np.random.default_rng(dseed)
        A = rng.standard_normal((m_r, n))
        B = rng.standard_normal((n, m_l))
        S = ref.apply_right(A, op)
        St = ref.apply_right_transposed(B, op)
        for bi, blk in enumerate(op.blocks):
            block_arrays(f"{name}/b{bi}/", blk, arrays)
        arrays[f"{name}/S"] = S
        arrays[f"{name}/St"] = St
        arrays[f"{name}/dense"] = ref.dense_rows(op, np.arange(n), np.arange(op.d))
        cases.append(dict(name=name, kind=kind, n=n,
                          blocks=[[r, seed_tuple(s)] for r, s in blocks],
                          alpha=alpha, construction=cons, m_right=m_r, m_left=m_l,
                          data_seed=dseed, sha_A=sha(A), sha_B=sha(B), d=op.d,
                          n_pad=getattr(op.blocks[0], "n_pad", None)))

    # ---- explicit patterns (sketching.py:277-284)
    worked = dict(name="worked_pattern", n=4, rows=3, alpha=2,
                  pos=[[0, 2], [1, 2], [0, 1], [0, 2]],
                  signs=[[1, -1], [-1, -1], [1, -1], [1, 1]])
    blk = ref.SjltBlock.from_pattern(4, 3, 2, worked["pos"], worked["signs"])
    st = blk.storage
    for f in ("plus_rowptr", "plus_cols", "minus_rowptr", "minus_cols",
              "plus_colptr", "plus_rows", "minus_colptr", "minus_rows"):
        arrays[f"worked_pattern/{f}"] = np.asarray(getattr(st, f), dtype=np.int64)
    A = np.random.default_rng(4).standard_normal((5, 4))
    arrays["worked_pattern/S"] = blk.apply_right(np.asfortranarray(A))
    arrays["worked_pattern/St"] = blk.apply_right_transposed(np.asfortranarray(A.T))
    arrays["worked_pattern/dense"] = blk.dense_rows(np.arange(4), np.arange(3))
    worked["data_seed"] = 4
    empty = dict(name="trailing_empty", n=2, rows=3, alpha=1, pos=[[0], [0]], signs=[[1], [-1]])
    blk = ref.SjltBlock.from_pattern(2, 3, 1, empty["pos"], empty["signs"])
    Ae = np.arange(6.0).reshape(2, 3)
    arrays["trailing_empty/St"] = blk.apply_right_transposed(np.asfortranarray(Ae))
    arrays["trailing_empty/S"] = blk.apply_right(np.asfortranarray(Ae.T))
    patterns = [worked, empty]

    # ---- operator draws at config sizes, pinned by hash only
    draws = []
    for (kind, n, d, seed, alpha, cons) in [
        ("sjlt", 4096, 256, [0, 0], 4, "graph"),        # C1 block 0 (compress seed 0)
        ("sjlt", 4096, 64, [0, 1], 4, "graph"),         # C1 first extension
        ("sjlt", 16384, 512, [0, 0], 4, "block"),       # C2 SJLT comparison
        ("sjlt", 65536, 64, [0, 5], 8, "block"),        # C3 increment 5
        ("sjlt", 131072, 2048, [0, 0], 8, "block"),     # C5
        ("gaussian", 2048, 64, [0, 0], None, None),
        ("srht", 65536, 512, [0, 0], None, None),       # C4
        ("srht", 5000, 64, [0, 3], None, None),
    ]:
        kw = dict(alpha=alpha, construction=cons) if kind == "sjlt" else {}
        op = ref.new_operator(kind, n, d, np.random.SeedSequence(tuple(seed)), **kw)
        b = op.blocks[0]
        if kind == "sjlt":
            h = dict(pos=sha(np.asarray(b._pos, dtype=np.int64)),
                     signs=sha(np.asarray(b._signs, dtype=np.int8)))
        elif kind == "gaussian":
            h = dict(matrix=sha(b.matrix))
        else:
            h = dict(signs=sha(b.signs), sample=sha(np.asarray(b.sample, dtype=np.int64)))
        draws.append(dict(kind=kind, n=n, d=d, seed_sequence=seed, alpha=alpha,
                          construction=cons, sha=h))

    # ---- FWHT known answers (sketching.py:100-112)
    arrays["fwht/const4"] = ref.fwht([1.0, 1.0, 1.0, 1.0])
    X = np.random.default_rng(1).standard_normal((3, 16))
    arrays["fwht/rows16"] = ref.fwht(X)

    # ---- np.add.reduceat segments (the summation the transposed SJLT uses)
    rng = np.random.default_rng(99)
    segs = []
    for L in (1, 2, 7, 8, 9, 15, 16, 17, 127, 128, 129, 130, 255, 256, 257, 1000):
        c = rng.standard_normal(L) * np.exp(3 * rng.standard_normal(L))
        arrays[f"reduceat/{L}/x"] = c
        arrays[f"reduceat/{L}/y"] = np.add.reduceat(np.concatenate([c, [0.0]]), [0, L])[:1]
        segs.append(L)

    manifest = dict(numpy=np.__version__, cases=cases, patterns=patterns, draws=draws,
                    reduceat_lengths=segs, scale_alpha={a: 1.0 / math.sqrt(a) for a in range(1, 9)})
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(manifest, f, indent=1)
    print("wrote", len(arrays), "arrays,", len(cases), "cases")


if __name__ == "__main__":
    main()
