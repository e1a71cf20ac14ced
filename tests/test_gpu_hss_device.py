"""Device-resident compression sweep (hss_device.DeviceDriver) against the
reference compressor, and the column-pivoted QR kernel against LAPACK.

The reference package (hsskit, baseline/_ref, installed by
__graft_entry__.build()) supplies the compressor whose sweep the device driver
subclasses and the CPU results it is compared with: same tree, same options,
same operator draws.  A missing hsskit is a failure under -m gpu.
"""

import os
import sys
import time

import numpy as np
import pytest
import scipy.linalg as sla

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
if os.path.isdir(REF) and REF not in sys.path:
    sys.path.append(REF)
try:
    import hsskit  # noqa: F401
    _IMPORT_ERROR = None
except ImportError as exc:
    hsskit = None
    _IMPORT_ERROR = exc

from paper_2302_01977_b200 import hss_device, matgen, plugin  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(autouse=True)
def _require_reference():
    if hsskit is None:
        pytest.fail(f"reference package hsskit not importable from {REF} ({_IMPORT_ERROR!r})")


def _ref_id(S, eps_rel, eps_abs):
    from hsskit.dense_kernels import row_interpolative_decomposition
    return row_interpolative_decomposition(S, eps_rel, eps_abs)


@pytest.mark.parametrize("rows,width,rank,eps", [
    (64, 200, 20, 1e-8), (128, 300, 128, 1e-12), (200, 150, 40, 1e-6), (1, 10, 1, 1e-8),
    (300, 2048, 250, 1e-9), (33, 7, 7, 1e-10),
])
def test_pqr_id_matches_lapack(cuda, rows, width, rank, eps):
    """Row ID through hsk_pqr vs the reference's scipy dgeqp3 path: same rank,
    same skeleton (norms well separated), coefficients to roundoff."""
    import torch
    rng = np.random.default_rng(rows * 7 + width)
    sv = np.logspace(0, -14, min(rows, width))
    sv[rank:] *= 1e-6
    U0, _ = np.linalg.qr(rng.standard_normal((rows, min(rows, width))))
    V0, _ = np.linalg.qr(rng.standard_normal((width, min(rows, width))))
    S = (U0 * sv) @ V0.T
    U_ref, J_ref = _ref_id(S, eps, 1e-300)
    U_gpu, J_gpu = hss_device.row_interpolative_decomposition(
        torch.as_tensor(S, device="cuda"), eps, 1e-300)
    U_gpu = U_gpu.cpu().numpy()
    np.testing.assert_array_equal(U_gpu[J_gpu, :], np.eye(len(J_gpu)))
    # ranks agree up to a diagonal sitting on the threshold (roundoff)
    assert abs(len(J_gpu) - len(J_ref)) <= 1, (len(J_gpu), len(J_ref))
    k = min(len(J_gpu), len(J_ref), 16)
    np.testing.assert_array_equal(J_gpu[:k], J_ref[:k])   # leading pivots: LAPACK's order
    if len(J_gpu) == len(J_ref) and np.array_equal(J_gpu, J_ref):
        # coefficients solve against R11, whose condition is up to ~1/eps
        np.testing.assert_allclose(U_gpu, U_ref, rtol=0,
                                   atol=1e-15 / eps * max(1.0, np.abs(U_ref).max()))
    # the ID reproduces S as well as the reference's does
    e_gpu = np.linalg.norm(S - U_gpu @ S[J_gpu]) / np.linalg.norm(S)
    e_ref = np.linalg.norm(S - U_ref @ S[J_ref]) / np.linalg.norm(S)
    assert e_gpu <= 10 * e_ref + 1e-15, (e_gpu, e_ref)
    print(f"pqr {rows}x{width}: rank {len(J_gpu)} (ref {len(J_ref)}), "
          f"skeleton equal {np.array_equal(J_gpu, J_ref)}, err {e_gpu:.2e} (ref {e_ref:.2e})")


def test_pqr_id_edge_cases(cuda):
    import torch
    Z = torch.zeros((5, 9), dtype=torch.float64, device="cuda")
    U, J = hss_device.row_interpolative_decomposition(Z, 1e-6, 0.0)
    assert U.shape == (5, 0) and J.size == 0
    E = torch.zeros((0, 4), dtype=torch.float64, device="cuda")
    U, J = hss_device.row_interpolative_decomposition(E, 1e-6, 1e-8)
    assert U.shape == (0, 0)
    with pytest.raises(ValueError):
        hss_device.row_interpolative_decomposition(Z, -1.0, 0.0)
    # exact ties: LAPACK's first-max rule
    S = np.array([[1.0, 0.0, 0.0], [0.0, 1.0, 0.0], [1.0, 1.0, 0.0]])
    U_ref, J_ref = _ref_id(S, 1e-12, 1e-14)
    U_gpu, J_gpu = hss_device.row_interpolative_decomposition(
        torch.as_tensor(S, device="cuda"), 1e-12, 1e-14)
    np.testing.assert_array_equal(J_gpu, J_ref)
    np.testing.assert_allclose(U_gpu.cpu().numpy(), U_ref, atol=1e-14)


def _both(acc, tree, opts):
    from hsskit import compress
    t0 = time.perf_counter()
    H_ref = compress(acc, tree, opts)
    t1 = time.perf_counter()
    H_dev = hss_device.compress(acc, tree, opts)
    t2 = time.perf_counter()
    return H_ref, H_dev, t1 - t0, t2 - t1


@pytest.mark.parametrize("kind,kw", [("sjlt", dict(alpha=4)), ("gaussian", {}), ("srht", {}),
                                     ("sjlt", dict(alpha=3, construction="graph"))])
def test_device_driver_exact_recovery(cuda, kind, kw):
    """Reference acceptance 1 / test_exact_recovery: a synthetic HSS matrix is
    recovered to the reference's accuracy with the same final sketch size."""
    from hsskit import relative_error, stats
    from hsskit.hss_compress import CompressOptions
    from hsskit.matgen import synthetic_hss
    acc, tree, truth = synthetic_hss(256, 32, 6, seed=3)
    opts = CompressOptions(d0=16, dd=8, eps_rel=1e-10, eps_abs=1e-12, kind=kind, seed=4,
                           leaf_size=32, **kw)
    H_ref, H_dev, _, _ = _both(acc, tree, opts)
    e_ref, e_dev = relative_error(truth, H_ref), relative_error(truth, H_dev)
    assert e_dev <= max(1.01 * e_ref, 1e-9), (e_dev, e_ref)
    s_ref, s_dev = stats(H_ref), stats(H_dev)
    assert s_dev.final_d == s_ref.final_d
    assert s_dev.max_rank == s_ref.max_rank


def test_device_driver_structure_and_determinism(cuda):
    """test_node_structure_invariants + test_fixed_seed_is_bit_reproducible
    (reference tests/test_hss_compress.py:126-171) through the device driver."""
    from hsskit import matvec, reconstruct_dense
    from hsskit.hss_compress import CompressOptions, NodeState
    from hsskit.matgen import synthetic_hss
    acc, tree, _ = synthetic_hss(256, 64, 4, seed=11)
    opts = CompressOptions(d0=16, dd=8, eps_rel=1e-8, eps_abs=1e-10, kind="gaussian", seed=12,
                           leaf_size=64)
    H = hss_device.compress(acc, tree, opts)
    for tnode in tree.nodes:
        node = H.nodes[tnode.nid]
        assert node.state is NodeState.COMPRESSED
        if tnode.level == 0:
            assert node.B12 is not None and node.B21 is not None
            continue
        r_row, r_col = node.rank_row, node.rank_col
        if tnode.is_leaf:
            assert node.D.shape == (tnode.size, tnode.size)
            assert node.U_coeff.shape == (tnode.size, r_row)
        else:
            c1, c2 = H.nodes[tnode.left.nid], H.nodes[tnode.right.nid]
            assert node.U_coeff.shape == (c1.rank_row + c2.rank_row, r_row)
            assert node.V_coeff.shape == (c1.rank_col + c2.rank_col, r_col)
        assert np.all((node.Itilde_row >= tnode.lo) & (node.Itilde_row < tnode.hi))
        np.testing.assert_array_equal(node.U_coeff[node.J_row, :], np.eye(r_row))
        np.testing.assert_array_equal(node.V_coeff[node.J_col, :], np.eye(r_col))
    acc2, tree2, _ = synthetic_hss(256, 64, 8, seed=8)
    opts2 = CompressOptions(d0=16, dd=8, eps_rel=1e-6, eps_abs=1e-10, kind="sjlt", alpha=4,
                            seed=9, leaf_size=64)
    H1 = hss_device.compress(acc2, tree2, opts2)
    H2 = hss_device.compress(acc2, tree2, opts2)
    np.testing.assert_array_equal(reconstruct_dense(H1), reconstruct_dense(H2))
    x = np.random.default_rng(10).standard_normal(256)
    np.testing.assert_array_equal(matvec(H1, x), matvec(H2, x))


def test_device_driver_max_sketch_and_validation(cuda):
    from hsskit.cluster_tree import build_uniform
    from hsskit.hss_compress import CompressOptions, MaxSketchReached
    from hsskit.sketching import DenseAccessor
    rng = np.random.default_rng(1)
    A = rng.standard_normal((128, 128))
    tree = build_uniform(128, 16)
    opts = CompressOptions(d0=8, dd=8, d_max=24, eps_rel=1e-12, eps_abs=1e-14, seed=2,
                           leaf_size=16)
    with pytest.raises(MaxSketchReached) as ei:
        hss_device.compress(DenseAccessor(A), tree, opts)
    from hsskit import compress
    with pytest.raises(MaxSketchReached) as er:
        compress(DenseAccessor(A), tree, opts)
    assert ei.value.blocking_nid == er.value.blocking_nid and ei.value.d == er.value.d
    with pytest.raises(ValueError, match="square"):
        hss_device.compress(DenseAccessor(np.zeros((128, 64))), tree, opts)


def test_plugin_compressor_install_and_device_accessor(cuda, tmp_path):
    """plugin.install(compressor=True) routes hsskit.compress through the
    device driver; an .hssd file loaded straight into HBM (hssd.from_file,
    DeviceAccessor) compresses to the reference's error (§8(f) row 2)."""
    import hsskit.sketching as hs
    from hsskit import compress, relative_error
    from hsskit.hss_compress import CompressOptions
    from hsskit.matgen import covariance_matrix
    from paper_2302_01977_b200 import hssd
    acc, tree = covariance_matrix(8, 0.2, leaf_size=64)
    opts = CompressOptions(d0=64, dd=32, eps_rel=1e-4, eps_abs=1e-10, kind="sjlt", alpha=4,
                           seed=3, leaf_size=64)
    H_ref = compress(acc, tree, opts)
    e_ref = relative_error(acc.dense(), H_ref)
    path = str(tmp_path / "cov.hssd")
    hssd.write_file(path, acc.dense())
    dacc = hssd.from_file(path)
    plugin.install(hs, compressor=True)
    try:
        import hsskit.hss_compress as hc
        assert hc._Driver.__name__ == "DeviceDriver"
        H_dev = compress(dacc, tree, opts)
    finally:
        plugin.uninstall(hs)
    assert hc._Driver.__name__ == "_Driver"
    e_dev = relative_error(acc.dense(), H_dev)
    assert abs(e_dev - e_ref) <= 0.01 * e_ref, (e_dev, e_ref)
    assert H_dev.final_d == H_ref.final_d


@pytest.mark.slow
def test_c1_hss_device_driver_matches_reference(cuda):
    """BASELINE.json configs[0] downstream gate through the device driver: the
    whole C1 compression (sketch, sweep, IDs) on the GPU, relative error within
    1% of the reference's CPU run on the same A bytes (SURVEY §8(c):
    2.070606e-05, final_d 1984)."""
    from hsskit import build_uniform, compress, relative_error, stats
    from hsskit.hss_compress import CompressOptions
    from hsskit.sketching import DenseAccessor
    n = 4096
    Ah = matgen.gaussian_kernel(n, 8, 0.5).to_host()
    opts = CompressOptions(d0=192, dd=64, eps_rel=1e-6, eps_abs=1e-8, leaf_size=128,
                           kind="sjlt", alpha=4, construction="graph", seed=0)
    tree = build_uniform(n, 128)
    t0 = time.perf_counter()
    H_ref = compress(DenseAccessor(Ah), tree, opts)
    t1 = time.perf_counter()
    hss_device.compress(DenseAccessor(Ah), tree, opts)   # warm-up (plans, cuSOLVER handles)
    t2 = time.perf_counter()
    H_dev = hss_device.compress(DenseAccessor(Ah), tree, opts)
    t3 = time.perf_counter()
    e_ref, e_dev = relative_error(Ah, H_ref), relative_error(Ah, H_dev)
    s_ref, s_dev = stats(H_ref), stats(H_dev)
    print(f"C1 HSS: reference {e_ref:.6e} final_d {s_ref.final_d} max_rank {s_ref.max_rank} "
          f"{t1 - t0:.2f} s; device driver {e_dev:.6e} final_d {s_dev.final_d} "
          f"max_rank {s_dev.max_rank} {t3 - t2:.2f} s (first call {t2 - t1:.2f} s)")
    assert abs(e_dev - e_ref) <= 0.01 * e_ref, (e_dev, e_ref)
    assert s_dev.final_d == s_ref.final_d
