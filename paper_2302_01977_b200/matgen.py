"""BASELINE.json configuration matrices, generated directly in HBM.

None of the configs' matrices exist in the reference's matgen.py, so they
are defined here:

  gaussian kernel  A_ij = exp(-|x_i - x_j|^2 / (2 h^2)) + 1e-2 * [i == j],
                   x_i ~ U[0,1]^D i.i.d. from default_rng(seed)   (C1,C2,C4,C5)
  toeplitz-sine    A_ij = 1/(1 + |i-j|) + 0.1 sin(i + 2j) / n      (C3)

The points are drawn on the host (bit-reproducible numpy stream) and the
entries are evaluated by libhsk kernels, so a 34-137 GB matrix never exists
on the host.  For parity checks the oracle must see the SAME bytes: copy
slabs back with DeviceMatrix.to_host / row_view (GPU and numpy exp/sin
differ in the last bits).
"""

from __future__ import annotations

import dataclasses

import numpy as np

from . import _lib
from . import device as _dev


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    n: int
    kind: str                 # primary sketch kind
    d: int
    alpha: int | None = None
    construction: str | None = None
    matrix: str = "gauss"     # "gauss" | "toeplitz_sin"
    dim: int = 8
    h: float = 0.5
    dd: int | None = None     # adaptive increment
    blocks: int = 1


CONFIGS = {
    "c1": Config("c1", 4096, "sjlt", 256, 4, "graph", "gauss", 8, 0.5),
    "c2": Config("c2", 16384, "gaussian", 512, None, None, "gauss", 8, 0.5),
    "c2_sjlt": Config("c2_sjlt", 16384, "sjlt", 512, 4, "block", "gauss", 8, 0.5),
    "c3": Config("c3", 65536, "sjlt", 1024, 8, "block", "toeplitz_sin", dd=64, blocks=16),
    "c4": Config("c4", 65536, "srht", 512, None, None, "gauss", 8, 0.25),
    "c5_sjlt": Config("c5_sjlt", 131072, "sjlt", 2048, 8, "block", "gauss", 16, 1.0),
    "c5_gauss": Config("c5_gauss", 131072, "gaussian", 512, None, None, "gauss", 16, 1.0),
}


def kernel_points(n: int, dim: int, seed: int = 0) -> np.ndarray:
    """x_i ~ U[0,1]^dim, i.i.d., from default_rng(seed) (n x dim, C order)."""
    return np.random.default_rng(seed).uniform(0.0, 1.0, (n, dim))


def gaussian_kernel(n: int, dim: int, h: float, diag: float = 1e-2, seed: int = 0,
                    row0: int = 0, nrows: int | None = None, ld: int | None = None,
                    points=None, stream=None) -> "_dev.DeviceMatrix":
    """Rows [row0, row0+nrows) of the n x n Gaussian-kernel matrix in HBM."""
    import torch
    nrows = n - row0 if nrows is None else nrows
    pts = kernel_points(n, dim, seed) if points is None else points
    dpts = torch.from_numpy(np.ascontiguousarray(pts, dtype=np.float64)).cuda()
    A = _dev.DeviceMatrix.empty(nrows, n, ld)
    st = _dev.current_stream_ptr() if stream is None else stream
    _lib.call("hsk_gen_gauss_kernel", dpts.data_ptr(), n, dim, float(h), float(diag), row0,
              nrows, 0, n, A.ptr, A.ld, st)
    torch.cuda.current_stream().synchronize()
    return A


def toeplitz_sin(n: int, row0: int = 0, nrows: int | None = None, ld: int | None = None,
                 stream=None) -> "_dev.DeviceMatrix":
    """Rows [row0, row0+nrows) of A_ij = 1/(1+|i-j|) + 0.1 sin(i+2j)/n in HBM."""
    nrows = n - row0 if nrows is None else nrows
    A = _dev.DeviceMatrix.empty(nrows, n, ld)
    st = _dev.current_stream_ptr() if stream is None else stream
    _lib.call("hsk_gen_toeplitz_sin", n, row0, nrows, 0, n, A.ptr, A.ld, st)
    return A


def config_matrix(cfg: Config, row0: int = 0, nrows: int | None = None,
                  seed: int = 0) -> "_dev.DeviceMatrix":
    if cfg.matrix == "toeplitz_sin":
        return toeplitz_sin(cfg.n, row0, nrows)
    return gaussian_kernel(cfg.n, cfg.dim, cfg.h, 1e-2, seed, row0, nrows)
