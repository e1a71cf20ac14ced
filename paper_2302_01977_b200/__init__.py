"""B200-native sketch engine for randomized HSS compression (arXiv 2302.01977).

The hot path -- S = A R^T and S' = A^T R^T for the SJLT, Gaussian and SRHT
operators, with adaptive Delta-d appends -- runs as hand-written sm_100a
CUDA kernels in libhsk.so (C ABI: include/hsk.h), bound with ctypes.

  sketching   drop-in for hsskit.sketching (same API, GPU products)
  plugin      install()/uninstall() into the reference package
  adaptive    DeviceSketch: preallocated S/S' grown by column appends
  distributed row-block sharding over GPUs + NCCL reduce-scatter of S'
  matgen      BASELINE.json config matrices generated in HBM
"""

from . import draws, operators, sketching  # noqa: F401

__version__ = "0.1.0"
