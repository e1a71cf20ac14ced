"""Shared pytest configuration.

Markers: `gpu` tests need a B200 (run with `-m gpu` on the GPU box); all
other tests run on CPU.  BLAS threads are pinned to 1 before numpy loads, as
the reference's suite does (reference tests/conftest.py:8-11), so the CPU
oracle comparisons are reproducible.
"""

import os
import sys

for _name in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_name, "1")

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import json  # noqa: E402

import numpy as np  # noqa: E402
import pytest  # noqa: E402

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device")
    config.addinivalue_line("markers", "slow: long-running")


# Modules that drive the reference package (hsskit from baseline/_ref, installed
# by __graft_entry__.build()).  Without it they FAIL (never skip); they run
# last so that, under `pytest -x`, a missing install cannot hide the results of
# the engine's own parity tests.
_REFERENCE_MODULES = ("test_gpu_plugin.py", "test_gpu_hss_device.py", "test_gpu_reference_suite.py")


def pytest_collection_modifyitems(session, config, items):
    def uses_reference(item):
        return os.path.basename(str(item.fspath)) in _REFERENCE_MODULES
    items.sort(key=uses_reference)   # stable: original order within each group


@pytest.fixture(scope="session")
def golden():
    arrays = np.load(os.path.join(GOLDEN_DIR, "golden.npz"))
    with open(os.path.join(GOLDEN_DIR, "golden.json")) as f:
        manifest = json.load(f)
    return arrays, manifest


@pytest.fixture(scope="session")
def cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("GPU test collected without a CUDA device (run -m 'not gpu' on CPU)")
    from paper_2302_01977_b200 import _lib
    _lib.load()
    return torch.device("cuda", 0)


def case_inputs(case):
    """Regenerate a golden case's seeded inputs (A: m_right x n, B: n x m_left)."""
    rng = np.random.default_rng(case["data_seed"])
    A = rng.standard_normal((case["m_right"], case["n"]))
    B = rng.standard_normal((case["n"], case["m_left"]))
    return A, B


def seed_of(s):
    return tuple(s) if isinstance(s, list) else s


@pytest.fixture
def tune(monkeypatch):
    """Set an HSK_* tuning variable for one test: libhsk reads them once and
    caches them, so every change (and the undo at teardown) is followed by
    hsk_tuning_reload()."""
    from paper_2302_01977_b200 import _lib

    def set_(name, value):
        monkeypatch.setenv(name, value)
        _lib.load().hsk_tuning_reload()
    yield set_
    monkeypatch.undo()
    _lib.load().hsk_tuning_reload()
