"""The reference's OWN test suite (hsskit tests/, copied next to the install in
baseline/_ref_tests by __graft_entry__.build()) run with the drop-in installed:
every sketch product through libhsk and the whole compression sweep through
hss_device.DeviceDriver (tests/refsuite_gpu_plugin.py).  The reference's
acceptance criteria print their verdicts as in its own runs.  Left out, because
they run the reference's CLI, which imports matplotlib (absent from this image;
they fail the same way without the drop-in, and the CLI subprocess would not
load it anyway): test_cli.py and acceptance criterion 9 (CLI reruns)."""

import os
import re
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITE = os.path.join(ROOT, "baseline", "_ref_tests")


def test_reference_suite_with_gpu_sketch_and_device_driver(cuda):
    if not os.path.isdir(SUITE):
        pytest.fail(f"reference tests not found at {SUITE}: run __graft_entry__.build() "
                    "where /root/reference exists")
    files = sorted(os.path.join(SUITE, f) for f in os.listdir(SUITE)
                   if f.startswith("test_") and f.endswith(".py") and f != "test_cli.py")
    env = dict(os.environ)
    env["PYTHONPATH"] = os.pathsep.join([ROOT, os.path.join(ROOT, "tests"),
                                         os.path.join(ROOT, "baseline", "_ref"),
                                         env.get("PYTHONPATH", "")])
    cmd = [sys.executable, "-m", "pytest", "-q", "-p", "refsuite_gpu_plugin",
           "-p", "no:cacheprovider", "-k", "not test_criterion_9_byte_identical_reruns",
           *files]
    res = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT, env=env, timeout=1800)
    tail = res.stdout[-4000:]
    print(tail)
    assert "DeviceDriver" in res.stdout, "drop-in not installed in the reference run"
    assert res.returncode == 0, tail + res.stderr[-2000:]
    assert re.search(r"\d+ passed", res.stdout)
    verdicts = [l for l in res.stdout.splitlines() if l.startswith("ACCEPTANCE")]
    assert all("PASS" in l for l in verdicts if not l.startswith("ACCEPTANCE 9")), verdicts
