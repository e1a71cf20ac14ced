"""bench.py's reference arm on CPU: `--impl reference` times the oracle C port
of SjltBlock.apply_right (the reference's CPU path) on a bounded slab of the
C2 workload and prints one JSON line with the contract's keys."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    env = dict(os.environ, HSK_REF_ROWS="64")
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True,
                         timeout=600, env=env, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    line = json.loads(res.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "GB/s" and line["value"] > 0
    assert line["warmup"] == 3 and line["steps"] == 2          # W >= 3 enforced
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]
    assert line["config"]["workload"] == "c2_sjlt_S" and line["config"]["rows_per_step"] == 64


def test_reference_arm_other_ranks_exit_quietly():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2")
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--gpus", "2", "--steps", "1"], capture_output=True, text=True,
                         timeout=300, env=env, cwd=ROOT)
    assert res.returncode == 0 and res.stdout.strip() == ""


def test_committed_ncu_summary_feeds_roofline_traffic():
    """bench.py's `roofline.traffic` is the headline kernel's per-launch DRAM
    bytes from the committed ncu capture (profiles/ncu_summary.json): the key
    must exist and sit near the algorithmic bytes (8 n^2 + 8 n d)."""
    sys.path.insert(0, ROOT)
    import bench
    traffic = bench._traffic_from_profiles("sjlt_apply_S")
    algorithmic = 8 * bench.N * bench.N + 8 * bench.N * bench.D
    assert traffic is not None and 0.9 * algorithmic <= traffic <= 1.5 * algorithmic
