"""bench.py's host-side pieces (no GPU): the BASELINE config labels, the tree
statistics of the line, and the reference arm's JSON line on a tiny workload."""

import json
import os
import subprocess
import sys
from types import SimpleNamespace

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_config_labels_name_the_baseline_configs():
    lab = lambda n, p, m: bench.baseline_config_label(SimpleNamespace(n=n, p=p, m=m))
    assert lab(1_000_000, 100, 200) == "BASELINE.json configs[2]"
    assert lab(100_000, 100, 200) == "BASELINE.json configs[1]"
    assert lab(10_000_000, 100, 200) == "BASELINE.json configs[3]"
    assert lab(1_000_000, 1000, 1000) == "BASELINE.json configs[4]"
    assert lab(12345, 3, 7) == "not a BASELINE.json config"


def test_tree_stats_counts_leaves_from_cutpoints():
    cut = np.zeros((3, 32), np.uint8)
    cut[1, 1] = 5                 # a stump: 2 leaves
    cut[2, [1, 2, 3]] = 7         # 4 leaves
    st = SimpleNamespace(forest=SimpleNamespace(cutpoint=cut), iteration=17)
    t = bench.tree_stats(st)
    assert t["mean_leaves"] == (1 + 2 + 4) / 3 and t["max_leaves"] == 4
    assert t["leaves_hist"] == {"1": 1, "2": 1, "4": 1} and t["iteration"] == 17


def test_reference_arm_line_on_a_tiny_workload():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--points", "2000",
                          "--p", "5", "--m", "10", "--steps", "20", "--warmup", "5"],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["unit"] == "iters/s" and d["value"] > 0
    assert d["steps"] == bench.REF_MAX_STEPS and d["steps_requested"] == 20 and d["warmup"] == 1
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    # the job's step is the slowest chain's full iteration: value = chains / step time
    assert abs(d["value"] - d["cpu_baseline"]["cores"] * 1e3 / d["ms_per_step"]) < 1e-6 * d["value"]
