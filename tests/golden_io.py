"""Loader for the golden step vectors in tests/golden/ (made by make_golden.py)."""

from __future__ import annotations

import glob
import os
from types import SimpleNamespace

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
STEP_CASES = sorted(os.path.basename(p)[5:-4] for p in glob.glob(os.path.join(GOLDEN, "step_*.npz")))


def load_case(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, f"step_{name}.npz")) as z:
        d = {k: z[k] for k in z.files}
    h, hi = d["hp"], d["hp_int"]
    d["hpns"] = SimpleNamespace(
        leaf_sd=float(h[0]), lam=float(h[1]), alpha=float(h[2]), beta=float(h[3]),
        leaf_mean=float(h[4]), nu=float(h[5]), p_grow=float(h[6]),
        n_trees=int(hi[0]), max_depth=int(hi[1]), update_sigma=bool(hi[2]),
    )
    d["steps"] = d["chi2"].shape[0]
    return d


def load(name: str) -> dict:
    with np.load(os.path.join(GOLDEN, name)) as z:
        return {k: z[k] for k in z.files}
