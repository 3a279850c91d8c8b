"""Golden BFORGE1 / BFTRACE1 files written by the REAL reference (`bforge`).

Test infrastructure only.  Run in the build container (the reference is
mounted read-only at /root/reference):

    python tests/golden/make_serialize_golden.py

Builds a small deterministic forest, grid and trace from `serialize_inputs()`
(shared with tests/test_serialize.py, which rebuilds the same objects with
this package's classes) and writes them with the reference's own
`bforge.serialize.save_forest` / `save_trace` (serialize.py:66-133).  The
tests check that this package reads the files and writes byte-identical ones.
"""

from __future__ import annotations

import io
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent


def serialize_inputs(with_test: bool):
    """Plain arrays of a 2-chain, 3-draw trace (depth 3, 4 trees, 2 axes)."""
    rng = np.random.default_rng(11)
    D, m, C, K, n, n_iter = 3, 4, 2, 3, 5, 6
    half, full = 2 ** (D - 1), 2 ** D
    cuts = [np.linspace(0.0, 1.0, 4), np.array([-2.0, 0.5, 3.25])]
    def forest_arrays():
        axis = np.zeros((m, half), np.uint8)
        cut = np.zeros((m, half), np.uint8)
        leaf = np.zeros((m, full), np.float32)
        for j in range(m):  # root split + one child split on some trees
            axis[j, 1], cut[j, 1] = j % 2, 1 + j % 3
            if j % 2 == 0:
                axis[j, 2], cut[j, 2] = 1, 1 + (j // 2) % 3
                leaf[j, [3, 4, 5]] = rng.normal(size=3).astype(np.float32)
            else:
                leaf[j, [2, 3]] = rng.normal(size=2).astype(np.float32)
        return axis, cut, leaf
    out = dict(D=D, m=m, C=C, K=K, n=n, n_iter=n_iter, cuts=cuts, forest=forest_arrays(),
               sigma=rng.gamma(2.0, 0.3, (C, K)), yhat_train=rng.normal(size=(C, K, n)),
               accepted=rng.random((C, n_iter, m)) < 0.4, mean_leaves=rng.normal(size=(C, K)) * 1e-3,
               forests=[[forest_arrays() for _ in range(K)] for _ in range(C)],
               center=1.25, scale=3.5)
    if with_test:
        out["x_test"] = rng.normal(size=(2, 2))
        out["yhat_test"] = rng.normal(size=(C, K, 2))
    return out


CONFIG = dict(n_trees=4, n_burn=3, n_kept=3, thinning=1, max_depth=3, grid="uniform", n_cutpoints=4, seed=5,
              k=2.0, q=0.9, nu=3.0, n_chains=2, alpha=0.95, beta=2.0, p_grow=0.5, keep_forests=None)


def main():
    os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="numba_golden_"))
    sys.dont_write_bytecode = True
    sys.path.insert(0, REF_SRC)
    from bforge import serialize
    from bforge.grid import CutpointGrid
    from bforge.regression import FitConfig, Trace, YScale
    from bforge.trees import Forest

    def forest(t, D):
        return Forest(axis=t[0], cutpoint=t[1], leaf_value=t[2], max_depth=D)

    a = serialize_inputs(False)
    buf = io.BytesIO()
    serialize.save_forest(buf, forest(a["forest"], a["D"]), CutpointGrid(a["cuts"]))
    (OUT / "ref_forest.bforge").write_bytes(buf.getvalue())
    for with_test in (False, True):
        a = serialize_inputs(with_test)
        trace = Trace(config=FitConfig(**CONFIG), yscale=YScale(center=a["center"], scale=a["scale"]),
                      grid=CutpointGrid(a["cuts"]), sigma=a["sigma"], yhat_train=a["yhat_train"],
                      yhat_test=a.get("yhat_test"), accepted=a["accepted"], mean_leaves=a["mean_leaves"],
                      forests=None if with_test else [[forest(t, a["D"]) for t in ch] for ch in a["forests"]],
                      x_test=a.get("x_test"))
        serialize.save_trace(str(OUT / ("ref_trace_test.bftrace" if with_test else "ref_trace.bftrace")), trace)
    print("wrote", sorted(p.name for p in OUT.glob("ref_*")))


if __name__ == "__main__":
    main()
