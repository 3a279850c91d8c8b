"""Golden quantize vectors for non-finite test rows, from the REAL reference.

Test infrastructure only (run in the build container, where /root/reference
is mounted read-only):  python tests/golden/make_grid_special.py

bforge.grid.quantize is np.searchsorted(cuts, x, side="right") per axis
(grid.py:121-134): NaN sorts after every cutpoint (-> len(cuts)), +inf goes
to len(cuts), -inf to 0.  fit()/predict() quantize test rows with it, so the
device quantize must agree on them.  Writes tests/golden/grid_special.npz.
"""
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="numba_golden_"))
sys.dont_write_bytecode = True
sys.path.insert(0, "/root/reference/pkg/src")

from bforge.grid import build_grid_uniform, quantize  # noqa: E402

OUT = Path(__file__).resolve().parent


def main():
    r = np.random.default_rng(21)
    X = r.normal(size=(300, 4))
    X[:, 2] = -0.25  # degenerate axis: no cutpoints
    grid = build_grid_uniform(X, 60)
    Xs = r.normal(scale=3.0, size=(64, 4))
    Xs[::5, 0] = np.nan
    Xs[1::7, 1] = np.inf
    Xs[2::7, 1] = -np.inf
    Xs[3::6, 2] = np.nan
    Xs[4::9, 3] = np.nan
    Xs[5, :] = np.nan
    np.savez_compressed(OUT / "grid_special.npz", X=X, counts=grid.counts,
                        cuts=np.concatenate(grid.cutpoints), X_special=Xs, q_special=quantize(Xs, grid).data)
    print("grid_special.npz written")


if __name__ == "__main__":
    main()
