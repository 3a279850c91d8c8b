"""Host binning (grid.py mirror of the reference's grid.py:77-134) against the
reference-generated fixtures tests/golden/grid.npz and grid_special.npz."""

import os

import numpy as np


def _golden(name):
    return np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", name))


def test_host_grid_matches_reference_golden():
    from paper_2410_23244_b200.grid import build_grid_midpoints, build_grid_uniform, quantize
    g = _golden("grid.npz")
    gu = build_grid_uniform(g["X"], 40)
    np.testing.assert_array_equal(gu.counts, g["uniform_counts"])
    np.testing.assert_array_equal(np.concatenate(gu.cutpoints), g["uniform_cuts"])
    np.testing.assert_array_equal(quantize(g["X"], gu).data, g["q_train"])
    np.testing.assert_array_equal(quantize(g["X_new"], gu).data, g["q_new"])
    gm = build_grid_midpoints(g["Xm"])
    np.testing.assert_array_equal(gm.counts, g["mid_counts"])
    np.testing.assert_array_equal(np.concatenate(gm.cutpoints), g["mid_cuts"])
    np.testing.assert_array_equal(quantize(g["Xm"], gm).data, g["qm"])


def test_host_quantize_non_finite_rows_match_reference():
    from paper_2410_23244_b200.grid import build_grid_uniform, quantize
    g = _golden("grid_special.npz")
    grid = build_grid_uniform(g["X"], 60)
    np.testing.assert_array_equal(grid.counts, g["counts"])
    np.testing.assert_array_equal(quantize(g["X_special"], grid).data, g["q_special"])

