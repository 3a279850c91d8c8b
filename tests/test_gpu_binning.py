"""GPU binning (csrc/binning.cu) against the reference's numpy semantics
(grid.py:77-95 uniform grid, grid.py:121-134 searchsorted side="right")."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_quantize_matches_numpy_with_ties_and_edges():
    from paper_2410_23244_b200.grid import build_grid_midpoints, build_grid_uniform, quantize
    rng = np.random.default_rng(0)
    X = rng.normal(size=(20011, 7)) * 10.0 ** rng.integers(-3, 4, size=7)
    X[:, 3] = np.round(X[:, 3])              # many ties
    X[:, 5] = 2.5                            # constant axis: no cutpoints
    X[:100, 0] = X[:100, 0].max()            # values equal to the top of the range
    for grid in (build_grid_uniform(X, 100), build_grid_uniform(X, 255), build_grid_midpoints(X)):
        want = quantize(X, grid).data
        got = quantize(X, grid, device=0).data
        np.testing.assert_array_equal(got, want)
        # exact cutpoint values go right (ties right, grid.py:127-128)
        cuts = grid.cutpoints[0]
        probe = np.tile(cuts[:, None], (1, 7))
        np.testing.assert_array_equal(quantize(probe, grid, device=0).data[:, 0], np.arange(1, cuts.size + 1))


def test_uniform_grid_ranges_on_device():
    from paper_2410_23244_b200.grid import build_grid_uniform
    rng = np.random.default_rng(1)
    X = rng.normal(size=(100003, 11))
    X[:, 2] = -np.abs(X[:, 2])               # all negative
    X[:, 4] = 0.0                            # constant
    a, b = build_grid_uniform(X, 100), build_grid_uniform(X, 100, device=0)
    for ca, cb in zip(a.cutpoints, b.cutpoints):
        np.testing.assert_array_equal(ca, cb)
    with pytest.raises(ValueError):
        X[7, 1] = np.nan
        build_grid_uniform(X, 100, device=0)


@pytest.mark.parametrize("nc", [1, 100, 255])
def test_one_upload_grid_and_binning_equal_the_two_calls(nc):
    """fit()'s binning (grid_uniform_quantize: X uploaded once, cutpoints from the
    device ranges) equals build_grid_uniform + quantize, on the device and in
    numpy, bit for bit -- including values exactly at cutpoints."""
    from paper_2410_23244_b200.grid import build_grid_uniform, grid_uniform_quantize, quantize
    rng = np.random.default_rng(nc)
    X = rng.normal(size=(30011, 9)) * 10.0 ** rng.integers(-3, 4, size=9)
    X[:, 4] = -1.25                                  # constant axis: no cutpoints
    ref = build_grid_uniform(X, nc)
    X[:nc, 0] = ref.cutpoints[0]                     # rows exactly at axis 0's cutpoints
    ref = build_grid_uniform(X, nc)
    grid, qm = grid_uniform_quantize(X, nc, 0)
    for ca, cb in zip(ref.cutpoints, grid.cutpoints):
        np.testing.assert_array_equal(ca, cb)
    np.testing.assert_array_equal(qm.data, quantize(X, ref).data)
    np.testing.assert_array_equal(qm.data, quantize(X, ref, device=0).data)
    with pytest.raises(ValueError):
        X[3, 2] = np.inf
        grid_uniform_quantize(X, nc, 0)


def _golden(name):
    import os
    return np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", name))


def test_device_binning_matches_reference_golden():
    """tests/golden/grid.npz was written by the reference's own
    build_grid_uniform / build_grid_midpoints / quantize (make_golden.py):
    the device min/max grid and device quantize reproduce it exactly."""
    from paper_2410_23244_b200.grid import CutpointGrid, build_grid_uniform, quantize
    g = _golden("grid.npz")
    gu = build_grid_uniform(g["X"], 40, device=0)
    np.testing.assert_array_equal(gu.counts, g["uniform_counts"])
    np.testing.assert_array_equal(np.concatenate(gu.cutpoints), g["uniform_cuts"])
    np.testing.assert_array_equal(quantize(g["X"], gu, device=0).data, g["q_train"])
    np.testing.assert_array_equal(quantize(g["X_new"], gu, device=0).data, g["q_new"])
    off = np.concatenate([[0], np.cumsum(g["mid_counts"])])
    gm = CutpointGrid([g["mid_cuts"][off[a]:off[a + 1]] for a in range(len(g["mid_counts"]))])
    np.testing.assert_array_equal(quantize(g["Xm"], gm, device=0).data, g["qm"])


def test_device_quantize_non_finite_rows_match_reference():
    """NaN -> len(cuts), +inf -> len(cuts), -inf -> 0, as the reference's
    np.searchsorted(side="right") (grid.py:121-134; grid_special.npz)."""
    from paper_2410_23244_b200.grid import CutpointGrid, quantize
    g = _golden("grid_special.npz")
    off = np.concatenate([[0], np.cumsum(g["counts"])])
    grid = CutpointGrid([g["cuts"][off[a]:off[a + 1]] for a in range(len(g["counts"]))])
    np.testing.assert_array_equal(quantize(g["X_special"], grid, device=0).data, g["q_special"])
