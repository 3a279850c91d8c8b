"""fit()'s host-side post-processing (no GPU)."""

import numpy as np


def test_yscale_inverse_in_place_is_bit_identical():
    """fit() unscales the (C, K, n) draws in place (YScale.inverse_): the same two
    roundings as inverse, bit for bit."""
    from paper_2410_23244_b200.regression import YScale
    rng = np.random.default_rng(4)
    ys = YScale(center=0.37, scale=13.25)
    f = rng.normal(size=(3, 5, 1001)) * 10.0 ** rng.integers(-8, 8, size=(3, 5, 1001))
    want = ys.inverse(f)
    got = ys.inverse_(f.copy())
    np.testing.assert_array_equal(got, want)
