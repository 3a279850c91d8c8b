"""Containers fed from the device: fit(..., trace_path=) streams the kept draws
into a BFTRACE1 file; checkpoints resume a chain bit-identically."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _data(n=700, p=5, seed=1):
    from paper_2410_23244_b200.dgp import friedman1
    X, y, _ = friedman1(n, p, seed=seed)
    return X, y


@pytest.mark.parametrize("with_test", [False, True])
def test_fit_streams_trace_file(tmp_path, with_test):
    """The streamed file holds exactly the draws a keep_train_draws fit returns,
    even when the returned trace keeps none of them in host memory."""
    from paper_2410_23244_b200 import serialize
    from paper_2410_23244_b200.regression import FitConfig, fit, predict
    X, y = _data()
    Xt = X[:40] * 0.97 if with_test else None
    base = dict(n_trees=20, n_burn=15, n_kept=9, thinning=2, n_chains=2, seed=4)
    full = fit(X, y, FitConfig(**base, keep_train_draws=True), X_test=Xt)
    path = tmp_path / "trace.bftrace"
    lean = fit(X, y, FitConfig(**base, keep_train_draws=False), X_test=Xt, trace_path=str(path))
    assert lean.yhat_train is None
    got = serialize.load_trace(str(path))
    np.testing.assert_array_equal(got.yhat_train, full.yhat_train)
    np.testing.assert_array_equal(got.sigma, full.sigma)
    np.testing.assert_array_equal(got.accepted, full.accepted)
    np.testing.assert_array_equal(got.mean_leaves, full.mean_leaves)
    if with_test:
        np.testing.assert_array_equal(got.yhat_test, full.yhat_test)
        np.testing.assert_array_equal(got.x_test, Xt)
    else:  # forests kept: predictions from the loaded trace reproduce the fit's
        np.testing.assert_array_equal(predict(got, X[:11]).values, predict(full, X[:11]).values)
    # a trace that kept its draws writes the same file through save_trace
    serialize.save_trace(str(tmp_path / "whole.bftrace"), full)
    whole = serialize.load_trace(str(tmp_path / "whole.bftrace"))
    np.testing.assert_array_equal(whole.yhat_train, got.yhat_train)


@pytest.mark.parametrize("rng_kind", ["device", "numpy"])
def test_checkpoint_resume_is_bit_identical(tmp_path, rng_kind):
    from paper_2410_23244_b200 import serialize
    from paper_2410_23244_b200.sampler import DeviceRNG, init_state, run, step
    from paper_2410_23244_b200.regression import FitConfig, derive_hyperparams
    from paper_2410_23244_b200 import grid as gridmod
    X, y = _data(n=900)
    g = gridmod.build_grid_uniform(X, 30)
    Xq = gridmod.quantize(X, g).data
    hp, ys = derive_hyperparams(y, FitConfig(n_trees=25, max_depth=5))
    rng = DeviceRNG(77) if rng_kind == "device" else np.random.default_rng(77)

    def advance(st, k):
        if rng_kind == "device":
            run(st, hp, k)
            st.sync()
        else:
            for _ in range(k):
                step(st, hp)

    a = init_state(Xq, g.counts, ys.forward(y).astype(np.float32), hp, rng)
    advance(a, 7)
    path = tmp_path / "chain.bfckpt"
    serialize.save_checkpoint(str(path), a, hp)
    advance(a, 6)
    b, hp_b = serialize.load_checkpoint(str(path))
    assert b.iteration == 7 and hp_b == hp
    advance(b, 6)
    assert b.iteration == a.iteration == 13
    fa, fb = a.forest, b.forest
    np.testing.assert_array_equal(fa.axis, fb.axis)
    np.testing.assert_array_equal(fa.cutpoint, fb.cutpoint)
    np.testing.assert_array_equal(fa.leaf_value, fb.leaf_value)
    np.testing.assert_array_equal(a.resid, b.resid)
    np.testing.assert_array_equal(a.leaf_index, b.leaf_index)
    assert a.sigma2 == b.sigma2
    a.close()
    b.close()
