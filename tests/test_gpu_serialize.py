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


def test_fit_streams_trace_through_device_ring(tmp_path, monkeypatch):
    """With a 4-draw device ring (the ring a huge n * n_kept would get), the
    streamed file still holds every kept draw: the ring is drained to the file
    as it fills (bounded device memory for streamed traces)."""
    from paper_2410_23244_b200 import regression, serialize
    from paper_2410_23244_b200.regression import FitConfig, fit
    X, y = _data()
    base = dict(n_trees=20, n_burn=10, n_kept=11, thinning=1, n_chains=2, seed=6)
    full = fit(X, y, FitConfig(**base, keep_train_draws=True))
    monkeypatch.setattr(regression, "_TRACE_RING_BYTES", 4 * 8 * X.shape[0])  # -> 4 rows per chain
    path = tmp_path / "ring.bftrace"
    fit(X, y, FitConfig(**base, keep_train_draws=False), trace_path=str(path))
    got = serialize.load_trace(str(path))
    np.testing.assert_array_equal(got.yhat_train, full.yhat_train)


def test_trace_ring_windows():
    """bart_trace_read_draws over a ring: windows still in it read back exactly
    (also across the wrap), older ones are refused, the whole-trace read too."""
    from paper_2410_23244_b200.sampler import DeviceRNG, Hyperparams, init_state, run
    rng = np.random.default_rng(3)
    X = rng.integers(0, 10, (500, 3)).astype(np.uint8)
    hp = Hyperparams(leaf_sd=0.3, lam=0.1, n_trees=5, max_depth=4)
    y = rng.normal(size=500).astype(np.float32)
    a = init_state(X, np.full(3, 9), y, hp, DeviceRNG(8), sigma2=1.0)
    b = init_state(X, np.full(3, 9), y, hp, DeviceRNG(8), sigma2=1.0)
    a.trace_begin(20, 10, store_train_draws=True)
    b.trace_begin(20, 10, store_train_draws=True, train_ring=3)
    got = []
    for k in range(10):
        for st in (a, b):
            run(st, hp, 2)
            st.trace_keep()
        if k % 3 == 2:  # drain b's ring every 3 draws
            got.append(b.trace_read_draws(k - 2, k + 1)[0])
    want = a.trace_read_draws(0, 10)[0]
    np.testing.assert_array_equal(np.concatenate(got), want[:9])
    np.testing.assert_array_equal(b.trace_read_draws(8, 10)[0], want[8:10])  # wraps the ring end
    with pytest.raises(ValueError):
        b.trace_read_draws(5, 8)  # overwritten
    with pytest.raises(RuntimeError):
        b.trace_read(train_draws=True)
    a.close()
    b.close()


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
