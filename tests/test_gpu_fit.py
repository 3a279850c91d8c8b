"""The gbart-style API on the device (regression.fit / predict / diagnostics;
reference regression.py:145-313), including the on-device trace."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _data(n=600, p=5, seed=0):
    from paper_2410_23244_b200.dgp import friedman1
    X, y, f = friedman1(n, p, seed=seed)
    return X, y, f


def test_device_trace_equals_host_trace():
    """Same chains (reference Generator stream): recording on the device gives
    the same trace as reading the state back every iteration."""
    from paper_2410_23244_b200.regression import FitConfig, fit
    X, y, _ = _data()
    Xt = X[:50] + 0.01
    base = dict(n_trees=30, n_burn=20, n_kept=15, thinning=2, n_chains=2, rng="host", seed=3)
    a = fit(X, y, FitConfig(**base, trace="device", keep_train_draws=True, keep_forests=True), X_test=Xt)
    b = fit(X, y, FitConfig(**base, trace="host", keep_forests=True), X_test=Xt)
    np.testing.assert_array_equal(a.accepted, b.accepted)
    np.testing.assert_array_equal(a.sigma, b.sigma)
    np.testing.assert_array_equal(a.yhat_train, b.yhat_train)
    np.testing.assert_array_equal(a.yhat_test, b.yhat_test)
    np.testing.assert_array_equal(a.mean_leaves, b.mean_leaves)
    for fa, fb in zip(a.forests[1], b.forests[1]):
        np.testing.assert_array_equal(fa.cutpoint, fb.cutpoint)
        np.testing.assert_array_equal(fa.leaf_value, fb.leaf_value)
    np.testing.assert_allclose(a.yhat_train_mean, b.yhat_train.mean(axis=1), rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(a.yhat_train_var, b.yhat_train.var(axis=1, ddof=1), rtol=1e-8, atol=1e-12)


def test_fit_recovers_friedman_and_diagnostics_without_draws():
    """Device RNG, moments-only trace: the posterior mean tracks the true
    function (reference A3-style recovery check) and diagnostics run on the
    recorded check-point draws."""
    from paper_2410_23244_b200.regression import FitConfig, diagnostics, fit, predict
    X, y, f = _data(n=2000, seed=1)
    tr = fit(X, y, FitConfig(n_trees=50, n_burn=100, n_kept=100, n_chains=2, keep_train_draws=False,
                             keep_forests=True))
    assert tr.yhat_train is None and tr.yhat_train_mean.shape == (2, 2000)
    rmse = float(np.sqrt(np.mean((tr.yhat_train_mean.mean(axis=0) - f) ** 2)))
    assert rmse < 1.0, rmse
    rep = diagnostics(tr)
    assert 0.0 < rep.acceptance_rate < 1.0 and rep.cross_chain_ks <= 1.0
    pr = predict(tr, X[:100])
    np.testing.assert_allclose(pr.mean, tr.yhat_train_mean.mean(axis=0)[:100], rtol=1e-9, atol=1e-9)
    assert tr.sigma.shape == (2, 100) and np.all(tr.sigma > 0)


def test_fit_matches_reference_golden():
    """Whole-API parity: the reference's own fit() (regression.py:145-216, host
    Philox streams) recorded in tests/golden/fit.npz, against fit(rng="host")
    here: identical accept decisions in every chain and iteration, and the kept
    draws to f32 rounding (the device sums in a different f64 order)."""
    import os
    from paper_2410_23244_b200.regression import FitConfig, fit
    d = np.load(os.path.join(os.path.dirname(__file__), "golden", "fit.npz"))
    n_trees, n_burn, n_kept, n_chains, seed = (int(v) for v in d["cfg"])
    cfg = FitConfig(n_trees=n_trees, n_burn=n_burn, n_kept=n_kept, n_chains=n_chains, seed=seed, rng="host",
                    keep_train_draws=True)
    for trace_mode in ("device", "host"):
        tr = fit(d["X"], d["y"], FitConfig(**{**cfg.__dict__, "trace": trace_mode}), X_test=d["X_test"])
        np.testing.assert_array_equal(tr.accepted, d["accepted"].astype(bool))
        np.testing.assert_allclose(tr.sigma, d["sigma"], rtol=1e-5)
        np.testing.assert_allclose(tr.yhat_train, d["yhat_train"], rtol=1e-5, atol=1e-5)
        np.testing.assert_allclose(tr.yhat_test, d["yhat_test"], rtol=1e-5, atol=1e-5)
        np.testing.assert_allclose(tr.mean_leaves, d["mean_leaves"], rtol=1e-12)
