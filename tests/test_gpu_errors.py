"""Device error reporting: the step never returns wrong results as success.

The sweep's cross-CTA exchange carries per-leaf sums as exact fixed point
(sweep.cu to_limbs).  A partial outside its range (an unstandardised y whose
sum of squared residuals is huge) or a NaN residual sets a sticky device flag;
the host reports it as BART_ERANGE -> RuntimeError at the next read instead of
returning decisions computed from zeroed partials.  The reference would carry
the NaN on and reject every move (sampler.py:570-576, 833-834); here the chain
fails loudly and stays failed until its state is reset.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _chain(y, n=3000, p=4, m=8, seed=0):
    from paper_2410_23244_b200.sampler import Hyperparams, init_state
    rng = np.random.default_rng(seed)
    X = rng.integers(0, 20, (n, p)).astype(np.uint8)
    hp = Hyperparams(leaf_sd=0.3, lam=0.1, n_trees=m, max_depth=5)
    st = init_state(X, np.full(p, 19), np.asarray(y, np.float32), hp, None, sigma2=1.0)
    return st, hp, rng


def _randoms(rng, hp, n):
    from paper_2410_23244_b200.sampler import StepRandoms
    return StepRandoms.draw(rng, hp.n_trees, 1 << hp.max_depth, hp.nu + n)


def test_huge_y_raises_instead_of_wrong_sums():
    from paper_2410_23244_b200.sampler import step
    n = 3000
    y = np.random.default_rng(1).normal(size=n) * 1e12
    st, hp, rng = _chain(y, n)
    step(st, hp, randoms=_randoms(rng, hp, n))
    with pytest.raises(RuntimeError, match="fixed-point range"):
        st.step_result()
    with pytest.raises(RuntimeError, match="fixed-point range"):
        _ = st.resid  # every synced read reports it (sticky)
    st.close()


def test_nan_residual_raises_then_reset_recovers():
    from paper_2410_23244_b200.sampler import step
    n = 3000
    y = np.random.default_rng(2).normal(size=n)
    st, hp, rng = _chain(y, n)
    step(st, hp, randoms=_randoms(rng, hp, n))
    st.step_result()
    good, good_forest = st.resid.copy(), st.forest
    bad = good.copy()
    bad[17] = np.nan
    st.resid = bad
    step(st, hp, randoms=_randoms(rng, hp, n))
    with pytest.raises(RuntimeError, match="fixed-point range"):
        st.step_result()
    with pytest.raises(RuntimeError):
        st.sync()
    # a state reset clears the flag: the chain steps normally again
    st.forest = good_forest
    st.resid = good
    st.sigma2 = 1.0  # the NaN step drew a NaN sigma2 (sampler.py:797-799)
    st.rebuild_structure_caches()
    step(st, hp, randoms=_randoms(rng, hp, n))
    acc, s2 = st.step_result()
    assert np.isfinite(s2) and s2 > 0
    assert np.isfinite(st.resid).all()
    st.close()


def test_device_rng_run_reports_range_error_at_sync():
    from paper_2410_23244_b200.sampler import DeviceRNG, Hyperparams, init_state, run
    n = 5000
    rng = np.random.default_rng(3)
    X = rng.integers(0, 20, (n, 3)).astype(np.uint8)
    y = (rng.normal(size=n) * 1e13).astype(np.float32)
    hp = Hyperparams(leaf_sd=0.3, lam=0.1, n_trees=6, max_depth=4)
    st = init_state(X, np.full(3, 19), y, hp, DeviceRNG(4), sigma2=1.0)
    run(st, hp, 2)
    with pytest.raises(RuntimeError, match="fixed-point range"):
        st.sync()
    st.close()
