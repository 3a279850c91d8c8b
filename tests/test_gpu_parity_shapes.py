"""GPU parity at the benchmarked shapes (BASELINE.json configs[1-4]).

The golden and seeded-chain parity tests (test_gpu_parity.py) run at n <= 3e4,
which selects the sweep's W=1 register layout on <= 30 CTAs.  These tests run
the shapes bench.py measures: the step kernel's W=2, W=4 (the n=1e6 headline
at 148 CTAs) and W=8 instantiations (sweep.cu sweep_words_per_thread), the
p=1000 / m=1000 width of configs[4] (uint16 axes, 1000-tree exchange), and
the 8-group exchange of an n-sharded chain at the n=1.25e6-per-shard shape of
configs[3] on 8 GPUs.

Protocol: the device chain burns in with its own Philox stream (so trees are
at posterior size, not the 1-2-leaf trees of a fresh chain); its state is
copied into the CPU oracle; then both take the same injected StepRandoms
(sampler.py:244-260) for a few steps.  Bars (north star): counts, leaf
indices, forests and accept decisions bit-exact; sums <= 1e-9 relative; leaf
values, residuals and sigma2 <= 1e-5 relative.  Reference contract:
sampler.py:878-912; test_acceptance.py:269-295 (the step-by-step naive
equivalence these mirror).
"""

import numpy as np
import pytest

from oracle.bart_oracle import OracleChain

pytestmark = pytest.mark.gpu


def _burned_pair(n, p, m, burn, seed, groups=1, exchange="flat", **fit_kw):
    from paper_2410_23244_b200.dgp import friedman1_binned
    from paper_2410_23244_b200.regression import FitConfig, derive_hyperparams
    from paper_2410_23244_b200.sampler import DeviceRNG, init_state, run
    Xq, y, _, grid = friedman1_binned(n, p, seed=seed)
    hp, ys = derive_hyperparams(y, FitConfig(n_trees=m, **fit_kw))
    y32 = ys.forward(y).astype(np.float32)
    st = init_state(Xq, grid.counts, y32, hp, DeviceRNG(seed + 100))
    if groups > 1:
        st.set_copy_groups(groups)
    st.set_exchange(exchange)
    run(st, hp, burn)
    f = st.forest
    ora = OracleChain(Xq, grid.counts, y32, hp, sigma2=st.sigma2, axis=f.axis, cut=f.cutpoint, leaf=f.leaf_value,
                      resid=st.resid, leaf_index=st.leaf_index)
    st.enable_taps(True)
    return st, ora, hp, n


def _compare_steps(st, ora, hp, n, steps, seed):
    from paper_2410_23244_b200.sampler import StepRandoms, step
    rng = np.random.default_rng(seed)
    size = 1 << hp.max_depth
    for s in range(steps):
        rnd = StepRandoms.draw(rng, hp.n_trees, size, hp.nu + n)
        taps = {}
        ora.step(rnd.move_u, rnd.accept_u, rnd.leaf_z, rnd.chi2_value, taps)
        step(st, hp, randoms=rnd)
        counts, sums = st.taps()
        np.testing.assert_array_equal(counts, taps["counts"], err_msg=f"step {s} counts")
        scale = np.abs(taps["sums"]).max() + 1e-30
        np.testing.assert_allclose(sums, taps["sums"], rtol=1e-9, atol=1e-12 * scale, err_msg=f"step {s} sums")
        np.testing.assert_array_equal(st.last_accepted, ora.last_accepted, err_msg=f"step {s} accept")
        f = st.forest
        np.testing.assert_array_equal(f.axis, ora.axis, err_msg=f"step {s} axis")
        np.testing.assert_array_equal(f.cutpoint, ora.cut, err_msg=f"step {s} cutpoint")
        np.testing.assert_allclose(f.leaf_value, ora.leaf, rtol=1e-5, atol=1e-6, err_msg=f"step {s} leaves")
        assert np.array_equal(st.leaf_index, ora.leaf_index), f"step {s} leaf_index"
        np.testing.assert_allclose(st.resid, ora.resid, rtol=1e-5, atol=1e-5, err_msg=f"step {s} resid")
        assert st.sigma2 == pytest.approx(ora.sigma2, rel=1e-5)
    return st.last_accepted


# (n, p, m, expected words per worker thread W, CTAs, burn-in, steps)
SHAPES = {
    "w2_n4e5": (400_000, 100, 200, 2, 148, 50, 3),
    "w4_headline_1e6": (1_000_000, 100, 200, 4, 148, 50, 3),
    "w8_n1p5e6": (1_500_000, 100, 200, 8, 148, 30, 3),
    "wide_p1000_m1000": (200_000, 1000, 1000, 1, 148, 20, 2),
}


def _words(chunk):
    """sweep_words_per_thread (csrc/sweep.cu): words per worker thread, 14 worker warps."""
    words = (chunk + 3) // 4
    for w in (1, 2, 4, 8):
        if w * 14 * 32 >= words:
            return w
    return 0


@pytest.mark.parametrize("shape", list(SHAPES))
def test_benchmark_shape_matches_oracle(shape):
    n, p, m, W, ctas, burn, steps = SHAPES[shape]
    st, ora, hp, n = _burned_pair(n, p, m, burn, seed=len(shape))
    cfg = st.sweep_config()
    assert cfg["ctas"] == ctas and not cfg["stream"]
    assert _words(cfg["chunk"]) == W, cfg
    leaves = (st.forest.cutpoint > 0).sum(axis=1) + 1
    assert leaves.mean() > 1.2, "burn-in should have grown the trees"
    _compare_steps(st, ora, hp, n, steps, seed=7)
    st.close()


@pytest.mark.parametrize("exchange", ["flat", "two_level"])
def test_eight_copy_groups_at_shard_shape(exchange):
    """One GPU standing in for an 8-way n-sharded chain of configs[3] (n=1e7
    over 8 GPUs = 1.25e6 points per shard): 148 CTAs in 8 copy groups, each
    polling its own exchange copy -- every CTA adding into all 8 copies (flat),
    or each group's forwarder adding its group's total (two_level; DESIGN.md
    §6) -- the W=8 instantiation with the sharded exchange."""
    st, ora, hp, n = _burned_pair(1_250_000, 100, 200, 30, seed=3, groups=8, exchange=exchange)
    cfg = st.sweep_config()
    assert cfg["ctas"] == 148 and _words(cfg["chunk"]) == 8
    _compare_steps(st, ora, hp, n, 3, seed=8)
    st.close()


def test_stream_mode_at_stream_size_matches_oracle():
    """n = 2.5e6 exceeds the register budget (2.1M points per GPU), so the
    sweep runs in stream mode by itself -- residuals in L2, refreshed rows in
    the Lref ring -- the mode n=1e7 on 1-4 GPUs uses."""
    st, ora, hp, n = _burned_pair(2_500_000, 20, 60, 30, seed=12)
    assert st.sweep_config()["stream"] and st.sweep_config()["ctas"] == 148
    _compare_steps(st, ora, hp, n, 2, seed=9)
    st.close()


def test_deep_wide_trees_match_oracle():
    """D = 8 (256-slot leaf rows) with a prior that grows deep, bushy trees:
    after burn-in some trees' larger trees have more than 8 leaves (the A
    pass's multi-pass sums) and the decision's wide path; 148 CTAs."""
    st, ora, hp, n = _burned_pair(600_000, 10, 40, 150, seed=21, max_depth=8, alpha=0.99, beta=0.3)
    leaves = (st.forest.cutpoint > 0).sum(axis=1) + 1
    assert leaves.max() > 8, leaves.max()
    _compare_steps(st, ora, hp, n, 3, seed=10)
    st.close()
