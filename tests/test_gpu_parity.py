"""GPU parity: the sm_100a step vs the reference, through the C ABI.

Each golden case (tests/golden, produced by running the real reference) is
replayed on the device with the reference's own injected random blocks.
Bars (north star, BASELINE.json): leaf indices, counts, proposals and
accept/reject decisions bit-exact; residual sums, leaf values, residuals and
sigma2 within 1e-5 relative (float32 quantities) — in practice the f64 sums
differ from the reference's point-order sums only in the last bits.
"""

import numpy as np
import pytest

from golden_io import STEP_CASES, load_case
from oracle.bart_oracle import OracleChain, propose as oracle_propose

pytestmark = pytest.mark.gpu

PROP_FIELDS = [("kind", "kind"), ("node", "node"), ("axis_p", "axis"), ("cut_p", "cut"), ("depth_p", "depth"),
               ("n_axes", "n_axes"), ("n_splits", "n_splits"), ("w_small", "w_small"),
               ("w_prime_big", "w_prime_big"), ("growable_big", "growable_big"),
               ("gl", "left_child_growable"), ("gr", "right_child_growable")]


def _hp(ns):
    from paper_2410_23244_b200.sampler import Hyperparams
    return Hyperparams(leaf_sd=ns.leaf_sd, lam=ns.lam, n_trees=ns.n_trees, alpha=ns.alpha, beta=ns.beta,
                       leaf_mean=ns.leaf_mean, nu=ns.nu, max_depth=ns.max_depth, p_grow=ns.p_grow,
                       update_sigma=ns.update_sigma)


def device_chain(d):
    from paper_2410_23244_b200.sampler import init_state
    from paper_2410_23244_b200.trees import Forest
    hp = _hp(d["hpns"])
    st = init_state(d["X"], d["max_cuts"], d["y"], hp, None, sigma2=float(d["sigma2_0"]))
    st.forest = Forest(d["axis0"].copy(), d["cutpoint0"].copy(), d["leaf_value0"].copy(), hp.max_depth)
    st.leaf_index = d["leaf_index0"].copy()
    st.resid = d["resid0"].copy()
    st.sigma2 = float(d["sigma2_0"])
    st.enable_taps(True)
    return st, hp


def randoms(d, s):
    from paper_2410_23244_b200.sampler import StepRandoms
    return StepRandoms(d["move_u"][s], d["accept_u"][s], d["leaf_z"][s], float(d["chi2"][s]))


@pytest.mark.parametrize("case", STEP_CASES)
def test_step_matches_reference_golden(case):
    from paper_2410_23244_b200.sampler import step
    d = load_case(case)
    st, hp = device_chain(d)
    for s in range(d["steps"]):
        step(st, hp, randoms=randoms(d, s))
        props = st.last_proposals
        for gk, ak in PROP_FIELDS:
            np.testing.assert_array_equal(getattr(props, ak), d[gk][s], err_msg=f"{case} step {s} proposal {gk}")
        np.testing.assert_allclose(props.struct_log, d["struct_log"][s], rtol=1e-13, atol=1e-14)
        counts, sums = st.taps()
        np.testing.assert_array_equal(counts, d["counts"][s], err_msg=f"{case} step {s} counts")
        scale = np.abs(d["sums"][s]).max() + 1e-30
        np.testing.assert_allclose(sums, d["sums"][s], rtol=1e-10, atol=1e-12 * scale, err_msg=f"{case} step {s} sums")
        np.testing.assert_array_equal(st.last_accepted, d["accepted"][s], err_msg=f"{case} step {s} accept")
        f = st.forest
        np.testing.assert_array_equal(f.axis, d["axis"][s])
        np.testing.assert_array_equal(f.cutpoint, d["cutpoint"][s])
        np.testing.assert_array_equal(st.leaf_index, d["leaf_index"][s], err_msg=f"{case} step {s} leaf_index")
        np.testing.assert_allclose(f.leaf_value, d["leaf_value"][s], rtol=1e-5, atol=1e-6)
        np.testing.assert_allclose(st.resid, d["resid"][s], rtol=1e-5, atol=1e-5)
        assert st.sigma2 == pytest.approx(float(d["sigma2"][s]), rel=1e-5)
    st.close()


@pytest.mark.parametrize("case", ["a8", "wide", "depth8"])
def test_golden_stream_mode(case, monkeypatch):
    """The stream-mode sweep (large n) against the reference's golden steps."""
    monkeypatch.setenv("BART_FORCE_STREAM", "1")
    test_step_matches_reference_golden(case)


@pytest.mark.parametrize("case", ["a8", "friedman", "wide", "depth8"])
def test_first_step_bitwise(case):
    """From an identical start, one step reproduces the reference bit for bit."""
    from paper_2410_23244_b200.sampler import step
    d = load_case(case)
    st, hp = device_chain(d)
    step(st, hp, randoms=randoms(d, 0))
    _, sums = st.taps()
    frac_sums = np.mean(sums == d["sums"][0])
    assert frac_sums > 0.9, f"sums bit-identical fraction {frac_sums}"
    np.testing.assert_array_equal(st.forest.leaf_value, d["leaf_value"][0])
    np.testing.assert_array_equal(st.resid, d["resid"][0])
    st.close()


def test_propose_matches_oracle_on_prior_forests():
    """Phase 1 alone on many prior-drawn forests, p=300 (uint16 axes) and D=8."""
    from paper_2410_23244_b200.sampler import Hyperparams, init_state, propose_moves, sample_prior_tree
    from paper_2410_23244_b200.trees import Forest
    rng = np.random.default_rng(5)
    for D, p, m, alpha, beta in ((6, 300, 64, 0.95, 1.0), (8, 4, 40, 0.99, 0.5), (3, 2, 200, 0.9, 1.0), (2, 3, 30, 0.9, 0.0)):
        hp = Hyperparams(leaf_sd=0.2, lam=0.1, n_trees=m, alpha=alpha, beta=beta, max_depth=D)
        max_cuts = rng.integers(0, 12, p)
        max_cuts[0] = 11
        ts = [sample_prior_tree(max_cuts, hp, rng) for _ in range(m)]
        forest = Forest(np.stack([t.axis for t in ts]), np.stack([t.cutpoint for t in ts]),
                        np.stack([t.leaf_value for t in ts]), D)
        X = rng.integers(0, 12, (50, p)).astype(np.uint8)
        st = init_state(X, max_cuts, rng.normal(size=50), hp, None, sigma2=1.0)
        st.forest = forest
        for _ in range(5):
            u = rng.random((m, 5))
            got = propose_moves(st, hp, uniforms=u)
            want = oracle_propose(forest.axis, forest.cutpoint, D, max_cuts, alpha, beta, hp.p_grow, u)
            for _, ak in PROP_FIELDS:
                ok = {"left_child_growable": "gl", "right_child_growable": "gr"}.get(ak, ak)
                np.testing.assert_array_equal(getattr(got, ak), getattr(want, ok), err_msg=f"D={D} {ak}")
            np.testing.assert_allclose(got.struct_log, want.struct_log, rtol=1e-13, atol=1e-14)
        st.close()


@pytest.mark.parametrize("case", STEP_CASES)
def test_forest_kernels_match_reference(case):
    """traverse_forest / sum_leaf_values / evaluate_forest vs reference outputs (trees.py:174-223)."""
    from paper_2410_23244_b200.trees import Forest, evaluate_forest, sum_leaf_values, traverse_forest
    d = load_case(case)
    D = d["hpns"].max_depth
    f = Forest(d["axis"][-1], d["cutpoint"][-1], d["leaf_value"][-1], D)
    L = traverse_forest(f, d["X"])
    np.testing.assert_array_equal(L, d["leaf_index"][-1])
    np.testing.assert_array_equal(sum_leaf_values(f.leaf_value, L), d["yhat"])
    np.testing.assert_array_equal(evaluate_forest(f, d["X"]), d["yhat"])


@pytest.mark.parametrize("n,F", [(301, 37), (70001, 9)])
def test_evaluate_forests_batches_match_single(n, F):
    """Stacked forests evaluated a batch per launch (grid y = forest) equal one
    evaluate_forest per forest, bit for bit, across batch boundaries; and the
    tree-group traversal equals the cached sum (trees.py:206-223)."""
    from paper_2410_23244_b200.sampler import Hyperparams, init_state, run, DeviceRNG
    from paper_2410_23244_b200.trees import evaluate_forest, evaluate_forests, sum_leaf_values, traverse_forest
    rng = np.random.default_rng(n)
    p = 7
    X = rng.integers(0, 30, (n, p)).astype(np.uint8)
    y = rng.normal(size=n).astype(np.float32)
    hp = Hyperparams(leaf_sd=0.3, lam=0.1, n_trees=13, max_depth=6)
    st = init_state(X, np.full(p, 29), y, hp, DeviceRNG(5))
    forests = []
    for _ in range(F):
        run(st, hp, 3)
        forests.append(st.forest)
    st.close()
    got = evaluate_forests(forests, X)
    for k in (0, F // 2, F - 1):
        np.testing.assert_array_equal(got[k], evaluate_forest(forests[k], X))
        L = traverse_forest(forests[k], X)
        np.testing.assert_array_equal(sum_leaf_values(forests[k].leaf_value, L), got[k])


@pytest.fixture(params=["register", "stream"])
def sweep_mode(request, monkeypatch):
    """Run a test in both sweep modes: register-resident points (the default at
    these sizes) and the stream mode large n uses, forced at small n."""
    if request.param == "stream":
        monkeypatch.setenv("BART_FORCE_STREAM", "1")
    return request.param


@pytest.mark.parametrize("max_ctas", [None, 5])
def test_chain_matches_oracle_friedman_multi_cta(sweep_mode, max_ctas):
    """n=20000 spans many CTAs: 12 steps vs the oracle with the same injected randoms
    (max_ctas: the chain squeezed onto 5 SMs, as multi-chain batching does)."""
    from paper_2410_23244_b200.dgp import friedman1
    from paper_2410_23244_b200.grid import build_grid_uniform, quantize
    from paper_2410_23244_b200.regression import FitConfig, derive_hyperparams
    from paper_2410_23244_b200.sampler import StepRandoms, init_state, step
    X, y, _ = friedman1(20003, 10, seed=3)
    g = build_grid_uniform(X, 100)
    Xq = quantize(X, g).data
    hp, ys = derive_hyperparams(y, FitConfig(n_trees=40))
    y32 = ys.forward(y).astype(np.float32)
    st = init_state(Xq, g.counts, y32, hp, None, max_ctas=max_ctas)
    assert st.sweep_config()["ctas"] == (5 if max_ctas else 20)
    assert st.sweep_config()["stream"] == (sweep_mode == "stream")
    st.enable_taps(True)
    ora = OracleChain(Xq, g.counts, y32, hp)
    rng = np.random.default_rng(0)
    for s in range(12):
        rnd = StepRandoms.draw(rng, hp.n_trees, 1 << hp.max_depth, hp.nu + y.size)
        taps = {}
        ora.step(rnd.move_u, rnd.accept_u, rnd.leaf_z, rnd.chi2_value, taps)
        step(st, hp, randoms=rnd)
        counts, sums = st.taps()
        np.testing.assert_array_equal(counts, taps["counts"])
        np.testing.assert_allclose(sums, taps["sums"], rtol=1e-9, atol=1e-9)
        np.testing.assert_array_equal(st.last_accepted, ora.last_accepted, err_msg=f"step {s}")
        np.testing.assert_array_equal(st.forest.cutpoint, ora.cut)
        np.testing.assert_array_equal(st.leaf_index, ora.leaf_index)
        np.testing.assert_allclose(st.forest.leaf_value, ora.leaf, rtol=1e-5, atol=1e-6)
        np.testing.assert_allclose(st.resid, ora.resid, rtol=1e-5, atol=1e-5)
        assert st.sigma2 == pytest.approx(ora.sigma2, rel=1e-5)
    st.close()


@pytest.mark.parametrize("n", [1, 7, 16, 17, 1025, 4099])
def test_ragged_sizes(n, sweep_mode):
    """Chunk edges: n not a multiple of 16, a single point, several CTAs."""
    from paper_2410_23244_b200.sampler import Hyperparams, StepRandoms, init_state, step
    rng = np.random.default_rng(n)
    p, m = 3, 6
    X = rng.integers(0, 9, (n, p)).astype(np.uint8)
    y = rng.normal(size=n).astype(np.float32)
    hp = Hyperparams(leaf_sd=0.3, lam=0.1, n_trees=m, max_depth=4)
    st = init_state(X, np.full(p, 8), y, hp, None, sigma2=1.0)
    ora = OracleChain(X, np.full(p, 8), y, hp, sigma2=1.0)
    for _ in range(10):
        rnd = StepRandoms.draw(rng, m, 16, hp.nu + n)
        step(st, hp, randoms=rnd)
        ora.step(rnd.move_u, rnd.accept_u, rnd.leaf_z, rnd.chi2_value)
        np.testing.assert_array_equal(st.last_accepted, ora.last_accepted)
        np.testing.assert_array_equal(st.leaf_index, ora.leaf_index)
        np.testing.assert_allclose(st.resid, ora.resid, rtol=1e-5, atol=1e-5)
    st.close()


def test_stream_mode_large_n_invariants():
    """n = 3e6 exceeds the register budget (stream mode by default): after a
    few device-RNG steps the cache equals a fresh traversal of the forest and
    the residuals equal y minus the forest's prediction (sampler.py:125-130)."""
    from paper_2410_23244_b200.dgp import friedman1_binned
    from paper_2410_23244_b200.regression import FitConfig, derive_hyperparams
    from paper_2410_23244_b200.sampler import DeviceRNG, init_state, run
    from paper_2410_23244_b200.trees import evaluate_forest, traverse_forest
    n = 3_000_000
    Xq, y, _, grid = friedman1_binned(n, 10, seed=4)
    hp, ys = derive_hyperparams(y, FitConfig(n_trees=50))
    y32 = ys.forward(y).astype(np.float32)
    st = init_state(Xq, grid.counts, y32, hp, DeviceRNG(9))
    assert st.sweep_config()["stream"]
    run(st, hp, 6)
    f = st.forest
    sub = np.random.default_rng(0).choice(n, 20000, replace=False)
    np.testing.assert_array_equal(st.leaf_index[sub], traverse_forest(f, Xq[sub]))
    pred = evaluate_forest(f, Xq[sub])
    np.testing.assert_allclose(st.resid[sub], (y32[sub] - pred).astype(np.float32), atol=1e-4)
    assert 0 < st.sigma2 < 10
    assert (f.cutpoint > 0).sum() > 0
    st.close()


@pytest.mark.parametrize("mode", ["flat", "two_level"])
@pytest.mark.parametrize("groups", [2, 3, 8])
def test_sharded_exchange_emulated(groups, mode):
    """n-sharding's exchange protocol (every shard adds into every shard's
    words, each polls its own copy), emulated by splitting one
    launch's CTAs into `groups` copy groups: decisions, counts and indices stay
    bit-exact against the oracle."""
    from paper_2410_23244_b200.dgp import friedman1
    from paper_2410_23244_b200.grid import build_grid_uniform, quantize
    from paper_2410_23244_b200.regression import FitConfig, derive_hyperparams
    from paper_2410_23244_b200.sampler import StepRandoms, init_state, step
    X, y, _ = friedman1(30011, 8, seed=11)
    g = build_grid_uniform(X, 100)
    Xq = quantize(X, g).data
    hp, ys = derive_hyperparams(y, FitConfig(n_trees=30))
    y32 = ys.forward(y).astype(np.float32)
    st = init_state(Xq, g.counts, y32, hp, None)
    st.set_copy_groups(groups)
    st.set_exchange(mode)
    st.enable_taps(True)
    ora = OracleChain(Xq, g.counts, y32, hp)
    rng = np.random.default_rng(groups)
    for s in range(6):
        rnd = StepRandoms.draw(rng, hp.n_trees, 1 << hp.max_depth, hp.nu + y.size)
        taps = {}
        ora.step(rnd.move_u, rnd.accept_u, rnd.leaf_z, rnd.chi2_value, taps)
        step(st, hp, randoms=rnd)
        counts, sums = st.taps()
        np.testing.assert_array_equal(counts, taps["counts"])
        np.testing.assert_allclose(sums, taps["sums"], rtol=1e-9, atol=1e-9)
        np.testing.assert_array_equal(st.last_accepted, ora.last_accepted, err_msg=f"step {s}")
        np.testing.assert_array_equal(st.leaf_index, ora.leaf_index)
        np.testing.assert_allclose(st.resid, ora.resid, rtol=1e-5, atol=1e-5)
        assert st.sigma2 == pytest.approx(ora.sigma2, rel=1e-5)
    st.close()


def test_unconnected_shard_refuses_to_step():
    from paper_2410_23244_b200.sampler import DeviceRNG, Hyperparams, SamplerState, step
    rng = np.random.default_rng(0)
    X = rng.integers(0, 9, (500, 3)).astype(np.uint8)
    y = rng.normal(size=500).astype(np.float32)
    hp = Hyperparams(leaf_sd=0.3, lam=0.1, n_trees=4, max_depth=4)
    st = SamplerState(X, np.full(3, 8), y, hp, DeviceRNG(1), 1.0, 0, shard=(1000, 0, 2))
    assert len(st.shard_export()) == 256
    with pytest.raises(RuntimeError, match="not connected"):
        step(st, hp)
    with pytest.raises(ValueError):
        st.shard_connect([st.shard_export()])  # one handle for two shards
    st.close()


def test_pipelined_step_results_match_synchronous_reads():
    """state.step_result(k), read after step k+1 was launched (the e2e loop),
    equals what a synchronous read right after step k returns."""
    from paper_2410_23244_b200.sampler import Hyperparams, StepRandoms, init_state, step
    rng = np.random.default_rng(11)
    n, p, m = 2500, 5, 9
    X = rng.integers(0, 12, (n, p)).astype(np.uint8)
    y = rng.normal(size=n).astype(np.float32)
    hp = Hyperparams(leaf_sd=0.3, lam=0.1, n_trees=m, max_depth=5)
    blocks = [StepRandoms.draw(rng, m, 32, hp.nu + n) for _ in range(8)]
    a = init_state(X, np.full(p, 11), y, hp, None, sigma2=1.0)
    want = []
    for rnd in blocks:
        step(a, hp, randoms=rnd)
        want.append((a.last_accepted.copy(), a.sigma2))
    b = init_state(X, np.full(p, 11), y, hp, None, sigma2=1.0)
    got = []
    for k, rnd in enumerate(blocks):
        step(b, hp, randoms=rnd)
        if k > 0:
            got.append(b.step_result(b.iteration - 2))
    got.append(b.step_result())
    for (wa, ws), (ga, gs) in zip(want, got):
        np.testing.assert_array_equal(wa, ga)
        assert ws == gs
    with pytest.raises(ValueError):
        b.step_result(0)  # only the last two steps are kept
    a.close()
    b.close()


@pytest.mark.parametrize("groups", [1, 2, 8])
def test_two_level_exchange_bit_identical_to_flat(groups, sweep_mode):
    """The two-level exchange (per-shard stage words + one forwarder per shard)
    sums the same integers as the flat one: a device-RNG chain takes the same
    decisions and ends in the same state, bit for bit, in both modes."""
    from paper_2410_23244_b200.dgp import friedman1_binned
    from paper_2410_23244_b200.regression import FitConfig, derive_hyperparams
    from paper_2410_23244_b200.sampler import DeviceRNG, init_state, run
    Xq, y, _, grid = friedman1_binned(60_013, 12, seed=5)
    hp, ys = derive_hyperparams(y, FitConfig(n_trees=40))
    y32 = ys.forward(y).astype(np.float32)
    out = []
    for mode in ("flat", "two_level"):
        st = init_state(Xq, grid.counts, y32, hp, DeviceRNG(77))
        if groups > 1:
            st.set_copy_groups(groups)
        st.set_exchange(mode)
        run(st, hp, 3)
        st.set_exchange("flat" if mode == "two_level" else "two_level")  # switching between launches
        run(st, hp, 3)
        f = st.forest
        out.append((f.axis.copy(), f.cutpoint.copy(), f.leaf_value.copy(), st.resid.copy(), st.sigma2))
        st.close()
    for a, b in zip(out[0], out[1]):
        assert np.array_equal(a, b)
