"""Posterior agreement with the reference algorithm on independent random
streams (the statistical check of the north star): device chains (Philox
streams) and oracle chains (numpy streams; oracle/bart_oracle.py restates
bforge.sampler.step) run long enough to forget their streams.  BART chains
mix slowly, so the yardstick is the spread between independent chains of the
same sampler: a device chain must sit as close to an oracle chain as two
device (or two oracle) chains sit to each other, and all must track the true
function."""

import numpy as np
import pytest

from oracle.bart_oracle import OracleChain, sum_leaf_values

pytestmark = pytest.mark.gpu

BURN, KEPT = 400, 800


def _data():
    from paper_2410_23244_b200.dgp import friedman1
    from paper_2410_23244_b200.grid import build_grid_uniform, quantize
    from paper_2410_23244_b200.regression import FitConfig, derive_hyperparams
    X, y, f = friedman1(250, 5, seed=8, noise_sd=0.5)
    g = build_grid_uniform(X, 30)
    Xq = quantize(X, g).data
    hp, ys = derive_hyperparams(y, FitConfig(n_trees=20, max_depth=5))
    return Xq, g.counts, ys.forward(y).astype(np.float32), hp, ys.forward(f)


def _device_mean(Xq, counts, y32, hp, seed):
    from paper_2410_23244_b200.sampler import DeviceRNG, init_state, run
    st = init_state(Xq, counts, y32, hp, DeviceRNG(seed))
    run(st, hp, BURN)
    acc = np.zeros(y32.size)
    for _ in range(KEPT):
        run(st, hp, 1)
        acc += sum_leaf_values(st.forest.leaf_value, np.ascontiguousarray(st.leaf_index.T))
    st.close()
    return acc / KEPT


def _oracle_mean(Xq, counts, y32, hp, seed):
    from paper_2410_23244_b200.sampler import StepRandoms
    ora = OracleChain(Xq, counts, y32, hp)
    rng = np.random.default_rng(seed)
    acc = np.zeros(y32.size)
    for it in range(BURN + KEPT):
        rnd = StepRandoms.draw(rng, hp.n_trees, 1 << hp.max_depth, hp.nu + y32.size)
        ora.step(rnd.move_u, rnd.accept_u, rnd.leaf_z, rnd.chi2_value)
        if it >= BURN:
            acc += sum_leaf_values(ora.leaf, ora.Lt)
    return acc / KEPT


def test_posterior_means_agree_with_oracle_chains():
    Xq, counts, y32, hp, truth = _data()
    d1, d2 = (_device_mean(Xq, counts, y32, hp, s) for s in (21, 22))
    o1, o2 = (_oracle_mean(Xq, counts, y32, hp, s) for s in (99, 100))
    rms = lambda a, b: float(np.sqrt(np.mean((a - b) ** 2)))
    within = max(rms(d1, d2), rms(o1, o2))          # same sampler, independent streams
    across = np.mean([rms(d, o) for d in (d1, d2) for o in (o1, o2)])  # device vs oracle
    print(f"posterior means: device-vs-oracle rms {across:.4f}, within-sampler rms {within:.4f}, "
          f"sd(truth) {np.std(truth):.4f}")
    assert across < 1.5 * within, f"device-vs-oracle spread {across:.4f} vs within-sampler {within:.4f}"
    pooled_d, pooled_o = (d1 + d2) / 2, (o1 + o2) / 2
    assert np.corrcoef(pooled_d, pooled_o)[0, 1] > 0.98
    for mu in (pooled_d, pooled_o):
        assert rms(mu, truth) < 0.35 * np.std(truth)
