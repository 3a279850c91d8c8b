"""Generate golden step vectors by running the REAL reference (`bforge`) here.

Test infrastructure only.  Run in the build container, where the reference is
mounted read-only at /root/reference:

    python tests/golden/make_golden.py

It imports `bforge` from /root/reference/pkg/src (numba cache redirected to a
temp dir so nothing is written into the reference tree), runs a set of chains
chosen to cover the hot-path edge cases the reference's own tests exercise
(SURVEY.md §4 / §8c), and records per step:

* the state before the step (forest, leaf_index (n,m), resid, sigma2),
* the exact `StepRandoms` the step consumed (captured by replaying a deepcopy
  of the chain's Generator, which is the only RNG use inside `step`,
  sampler.py:891),
* phase taps: the proposals (sampler.py:469-526), the per-tree counts after
  the grow refresh (sampler.py:894-897), and the tree-excluded residual sums
  each `_resolve_tree` computed (sampler.py:828, recorded before the collapse
  at :861-866 mutates them),
* the state after the step and `last_accepted`.

Fixtures land in tests/golden/*.npz; the GPU box never needs /root/reference.
"""

from __future__ import annotations

import copy
import os
import sys
import tempfile
from pathlib import Path

import numpy as np

REF_SRC = "/root/reference/pkg/src"
OUT = Path(__file__).resolve().parent

os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="numba_golden_"))
sys.dont_write_bytecode = True
sys.path.insert(0, REF_SRC)

from bforge import sampler, trees  # noqa: E402
from bforge.grid import build_grid_uniform, quantize  # noqa: E402
from bforge.regression import FitConfig, derive_hyperparams, fit  # noqa: E402


def _friedman(n, p, seed):
    rng = np.random.default_rng(seed)
    X = rng.uniform(0.0, 1.0, size=(n, p))
    f = 10 * np.sin(np.pi * X[:, 0] * X[:, 1]) + 20 * (X[:, 2] - 0.5) ** 2 + 10 * X[:, 3] + 5 * X[:, 4]
    y = f + rng.normal(0.0, 1.0, size=n)
    return X, y


class _SumsTap:
    """Wraps sampler.sum_residuals_per_leaf to record each tree's sums."""

    def __init__(self):
        self.rows = []
        self._orig = sampler.sum_residuals_per_leaf

    def __enter__(self):
        orig = self._orig

        def wrapped(*a, **k):
            out = orig(*a, **k)
            self.rows.append(out.copy())
            return out

        sampler.sum_residuals_per_leaf = wrapped
        return self

    def __exit__(self, *exc):
        sampler.sum_residuals_per_leaf = self._orig


def record(name, X, max_cuts, y, hp, rng, steps, burn=0, sigma2=None, forest=None):
    X = np.asarray(X, np.uint8)
    state = sampler.init_state(X, max_cuts, y, hp, rng, sigma2=sigma2)
    if forest is not None:
        state.forest = forest
        state.leaf_index = trees.traverse_forest(forest, state.X)
        state.rebuild_structure_caches()
        pred = np.zeros(state.n_points)
        for j in range(forest.n_trees):
            pred += forest.leaf_value[j, state.leaf_index[:, j]]
        state.resid = (state.y.astype(np.float64) - pred).astype(np.float32)
    for _ in range(burn):
        sampler.step(state, hp)

    m = hp.n_trees
    size = trees.heap_size(hp.max_depth)
    n = X.shape[0]
    rec = {k: [] for k in (
        "move_u", "accept_u", "leaf_z", "chi2",
        "kind", "node", "axis_p", "cut_p", "depth_p", "n_axes", "n_splits", "w_small",
        "w_prime_big", "growable_big", "gl", "gr", "struct_log",
        "counts", "sums",
        "axis", "cutpoint", "leaf_value", "resid", "leaf_index", "sigma2", "accepted",
    )}
    init = dict(
        axis0=state.forest.axis.copy(), cutpoint0=state.forest.cutpoint.copy(),
        leaf_value0=state.forest.leaf_value.copy(), resid0=state.resid.copy(),
        leaf_index0=state.leaf_index.copy(), sigma2_0=np.float64(state.sigma2),
    )
    for _ in range(steps):
        rnd = sampler.StepRandoms.draw(copy.deepcopy(state.rng), m, size, hp.nu + n)
        probe = copy.deepcopy(state)
        props = sampler.propose_moves(probe, hp, uniforms=rnd.move_u)
        sampler.refresh_leaf_indices(probe, props)
        counts = np.stack([sampler.count_points_per_leaf(probe.leaf_index[:, j], size) for j in range(m)])
        with _SumsTap() as tap:
            sampler.step(state, hp)
        assert len(tap.rows) == m
        rec["move_u"].append(rnd.move_u)
        rec["accept_u"].append(rnd.accept_u)
        rec["leaf_z"].append(rnd.leaf_z)
        rec["chi2"].append(rnd.chi2_value)
        rec["kind"].append(props.kind)
        rec["node"].append(props.node)
        rec["axis_p"].append(props.axis)
        rec["cut_p"].append(props.cut)
        rec["depth_p"].append(props.depth)
        rec["n_axes"].append(props.n_axes)
        rec["n_splits"].append(props.n_splits)
        rec["w_small"].append(props.w_small)
        rec["w_prime_big"].append(props.w_prime_big)
        rec["growable_big"].append(props.growable_big)
        rec["gl"].append(props.left_child_growable)
        rec["gr"].append(props.right_child_growable)
        rec["struct_log"].append(props.struct_log)
        rec["counts"].append(counts)
        rec["sums"].append(np.stack(tap.rows))
        rec["axis"].append(state.forest.axis.copy())
        rec["cutpoint"].append(state.forest.cutpoint.copy())
        rec["leaf_value"].append(state.forest.leaf_value.copy())
        rec["resid"].append(state.resid.copy())
        rec["leaf_index"].append(state.leaf_index.copy())
        rec["sigma2"].append(state.sigma2)
        rec["accepted"].append(state.last_accepted.copy())
        # per-step invariant the reference guarantees (sampler.py:125-130)
        assert np.array_equal(state.leaf_index, trees.traverse_forest(state.forest, state.X))

    out = {k: np.asarray(v) for k, v in rec.items()}
    out.update(init)
    out.update(
        X=X, max_cuts=np.asarray(max_cuts, np.int64), y=np.asarray(y, np.float32),
        hp=np.array([hp.leaf_sd, hp.lam, hp.alpha, hp.beta, hp.leaf_mean, hp.nu, hp.p_grow], np.float64),
        hp_int=np.array([hp.n_trees, hp.max_depth, int(hp.update_sigma)], np.int64),
        yhat=trees.sum_leaf_values(state.forest.leaf_value, state.leaf_index),
    )
    np.savez_compressed(OUT / f"step_{name}.npz", **out)
    n_acc = int(out["accepted"].sum())
    kinds = np.bincount(out["kind"].ravel().astype(np.int64), minlength=3)
    print(f"{name}: n={n} p={X.shape[1]} m={m} D={hp.max_depth} steps={steps} "
          f"accepted={n_acc} kinds(none,grow,prune)={kinds.tolist()}")


def H(**kw):
    base = dict(leaf_sd=0.3, lam=0.1, n_trees=1, alpha=0.95, beta=2.0, nu=3.0, max_depth=3)
    base.update(kw)
    return sampler.Hyperparams(**base)


def main():
    # A8 shape (test_acceptance.py:269-295)
    r = np.random.default_rng(808)
    X = r.integers(0, 12, (100, 3)).astype(np.uint8)
    y = r.normal(0, 1, 100).astype(np.float32)
    hp = sampler.Hyperparams(leaf_sd=0.15, lam=0.2, n_trees=10, max_depth=4, nu=3.0)
    record("a8", X, np.full(3, 11), y, hp, np.random.default_rng(909), steps=40,
           sigma2=float(np.var(y, ddof=1)))

    # naive-equivalence short (test_sampler.py:485-503)
    r = np.random.default_rng(33)
    X = r.integers(0, 6, (30, 2)).astype(np.uint8)
    y = r.normal(0, 1, 30).astype(np.float32)
    record("short", X, np.array([5, 5]), y, H(n_trees=3, max_depth=4, leaf_sd=0.2, lam=0.1),
           np.random.default_rng(7), steps=30, sigma2=float(np.var(y, ddof=1)))

    # Friedman #1, BASELINE configs[0] shape (n=1e3, p=10, m=50), default D=6 after burn-in
    Xr, yr = _friedman(1000, 10, 0)
    grid = build_grid_uniform(Xr, 100)
    Xq = quantize(Xr, grid).data
    cfg = FitConfig(n_trees=50, n_chains=1)
    hp, ys = derive_hyperparams(yr, cfg)
    record("friedman", Xq, grid.counts, ys.forward(yr).astype(np.float32), hp,
           np.random.Generator(np.random.Philox(np.random.SeedSequence(0))), steps=8, burn=30)

    # depth 8 (test_sampler.py:611-620): uint8 leaf index at its limit
    r = np.random.default_rng(52)
    X = r.integers(0, 200, (150, 2)).astype(np.uint8)
    y = r.normal(0, 1, 150).astype(np.float32)
    record("depth8", X, np.array([199, 199]), y,
           H(n_trees=3, max_depth=8, leaf_sd=0.1, alpha=0.99, beta=0.5), r, steps=30, burn=30)

    # wide X: p=300 -> uint16 axis path (trees.py:53-55)
    r = np.random.default_rng(5)
    X = r.integers(0, 20, (400, 300)).astype(np.uint8)
    y = (0.5 * (X[:, 7] > 9) - 0.3 * (X[:, 250] > 4) + r.normal(0, 0.2, 400)).astype(np.float32)
    record("wide", X, np.full(300, 19), y, H(n_trees=8, max_depth=5, leaf_sd=0.1, lam=0.05),
           r, steps=12, burn=10)

    # depth edges (test_sampler.py:581-609)
    r = np.random.default_rng(51)
    X = r.integers(0, 6, (20, 1)).astype(np.uint8)
    y = r.normal(0, 1, 20).astype(np.float32)
    record("depth1", X, np.array([5]), y, H(n_trees=3, max_depth=1, leaf_sd=0.2), r, steps=5)
    r = np.random.default_rng(50)
    X = r.integers(0, 6, (60, 2)).astype(np.uint8)
    y = r.normal(0, 1, 60).astype(np.float32)
    record("depth2", X, np.array([5, 5]), y, H(n_trees=5, max_depth=2, leaf_sd=0.2), r, steps=20)

    # degenerate grid -> null proposals (test_sampler.py:179-188)
    X = np.zeros((4, 1), np.uint8)
    y = np.arange(4, dtype=np.float32)
    record("degenerate", X, np.array([0]), y, H(), np.random.default_rng(0), steps=3, sigma2=1.0)

    # flat response: exact-zero residual sums (test_sampler.py:426-437)
    r = np.random.default_rng(0)
    X = r.integers(0, 9, (100, 2)).astype(np.uint8)
    y = np.zeros(100, np.float32)
    record("flat", X, np.array([8, 8]), y, H(n_trees=10, max_depth=4, leaf_sd=0.05, lam=0.01),
           r, steps=20, sigma2=0.01)

    # fixed sigma (update_sigma=False) with hand-built multi-level forest
    r = np.random.default_rng(14)
    hp = H(n_trees=4, max_depth=4, leaf_sd=0.5, update_sigma=False)
    mc = np.array([6, 6])
    ts = [sampler.sample_prior_tree(mc, hp, r) for _ in range(4)]
    forest = trees.Forest(np.stack([t.axis for t in ts]), np.stack([t.cutpoint for t in ts]),
                          np.stack([t.leaf_value for t in ts]), 4)
    X = r.integers(0, 7, (60, 2)).astype(np.uint8)
    y = r.normal(0, 1, 60).astype(np.float32)
    record("prior_forest", X, mc, y, hp, r, steps=15, sigma2=1.0, forest=forest)

    # A6 shape (easy DGP n=500, p=5, m=200, D=6), after burn-in
    rng = np.random.default_rng(606)
    Xe = rng.uniform(-2.0, 2.0, size=(500, 5))
    ye = np.cos(np.pi * Xe).sum(axis=1) / np.sqrt(5) + rng.normal(0, 0.1, 500)
    g = build_grid_uniform(Xe, 100)
    hp, ys = derive_hyperparams(ye, FitConfig(n_trees=200, n_chains=1))
    record("easy200", quantize(Xe, g).data, g.counts, ys.forward(ye).astype(np.float32), hp,
           np.random.default_rng(606), steps=3, burn=60)

    # grid + quantize golden (grid.py:77-134)
    r = np.random.default_rng(11)
    Xg = r.normal(size=(257, 6))
    Xg[:, 3] = 1.5  # degenerate axis
    Xg[:5, 4] = np.nan_to_num(Xg[:5, 4])
    Xg_new = r.normal(scale=2.0, size=(50, 6))
    gu = build_grid_uniform(Xg, 40)
    from bforge.grid import build_grid_midpoints
    Xm = np.round(r.normal(size=(400, 3)) * 100)  # many distinct values -> thinning
    gm = build_grid_midpoints(Xm)
    np.savez_compressed(
        OUT / "grid.npz", X=Xg, X_new=Xg_new,
        uniform_counts=gu.counts, uniform_cuts=np.concatenate(gu.cutpoints),
        q_train=quantize(Xg, gu).data, q_new=quantize(Xg_new, gu).data,
        Xm=Xm, mid_counts=gm.counts, mid_cuts=np.concatenate(gm.cutpoints),
        qm=quantize(Xm, gm).data,
    )

    # whole-API golden: fit() with host Philox streams (regression.py:145-216)
    Xf, yf = _friedman(300, 6, 3)
    Xt, _ = _friedman(40, 6, 4)
    cfg = FitConfig(n_trees=20, n_burn=15, n_kept=10, n_chains=2, seed=5)
    tr = fit(Xf, yf, cfg, X_test=Xt)
    np.savez_compressed(
        OUT / "fit.npz", X=Xf, y=yf, X_test=Xt,
        cfg=np.array([cfg.n_trees, cfg.n_burn, cfg.n_kept, cfg.n_chains, cfg.seed], np.int64),
        sigma=tr.sigma, yhat_train=tr.yhat_train, yhat_test=tr.yhat_test,
        accepted=tr.accepted, mean_leaves=tr.mean_leaves,
    )
    print("grid.npz, fit.npz written")


if __name__ == "__main__":
    main()
