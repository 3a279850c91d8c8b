"""Drop-in for `bforge.sampler` whose `step` runs on the B200.

`init_state` / `step` keep the reference's signatures and state semantics
(sampler.py:201-241, 878-912): the chain state lives on the device behind an
opaque C handle (include/bart_b200.h) and `SamplerState` exposes it through
the reference's attribute names, fetched lazily in the reference's layouts.
One `step` = ONE kernel launch: the persistent sweep kernel proposes every
tree (phase 1, spread over all warps of the grid), then runs phases 2-11 tree
by tree and the sigma draw (csrc/sweep.cu).

Randomness.  With a numpy `Generator` (the reference's `rng`), `step` draws
the reference's `StepRandoms` block on the host in the reference's order and
injects it, so the device chain consumes exactly the random stream the
reference would.  With a `DeviceRNG`, the block is drawn on the device from
counter-based Philox4x32-10 (no host round trip; CUDA-graph replayable).

The scalar conjugate helpers at the end (`leaf_posterior`, `log_marginal_leaf`,
`accept_probability`, `sample_leaves`, `sample_sigma`, `sample_prior_tree`)
are host mirrors of the reference's test-facing formulas (sampler.py:579-621,
706-806, 915-952); they are not on the per-iteration path.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .trees import Forest, TreeHeap, check_depth, depth_table, heap_size, leaf_mask, min_axis_dtype, present_mask, split_slots

KIND_NONE = 0
KIND_GROW = 1
KIND_PRUNE = 2


@dataclass
class Hyperparams:
    """Model/sampler configuration, same fields and defaults as sampler.py:62-104."""

    leaf_sd: float
    lam: float
    n_trees: int = 200
    alpha: float = 0.95
    beta: float = 2.0
    leaf_mean: float = 0.0
    nu: float = 3.0
    max_depth: int = 6
    p_grow: float = 0.5
    update_sigma: bool = True


def depth_probabilities(hp: Hyperparams) -> np.ndarray:
    """alpha/(1+d)**beta per depth, 0 at the deepest level (sampler.py:107-118)."""
    d = np.arange(hp.max_depth, dtype=np.float64)
    out = hp.alpha / (1.0 + d) ** hp.beta
    out[-1] = 0.0
    return out


class DeviceRNG:
    """Key of the on-device Philox4x32-10 stream (counter = iteration, tree, slot)."""

    def __init__(self, seed: int = 0):
        self.seed = int(seed) & 0xFFFFFFFFFFFFFFFF

    @classmethod
    def from_seed_sequence(cls, ss: np.random.SeedSequence) -> "DeviceRNG":
        w = ss.generate_state(2, np.uint32)
        return cls(int(w[0]) | (int(w[1]) << 32))


@dataclass(frozen=True)
class StepRandoms:
    """One step's random block, drawn in the reference's order (sampler.py:244-260)."""

    move_u: np.ndarray
    accept_u: np.ndarray
    leaf_z: np.ndarray
    chi2_value: float

    @classmethod
    def draw(cls, rng: np.random.Generator, n_trees: int, heap: int, chi2_df: float) -> "StepRandoms":
        move_u = rng.random((n_trees, 5))
        accept_u = rng.random(n_trees)
        leaf_z = rng.standard_normal((n_trees, heap))
        return cls(move_u, accept_u, leaf_z, float(rng.chisquare(chi2_df)))


@dataclass(frozen=True)
class MoveProposal:
    tree: int
    kind: int
    node: int
    axis: int
    cut: int
    depth: int
    n_axes: int
    n_splits: int
    w_small: int
    w_prime_big: int
    growable_big: int
    left_child_growable: bool
    right_child_growable: bool


@dataclass
class Proposals:
    """Per-tree proposals (sampler.py:286-323), read back from the device."""

    kind: np.ndarray
    node: np.ndarray
    axis: np.ndarray
    cut: np.ndarray
    depth: np.ndarray
    n_axes: np.ndarray
    n_splits: np.ndarray
    w_small: np.ndarray
    w_prime_big: np.ndarray
    growable_big: np.ndarray
    left_child_growable: np.ndarray
    right_child_growable: np.ndarray
    struct_log: np.ndarray

    def tree(self, j: int) -> MoveProposal:
        return MoveProposal(j, int(self.kind[j]), int(self.node[j]), int(self.axis[j]), int(self.cut[j]),
                            int(self.depth[j]), int(self.n_axes[j]), int(self.n_splits[j]), int(self.w_small[j]),
                            int(self.w_prime_big[j]), int(self.growable_big[j]),
                            bool(self.left_child_growable[j]), bool(self.right_child_growable[j]))


def _hp_key(hp: Hyperparams) -> tuple:
    return (float(hp.leaf_sd), float(hp.lam), float(hp.alpha), float(hp.beta), float(hp.leaf_mean),
            float(hp.nu), float(hp.p_grow), bool(hp.update_sigma), int(hp.max_depth))


def availability_intervals(forest: Forest, max_cuts: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Host (lo, hi] availability per (tree, node, axis), uint8 like sampler.py:171-198.

    Not used by the device path (which walks ancestors); provided for callers
    that read `avail_lo`/`avail_hi`.  Only present nodes are meaningful.
    """
    m, half = forest.cutpoint.shape
    p = np.asarray(max_cuts).size
    lo = np.zeros((m, 2 * half, p), np.uint8)
    hi = np.zeros((m, 2 * half, p), np.uint8)
    hi[:, 1, :] = np.asarray(max_cuts, np.int64).astype(np.uint8)
    rows = np.arange(m)
    for t in range(1, half):
        lo[:, 2 * t] = lo[:, 2 * t + 1] = lo[:, t]
        hi[:, 2 * t] = hi[:, 2 * t + 1] = hi[:, t]
        ax = forest.axis[:, t].astype(np.int64)
        c = forest.cutpoint[:, t]
        hi[rows, 2 * t, ax] = c - np.uint8(1)
        lo[rows, 2 * t + 1, ax] = c
    return lo, hi


class SamplerState:
    """Device-resident chain state with the reference's attribute interface.

    Readable like `bforge.sampler.SamplerState` (sampler.py:121-147): `X`,
    `max_cuts`, `y`, `forest`, `resid`, `leaf_index` (n, m), `sigma2`, `rng`,
    node flags, `iteration`, `last_accepted`, `last_proposals`.  Assigning
    `forest`, `leaf_index`, `resid` or `sigma2` (or editing the returned host
    arrays in place and calling `rebuild_structure_caches()`) pushes the edit
    to the device before the next step, as tests/util.py:11-24 expects.
    """

    def __init__(self, X, max_cuts, y, hp: Hyperparams, rng, sigma2: float, device: int = 0,
                 shard: tuple[int, int, int] | None = None, max_ctas: int | None = None):
        self.X = X
        self.max_cuts = max_cuts
        self.y = y
        self.rng = rng
        self.device = int(device)
        self._m = int(hp.n_trees)
        self._D = int(hp.max_depth)
        self._hp_key = _hp_key(hp)
        self.iteration = 0
        self._cache: dict = {}
        self._dirty: set = set()
        self._h = C.c_void_p()
        seed = rng.seed if isinstance(rng, DeviceRNG) else 0
        d = N.dims(X.shape[0], X.shape[1], self._m, self._D)
        self.shard = shard  # (n_total, shard index, n_shards) for an n-sharded chain (paper_2410_23244_b200.shard)
        if shard is None:
            N.check(N.lib().bart_create_ex(d, N.hparams(hp, depth_probabilities(hp)), N.ptr(X), N.ptr(max_cuts),
                                           N.ptr(y), float(sigma2), seed, self.device, int(max_ctas or 0),
                                           C.byref(self._h)))
        else:
            n_total, k, n_shards = shard
            N.check(N.lib().bart_create_shard(d, int(n_total), int(k), int(n_shards),
                                              N.hparams(hp, depth_probabilities(hp)), N.ptr(X), N.ptr(max_cuts),
                                              N.ptr(y), float(sigma2), seed, self.device, C.byref(self._h)))

    # -- lifecycle
    def close(self) -> None:
        if getattr(self, "_h", None) and self._h.value:
            N.lib().bart_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    @property
    def n_points(self) -> int:
        """Points of the whole chain (all shards): the chi-square df is nu + n (sampler.py:259)."""
        return self.shard[0] if self.shard is not None else self.y.size

    # -- lazily fetched host mirrors
    def _fetch(self, key):
        if key in self._cache:
            return self._cache[key]
        L, h, m, D = N.lib(), self._h, self._m, self._D
        n = self.y.size
        if key == "forest":
            ax = np.empty((m, split_slots(D)), np.uint16)
            ct = np.empty((m, split_slots(D)), np.uint8)
            lv = np.empty((m, heap_size(D)), np.float32)
            N.check(L.bart_get_forest(h, N.ptr(ax), N.ptr(ct), N.ptr(lv)))
            val = Forest(ax.astype(min_axis_dtype(self.max_cuts.size)), ct, lv, D)
        elif key == "leaf_index":
            val = np.empty((n, m), np.uint8)
            N.check(L.bart_get_leaf_index(h, N.ptr(val)))
        elif key == "resid":
            val = np.empty(n, np.float32)
            N.check(L.bart_get_resid(h, N.ptr(val)))
        elif key in ("sigma2", "last_accepted"):
            if key == "last_accepted" and self.iteration == 0:
                return None
            # both in one synchronisation: a step's result is read as a pair
            v = np.empty(1, np.float64)
            a = np.empty(m, np.uint8) if self.iteration > 0 else None
            N.check(L.bart_get_step_result(h, N.ptr(a), N.ptr(v)))
            self._cache["sigma2"] = float(v[0])
            if a is not None:
                self._cache["last_accepted"] = a.astype(bool)
            val = self._cache[key]
        elif key == "last_proposals":
            if self.iteration == 0:
                return None
            val = self._read_proposals()
        else:
            raise KeyError(key)
        self._cache[key] = val
        return val

    def _read_proposals(self) -> Proposals:
        m = self._m
        rows = np.empty((N.PROPOSAL_ROWS, m), np.int64)
        sl = np.empty(m, np.float64)
        N.check(N.lib().bart_get_proposals(self._h, N.ptr(rows), N.ptr(sl)))
        return Proposals(kind=rows[0].astype(np.int8), node=rows[1], axis=rows[2], cut=rows[3], depth=rows[4],
                         n_axes=rows[5], n_splits=rows[6], w_small=rows[7], w_prime_big=rows[8],
                         growable_big=rows[9], left_child_growable=rows[10].astype(bool),
                         right_child_growable=rows[11].astype(bool), struct_log=sl)

    def _set(self, key, val):
        self._cache[key] = val
        self._dirty.add(key)

    forest = property(lambda s: s._fetch("forest"), lambda s, v: s._set("forest", v))
    leaf_index = property(lambda s: s._fetch("leaf_index"), lambda s, v: s._set("leaf_index", v))
    resid = property(lambda s: s._fetch("resid"), lambda s, v: s._set("resid", v))
    sigma2 = property(lambda s: s._fetch("sigma2"), lambda s, v: s._set("sigma2", float(v)))
    last_accepted = property(lambda s: s._fetch("last_accepted"))
    last_proposals = property(lambda s: s._fetch("last_proposals"))

    @property
    def node_present(self) -> np.ndarray:
        return present_mask(self.forest.cutpoint, self._D)

    @property
    def node_leaf(self) -> np.ndarray:
        return leaf_mask(self.forest.cutpoint, self._D)

    @property
    def avail_lo(self) -> np.ndarray:
        return availability_intervals(self.forest, self.max_cuts)[0]

    @property
    def avail_hi(self) -> np.ndarray:
        return availability_intervals(self.forest, self.max_cuts)[1]

    @property
    def node_can_split(self) -> np.ndarray:
        lo, hi = availability_intervals(self.forest, self.max_cuts)
        return (hi > lo).any(axis=2)

    # -- results without waiting for the next step
    def step_result(self, iteration: int | None = None) -> tuple[np.ndarray, float]:
        """(last_accepted, sigma2) of step `iteration` (default: the latest) for
        either of the last two `step` calls, from the pinned copy each step
        enqueues behind itself: read step k after launching step k+1 and the
        host's work for k+1 overlaps the device's step k."""
        it = self.iteration - 1 if iteration is None else int(iteration)
        a = np.empty(self._m, np.uint8)
        v = np.empty(1, np.float64)
        N.check(N.lib().bart_read_step_result(self._h, it, N.ptr(a), N.ptr(v)))
        return a.astype(bool), float(v[0])

    # -- resume
    def restore(self, forest: Forest, leaf_index: np.ndarray, resid: np.ndarray, sigma2: float,
                iteration: int) -> None:
        """Install a saved chain state (serialize.load_checkpoint): the forest,
        the (n, m) leaf-index cache, residuals, sigma^2 and the iteration (the
        device random stream's counter)."""
        self.forest = forest
        self.leaf_index = leaf_index
        self.resid = resid
        self.sigma2 = sigma2
        self._push()
        N.check(N.lib().bart_set_iteration(self._h, int(iteration)))
        self.iteration = int(iteration)

    # -- pushing host edits
    def rebuild_structure_caches(self) -> None:
        """Make the device state match the host mirrors (sampler.py:157-168)."""
        if "forest" in self._cache:
            self._dirty.add("forest")
        self._push()

    def _push(self) -> None:
        if not self._dirty:
            return
        L, h = N.lib(), self._h
        if self._dirty & {"forest", "leaf_index", "resid"}:
            f = self.forest
            if f.n_trees != self._m or f.max_depth != self._D:
                raise ValueError("forest shape does not match the chain (n_trees, max_depth)")
            li = self._cache.get("leaf_index") if "leaf_index" in self._dirty else None
            if li is None and "forest" not in self._dirty:
                li = self.leaf_index
            rs = self._cache.get("resid") if "resid" in self._dirty else None
            if rs is None:
                rs = self.resid
            li = None if li is None else np.ascontiguousarray(li, np.uint8)
            rs = np.ascontiguousarray(rs, np.float32)
            s2 = float(self._cache["sigma2"]) if "sigma2" in self._dirty else -1.0
            N.check(L.bart_set_state(h, N.ptr(np.ascontiguousarray(f.axis, np.uint16)),
                                     N.ptr(np.ascontiguousarray(f.cutpoint, np.uint8)),
                                     N.ptr(np.ascontiguousarray(f.leaf_value, np.float32)),
                                     N.ptr(li), N.ptr(rs), s2))
        elif "sigma2" in self._dirty:
            N.check(L.bart_set_sigma2(h, float(self._cache["sigma2"])))
        self._dirty.clear()
        self._cache.clear()

    def _ensure_hp(self, hp: Hyperparams) -> None:
        if int(hp.n_trees) != self._m or int(hp.max_depth) != self._D:
            raise ValueError("hyperparameters do not match the chain's (n_trees, max_depth)")
        key = _hp_key(hp)
        if key != self._hp_key:
            N.check(N.lib().bart_set_hparams(self._h, N.hparams(hp, depth_probabilities(hp))))
            self._hp_key = key

    def _after_step(self, n: int = 1) -> None:
        self._cache.clear()
        self.iteration += n

    # -- taps and measurement
    def enable_taps(self, on: bool = True) -> None:
        N.check(N.lib().bart_set_taps(self._h, 1 if on else 0))

    def taps(self) -> tuple[np.ndarray, np.ndarray]:
        """(counts, sums) of the last step, each (m, 2**D): post-refresh counts
        (sampler.py:894-897) and the tree-excluded sums each tree was resolved
        with (sampler.py:828)."""
        size = heap_size(self._D)
        cnt = np.empty((self._m, size), np.int64)
        sums = np.empty((self._m, size), np.float64)
        N.check(N.lib().bart_get_taps(self._h, N.ptr(cnt), N.ptr(sums)))
        return cnt, sums

    def last_randoms(self) -> "StepRandoms":
        """The StepRandoms block (sampler.py:244-260) the latest step consumed:
        the injected one, or the one the device drew from Philox4x32-10."""
        m, size = self._m, heap_size(self._D)
        mu, au = np.empty((m, 5)), np.empty(m)
        z, c2 = np.empty((m, size)), np.empty(1)
        N.check(N.lib().bart_get_randoms(self._h, N.ptr(mu), N.ptr(au), N.ptr(z), N.ptr(c2)))
        return StepRandoms(mu, au, z, float(c2[0]))

    def predict_train(self) -> np.ndarray:
        """trees.sum_leaf_values(forest.leaf_value, leaf_index) from the device cache."""
        out = np.empty(self.y.size, np.float64)
        N.check(N.lib().bart_predict_cached(self._h, N.ptr(out)))
        return out

    def predict(self, Xq: np.ndarray) -> np.ndarray:
        """evaluate_forest(current forest, Xq) on the device."""
        Xq = np.ascontiguousarray(Xq, np.uint8)
        out = np.empty(Xq.shape[0], np.float64)
        N.check(N.lib().bart_predict_matrix(self._h, N.ptr(Xq), Xq.shape[0], N.ptr(out)))
        return out

    # -- n-sharding (paper_2410_23244_b200.shard)
    def shard_export(self) -> bytes:
        buf = (C.c_uint8 * N.SHARD_HANDLE_BYTES)()
        N.check(N.lib().bart_shard_export(self._h, C.cast(buf, C.c_void_p)))
        return bytes(buf)

    def shard_connect(self, handles: list[bytes]) -> None:
        blob = b"".join(handles)
        if self.shard is None or len(handles) != self.shard[2] or len(blob) != len(handles) * N.SHARD_HANDLE_BYTES:
            raise ValueError("need one exported handle per shard, in shard order")
        buf = (C.c_uint8 * len(blob)).from_buffer_copy(blob)
        N.check(N.lib().bart_shard_connect(self._h, C.cast(buf, C.c_void_p)))

    # -- fit() trace kept on the device (bart_trace_*)
    def trace_begin(self, n_iter: int, n_keep: int, Xq_test: np.ndarray | None = None,
                    store_train_draws: bool = False, store_forests: bool = False, train_ring: int = 0) -> None:
        """train_ring > 0: keep only that many training-row draws on the device
        (a ring; drain it with trace_read_draws before it wraps)."""
        X = None if Xq_test is None else np.ascontiguousarray(Xq_test, np.uint8)
        opts = N.TraceOpts(int(n_iter), int(n_keep), 0 if X is None else int(X.shape[0]),
                           int(bool(store_train_draws)), int(bool(store_forests)), int(train_ring))
        N.check(N.lib().bart_trace_begin(self._h, C.byref(opts), N.ptr(X)))
        self._trace = dict(n_test=opts.n_test, store_train=bool(store_train_draws), store_forests=bool(store_forests))

    def trace_keep(self) -> None:
        """Record the current state as a kept draw (asynchronous)."""
        N.check(N.lib().bart_trace_keep(self._h))

    def trace_read(self, train_draws: bool = True, train_out: np.ndarray | None = None) -> dict:
        """Everything recorded since trace_begin, in the reference's layouts (scaled units);
        train_draws=False leaves the (n_keep, n) draws on the device (trace_read_draws);
        train_out: a C-contiguous (n_keep, n) float64 array to read the draws into."""
        ni, nk = C.c_int64(), C.c_int64()
        N.check(N.lib().bart_trace_counts(self._h, C.byref(ni), C.byref(nk)))
        ni, nk, n, m, D = ni.value, nk.value, self.y.size, self._m, self._D
        o = self._trace
        out = dict(
            accepted=np.empty((ni, m), np.uint8), sigma2_iter=np.empty(ni), sigma2_keep=np.empty(nk),
            train_mean=np.empty(n), train_var=np.empty(n),
            train_draws=(None if not (o["store_train"] and train_draws) else
                         train_out if train_out is not None else np.empty((nk, n))),
            train_points=np.empty((nk, min(n, N.TRACE_POINTS))),
            test_draws=np.empty((nk, o["n_test"])) if o["n_test"] else None,
            mean_leaves=np.empty(nk),
            axis=np.empty((nk, m, split_slots(D)), np.uint16) if o["store_forests"] else None,
            cutpoint=np.empty((nk, m, split_slots(D)), np.uint8) if o["store_forests"] else None,
            leaf_value=np.empty((nk, m, heap_size(D)), np.float32) if o["store_forests"] else None)
        keys = ["accepted", "sigma2_iter", "sigma2_keep", "train_mean", "train_var", "train_draws", "train_points",
                "test_draws", "mean_leaves", "axis", "cutpoint", "leaf_value"]
        N.check(N.lib().bart_trace_read(self._h, *[N.ptr(out[k]) for k in keys]))
        out["accepted"] = out["accepted"].astype(bool)
        return out

    def trace_read_draws(self, k0: int, k1: int, train: bool = True, test: bool = False):
        """Kept draws [k0, k1) of the training-row (and test-row) predictions, scaled units."""
        n_test = self._trace["n_test"]
        tr = np.empty((k1 - k0, self.y.size)) if train else None
        te = np.empty((k1 - k0, n_test)) if test else None
        N.check(N.lib().bart_trace_read_draws(self._h, int(k0), int(k1), N.ptr(tr), N.ptr(te)))
        return tr, te

    def trace_end(self) -> None:
        N.check(N.lib().bart_trace_end(self._h))

    def set_exchange(self, mode: str) -> None:
        """The cross-CTA / cross-shard exchange: "flat" (every CTA adds into
        every shard's words) or "two_level" (per-shard stage, one forwarder
        per shard); bit-identical results (include/bart_b200.h)."""
        modes = {"flat": 0, "two_level": 1}
        if mode not in modes:
            raise ValueError(f"exchange mode must be one of {sorted(modes)}")
        N.check(N.lib().bart_set_exchange(self._h, modes[mode]))

    def set_copy_groups(self, groups: int) -> None:
        """Test hook: emulate `groups` shards inside one launch on one device."""
        N.check(N.lib().bart_set_copy_groups(self._h, int(groups)))

    def kernel_launches(self) -> int:
        return int(N.lib().bart_kernel_launches(self._h))

    def sweep_config(self) -> dict:
        out = np.zeros(5, np.int32)
        N.check(N.lib().bart_sweep_config(self._h, N.ptr(out)))
        return dict(ctas=int(out[0]), threads=int(out[1]), chunk=int(out[2]), smem_bytes=int(out[3]),
                    stream=bool(out[4]))

    def sync(self) -> None:
        N.check(N.lib().bart_sync(self._h))


def init_state(X: np.ndarray, max_cuts: np.ndarray, y: np.ndarray, hp: Hyperparams, rng,
               sigma2: float | None = None, device: int = 0, max_ctas: int | None = None) -> SamplerState:
    """Fresh chain on the device: root-only zero forest, resid = y (sampler.py:201-241).

    max_ctas limits the chain's sweep to that many SMs, so several chains on
    their own streams run side by side (multi-chain batching)."""
    X = np.ascontiguousarray(X, np.uint8)
    y32 = np.ascontiguousarray(y, np.float32)
    max_cuts = np.ascontiguousarray(max_cuts, np.int64)
    if X.ndim != 2:
        raise ValueError(f"X must be 2-d, got shape {X.shape}")
    n, p = X.shape
    if y32.shape != (n,):
        raise ValueError(f"y has shape {y32.shape}, expected ({n},)")
    if max_cuts.shape != (p,):
        raise ValueError(f"max_cuts has shape {max_cuts.shape}, expected ({p},)")
    check_depth(hp.max_depth)
    if hp.n_trees < 1:
        raise ValueError(f"n_trees must be >= 1, got {hp.n_trees}")
    if sigma2 is None:
        sigma2 = float(np.var(y32, ddof=1)) if n >= 2 else 1.0
    return SamplerState(X, max_cuts, y32, hp, rng, float(sigma2), device, max_ctas=max_ctas)


def philox4x32_10(ctr: np.ndarray, key: np.ndarray, device: int = 0) -> np.ndarray:
    """The device RNG's Philox4x32-10 bijection (Random123 philox4x32_10) on
    explicit counters (k, 4) and keys (k, 2), uint32 -> (k, 4) uint32."""
    ctr = np.ascontiguousarray(ctr, np.uint32).reshape(-1, 4)
    key = np.ascontiguousarray(key, np.uint32).reshape(-1, 2)
    if ctr.shape[0] != key.shape[0]:
        raise ValueError("one key per counter")
    out = np.empty_like(ctr)
    N.check(N.lib().bart_philox4x32_10(N.ptr(ctr), N.ptr(key), N.ptr(out), ctr.shape[0], int(device)))
    return out


def _randoms_struct(rnd: StepRandoms):
    arrs = (np.ascontiguousarray(rnd.move_u, np.float64), np.ascontiguousarray(rnd.accept_u, np.float64),
            np.ascontiguousarray(rnd.leaf_z, np.float64))
    return N.Randoms(N.ptr(arrs[0]), N.ptr(arrs[1]), N.ptr(arrs[2]), float(rnd.chi2_value)), arrs


def step(state: SamplerState, hp: Hyperparams, rng=None, randoms: StepRandoms | None = None) -> SamplerState:
    """One sampler iteration on the device; mutates and returns `state` (sampler.py:878-912).

    `randoms` injects an explicit random block (parity tests); otherwise a
    numpy Generator (`rng` or `state.rng`) supplies the reference's block and
    a `DeviceRNG` (or None) draws it on the device.
    """
    state._ensure_hp(hp)
    state._push()
    gen = rng if rng is not None else state.rng
    if randoms is None and isinstance(gen, np.random.Generator):
        randoms = StepRandoms.draw(gen, state._m, heap_size(state._D), hp.nu + state.n_points)
    if randoms is not None:
        rs, _keep = _randoms_struct(randoms)
        N.check(N.lib().bart_step(state.handle, C.byref(rs)))
    else:
        N.check(N.lib().bart_step(state.handle, None))
    state._after_step()
    return state


def run(state: SamplerState, hp: Hyperparams, n_iter: int) -> SamplerState:
    """n_iter device-RNG iterations back to back (CUDA-graph replay, asynchronous)."""
    state._ensure_hp(hp)
    state._push()
    N.check(N.lib().bart_run(state.handle, int(n_iter)))
    state._after_step(int(n_iter))
    return state


def propose_moves(state: SamplerState, hp: Hyperparams, rng=None, uniforms: np.ndarray | None = None) -> Proposals:
    """Phase 1 alone on the device (sampler.py:469-526); the state is unchanged."""
    state._ensure_hp(hp)
    state._push()
    if uniforms is None:
        uniforms = (rng if rng is not None else state.rng).random((state._m, 5))
    u = np.ascontiguousarray(uniforms, np.float64)
    N.check(N.lib().bart_propose(state.handle, N.ptr(u)))
    props = state._read_proposals()
    props.depth = depth_table(state._D)[props.node]
    return props


# ---------------------------------------------------------------- host scalar helpers

def leaf_posterior(count, rsum, sigma2, hp: Hyperparams):
    """Conjugate (mean, precision) of a leaf (sampler.py:579-590)."""
    tau = 1.0 / sigma2
    tau_mu = 1.0 / (hp.leaf_sd * hp.leaf_sd)
    prec = tau_mu + count * tau
    return (tau_mu * hp.leaf_mean + tau * rsum) / prec, prec


def draw_leaf_values(mean, prec, z):
    return mean + z / np.sqrt(prec)


def log_marginal_leaf(count, rsum, sigma, hp: Hyperparams):
    """Leaf log marginal up to cancelling terms (sampler.py:598-621); empty leaf -> 0."""
    s2 = sigma * sigma
    tau_mu = 1.0 / (hp.leaf_sd * hp.leaf_sd)
    mean, prec = leaf_posterior(count, rsum, s2, hp)
    return 0.5 * np.log(tau_mu / prec) - 0.5 * hp.leaf_mean * hp.leaf_mean * tau_mu + 0.5 * mean * mean * prec


def _lik_ratio(nl, nr, sl, sr, sigma2, hp):
    tau = 1.0 / sigma2
    tau_mu = 1.0 / (hp.leaf_sd * hp.leaf_sd)
    pl, pr, pp = tau_mu + nl * tau, tau_mu + nr * tau, tau_mu + (nl + nr) * tau
    count_part = 0.5 * np.log(tau_mu * pp / (pl * pr)) - 0.5 * hp.leaf_mean * hp.leaf_mean * tau_mu
    shift = tau_mu * hp.leaf_mean

    def q(prec, s):
        mu = (shift + tau * s) / prec
        return mu * mu * prec

    return count_part + 0.5 * (q(pl, sl) + q(pr, sr) - q(pp, sl + sr))


def accept_probability(proposal: MoveProposal, counts, sums, sigma: float, hp: Hyperparams) -> float:
    """Metropolis acceptance probability of one proposal (sampler.py:706-734)."""
    if proposal.kind == KIND_NONE:
        return 0.0
    c2, c3 = 2 * proposal.node, 2 * proposal.node + 1
    lik = _lik_ratio(int(counts[c2]), int(counts[c3]), float(sums[c2]), float(sums[c3]), sigma * sigma, hp)
    probs = depth_probabilities(hp)
    dp = probs[proposal.depth]
    cp = probs[min(proposal.depth + 1, hp.max_depth - 1)]
    ppe = 1.0 if proposal.growable_big == 0 else 1.0 - hp.p_grow
    pge = 1.0 if proposal.node == 1 else hp.p_grow
    core = dp * ppe * max(proposal.w_small, 1) / ((1.0 - dp) * pge * max(proposal.w_prime_big, 1))
    struct = (math.log(core) + math.log1p(-cp * float(proposal.left_child_growable))
              + math.log1p(-cp * float(proposal.right_child_growable)))
    total = (1.0 if proposal.kind == KIND_GROW else -1.0) * (struct + float(lik))
    return 1.0 if total >= 0 else math.exp(total)


def sample_leaves(tree: TreeHeap, counts, sums, sigma: float, hp: Hyperparams, rng=None, z=None) -> np.ndarray:
    """Redraw every leaf of one tree (sampler.py:764-787)."""
    size = heap_size(tree.max_depth)
    if z is None:
        z = rng.standard_normal(size)
    mask = leaf_mask(tree.cutpoint[None, :], tree.max_depth)[0]
    mean, prec = leaf_posterior(counts, sums, sigma * sigma, hp)
    return (draw_leaf_values(mean, prec, z) * mask).astype(np.float32)


def sum_squares(x: np.ndarray) -> float:
    return float(np.add.reduce(np.square(np.asarray(x, np.float64))))


def sigma2_draw(resid: np.ndarray, hp: Hyperparams, chi2_value: float) -> float:
    return (hp.nu * hp.lam + sum_squares(resid)) / chi2_value


def sample_sigma(resid: np.ndarray, hp: Hyperparams, rng, chi2_value: float | None = None) -> float:
    if chi2_value is None:
        chi2_value = float(rng.chisquare(hp.nu + resid.size))
    return math.sqrt(sigma2_draw(resid, hp, chi2_value))


def sample_prior_tree(max_cuts: np.ndarray, hp: Hyperparams, rng: np.random.Generator) -> TreeHeap:
    """One tree from the generative prior, consuming `rng` in the order of sampler.py:915-952:
    per visited node one uniform (only if some axis is open), then axis and
    cut uniforms for a split or one normal for a leaf, left subtree first."""
    max_cuts = np.asarray(max_cuts, np.int64)
    tree = TreeHeap.root_only(hp.max_depth, n_axes=max_cuts.size)
    probs = depth_probabilities(hp)
    bounds = np.stack([np.zeros_like(max_cuts), max_cuts])  # rows: lo, hi

    def visit(t: int, depth: int) -> None:
        open_ = np.flatnonzero(bounds[1] > bounds[0])
        if open_.size and rng.random() < probs[depth]:
            a = int(open_[min(int(rng.random() * open_.size), open_.size - 1)])
            width = int(bounds[1, a] - bounds[0, a])
            c = int(bounds[0, a]) + 1 + min(int(rng.random() * width), width - 1)
            tree.axis[t], tree.cutpoint[t] = a, c
            for child, row, val in ((2 * t, 1, c - 1), (2 * t + 1, 0, c)):
                keep = bounds[row, a]
                bounds[row, a] = val
                visit(child, depth + 1)
                bounds[row, a] = keep
        else:
            tree.leaf_value[t] = rng.normal(hp.leaf_mean, hp.leaf_sd)

    visit(1, 0)
    return tree
