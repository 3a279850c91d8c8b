"""CPU oracle for the BART MCMC step — TEST INFRASTRUCTURE ONLY.

Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` legs may import this module, and only as the checker or as
the timed CPU baseline.  The product path (`paper_2410_23244_b200`) never
imports it and fails loudly when its CUDA library is missing.

What it is: a restatement of the reference sampler (`bforge`, pure
numpy + numba, /root/reference/pkg/src/bforge) written as array code over a
tree-major layout (leaf index stored (m, n), predictors (p, n)), so that each
tree's column is contiguous.  Every function cites the reference lines whose
semantics it reproduces.  The per-tree proposal bookkeeping, a scalar numba
loop in the reference (sampler.py:326-466), is restated here as masked array
operations over all trees at once; availability intervals are recomputed from
the forest every step instead of being cached incrementally (equal on every
present node, which is all the reference ever reads).

Parity of this oracle is PINNED: tests/test_oracle_golden.py replays the
golden vectors in tests/golden/*.npz — produced by running the real reference
here (tests/golden/make_golden.py) — and requires bit-identical proposals,
counts, sums, accept decisions, forests, leaf indices and residuals.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

NONE, GROW, PRUNE = 0, 1, 2


# ---------------------------------------------------------------- structure

def heap_depths(size: int) -> np.ndarray:
    """Depth per heap index, index 0 mapped to 0 (trees.py:44-48)."""
    idx = np.arange(size)
    idx[0] = 1
    return np.floor(np.log2(idx)).astype(np.int64)


def depth_probs(alpha: float, beta: float, max_depth: int) -> np.ndarray:
    """alpha/(1+d)**beta with the deepest level forced to 0 (sampler.py:107-113)."""
    d = np.arange(max_depth, dtype=np.float64)
    probs = alpha / (1.0 + d) ** beta
    probs[-1] = 0.0
    return probs


def structure(cut: np.ndarray, max_depth: int) -> tuple[np.ndarray, np.ndarray]:
    """(present, leaf) masks of shape (m, 2**D) (trees.py:226-250)."""
    m, half = cut.shape
    size = 2 * half
    present = np.zeros((m, size), bool)
    present[:, 1] = True
    internal = np.zeros((m, size), bool)
    internal[:, :half] = cut > 0
    for t in range(1, half):
        both = present[:, t] & internal[:, t]
        present[:, 2 * t] = both
        present[:, 2 * t + 1] = both
    return present, present & ~internal


def availability(axis: np.ndarray, cut: np.ndarray, max_cuts: np.ndarray, max_depth: int):
    """Per (tree, node, axis) open interval (lo, hi] of cutpoint indices.

    Same values as the reference's cached `avail_lo/avail_hi` on every
    present node (sampler.py:171-198, refreshed at :850-859); int16 here, so
    entries at absent nodes are simply junk of a different kind.
    """
    m, half = cut.shape
    p = max_cuts.size
    lo = np.zeros((m, 2 * half, p), np.int16)
    hi = np.zeros((m, 2 * half, p), np.int16)
    hi[:, 1, :] = max_cuts
    rows = np.arange(m)
    for t in range(1, half):
        a = axis[:, t].astype(np.int64)
        c = cut[:, t].astype(np.int16)
        for child in (2 * t, 2 * t + 1):
            lo[:, child] = lo[:, t]
            hi[:, child] = hi[:, t]
        hi[rows, 2 * t, a] = c - 1
        lo[rows, 2 * t + 1, a] = c
    return lo, hi


def traverse_forest(axis, cut, max_depth, Xt) -> np.ndarray:
    """Leaf heap index per (tree, point), shape (m, n) uint8 (trees.py:174-203).

    D-1 fixed levels; a point stops at the first node whose cutpoint is 0;
    it goes right iff x[axis] >= cutpoint (trees.py:154-171).
    """
    m, half = cut.shape
    n = Xt.shape[1]
    out = np.ones((m, n), np.int64)
    for j in range(m):
        idx = np.ones(n, np.int64)
        done = np.zeros(n, bool)
        for _ in range(max_depth - 1):
            split = cut[j][np.minimum(idx, half - 1)].astype(np.int64)
            split = np.where(idx < half, split, 0)
            done |= split == 0
            ax = axis[j][np.minimum(idx, half - 1)].astype(np.int64)
            x = Xt[ax, np.arange(n)]
            idx = np.where(done, idx, 2 * idx + (x >= split))
        out[j] = idx
    return out.astype(np.uint8)


def sum_leaf_values(leaf_value: np.ndarray, Lt: np.ndarray) -> np.ndarray:
    """f64 sum of per-tree leaf values, tree by tree (trees.py:206-218)."""
    total = np.zeros(Lt.shape[1], np.float64)
    for j in range(leaf_value.shape[0]):
        total += leaf_value[j, Lt[j]]
    return total


# ---------------------------------------------------------------- proposals

@dataclass
class Proposals:
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
    gl: np.ndarray
    gr: np.ndarray
    struct_log: np.ndarray


def _kth_true(mask: np.ndarray, k: np.ndarray) -> np.ndarray:
    """Column of the k-th (0-based) True per row; 0 where the row has fewer."""
    cum = np.cumsum(mask, axis=1)
    hit = (cum == (k[:, None] + 1)) & mask
    return np.where(hit.any(axis=1), np.argmax(hit, axis=1), 0)


def _pick(u: np.ndarray, count: np.ndarray) -> np.ndarray:
    """floor(u * count) clamped to count-1 (sampler.py:377-379, 402-404, 418-420)."""
    return np.minimum((u * count).astype(np.int64), count - 1)


def propose(axis, cut, max_depth, max_cuts, alpha, beta, p_grow, u) -> Proposals:
    """One move per tree, all trees at once (reference: sampler.py:326-466).

    Growable leaf: leaf, depth < D-1, some open axis (:344-348).  Prunable
    node: decision node whose children are both leaves (:350-360).  Null
    move iff neither exists (:362-369); GROW iff w>0 and (wp==0 or
    u0 < p_grow) (:371).  Target, axis and cut are floor(u*k)-th
    candidates in index order; PRUNE keeps the node's own axis/cut.
    """
    m, half = cut.shape
    size = 2 * half
    D = max_depth
    dep = heap_depths(size)
    probs = depth_probs(alpha, beta, D)
    _, leaf = structure(cut, D)
    lo, hi = availability(axis, cut, max_cuts, D)
    open_ = hi > lo
    growable = leaf & (dep < D - 1)[None, :] & open_.any(axis=2)
    internal = cut > 0
    kid_internal = np.zeros((m, half), bool)
    for t in range(1, half // 2):
        kid_internal[:, t] = internal[:, 2 * t] | internal[:, 2 * t + 1]
    prunable = internal & ~kid_internal
    prunable[:, 0] = False
    w = growable.sum(axis=1)
    wp = prunable.sum(axis=1)

    null = (w == 0) & (wp == 0)
    grow = (w > 0) & ((wp == 0) | (u[:, 0] < p_grow))
    kind = np.where(null, NONE, np.where(grow, GROW, PRUNE)).astype(np.int8)

    t_grow = _kth_true(growable, _pick(u[:, 1], w))
    t_prune = _kth_true(prunable, _pick(u[:, 4], wp))
    t = np.where(grow, t_grow, t_prune)
    rows = np.arange(m)
    open_t = open_[rows, t]                      # (m, p)
    na = open_t.sum(axis=1)
    a = np.where(grow, _kth_true(open_t, _pick(u[:, 2], na)), axis[rows, t].astype(np.int64))
    la = lo[rows, t, a].astype(np.int64)
    ha = hi[rows, t, a].astype(np.int64)
    ns = ha - la
    c = np.where(grow, la + 1 + _pick(u[:, 3], ns), cut[rows, t].astype(np.int64))

    d = dep[t]
    child_ok = d < D - 2
    other = na >= 2
    gl_g = child_ok & (other | (c - 1 > la))
    gr_g = child_ok & (other | (ha > c))
    kids = np.minimum(2 * t, size - 2)
    gl_p = growable[rows, kids]
    gr_p = growable[rows, kids + 1]
    gl = np.where(grow, gl_g, gl_p)
    gr = np.where(grow, gr_g, gr_p)
    parent_prunable = (t > 1) & prunable[rows, t >> 1]
    w_small = np.where(grow, w, w - gl_p - gr_p + 1)
    w_prime_big = np.where(grow, wp + 1 - parent_prunable, wp)
    growable_big = np.where(grow, w - 1 + gl_g + gr_g, w)

    struct = np.zeros(m)
    for j in np.flatnonzero(~null):
        dj = int(d[j])
        dp = probs[dj]
        cp = probs[min(dj + 1, D - 1)]
        p_prune_eff = 1.0 if growable_big[j] == 0 else 1.0 - p_grow
        p_grow_eff = 1.0 if t[j] == 1 else p_grow
        core = dp * p_prune_eff * max(int(w_small[j]), 1) / ((1.0 - dp) * p_grow_eff * max(int(w_prime_big[j]), 1))
        struct[j] = (math.log(core) + math.log1p(-cp * (1.0 if gl[j] else 0.0))
                     + math.log1p(-cp * (1.0 if gr[j] else 0.0)))

    def z(x):  # null proposals report zeros everywhere (sampler.py:362-369)
        return np.where(null, 0, x).astype(np.int64)

    node = z(t)
    return Proposals(
        kind=kind, node=node, axis=z(a), cut=z(c), depth=dep[node], n_axes=z(na),
        n_splits=z(ns), w_small=z(w_small), w_prime_big=z(w_prime_big),
        growable_big=z(growable_big), gl=np.where(null, False, gl), gr=np.where(null, False, gr),
        struct_log=struct,
    )


# ---------------------------------------------------------------- chain

class OracleChain:
    """Chain state in tree-major layout plus the reference's `step`.

    Attributes mirror `bforge.sampler.SamplerState` (sampler.py:121-147):
    forest rows `axis`, `cut`, `leaf`; residuals `resid` (float32); leaf
    index `Lt` = reference `leaf_index.T`; `sigma2` (float64).
    """

    def __init__(self, X, max_cuts, y, hp, sigma2=None, axis=None, cut=None, leaf=None,
                 resid=None, leaf_index=None):
        self.Xt = np.ascontiguousarray(np.asarray(X, np.uint8).T)
        self.max_cuts = np.asarray(max_cuts, np.int64)
        self.y = np.asarray(y, np.float32)
        self.hp = hp
        m, D = hp.n_trees, hp.max_depth
        half, size = 1 << (D - 1), 1 << D
        n = self.y.size
        adt = np.uint8 if self.max_cuts.size <= 256 else np.uint16
        self.axis = np.zeros((m, half), adt) if axis is None else np.array(axis)
        self.cut = np.zeros((m, half), np.uint8) if cut is None else np.array(cut, np.uint8)
        self.leaf = np.zeros((m, size), np.float32) if leaf is None else np.array(leaf, np.float32)
        if leaf_index is None:
            self.Lt = traverse_forest(self.axis, self.cut, D, self.Xt)
        else:
            self.Lt = np.ascontiguousarray(np.asarray(leaf_index, np.uint8).T)
        if resid is None:
            if axis is None and leaf is None:
                self.resid = self.y.copy()  # init_state, sampler.py:232
            else:  # tests/util.py:19-23 recomputation
                self.resid = (self.y.astype(np.float64) - sum_leaf_values(self.leaf, self.Lt)).astype(np.float32)
        else:
            self.resid = np.array(resid, np.float32)
        if sigma2 is None:
            sigma2 = float(np.var(self.y, ddof=1)) if n >= 2 else 1.0  # sampler.py:222-223
        self.sigma2 = float(sigma2)
        self.last_accepted = np.zeros(m, bool)

    @property
    def leaf_index(self) -> np.ndarray:
        return self.Lt.T

    def step(self, move_u, accept_u, leaf_z, chi2, taps: dict | None = None) -> None:
        """One sampler iteration with the given random block (sampler.py:878-912)."""
        hp = self.hp
        D, m = hp.max_depth, hp.n_trees
        size = 1 << D
        props = propose(self.axis, self.cut, D, self.max_cuts, hp.alpha, hp.beta, hp.p_grow, move_u)

        # phase 2: index cache follows the larger tree (sampler.py:529-547)
        for j in np.flatnonzero(props.kind == GROW):
            t, a, c = int(props.node[j]), int(props.axis[j]), int(props.cut[j])
            col = self.Lt[j]
            hit = col == t
            col[hit] = (2 * t + (self.Xt[a][hit] >= c)).astype(np.uint8)
        # phase 3 (sampler.py:550-553, 895-897)
        counts = np.stack([np.bincount(self.Lt[j], minlength=size) for j in range(m)]).astype(np.int64)
        if taps is not None:
            taps["props"] = props
            taps["counts"] = counts.copy()
            taps["sums"] = np.zeros((m, size))

        tau = 1.0 / self.sigma2
        tau_mu = 1.0 / (hp.leaf_sd * hp.leaf_sd)
        _, leaf_mask = structure(self.cut, D)
        for j in range(m):
            self.last_accepted[j] = self._resolve(j, props, counts[j], tau, tau_mu, accept_u[j],
                                                  leaf_z[j], leaf_mask[j], taps)

        # sigma^2 | resid (sampler.py:790-799, 906-908)
        rss = float(np.add.reduce(np.square(self.resid.astype(np.float64))))
        s2 = (hp.nu * hp.lam + rss) / chi2
        if hp.update_sigma:
            self.sigma2 = s2

    def _resolve(self, j, props, cnt, tau, tau_mu, accept_u, z, leaf_row, taps) -> bool:
        """Phases 7-11 of one tree (sampler.py:809-875)."""
        hp = self.hp
        kind = int(props.kind[j])
        t = int(props.node[j])
        grow = kind == GROW
        c2, c3 = 2 * t, 2 * t + 1
        old_leaf = self.leaf[j].copy()
        col = self.Lt[j]

        # tree-excluded sums (sampler.py:556-576)
        raw = np.bincount(col, weights=self.resid, minlength=cnt.size)
        adj = old_leaf.astype(np.float64)
        if grow:
            adj[c2] = adj[c3] = float(old_leaf[t])
        sums = raw + cnt * adj
        if taps is not None:
            taps["sums"][j] = sums

        # acceptance (sampler.py:624-645, 669-684, 829-834)
        accepted = False
        if kind != NONE:
            nl, nr = int(cnt[c2]), int(cnt[c3])
            prec_l = tau_mu + nl * tau
            prec_r = tau_mu + nr * tau
            prec_p = tau_mu + (nl + nr) * tau
            count_part = 0.5 * math.log(tau_mu * prec_p / (prec_l * prec_r)) - 0.5 * hp.leaf_mean * hp.leaf_mean * tau_mu
            partial = float(props.struct_log[j]) + count_part
            shift = tau_mu * hp.leaf_mean

            def term(count, s):
                prec = tau_mu + count * tau
                mean = (shift + tau * s) / prec
                return mean * mean * prec

            sl, sr = float(sums[c2]), float(sums[c3])
            sum_part = 0.5 * (term(nl, sl) + term(nr, sr) - term(nl + nr, sl + sr))
            log_alpha = (1.0 if grow else -1.0) * (partial + sum_part)
            accepted = bool(accept_u < math.exp(min(log_alpha, 0.0)))

        leaf_row = leaf_row.copy()
        if accepted:  # structure write (sampler.py:836-848)
            if grow:
                self.axis[j, t] = props.axis[j]
                self.cut[j, t] = props.cut[j]
                leaf_row[t] = False
                leaf_row[c2] = leaf_row[c3] = True
            else:
                self.axis[j, t] = 0
                self.cut[j, t] = 0
                leaf_row[t] = True
                leaf_row[c2] = leaf_row[c3] = False

        final_small = (accepted != grow) and kind != NONE  # sampler.py:861-866
        cnt = cnt.copy()
        if final_small:
            cnt[t] = cnt[c2] + cnt[c3]
            cnt[c2] = cnt[c3] = 0
            sums[t] = sums[c2] + sums[c3]
            sums[c2] = sums[c3] = 0.0

        # leaf redraw (sampler.py:579-595, 868-870)
        prec = tau_mu + cnt * tau
        mean = (tau_mu * hp.leaf_mean + tau * sums) / prec
        new_leaf = ((mean + z / np.sqrt(prec)) * leaf_row).astype(np.float32)

        # cache + residual update (sampler.py:737-761)
        collapsed = np.where((col >> 1) == t, np.uint8(t), col)
        final = collapsed if final_small else col
        old_idx = collapsed if grow else col
        self.resid += old_leaf[old_idx] - new_leaf[final]
        self.Lt[j] = final
        self.leaf[j] = new_leaf
        return accepted
