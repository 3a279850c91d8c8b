"""Heap-layout forests (reference: bforge/trees.py) with device traversal.

Layout is the reference's, unchanged (trees.py:1-17): root at heap index 1,
children 2t and 2t+1, index 0 unused; `axis`/`cutpoint` cover the first
2**(D-1) slots, `leaf_value` all 2**D; `cutpoint == 0` marks a leaf; points
go right iff grid index >= cutpoint.  `traverse_forest`, `sum_leaf_values`
and `evaluate_forest` run as sm_100a kernels through the C ABI; the scalar
helpers (`traverse`, masks, `validate`) are host utilities.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _native as N

MAX_SUPPORTED_DEPTH = 8  # trees.py:27-28


def heap_size(max_depth: int) -> int:
    return 1 << max_depth


def split_slots(max_depth: int) -> int:
    return 1 << (max_depth - 1)


def node_depth(index: int) -> int:
    return int(index).bit_length() - 1


def depth_table(max_depth: int) -> np.ndarray:
    """Depth per heap index; index 0 reports 0 (trees.py:44-48)."""
    return np.array([max(node_depth(t), 0) for t in range(heap_size(max_depth))], np.int64)


def min_axis_dtype(n_axes: int) -> np.dtype:
    """uint8 up to 256 axes, uint16 above (trees.py:53-55)."""
    return np.min_scalar_type(max(int(n_axes) - 1, 0))


def serialized_tree_nbytes(max_depth: int) -> int:
    return 4 * (2 * split_slots(max_depth) + heap_size(max_depth))


def check_depth(max_depth: int) -> None:
    if not 1 <= max_depth <= MAX_SUPPORTED_DEPTH:
        raise ValueError(f"max_depth must be in [1, {MAX_SUPPORTED_DEPTH}], got {max_depth}")


@dataclass
class TreeHeap:
    axis: np.ndarray
    cutpoint: np.ndarray
    leaf_value: np.ndarray
    max_depth: int

    @classmethod
    def root_only(cls, max_depth: int, n_axes: int = 1, value: float = 0.0) -> "TreeHeap":
        check_depth(max_depth)
        t = cls(np.zeros(split_slots(max_depth), min_axis_dtype(n_axes)),
                np.zeros(split_slots(max_depth), np.uint8),
                np.zeros(heap_size(max_depth), np.float32), max_depth)
        t.leaf_value[1] = value
        return t

    def copy(self) -> "TreeHeap":
        return TreeHeap(self.axis.copy(), self.cutpoint.copy(), self.leaf_value.copy(), self.max_depth)


@dataclass
class Forest:
    axis: np.ndarray        # (m, 2**(D-1))
    cutpoint: np.ndarray    # (m, 2**(D-1)) uint8
    leaf_value: np.ndarray  # (m, 2**D) float32
    max_depth: int

    @property
    def n_trees(self) -> int:
        return self.axis.shape[0]

    @classmethod
    def root_only(cls, n_trees: int, max_depth: int, n_axes: int = 1) -> "Forest":
        check_depth(max_depth)
        if n_trees < 1:
            raise ValueError(f"n_trees must be >= 1, got {n_trees}")
        return cls(np.zeros((n_trees, split_slots(max_depth)), min_axis_dtype(n_axes)),
                   np.zeros((n_trees, split_slots(max_depth)), np.uint8),
                   np.zeros((n_trees, heap_size(max_depth)), np.float32), max_depth)

    def tree(self, j: int) -> TreeHeap:
        return TreeHeap(self.axis[j], self.cutpoint[j], self.leaf_value[j], self.max_depth)

    def copy(self) -> "Forest":
        return Forest(self.axis.copy(), self.cutpoint.copy(), self.leaf_value.copy(), self.max_depth)


def traverse(tree: TreeHeap, x: np.ndarray) -> int:
    """Scalar leaf lookup for one point (trees.py:154-171 semantics)."""
    half = split_slots(tree.max_depth)
    t = 1
    while t < half and int(tree.cutpoint[t]) != 0:
        t = 2 * t + (1 if int(x[int(tree.axis[t])]) >= int(tree.cutpoint[t]) else 0)
    return t


def _u16(a: np.ndarray) -> np.ndarray:
    return np.ascontiguousarray(a, np.uint16)


def traverse_forest(forest: Forest, X: np.ndarray, device: int = 0) -> np.ndarray:
    """(n, m) uint8 leaf index of every (point, tree) pair, on the GPU."""
    check_depth(forest.max_depth)
    X = np.ascontiguousarray(X, np.uint8)
    n, p = X.shape
    m = forest.n_trees
    out = np.empty((n, m), np.uint8)
    if n == 0:
        return out
    d = N.dims(n, p, m, forest.max_depth)
    N.check(N.lib().bart_traverse(d, N.ptr(_u16(forest.axis)),
                                  N.ptr(np.ascontiguousarray(forest.cutpoint, np.uint8)), N.ptr(X), N.ptr(out), device))
    return out


def sum_leaf_values(leaf_value: np.ndarray, leaf_index: np.ndarray, device: int = 0) -> np.ndarray:
    """Sum of per-tree leaf values, f64, tree order (trees.py:206-218), on the GPU."""
    leaf_value = np.ascontiguousarray(leaf_value, np.float32)
    leaf_index = np.ascontiguousarray(leaf_index, np.uint8)
    n, m = leaf_index.shape
    out = np.empty(n, np.float64)
    if n == 0:
        return out
    D = int(leaf_value.shape[1]).bit_length() - 1
    d = N.dims(n, 1, m, D)
    N.check(N.lib().bart_sum_leaf_values(d, N.ptr(leaf_value), N.ptr(leaf_index), N.ptr(out), device))
    return out


def evaluate_forest(forest: Forest, X: np.ndarray, device: int = 0) -> np.ndarray:
    """Sum-of-trees predictions at the rows of X (trees.py:221-223), fused on the GPU."""
    check_depth(forest.max_depth)
    X = np.ascontiguousarray(X, np.uint8)
    n, p = X.shape
    out = np.empty(n, np.float64)
    if n == 0:
        return out
    d = N.dims(n, p, forest.n_trees, forest.max_depth)
    N.check(N.lib().bart_evaluate(d, N.ptr(_u16(forest.axis)), N.ptr(np.ascontiguousarray(forest.cutpoint, np.uint8)),
                                  N.ptr(np.ascontiguousarray(forest.leaf_value, np.float32)), N.ptr(X),
                                  N.ptr(out), device))
    return out


def evaluate_forests(forests: list[Forest], X: np.ndarray, device: int = 0) -> np.ndarray:
    """(F, n) predictions of F same-shape forests on one matrix (X uploaded once)."""
    X = np.ascontiguousarray(X, np.uint8)
    n, p = X.shape
    F = len(forests)
    out = np.empty((F, n), np.float64)
    if F == 0 or n == 0:
        return out
    f0 = forests[0]
    ax = np.ascontiguousarray(np.stack([f.axis for f in forests]), np.uint16)
    ct = np.ascontiguousarray(np.stack([f.cutpoint for f in forests]), np.uint8)
    lv = np.ascontiguousarray(np.stack([f.leaf_value for f in forests]), np.float32)
    d = N.dims(n, p, f0.n_trees, f0.max_depth)
    N.check(N.lib().bart_evaluate_many(d, F, N.ptr(ax), N.ptr(ct), N.ptr(lv), N.ptr(X), N.ptr(out), device))
    return out


def present_mask(cutpoint: np.ndarray, max_depth: int) -> np.ndarray:
    """(m, 2**D) existence flags: a node exists iff all its ancestors split."""
    m, half = cutpoint.shape
    out = np.zeros((m, 2 * half), bool)
    out[:, 1] = True
    for t in range(1, half):
        alive = out[:, t] & (cutpoint[:, t] > 0)
        out[:, 2 * t] = alive
        out[:, 2 * t + 1] = alive
    return out


def leaf_mask(cutpoint: np.ndarray, max_depth: int) -> np.ndarray:
    pres = present_mask(cutpoint, max_depth)
    split = np.zeros_like(pres)
    split[:, : cutpoint.shape[1]] = cutpoint > 0
    return pres & ~split


def validate(tree: TreeHeap, n_axes: int | None = None, grid_counts: np.ndarray | None = None) -> str | None:
    """First violated heap invariant of one tree, or None (trees.py:253-299)."""
    D = tree.max_depth
    if not isinstance(D, (int, np.integer)) or D < 1:
        return f"max_depth must be a positive integer, got {D!r}"
    half, size = split_slots(D), heap_size(D)
    for name, arr, want in (("axis", tree.axis, half), ("cutpoint", tree.cutpoint, half),
                            ("leaf_value", tree.leaf_value, size)):
        if arr.shape != (want,):
            return f"{name} array has shape {arr.shape}, expected ({want},)"
    pres = present_mask(tree.cutpoint[None, :], D)[0]
    split = np.zeros(size, bool)
    split[:half] = tree.cutpoint > 0
    leaves = pres & ~split
    bad = np.flatnonzero(split & ~pres)
    if bad.size:
        return f"orphan internal node at index {bad[0]}"
    if split[0] or tree.axis[0] != 0 or tree.leaf_value[0] != 0:
        return "index 0 must be unused (zero entries)"
    bad = np.flatnonzero(~split[:half] & (tree.axis != 0))
    if bad.size:
        return f"non-decision node {bad[0]} has a nonzero axis entry"
    bad = np.flatnonzero(~leaves & (tree.leaf_value != 0))
    if bad.size:
        return f"non-leaf node {bad[0]} has a nonzero leaf value"
    nodes = np.flatnonzero(split[:half])
    if n_axes is not None:
        bad = nodes[tree.axis[nodes] >= n_axes]
        if bad.size:
            return f"decision node {bad[0]} splits on axis {tree.axis[bad[0]]} >= {n_axes}"
    if grid_counts is not None and nodes.size:
        over = nodes[tree.cutpoint[nodes] > np.asarray(grid_counts)[tree.axis[nodes]]]
        if over.size:
            return f"decision node {over[0]} uses cutpoint {tree.cutpoint[over[0]]} beyond its axis grid"
    return None
