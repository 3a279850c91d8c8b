"""Forest kernels on random forests of every depth, against the oracle
(trees.py:174-223 restated in oracle/bart_oracle.py): traversal bit-exact,
predictions bit-exact (f64, trees in ascending order).  The shapes cross the
fused evaluation's chunk boundaries (64 trees per leaf chunk at D=6, 16 at
D=8, 1024 at D=1), include trees without any split, axes above 255, point
counts that are not a multiple of the per-thread vector, and forests whose
every tree is full to max depth."""

import numpy as np
import pytest

from oracle.bart_oracle import sum_leaf_values as oracle_sum, traverse_forest as oracle_traverse

pytestmark = pytest.mark.gpu


def random_forest(rng, m, D, p, max_cut, q):
    """Well-formed heap trees: node t splits with probability q if its parent split."""
    from paper_2410_23244_b200.trees import Forest
    half = 1 << (D - 1)
    axis = np.zeros((m, half), np.uint16)
    cut = np.zeros((m, half), np.uint8)
    for j in range(m):
        for t in range(1, half):
            if (t == 1 or cut[j, t // 2] > 0) and rng.random() < q:
                cut[j, t] = rng.integers(1, max_cut + 1)
                axis[j, t] = rng.integers(0, p)
    leaf = rng.normal(size=(m, 2 * half)).astype(np.float32)
    return Forest(axis, cut, leaf, D)


CASES = [  # (D, m, n, p, q)
    (1, 1100, 777, 3, 0.0),
    (2, 9, 1, 5, 0.7),
    (3, 70, 5003, 300, 0.7),
    (6, 150, 5003, 300, 0.6),
    (6, 64, 4096, 20, 1.0),
    (6, 129, 37, 20, 0.0),
    (7, 40, 2049, 9, 0.8),
    (8, 33, 1031, 400, 0.9),
]


@pytest.mark.parametrize("D,m,n,p,q", CASES)
def test_random_forests_match_oracle(D, m, n, p, q):
    from paper_2410_23244_b200.trees import evaluate_forest, evaluate_forests, sum_leaf_values, traverse_forest
    rng = np.random.default_rng(1000 * D + m)
    X = rng.integers(0, 31, (n, p)).astype(np.uint8)
    f = random_forest(rng, m, D, p, 30, q)
    Lt = oracle_traverse(f.axis, f.cutpoint, D, np.ascontiguousarray(X.T))
    want = oracle_sum(f.leaf_value, Lt)
    np.testing.assert_array_equal(traverse_forest(f, X), Lt.T)
    np.testing.assert_array_equal(sum_leaf_values(f.leaf_value, Lt.T), want)
    np.testing.assert_array_equal(evaluate_forest(f, X), want)
    g = random_forest(rng, m, D, p, 30, q)
    got = evaluate_forests([f, g], X)
    np.testing.assert_array_equal(got[0], want)
    np.testing.assert_array_equal(got[1], oracle_sum(g.leaf_value, oracle_traverse(g.axis, g.cutpoint, D,
                                                                                      np.ascontiguousarray(X.T))))
