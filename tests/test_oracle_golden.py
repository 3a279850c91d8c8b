"""Pin the CPU oracle against golden vectors produced by the real reference.

Every hot-path quantity must be bit-identical: proposals (sampler.py:469-526),
post-refresh counts (:894-897), tree-excluded sums (:556-576), accept
decisions, forests, leaf-index caches, residuals and sigma2 (:878-912).
"""

import numpy as np
import pytest

from golden_io import STEP_CASES, load_case
from oracle.bart_oracle import OracleChain, traverse_forest, sum_leaf_values

PROP_FIELDS = [("kind", "kind"), ("node", "node"), ("axis_p", "axis"), ("cut_p", "cut"),
               ("depth_p", "depth"), ("n_axes", "n_axes"), ("n_splits", "n_splits"),
               ("w_small", "w_small"), ("w_prime_big", "w_prime_big"),
               ("growable_big", "growable_big"), ("gl", "gl"), ("gr", "gr")]


def chain_from(d):
    return OracleChain(d["X"], d["max_cuts"], d["y"], d["hpns"], sigma2=float(d["sigma2_0"]),
                       axis=d["axis0"], cut=d["cutpoint0"], leaf=d["leaf_value0"],
                       resid=d["resid0"], leaf_index=d["leaf_index0"])


@pytest.mark.parametrize("case", STEP_CASES)
def test_oracle_replays_reference_bit_exact(case):
    d = load_case(case)
    ch = chain_from(d)
    for s in range(d["steps"]):
        taps = {}
        ch.step(d["move_u"][s], d["accept_u"][s], d["leaf_z"][s], float(d["chi2"][s]), taps)
        props = taps["props"]
        for gk, ok in PROP_FIELDS:
            np.testing.assert_array_equal(getattr(props, ok), d[gk][s], err_msg=f"{case} step {s} {gk}")
        np.testing.assert_allclose(props.struct_log, d["struct_log"][s], rtol=1e-14, atol=1e-15)
        np.testing.assert_array_equal(taps["counts"], d["counts"][s])
        np.testing.assert_array_equal(taps["sums"], d["sums"][s])
        np.testing.assert_array_equal(ch.last_accepted, d["accepted"][s])
        np.testing.assert_array_equal(ch.axis, d["axis"][s])
        np.testing.assert_array_equal(ch.cut, d["cutpoint"][s])
        np.testing.assert_array_equal(ch.leaf, d["leaf_value"][s])
        np.testing.assert_array_equal(ch.leaf_index, d["leaf_index"][s])
        np.testing.assert_array_equal(ch.resid, d["resid"][s])
        assert ch.sigma2 == float(d["sigma2"][s])


@pytest.mark.parametrize("case", STEP_CASES)
def test_oracle_traversal_and_prediction(case):
    d = load_case(case)
    D = int(d["hpns"].max_depth)
    Xt = np.ascontiguousarray(d["X"].T)
    L = traverse_forest(d["axis"][-1], d["cutpoint"][-1], D, Xt)
    np.testing.assert_array_equal(L.T, d["leaf_index"][-1])
    np.testing.assert_array_equal(sum_leaf_values(d["leaf_value"][-1], L), d["yhat"])
