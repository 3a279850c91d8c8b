"""INTEGRATION.md §2's ctypes stub, executed as written.

The block is what a bforge maintainer would paste into bforge/sampler.py: it
binds include/bart_b200.h with ctypes against bforge's own SamplerState.
Here it runs against a bforge-shaped state (the attributes sampler.py:121-147
defines), with StepRandoms / depth_probabilities from this package's mirrors
of the reference's, and must reproduce paper_2410_23244_b200.sampler.step --
same random stream, so the same decisions and sigma2 -- step for step.
"""

import os
import re
from types import SimpleNamespace

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _stub_source() -> str:
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    section = text[text.index("## 2. Minimal ctypes stub"):text.index("## 3.")]
    return re.search(r"```python\n(.*?)```", section, re.S).group(1)


def test_integration_stub_reproduces_step():
    from paper_2410_23244_b200 import _native
    from paper_2410_23244_b200.dgp import friedman1
    from paper_2410_23244_b200.grid import build_grid_uniform, quantize
    from paper_2410_23244_b200.regression import FitConfig, derive_hyperparams
    from paper_2410_23244_b200.sampler import StepRandoms, depth_probabilities, init_state, step
    from paper_2410_23244_b200.trees import Forest

    ns = {"StepRandoms": StepRandoms, "depth_probabilities": depth_probabilities}
    exec(_stub_source().replace('"libbart_b200.so"', repr(_native.LIB)), ns)

    X, y, _ = friedman1(5000, 6, seed=12)
    g = build_grid_uniform(X, 50)
    Xq = quantize(X, g).data
    hp, ys = derive_hyperparams(y, FitConfig(n_trees=30))
    y32 = ys.forward(y).astype(np.float32)
    ours = init_state(Xq, g.counts, y32, hp, np.random.default_rng(5))
    m, D = hp.n_trees, hp.max_depth
    # what bforge's init_state leaves behind (sampler.py:201-241): root-only forest, L == 1, resid = y
    ref_state = SimpleNamespace(
        X=Xq, max_cuts=np.asarray(g.counts, np.int64), y=y32, resid=y32.copy(), sigma2=ours.sigma2,
        forest=Forest(np.zeros((m, 1 << (D - 1)), np.uint16), np.zeros((m, 1 << (D - 1)), np.uint8),
                      np.zeros((m, 1 << D), np.float32), D),
        leaf_index=np.ones((Xq.shape[0], m), np.uint8), rng=np.random.default_rng(5), n_points=Xq.shape[0],
        iteration=0, last_accepted=None)
    ns["attach_device"](ref_state, hp)
    for _ in range(4):
        ns["step"](ref_state, hp)
        step(ours, hp)
        np.testing.assert_array_equal(ref_state.last_accepted, ours.last_accepted)
        assert ref_state.sigma2 == ours.sigma2
    ours.close()
