"""Step rate and tree size along one chain (n=1e6, p=100, m=200, device RNG):
how far the bench's 200-iteration burn-in is from a longer-run steady state.

usage: python tools/drift.py [iterations]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_23244_b200 import _native as N  # noqa: E402
from paper_2410_23244_b200.dgp import friedman1_binned  # noqa: E402
from paper_2410_23244_b200.regression import FitConfig, derive_hyperparams  # noqa: E402
from paper_2410_23244_b200.sampler import DeviceRNG, init_state, run  # noqa: E402

total = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
Xq, y, _, grid = friedman1_binned(1_000_000, 100, seed=0)
hp, ys = derive_hyperparams(y, FitConfig(n_trees=200))
st = init_state(Xq, grid.counts, ys.forward(y).astype(np.float32), hp, DeviceRNG(1000))
done = 0
for upto in (5, 25, 100, 200, 300, 500, 1000, 1500, 2000, 3000, 5000):
    if upto > total:
        break
    run(st, hp, upto - done)
    done = upto
    ms = C = None
    import ctypes as C
    ms = C.c_float()
    N.check(N.lib().bart_run_timed(st.handle, 50, C.byref(ms)))
    done += 50
    leaves = ((st.forest.cutpoint > 0).sum(axis=1) + 1).mean()
    print(f"after {upto:5d} iterations: {50e3 / ms.value:7.1f} it/s over the next 50, mean leaves {leaves:.3f}", flush=True)
