"""Injected-randoms vs device-RNG step kernels, alternating on one burned-in
chain: run under ncu --metrics gpu__time_duration.sum to compare per-launch
durations (the e2e path injects; bench's value uses device randoms).

usage: python tools/inject_vs_device.py [burn] [pairs]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_23244_b200 import _native as N  # noqa: E402
from paper_2410_23244_b200.dgp import friedman1_binned  # noqa: E402
from paper_2410_23244_b200.regression import FitConfig, derive_hyperparams  # noqa: E402
from paper_2410_23244_b200.sampler import DeviceRNG, StepRandoms, init_state, run, step  # noqa: E402

burn = int(sys.argv[1]) if len(sys.argv) > 1 else 200
pairs = int(sys.argv[2]) if len(sys.argv) > 2 else 10
Xq, y, _, grid = friedman1_binned(1_000_000, 100, seed=0)
hp, ys = derive_hyperparams(y, FitConfig(n_trees=200))
st = init_state(Xq, grid.counts, ys.forward(y).astype(np.float32), hp, DeviceRNG(5))
run(st, hp, burn)
st.sync()
rng = np.random.default_rng(0)
for _ in range(pairs):
    step(st, hp, randoms=StepRandoms.draw(rng, 200, 64, hp.nu + 1_000_000))
    st.sync()
    N.check(N.lib().bart_step(st.handle, None))
    st._after_step()
    st.sync()
print("done")
