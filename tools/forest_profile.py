"""Forest kernels (traverse / cached predict / fused evaluate) on a burned-in
n=1e6 p=100 m=200 chain: per-launch CUDA-event times (bart_profile_forest).
Used under ncu for the forest-kernel captures in profiles/.

usage: python tools/forest_profile.py [burn] [reps]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_23244_b200 import _native as N  # noqa: E402
from paper_2410_23244_b200.dgp import friedman1_binned  # noqa: E402
from paper_2410_23244_b200.regression import FitConfig, derive_hyperparams  # noqa: E402
from paper_2410_23244_b200.sampler import DeviceRNG, init_state, run  # noqa: E402

burn = int(sys.argv[1]) if len(sys.argv) > 1 else 200
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
Xq, y, _, grid = friedman1_binned(1_000_000, 100, seed=0)
hp, ys = derive_hyperparams(y, FitConfig(n_trees=200))
st = init_state(Xq, grid.counts, ys.forward(y).astype(np.float32), hp, DeviceRNG(1000))
run(st, hp, burn)
st.sync()
ms = np.zeros(3, np.float32)
N.check(N.lib().bart_profile_forest(st.handle, reps, N.ptr(ms)))
print(f"burn {burn}: traverse {ms[0]*1e3:.1f} us  predict_cached {ms[1]*1e3:.1f} us  evaluate {ms[2]*1e3:.1f} us")
