"""The step kernel with its exchange split into G copy groups (one-device
emulation of G n-shards, bart_set_copy_groups), flat vs two-level exchange
(bart_set_exchange): per-iteration time at steady state.  The groups share
one GPU's 148 CTAs, so this measures the protocols' on-chip cost (arrivals,
the forwarder hop), not NVLink.

usage: python tools/exchange_emulation.py [n] [burn] [steps]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_23244_b200 import _native as N  # noqa: E402
from paper_2410_23244_b200.dgp import friedman1_binned  # noqa: E402
from paper_2410_23244_b200.regression import FitConfig, derive_hyperparams  # noqa: E402
from paper_2410_23244_b200.sampler import DeviceRNG, init_state, run  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000
burn = int(sys.argv[2]) if len(sys.argv) > 2 else 200
steps = int(sys.argv[3]) if len(sys.argv) > 3 else 50
Xq, y, _, grid = friedman1_binned(n, 100, seed=0)
hp, ys = derive_hyperparams(y, FitConfig(n_trees=200))
y32 = ys.forward(y).astype(np.float32)
print(f"n={n} p=100 m=200, burn {burn}, {steps} timed steps; ms per iteration (us per tree)")
for groups in (1, 2, 4, 8):
    row = []
    for mode in ("flat", "two_level"):
        st = init_state(Xq, grid.counts, y32, hp, DeviceRNG(1000))
        if groups > 1:
            st.set_copy_groups(groups)
        st.set_exchange(mode)
        run(st, hp, burn)
        st.sync()
        ms = np.zeros(1, np.float32)
        N.check(N.lib().bart_run_timed(st.handle, steps, N.ptr(ms)))
        st._after_step(steps)
        per = float(ms[0]) / steps
        row.append(f"{mode:9s} {per:.4f} ms ({per / 200 * 1e3:.2f} us)")
        st.close()
    print(f"  groups {groups}: " + "   ".join(row), flush=True)
