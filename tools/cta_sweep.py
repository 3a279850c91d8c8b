"""One chain's rate against its CTA count (bart_create_ex max_ctas).

usage: python tools/cta_sweep.py [n] [caps...]
"""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_23244_b200 import _native as N
from paper_2410_23244_b200.dgp import friedman1_binned
from paper_2410_23244_b200.regression import FitConfig, derive_hyperparams
from paper_2410_23244_b200.sampler import DeviceRNG, init_state, run

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000
caps = [int(c) for c in sys.argv[2:]] or [0, 16, 32, 48, 64, 98]
Xq, y, _, grid = friedman1_binned(n, 100, seed=0)
hp, ys = derive_hyperparams(y, FitConfig(n_trees=200))
y32 = ys.forward(y).astype(np.float32)
for cap in caps:
    st = init_state(Xq, grid.counts, y32, hp, DeviceRNG(7), max_ctas=cap)
    run(st, hp, 5)
    st.sync()
    ms = np.zeros(1, np.float32)
    N.check(N.lib().bart_run_timed(st.handle, 200, N.ptr(ms)))
    cfg = st.sweep_config()
    print(f"n={n} cap={cap:4d} ctas={cfg['ctas']:4d} chunk={cfg['chunk']:6d} stream={cfg['stream']}: "
          f"{200 / (ms[0] / 1e3):8.1f} it/s", flush=True)
    st.close()
