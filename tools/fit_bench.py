"""Wall time of regression.fit on BASELINE configs[0] (gbart Friedman n=1000,
p=10, ntree=50, ndpost=100, nskip=100): the reference's own CPU fit took 3.1 s
for one chain here.

usage: python tools/fit_bench.py [n] [p] [m] [chains]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_23244_b200.dgp import friedman1
from paper_2410_23244_b200.regression import FitConfig, fit

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1000
p = int(sys.argv[2]) if len(sys.argv) > 2 else 10
m = int(sys.argv[3]) if len(sys.argv) > 3 else 50
chains = int(sys.argv[4]) if len(sys.argv) > 4 else 1
X, y, f = friedman1(n, p, seed=0)
for trace in ("device", "host"):
    cfg = FitConfig(n_trees=m, n_burn=100, n_kept=100, n_chains=chains, trace=trace, keep_forests=False)
    fit(X, y, cfg)  # warm-up (build, context, graph capture)
    t0 = time.perf_counter()
    tr = fit(X, y, cfg)
    dt = time.perf_counter() - t0
    rmse = float(np.sqrt(np.mean((tr.yhat_train_mean.mean(axis=0) - f) ** 2)))
    print(f"fit n={n} p={p} m={m} chains={chains} trace={trace}: {dt:.3f} s "
          f"({chains * 200 / dt:.0f} chain-iterations/s), rmse vs f {rmse:.3f}")
