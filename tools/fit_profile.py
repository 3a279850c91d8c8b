"""Where regression.fit's wall time goes at n=1e6 (host-side cProfile, one chain,
device trace): setup, sampling, kept-draw readback.

usage: python tools/fit_profile.py [n] [chains]
"""
import cProfile
import os
import pstats
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_23244_b200.dgp import friedman1  # noqa: E402
from paper_2410_23244_b200.regression import FitConfig, fit  # noqa: E402

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000
chains = int(sys.argv[2]) if len(sys.argv) > 2 else 1
X, y, f = friedman1(n, 100, seed=0)
cfg = FitConfig(n_trees=200, n_burn=100, n_kept=100, n_chains=chains, keep_forests=False)
fit(X[:2000], y[:2000], cfg)  # warm-up: context, build
t0 = time.perf_counter()
pr = cProfile.Profile()
pr.enable()
tr = fit(X, y, cfg)
pr.disable()
print(f"fit n={n} chains={chains}: {time.perf_counter() - t0:.3f} s")
pstats.Stats(pr).sort_stats("cumulative").print_stats(30)
