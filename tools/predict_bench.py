"""regression.predict's device work: F posterior forests evaluated on new rows
(trees.evaluate_forests -> bart_evaluate_many), wall time incl. transfers.

usage: python tools/predict_bench.py [n_new] [forests] [trees]
"""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_23244_b200.dgp import friedman1_binned
from paper_2410_23244_b200.regression import FitConfig, derive_hyperparams
from paper_2410_23244_b200.sampler import DeviceRNG, init_state, run
from paper_2410_23244_b200 import trees

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000
F = int(sys.argv[2]) if len(sys.argv) > 2 else 200
m = int(sys.argv[3]) if len(sys.argv) > 3 else 200
Xq, y, _, grid = friedman1_binned(n, 100, seed=0)
hp, ys = derive_hyperparams(y, FitConfig(n_trees=m))
st = init_state(Xq, grid.counts, ys.forward(y).astype(np.float32), hp, DeviceRNG(3))
forests = []
for k in range(F):  # distinct forests along the chain
    run(st, hp, 1)
    forests.append(st.forest)
st.close()
trees.evaluate_forests(forests[:2], Xq[:1000])  # warm-up
t0 = time.perf_counter()
out = trees.evaluate_forests(forests, Xq)
dt = time.perf_counter() - t0
ref = trees.evaluate_forests(forests[-1:], Xq)
assert np.array_equal(out[-1], ref[0])
print(f"evaluate_forests: {F} forests x {m} trees on n={n}: {dt * 1e3:.1f} ms "
      f"({dt / F * 1e3:.3f} ms per forest, output {out.nbytes / 1e6:.0f} MB)")
