import sys, os, numpy as np
sys.path.insert(0, os.getcwd())
from paper_2410_23244_b200 import _native as N
from paper_2410_23244_b200.sampler import DeviceRNG, init_state, run
from paper_2410_23244_b200.regression import FitConfig, derive_hyperparams
n, p, m = 1_000_000, 100, 200
rng = np.random.default_rng(0)
Xq = rng.integers(0, 101, (n, p), dtype=np.uint8)
y = 10 * np.sin(np.pi * Xq[:, 0] * Xq[:, 1] / 1e4) + 20 * (Xq[:, 2] / 100 - .5) ** 2 + 10 * Xq[:, 3] / 100 + rng.normal(size=n)
hp, ys = derive_hyperparams(y, FitConfig(n_trees=m))
st = init_state(Xq, np.full(p, 100), ys.forward(y).astype(np.float32), hp, DeviceRNG(1))
for it in [20, 100, 300]:
    run(st, hp, it if it == 20 else it - (20 if it == 100 else 100)); st.sync()
    rows = np.zeros((12, m), np.int64); sl = np.zeros(m)
    N.check(N.lib().bart_get_proposals(st.handle, N.ptr(rows), N.ptr(sl)))
    ax = np.zeros((m, 32), np.uint16); cut = np.zeros((m, 32), np.uint8); lv = np.zeros((m, 64), np.float32)
    N.check(N.lib().bart_get_forest(st.handle, N.ptr(ax), N.ptr(cut), N.ptr(lv)))
    # leaves: nodes present whose children are absent; a node h is internal iff cut/axis set?  count via cutpoint>0
    internal = (cut > 0)
    leaves = internal.sum(1) + 1
    print("iter", it, "leaves per tree hist", np.bincount(leaves)[1:12], "mean", leaves.mean())
