import sys, os, numpy as np
sys.path.insert(0, os.getcwd())
from paper_2410_23244_b200.sampler import Hyperparams, StepRandoms, init_state, step, DeviceRNG, run
from paper_2410_23244_b200 import trees
rng = np.random.default_rng(3)
n, p, m = 3001, 4, 8
X = rng.integers(0, 9, (n, p)).astype(np.uint8)
y = rng.normal(size=n).astype(np.float32)
hp = Hyperparams(leaf_sd=0.3, lam=0.1, n_trees=m, max_depth=5)
st = init_state(X, np.full(p, 8), y, hp, None, sigma2=1.0)
for _ in range(3):
    step(st, hp, randoms=StepRandoms.draw(rng, m, 32, hp.nu + n))
st.sync(); print("steps ok", st.last_accepted.sum())
f = st.forest
L = trees.traverse_forest(f, X); print("traverse ok", L.shape)
print("pred", st.resid[:3])
st.close()
st2 = init_state(X, np.full(p, 8), y, hp, DeviceRNG(1))
run(st2, hp, 3); st2.sync(); print("run ok"); st2.close()
