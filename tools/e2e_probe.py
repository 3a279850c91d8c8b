import os, sys, time
import numpy as np
sys.path.insert(0, os.getcwd())
from paper_2410_23244_b200 import _native as N
from paper_2410_23244_b200.dgp import friedman1_binned
from paper_2410_23244_b200.regression import FitConfig, derive_hyperparams
from paper_2410_23244_b200.sampler import DeviceRNG, StepRandoms, init_state, run, step
n = 1_000_000
Xq, y, _, grid = friedman1_binned(n, 100, seed=0)
hp, ys = derive_hyperparams(y, FitConfig(n_trees=200))
st = init_state(Xq, grid.counts, ys.forward(y).astype(np.float32), hp, DeviceRNG(5))
run(st, hp, 200); st.sync()
rng = np.random.default_rng(0)
m, size = hp.n_trees, 64
K = 50
pre = [StepRandoms.draw(rng, m, size, hp.nu + n) for _ in range(K * 6)]
it = iter(pre)
def timed(f, k=K):
    st.sync(); t0 = time.perf_counter()
    for _ in range(k): f()
    st.sync(); return (time.perf_counter() - t0) / k * 1e6
print("device run(1) x K        ", round(timed(lambda: run(st, hp, 1))))
print("device run(K) once       ", round(timed(lambda: run(st, hp, K), 1) / K))
print("step(randoms) x K        ", round(timed(lambda: step(st, hp, randoms=next(it)))))
print("step(randoms)+sync x K   ", round(timed(lambda: (step(st, hp, randoms=next(it)), st.sync()))))
print("step(None=device) x K    ", round(timed(lambda: step(st, hp, rng=DeviceRNG(1)) if False else N.check(N.lib().bart_step(st.handle, None)))))
print("step(randoms) x K again  ", round(timed(lambda: step(st, hp, randoms=next(it)))))
print("device run(1) x K again  ", round(timed(lambda: run(st, hp, 1))))
