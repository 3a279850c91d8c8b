"""Host-side timing of bench.py's e2e loop (n=1e6, p=100, m=200, steady
state): per iteration, the StepRandoms draw, the step() call (stage write +
graph launch) and the wait for the previous step's result.

usage: python tools/e2e_timing.py [steps]
"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_23244_b200.dgp import friedman1_binned  # noqa: E402
from paper_2410_23244_b200.regression import FitConfig, derive_hyperparams  # noqa: E402
from paper_2410_23244_b200.sampler import DeviceRNG, StepRandoms, init_state, run, step  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 100
Xq, y, _, grid = friedman1_binned(1_000_000, 100, seed=0)
hp, ys = derive_hyperparams(y, FitConfig(n_trees=200))
st = init_state(Xq, grid.counts, ys.forward(y).astype(np.float32), hp, DeviceRNG(1000))
run(st, hp, 200)
st.sync()
rng = np.random.default_rng(0)
m, size, df = 200, 64, hp.nu + 1_000_000
for _ in range(3):
    step(st, hp, rng=rng)
st.step_result()
t_draw, t_call, t_wait = [], [], []
t0 = time.perf_counter()
for k in range(K):
    a = time.perf_counter()
    rnd = StepRandoms.draw(rng, m, size, df)
    b = time.perf_counter()
    step(st, hp, randoms=rnd)
    c = time.perf_counter()
    st.step_result(st.iteration - 2)
    d = time.perf_counter()
    t_draw.append(b - a)
    t_call.append(c - b)
    t_wait.append(d - c)
st.step_result()
tot = time.perf_counter() - t0
f = lambda v: f"{np.median(v) * 1e6:6.0f} us (mean {np.mean(v) * 1e6:6.0f})"
print(f"e2e loop: {tot / K * 1e6:.0f} us per step ({K / tot:.0f} it/s)")
print(f"  StepRandoms.draw  {f(t_draw)}")
print(f"  step() call       {f(t_call)}")
print(f"  wait for k-1      {f(t_wait)}")
