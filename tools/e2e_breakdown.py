"""Where the end-to-end step time goes (bench.py's e2e path) at the bench workload.

usage: python tools/e2e_breakdown.py [n] [steps]
"""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_23244_b200.dgp import friedman1_binned
from paper_2410_23244_b200.regression import FitConfig, derive_hyperparams
from paper_2410_23244_b200.sampler import DeviceRNG, StepRandoms, init_state, run, step

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000
K = int(sys.argv[2]) if len(sys.argv) > 2 else 100
Xq, y, _, grid = friedman1_binned(n, 100, seed=0)
hp, ys = derive_hyperparams(y, FitConfig(n_trees=200))
st = init_state(Xq, grid.counts, ys.forward(y).astype(np.float32), hp, DeviceRNG(5))
run(st, hp, 20)
st.sync()
rng = np.random.default_rng(0)
m, size = hp.n_trees, 1 << hp.max_depth


def timed(f):
    t0 = time.perf_counter()
    for _ in range(K):
        f()
    st.sync()
    return (time.perf_counter() - t0) / K * 1e6


pre = [StepRandoms.draw(rng, m, size, hp.nu + n) for _ in range(K)]
it = iter(pre * 2)
t_draw = timed(lambda: StepRandoms.draw(rng, m, size, hp.nu + n))
t_dev = timed(lambda: run(st, hp, 1))
t_step = timed(lambda: step(st, hp, randoms=next(it)))
def full():
    step(st, hp, rng=rng)
    _ = st.last_accepted
    _ = st.sigma2
t_full = timed(full)
def reads():
    _ = st._fetch("last_accepted"); st._cache.clear()
t_reads = timed(lambda: (st._cache.clear(), st.last_accepted, st.sigma2))
print(f"n={n}: per step (us): host StepRandoms.draw {t_draw:.0f} | device step (graph, device RNG) {t_dev:.0f} | "
      f"step(randoms) {t_step:.0f} | full e2e {t_full:.0f} | accepted+sigma2 reads {t_reads:.0f}")


def pipelined():  # bench.py's e2e loop: read step k-1 after launching step k
    step(st, hp, rng=rng)
    if st.iteration >= 2:
        st.step_result(st.iteration - 2)


t_pipe = timed(pipelined)
def host_only():  # the host's share of one pipelined iteration, device work excluded
    t0 = time.perf_counter()
    StepRandoms.draw(rng, m, size, hp.nu + n)
    return time.perf_counter() - t0
print(f"pipelined e2e loop {t_pipe:.0f} us per step (device step {t_dev:.0f} us)")
