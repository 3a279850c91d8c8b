"""Multi-chain batching: C chains of n points on one GPU,
each on its own stream, with and without splitting the SMs between them.

usage: python tools/multichain_bench.py [n] [chains] [iters]
Prints chain-iterations per second for: one chain alone (all SMs), the C
chains sharing the GPU unsplit (their cooperative sweeps take turns), and the
C chains each limited to SMs // C (they run side by side).
"""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_23244_b200 import _native as N
from paper_2410_23244_b200.dgp import friedman1_binned
from paper_2410_23244_b200.regression import FitConfig, derive_hyperparams
from paper_2410_23244_b200.sampler import DeviceRNG, init_state, run

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 100_000
C = int(sys.argv[2]) if len(sys.argv) > 2 else 4
iters = int(sys.argv[3]) if len(sys.argv) > 3 else 200
Xq, y, _, grid = friedman1_binned(n, 10, seed=0)
hp, ys = derive_hyperparams(y, FitConfig(n_trees=200))
y32 = ys.forward(y).astype(np.float32)
sms = N.lib().bart_device_sms(0)


def chains(k, cap):
    sts = [init_state(Xq, grid.counts, y32, hp, DeviceRNG(100 + i), max_ctas=cap) for i in range(k)]
    for st in sts:  # warm-up: graph capture, first launches
        run(st, hp, 5)
    for st in sts:
        st.sync()
    t0 = time.perf_counter()
    for st in sts:
        run(st, hp, iters)
    for st in sts:
        st.sync()
    dt = time.perf_counter() - t0
    cfg = sts[0].sweep_config()
    for st in sts:
        st.close()
    return k * iters / dt, cfg


one, c1 = chains(1, 0)
print(f"n={n} chains={C} sms={sms} iters={iters}")
print(f"one chain, all SMs          : {one:9.1f} chain-it/s  ({c1['ctas']} CTAs, stream={c1['stream']})")
tog, c2 = chains(C, 0)
print(f"{C} chains, unsplit           : {tog:9.1f} chain-it/s  ({c2['ctas']} CTAs each)")
cap = max(1, sms // C)
split, c3 = chains(C, cap)
print(f"{C} chains, {cap} SMs each       : {split:9.1f} chain-it/s  ({c3['ctas']} CTAs each, stream={c3['stream']})")
print(f"speed-up of splitting over taking turns: {split / tog:.2f}x")
