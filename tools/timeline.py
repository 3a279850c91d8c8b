"""Per-phase breakdown of the sweep kernel from on-device clock64 stamps.

usage: python tools/timeline.py [n] [p] [m]
"""
import sys, os, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_23244_b200 import _build, _native as N
from paper_2410_23244_b200.sampler import DeviceRNG, init_state, run
from paper_2410_23244_b200.regression import FitConfig, derive_hyperparams

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000
p = int(sys.argv[2]) if len(sys.argv) > 2 else 100
m = int(sys.argv[3]) if len(sys.argv) > 3 else 200
_build.build()
rng = np.random.default_rng(0)
Xq = rng.integers(0, 101, (n, p), dtype=np.uint8)
y = 10 * np.sin(np.pi * Xq[:, 0] * Xq[:, 1] / 1e4) + 20 * (Xq[:, 2] / 100 - .5) ** 2 + 10 * Xq[:, 3] / 100 + rng.normal(size=n)
hp, ys = derive_hyperparams(y, FitConfig(n_trees=m))
st = init_state(Xq, np.full(p, 100), ys.forward(y).astype(np.float32), hp, DeviceRNG(1))
run(st, hp, 20); st.sync()
N.check(N.lib().bart_set_timeline(st.handle, 1))
ms = np.zeros(3, np.float32)
N.check(N.lib().bart_profile(st.handle, 3, N.ptr(ms)))
tl = np.zeros((3, m + 1, 8), np.int64)
N.check(N.lib().bart_get_timeline(st.handle, N.ptr(tl)))
print(f"n={n} p={p} m={m} sweep {ms[1]/3:.3f} ms/launch, {ms[1]/3/m*1e3:.2f} us/tree; cfg {st.sweep_config()}")
names = ["wait_data", "pass", "sync+exchange+decide"]
for c, lab in ((0, "CTA0"), (1, "CTAlast")):
    t = tl[c]
    d = np.diff(t[:m, :4], axis=1)          # phases within tree
    nxt = t[1:m + 1, 0] - t[:m, 3]           # end -> next start
    med = np.median(d, axis=0)
    print(lab, " ".join(f"{nm}={v:.0f}" for nm, v in zip(names, med)), f"loop={np.median(nxt):.0f}",
          f"total/tree={np.median(t[1:m+1,0]-t[:m,0]):.0f} cyc")
    print("   p90:", " ".join(f"{nm}={v:.0f}" for nm, v in zip(names, np.percentile(d, 90, axis=0))))
dd = np.diff(tl[2, :m, :4], axis=1)
print("control warp CTA0 (cyc):", *[f"{v:.0f}" for v in np.median(dd, axis=0)], "[exchange, decide, prepare+post]")
nb = st.sweep_config()["ctas"]
tr = np.zeros((m + 1, nb, 2), np.int64)
N.check(N.lib().bart_get_trace(st.handle, N.ptr(tr)))
done = tr[:m, :, 1].astype(float)
spread = done.max(1) - done.min(1)
period = np.diff(done.max(1))
q = lambda a: f"median {np.median(a):.0f} p90 {np.percentile(a, 90):.0f} ns"
print("control-done spread over CTAs:", q(spread))
print("tree period:", q(period))
st.close()
