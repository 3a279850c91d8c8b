"""Per-phase breakdown of the sweep kernel from on-device clock64 stamps (CTA 0, cycles).

usage: python tools/timeline.py [n] [p] [m]
Worker thread 0: A start, A published, B done, decision received.
Control lane 0: partials synced, exchange complete, decision published; helper: next tree prepared.
"""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2410_23244_b200 import _build
os.environ["BART_LIB"] = _build.build_timeline(tuple(os.environ.get("BART_TL_DEFINES", "").split()))  # instrumented variant
from paper_2410_23244_b200 import _native as N
from paper_2410_23244_b200.sampler import DeviceRNG, init_state, run
from paper_2410_23244_b200.regression import FitConfig, derive_hyperparams

n = int(float(sys.argv[1])) if len(sys.argv) > 1 else 1_000_000
p = int(sys.argv[2]) if len(sys.argv) > 2 else 100
m = int(sys.argv[3]) if len(sys.argv) > 3 else 200
rng = np.random.default_rng(0)
Xq = rng.integers(0, 101, (n, p), dtype=np.uint8)
y = 10 * np.sin(np.pi * Xq[:, 0] * Xq[:, 1] / 1e4) + 20 * (Xq[:, 2] / 100 - .5) ** 2 + 10 * Xq[:, 3] / 100 + rng.normal(size=n)
hp, ys = derive_hyperparams(y, FitConfig(n_trees=m))
st = init_state(Xq, np.full(p, 100), ys.forward(y).astype(np.float32), hp, DeviceRNG(1))
burn = int(os.environ.get("BART_TL_BURN", "20"))
run(st, hp, burn); st.sync()
lv = (st.forest.cutpoint > 0).sum(axis=1) + 1
print(f"burn-in {burn} iterations: mean leaves/tree {lv.mean():.2f}, max {lv.max()}")
N.check(N.lib().bart_set_timeline(st.handle, 1))
ms = np.zeros(3, np.float32)
N.check(N.lib().bart_profile(st.handle, 3, N.ptr(ms)))
tl = np.zeros((4, m + 2, 8), np.int64)
N.check(N.lib().bart_get_timeline(st.handle, N.ptr(tl)))
print(f"n={n} p={p} m={m} sweep {ms[1]/3:.3f} ms/launch, {ms[1]/3/m*1e3:.2f} us/tree, propose {ms[2]/3*1e3:.1f} us; cfg {st.sweep_config()}")
t = tl.reshape(-1)[: (m + 2) * 32].reshape(m + 2, 32)[1:m + 1].astype(float)  # rows: trees 0..m-1
q = lambda a: f"{np.median(a):6.0f} (p90 {np.percentile(a, 90):6.0f})"
print("worker  A pass                ", q(t[:, 1] - t[:, 0]))
print("worker  B pass                ", q(t[:, 2] - t[:, 1]))
print("worker0 published -> fold done", q(t[:, 14] - t[:, 1]))
print("fold -> limbs                 ", q(t[:, 15] - t[:, 14]))
print("limbs -> adds issued          ", q(t[:, 5] - t[:, 15]))
print("  limbs -> red issued          ", q(t[:, 30] - t[:, 15]))
print("  red issued -> add loop exit  ", q(t[:, 5] - t[:, 30]))
print("adds -> prep loaded           ", q(t[:, 6] - t[:, 5]))
print("prep -> poll complete         ", q(t[:, 7] - t[:, 6]))
print("poll -> totals (gather/limbs) ", q(t[:, 8] - t[:, 7]))
print("decide: poll -> accept known   ", q(t[:, 10] - t[:, 8]))
print("decide: deltas + arrive       ", q(t[:, 11] - t[:, 10]))
print("worker: decision->A start     ", q(t[:, 0][1:] - t[:, 11][:-1]))
print("  ctrl arrive -> worker sync ret", q(t[:, 3] - t[:, 11]))
print("  worker sync ret -> A start    ", q(t[:, 0][1:] - t[:, 3][:-1]))
print("  worker B done -> ctrl arrive  ", q(t[:, 11] - t[:, 2]))
wa = t[:, 16:24]
print("  A setup (flags, slots)       ", q(t[:, 26] - t[:, 0]))
print("  A word loop (update + sums)  ", q(t[:, 24] - t[:, 26]))
print("  A warp reductions            ", q(t[:, 25] - t[:, 24]))
print("  A reductions -> published    ", q(t[:, 1] - t[:, 25]))
print("A end spread over worker warps ", q(wa.max(1) - wa.min(1)))
print("A start -> last warp A end     ", q(wa.max(1) - t[:, 0]))
print("last warp A end -> ctrl synced ", q(t[:, 4] - wa.max(1)))
print("A end by warp (median rel. to first):", np.median(wa - wa.min(1, keepdims=True), axis=0).astype(int))
print("helper prepare(e+1) done      ", q(t[:, 13] - t[:, 12]))
print("tree period (cycles)          ", q(np.diff(t[:, 4])))
nb = st.sweep_config()["ctas"]
tr = np.zeros((m + 2, nb, 2), np.int64)
N.check(N.lib().bart_get_trace(st.handle, N.ptr(tr)))
pub = tr[1:m + 1, :, 0].astype(float)
done = tr[1:m + 1, :, 1].astype(float)
print("arrival skew (ns): last publish - first publish ", q(pub.max(1) - pub.min(1)))
print("detection jitter (ns): last done - first done  ", q(done.max(1) - done.min(1)))
print("exchange latency (ns): first done - last publish", q(done.min(1) - pub.max(1)))
late = np.argmax(pub, axis=1)
hist = np.bincount(late, minlength=nb)
top = hist.argsort()[::-1][:5]
print("latest publisher CTAs (top 5, share of trees):", [(int(c), round(float(hist[c]) / m, 2)) for c in top])
# per-CTA systematics (ns, averaged over trees): when it published relative to
# the first publisher; when it saw the exchange complete relative to the first
# CTA that did; and its own A-pass-to-publish time (publish e - done e-1)
lat_pub = (pub - pub.min(1, keepdims=True)).mean(0)
lat_done = (done - done.min(1, keepdims=True)).mean(0)
work = (pub[1:] - done[:-1]).mean(0)
order = lat_pub.argsort()[::-1]
print("per-CTA mean publish lateness (ns): max %.0f, median %.0f, min %.0f" % (lat_pub.max(), np.median(lat_pub), lat_pub.min()))
print("per-CTA mean detection lateness (ns): max %.0f, median %.0f, min %.0f" % (lat_done.max(), np.median(lat_done), lat_done.min()))
print("per-CTA done(e-1) -> publish(e) (ns): max %.0f, median %.0f, min %.0f" % (work.max(), np.median(work), work.min()))
print("latest 8 CTAs: publish lateness / detection lateness / A-to-publish (ns):")
for ci in order[:8]:
    print(f"  CTA {ci:3d}: {lat_pub[ci]:6.0f} / {lat_done[ci]:6.0f} / {work[ci]:6.0f}")
print("corr(publish lateness, detection lateness) = %.2f, corr(publish lateness, A-to-publish) = %.2f" % (
    np.corrcoef(lat_pub, lat_done)[0, 1], np.corrcoef(lat_pub, work)[0, 1]))
st.close()
