#!/usr/bin/env python
"""Benchmark: BART MCMC iterations/s on B200 (BASELINE.json metric).

Workload (default, BASELINE configs[2], the metric's config): gbart on
synthetic Friedman #1 data, n=1e6, p=100, ntree=200, D=6, 100 uniform
cutpoints.  A "step" is one full MCMC iteration (propose + sequential sweep
over all 200 trees + sigma draw) on resident device state.  The chain is
burned in (--burn, default 2000 iterations; the reference's own protocol
warms up 3, bench.py:114-122) before the W warm-up and K timed steps, so the
number is a steady-state one: trees keep growing for ~1500 iterations
(mean leaves 2.3 after 5, 3.7 after 200, 4.5-4.6 from ~1500 on, where the
rate stops falling; tools/drift.py), reported as "trees" in the line.  The
fresh-chain rate (iterations 5..25) is reported beside it.

  value     iterations/s of CUDA-graph-replayed device-RNG steps, CUDA events
            on the chain's stream, max over ranks; inputs (X 100 MB, leaf
            index 200 MB) exceed the 126 MB L2, no flush needed.
  e2e       the same metric through the reference-facing call
            `step(state, hp, rng=numpy Generator)`: host StepRandoms draw
            into the pinned stage the kernel reads (zero-copy H2D), the step,
            and its accept flags + sigma2 read back (zero-copy D2H) every step.
  roofline  the sweep kernel: algorithmic bytes 10*n*m per launch (SURVEY.md
            §8d) / mean per-launch CUDA-event duration, vs measured HBM peak.
  cpu_baseline  the CPU oracle (numpy port of the reference, oracle/), one
            core, full workload (n, p, all 200 trees): 1 warm-up + 3 timed
            steps, median.

`--impl reference` times the CPU oracle port with all host cores
(independent chains, one per core, each running full 200-tree steps) on the
same workload and prints the same JSON line with "impl": "reference".
"""

from __future__ import annotations

import argparse
import json
import multiprocessing as mp
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "MCMC iters/sec at n=1e6,p=100,ntree=200 (1/2/4/8 B200) vs host CPU; HBM GB/s"
CPU_TIMED_STEPS = 3  # per chain, after one warm-up step: full-workload iterations
REF_MAX_STEPS = 8    # reference arm: timed steps actually run (each ~3 s at n=1e6)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--burn", type=int, default=2000,
                    help="iterations run before warm-up so the timed chain is at steady state")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", "--points", dest="n", type=int, default=1_000_000)  # --points: under torchrun (--n is ambiguous there)
    ap.add_argument("--p", type=int, default=100)
    ap.add_argument("--m", type=int, default=200)
    ap.add_argument("--depth", type=int, default=6)
    ap.add_argument("--e2e-steps", type=int, default=100)
    ap.add_argument("--cpu-steps", type=int, default=CPU_TIMED_STEPS)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--max-ctas", type=int, default=0, help="cap the sweep's CTAs (0: one per SM)")
    ap.add_argument("--shard", action="store_true",
                    help="N>1: shard ONE chain's points across the ranks (in-kernel NVLink exchange, strong "
                         "scaling; BASELINE configs[3] with --n 10000000) instead of independent replicas")
    return ap.parse_args()


def workload(args):
    from paper_2410_23244_b200.dgp import friedman1_binned
    from paper_2410_23244_b200.regression import FitConfig, derive_hyperparams

    Xq, y, _, grid = friedman1_binned(args.n, args.p, seed=args.seed)
    hp, ys = derive_hyperparams(y, FitConfig(n_trees=args.m, max_depth=args.depth))
    return Xq, grid.counts, ys.forward(y).astype(np.float32), hp


def baseline_config_label(args) -> str:
    """Which BASELINE.json config this workload is."""
    shape = (args.n, args.p, args.m)
    if shape == (100_000, 100, 200):
        return "BASELINE.json configs[1]"
    if shape == (1_000_000, 100, 200):
        return "BASELINE.json configs[2]"
    if shape == (10_000_000, 100, 200):
        return "BASELINE.json configs[3]"
    if shape == (1_000_000, 1000, 1000):
        return "BASELINE.json configs[4]"
    if shape == (1000, 10, 50):
        return "BASELINE.json configs[0] shape"
    return "not a BASELINE.json config"


def config_dict(args, parallelism):
    return {
        "workload": f"gbart Friedman#1 n={args.n:g} p={args.p} ntree={args.m} D={args.depth} "
                    f"({baseline_config_label(args)})",
        "n": args.n, "p": args.p, "ntree": args.m, "max_depth": args.depth, "n_cutpoints": 100,
        "parallelism": parallelism,
        "l2": "no flush: X (n*p B) + leaf index (n*m B) per iteration exceed the 126 MB L2",
    }


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu, self.rows, self._stop = gpu, [], threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0:
                    self.rows.append([x.strip() for x in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.1)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 2 + i and r[2 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def measured_peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def committed_traffic():
    """dram bytes per sweep launch from the committed ncu summary, if any."""
    try:
        with open(os.path.join(ROOT, "profiles", "sweep_ncu_summary.json")) as f:
            return json.load(f).get("dram_bytes_per_launch")
    except Exception:
        return None


# ---------------------------------------------------------------- CPU side
def _cpu_worker(args_tuple):
    """One CPU chain of the full workload: `warm` untimed then `steps` timed
    full iterations (all m trees) of the oracle port; per-step seconds."""
    Xq, max_cuts, y32, hp_fields, warm, steps, seed = args_tuple
    from types import SimpleNamespace

    from oracle.bart_oracle import OracleChain

    hp = SimpleNamespace(**hp_fields)
    m = hp.n_trees
    ch = OracleChain(Xq, max_cuts, y32, hp)
    rng = np.random.default_rng(seed)
    size = 1 << hp.max_depth
    times = []
    for s in range(warm + steps):
        u = rng.random((m, 5))
        acc = rng.random(m)
        z = rng.standard_normal((m, size))
        chi2 = float(rng.chisquare(hp.nu + y32.size))
        t0 = time.perf_counter()
        ch.step(u, acc, z, chi2)
        if s >= warm:
            times.append(time.perf_counter() - t0)
    return times


def _hp_fields(hp):
    return dict(leaf_sd=hp.leaf_sd, lam=hp.lam, n_trees=hp.n_trees, alpha=hp.alpha, beta=hp.beta,
                leaf_mean=hp.leaf_mean, nu=hp.nu, max_depth=hp.max_depth, p_grow=hp.p_grow,
                update_sigma=hp.update_sigma)


def cpu_oracle_times(Xq, max_cuts, y32, hp, warm, steps, procs=1):
    """Per-step seconds of `procs` concurrent oracle chains of the full
    workload (one process per chain), each `warm` + `steps` iterations."""
    job = (Xq, max_cuts, y32, _hp_fields(hp), warm, steps)
    if procs <= 1:
        return [_cpu_worker(job + (0,))]
    ctx = mp.get_context("fork")
    with ctx.Pool(procs) as pool:
        return pool.map(_cpu_worker, [job + (k,) for k in range(procs)])


def tree_stats(st) -> dict:
    """Leaves per tree of the chain's forest at the start of the timed region
    (a leaf-less heap slot has cutpoint 0: trees.py:174-203)."""
    f = st.forest
    leaves = (f.cutpoint > 0).sum(axis=1) + 1
    hist = np.bincount(leaves, minlength=leaves.max() + 1)
    return {"mean_leaves": float(leaves.mean()), "max_leaves": int(leaves.max()),
            "leaves_hist": {str(k): int(v) for k, v in enumerate(hist) if v},
            "iteration": int(st.iteration)}


# ---------------------------------------------------------------- GPU side
def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist

        ndev = max(1, torch.cuda.device_count())
        local = local % ndev  # one GPU per rank; several ranks per GPU only on a box with fewer GPUs
        torch.cuda.set_device(local)
        # the bench's collectives carry only timings (no data path); NCCL refuses
        # two ranks on one GPU, so ranks sharing GPUs use gloo
        backend = os.environ.get("BENCH_DIST_BACKEND", "nccl" if world <= ndev else "gloo")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return world, rank, local


def allreduce_max(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda" if dist.get_backend() == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(world: int):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def profile_forest_kernels(st, N, args, reps: int = 10) -> dict:
    """The reference's traverse_forest / sum_leaf_values / evaluate_forest
    kernels (trees.py:174-223) on the chain's current forest, per launch, with
    their algorithmic bytes: traverse reads each split column a tree uses once
    (n B per distinct axis) and writes the (m, n) u8 cache; the cached sum reads
    the cache and writes n f64; the fused one reads the columns and writes n f64."""
    ms = np.zeros(3, np.float32)
    N.check(N.lib().bart_profile_forest(st.handle, reps, N.ptr(ms)))
    f = st.forest
    n, m = args.n, args.m
    cols = sum(len(set(int(a) for a, c in zip(f.axis[j], f.cutpoint[j]) if c > 0)) for j in range(m))
    peak, _ = measured_peak()
    out = {}
    for k, (name, nbytes) in enumerate([("traverse", n * cols + n * m), ("predict_cached", n * m + 8 * n),
                                        ("evaluate", n * cols + 8 * n)]):
        gbs = nbytes / (float(ms[k]) / 1e3) / 1e9
        out[name] = {"ms": float(ms[k]), "algorithmic_bytes": nbytes, "achieved_gbs": gbs, "frac": gbs / peak}
    out["split_columns_in_forest"] = cols
    return out


def run_ours(args):
    world, rank, local = dist_setup(args)
    from paper_2410_23244_b200 import _build

    if rank == 0:
        _build.build()
    barrier(world)
    from paper_2410_23244_b200 import _native as N
    from paper_2410_23244_b200.sampler import DeviceRNG, init_state, run, step

    Xq, max_cuts, y32, hp = workload(args)
    sharded = args.shard and world > 1
    if sharded:
        # one chain: this rank holds a contiguous slice of the points; same
        # device seed everywhere, so every shard takes identical decisions
        from paper_2410_23244_b200.shard import ShardPlan, init_sharded_state, torch_all_gather
        plan = ShardPlan(args.n, world)
        lo, hi = plan.bounds(rank)
        st = init_sharded_state(Xq[lo:hi], max_cuts, y32[lo:hi], hp, DeviceRNG(1000), plan, rank,
                                float(np.var(y32, ddof=1)), torch_all_gather(), device=local)
    else:
        # replicas: every rank runs an independent chain of the full workload
        st = init_state(Xq, max_cuts, y32, hp, DeviceRNG(1000 + rank), device=local, max_ctas=args.max_ctas or None)
    cfg = st.sweep_config()
    # the round-1 protocol (5 warm-up, then 20 timed iterations of a fresh chain,
    # 1-2-leaf trees), kept for comparison; then on to steady state
    fresh = None
    if args.burn >= 25:
        run(st, hp, 5)
        ms_f = np.zeros(1, np.float32)
        N.check(N.lib().bart_run_timed(st.handle, 20, N.ptr(ms_f)))
        st._after_step(20)
        fresh_rate = 20 / (float(ms_f[0]) / 1e3)
        fresh = {"iters_per_s": fresh_rate, "iterations": "5..25",
                 "frac": 10.0 * args.n * args.m * fresh_rate / 1e9 / measured_peak()[0]}
        run(st, hp, args.burn - 25)
    else:
        run(st, hp, args.burn)  # to steady state (trees at posterior size)
    st.sync()
    trees = tree_stats(st)
    run(st, hp, args.warmup)
    st.sync()
    launches0 = st.kernel_launches()
    barrier(world)
    ms = np.zeros(1, np.float32)
    with ClockSampler(local) as clk:
        N.check(N.lib().bart_run_timed(st.handle, args.steps, N.ptr(ms)))
    gpu_launches = st.kernel_launches() - launches0
    st._after_step(args.steps)
    barrier(world)
    t_max = allreduce_max(float(ms[0]) / 1e3, world)
    value = (1 if sharded else world) * args.steps / t_max

    # per-kernel durations (events around each launch, not graph-replayed)
    # The step is ONE kernel launch (sweep_kernel: in-kernel proposals, the
    # sequential tree sweep, sigma), so its average launch duration is the
    # timed region's per-step time on this rank (CUDA events, graph replay).
    # Events around individual non-graph launches are reported beside it.
    prof = np.zeros(3, np.float32)
    kp = 10  # few: the chain keeps evolving, and the e2e leg that follows should see the timed trees
    N.check(N.lib().bart_profile(st.handle, kp, N.ptr(prof)))
    st._after_step(kp)
    sweep_ms = float(ms[0]) / args.steps
    single_launch_ms = float(prof[1]) / kp
    alg_bytes = 10.0 * args.n * args.m
    peak, peak_src = measured_peak()
    achieved = alg_bytes / (sweep_ms / 1e3) / 1e9

    # e2e through the reference-facing call with host random blocks
    rng = np.random.default_rng(0 if sharded else rank)  # shards must inject identical random blocks
    m, size = args.m, 1 << args.depth
    h2d = 8 * (5 * m + m + m * size) + 8
    d2h = m + 8
    barrier(world)
    for _ in range(2):  # warm-up: the step pipeline's buffers and both slots' captured launches
        step(st, hp, rng=rng)
    st.step_result()
    barrier(world)
    t0 = time.perf_counter()
    for k in range(args.e2e_steps):
        step(st, hp, rng=rng)  # host StepRandoms into the pinned stage, launch
        if k > 0:  # the previous step's result, read while this step runs
            acc_prev, s2_prev = st.step_result(st.iteration - 2)
    acc_last, s2_last = st.step_result()
    e2e_s = allreduce_max(time.perf_counter() - t0, world)
    e2e = (1 if sharded else world) * args.e2e_steps / e2e_s
    graph = bool(N.lib().bart_graph_active(st.handle))
    forest_kernels = profile_forest_kernels(st, N, args) if rank == 0 and not sharded else None
    st.close()

    cpu = None
    if rank == 0 and not args.no_cpu:
        (times,) = cpu_oracle_times(Xq, max_cuts, y32, hp, 1, args.cpu_steps, procs=1)
        med = statistics.median(times)
        cpu = {"value": 1.0 / med, "unit": "iters/s", "cores": 1, "kind": "port",
               "sample": f"oracle/bart_oracle.py (numpy port of bforge.sampler.step), the full workload "
                         f"(n={args.n}, p={args.p}, all {args.m} trees): 1 warm-up + {len(times)} timed "
                         f"iterations of one chain on one core, median {med:.2f} s"}
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_max * 1e3 / args.steps, "higher_is_better": True,
            "scaling": "strong" if sharded else "weak", "vs_baseline": None,
            "dtype": "f32 resid / f64 sums / u8 indices",
            "data": "synthetic Friedman #1 (binned uint8), device Philox RNG",
            "config": config_dict(args, (f"one chain n-sharded over {world} GPUs (in-kernel NVLink exchange)"
                                         if sharded else (f"{world} independent chains (replicas)" if world > 1
                                                          else "single chain, 1 GPU"))),
            "e2e": {"value": e2e, "unit": "iters/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "path": "per step: sampler.step(state, hp, rng=numpy Generator) = host StepRandoms written into a "
                            "pinned stage that the step kernel reads over the host link (zero-copy H2D) + launch; "
                            "the kernel writes each step's accept flags + sigma2 into pinned host memory (zero-copy "
                            "D2H), read (state.step_result) after the next step is launched, so the host's draw for "
                            "step k+1 overlaps the device's step k"},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": committed_traffic(),
                         "kernel": "sweep_kernel (the whole step: one launch per iteration)",
                         "algorithmic_bytes_per_launch": alg_bytes,
                         "algorithmic_bytes_formula": "10*n*ntree: per point and tree 1 B leaf index + 1 B X "
                                                      "column + 2x4 B residual (SURVEY.md 8d)",
                         "kernel_ms": sweep_ms, "kernel_ms_single_launch_events": single_launch_ms,
                         "peak_source": peak_src,
                         "traffic_source": "ncu dram__bytes_read.sum + dram__bytes_write.sum per launch, "
                                           "profiles/sweep_ncu_summary.json"},
            "cpu_baseline": cpu,
            "gpu_launches": gpu_launches,
            "cuda_graph": graph,
            "sweep_grid": cfg,
            "burn_in": args.burn,
            "trees": trees,
            "fresh_chain": fresh,
            "clocks": clk.summary(),
            "forest_kernels": forest_kernels,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


def run_reference(args):
    """The reference arm: the CPU oracle port (the reference is pure Python and
    cannot travel to the GPU box) on every host core, one independent chain of
    the FULL workload per core.  Each step is one full m-tree iteration of
    every chain; min(K, REF_MAX_STEPS) timed steps after min(W, 1) warm-up
    (each step takes seconds), all reported as run."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    Xq, max_cuts, y32, hp = workload(args)
    procs = max(1, min(os.cpu_count() or 1, 64))
    steps = max(1, min(args.steps, REF_MAX_STEPS))
    warm = min(args.warmup, 1)
    t0 = time.perf_counter()
    per_chain = cpu_oracle_times(Xq, max_cuts, y32, hp, warm, steps, procs=procs)
    wall = time.perf_counter() - t0
    # chains run concurrently: step k of the job takes the slowest chain's step k
    step_s = [max(t[k] for t in per_chain) for k in range(steps)]
    ms_per_step = 1e3 * statistics.fmean(step_s)
    value = procs * 1e3 / ms_per_step
    sample = (f"oracle port (numpy restatement of bforge.sampler.step; the reference is pure Python and is not "
              f"buildable) at n={args.n}, p={args.p}, ntree={args.m}: {procs} independent chains (one process per "
              f"core), each {warm} warm-up + {steps} timed full iterations; job step = slowest chain's step")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": 0,
        "steps": steps, "steps_requested": args.steps, "warmup": warm, "ms_per_step": ms_per_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32 resid / f64 sums",
        "data": "synthetic Friedman #1 (binned uint8)", "config": config_dict(args, f"{procs} CPU chains"),
        "cpu_baseline": {"value": value, "unit": "iters/s", "cores": procs, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "wall_s": wall,
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
