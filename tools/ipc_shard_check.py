"""Two real processes, one n-sharded chain, over the CUDA IPC exchange.

Run with torchrun (gloo for the one-time handle all-gather):
    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 \
        --master-port 29561 tools/ipc_shard_check.py [n] [trees] [iters] [flat|two_level]

Every rank uses device LOCAL_RANK % device_count, so on a one-GPU box both
shards share the GPU: their sweeps then progress by time-slicing (one context
switch per exchange), which is slow but exercises exactly the cross-process
path -- IPC-mapped peer exchange words, system-scope atomics and polls.
Checks: both shards hold the same forest bit for bit, and it matches an
unsharded chain with the same device random stream (accept flags exact,
leaf values to f32 rounding).
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    import torch.distributed as dist
    from paper_2410_23244_b200.dgp import friedman1
    from paper_2410_23244_b200.grid import build_grid_uniform, quantize
    from paper_2410_23244_b200.regression import FitConfig, derive_hyperparams
    from paper_2410_23244_b200.sampler import DeviceRNG, init_state, run
    from paper_2410_23244_b200.shard import ShardPlan, init_sharded_state, torch_all_gather

    n = int(sys.argv[1]) if len(sys.argv) > 1 else 3000
    m = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    iters = int(sys.argv[3]) if len(sys.argv) > 3 else 3
    mode = sys.argv[4] if len(sys.argv) > 4 else "flat"
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    device = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    X, y, _ = friedman1(n, 6, seed=2)
    g = build_grid_uniform(X, 20)
    Xq = quantize(X, g).data
    hp, ys = derive_hyperparams(y, FitConfig(n_trees=m, max_depth=4))
    y32 = ys.forward(y).astype(np.float32)
    s2 = float(np.var(y32, ddof=1))
    plan = ShardPlan(n, world)
    lo, hi = plan.bounds(rank)
    st = init_sharded_state(Xq[lo:hi], g.counts, y32[lo:hi], hp, DeviceRNG(42), plan, rank, s2, torch_all_gather(),
                            device=device)
    st.set_exchange(mode)
    cfg = st.sweep_config()
    run(st, hp, iters)
    st.sync()
    f = st.forest
    mine = np.concatenate([f.axis.ravel().astype(np.float64), f.cutpoint.ravel().astype(np.float64),
                           f.leaf_value.ravel().astype(np.float64)])
    allf = [None] * world
    dist.all_gather_object(allf, mine)
    resid = st.resid.copy()
    allr = [None] * world
    dist.all_gather_object(allr, (lo, resid))
    st.close()
    if rank == 0:
        same = all(np.array_equal(allf[0], a) for a in allf[1:])
        ref = init_state(Xq, g.counts, y32, hp, DeviceRNG(42), sigma2=s2, device=device)
        run(ref, hp, iters)
        ref.sync()
        rf = ref.forest
        cut_ok = np.array_equal(rf.cutpoint, f.cutpoint) and np.array_equal(rf.axis, f.axis)
        leaf_ok = np.allclose(rf.leaf_value, f.leaf_value, rtol=1e-5, atol=1e-6)
        full_r = np.concatenate([r for _, r in sorted(allr, key=lambda t: t[0])])
        resid_ok = np.allclose(ref.resid, full_r, rtol=1e-5, atol=1e-5)
        ref.close()
        ok = same and cut_ok and leaf_ok and resid_ok
        print(f"ipc shard check: world={world} n={n} trees={m} iters={iters} exchange={mode} "
              f"ctas/shard={cfg['ctas']} chunk={cfg['chunk']}: shards identical={same} "
              f"structure==unsharded={cut_ok} leaves~={leaf_ok} resid~={resid_ok} -> {'OK' if ok else 'FAIL'}",
              flush=True)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
