"""Datapoint sharding of one chain across GPUs.

The reference has no multi-device path (sharding along the
observations "is straightforward ... I simply have not put in the work").
Here one process per GPU holds a contiguous range of the points; the forest,
the proposals and the device random stream are replicated (same seed on every
shard), so every shard takes identical decisions from identical totals.  The
per-tree leaf statistics are combined INSIDE the sweep kernel: each shard
adds its fixed-point partials into every shard's exchange words over NVLink
(peer-mapped through CUDA IPC) and polls its own copy -- no collective launch
per tree.  The host side below only plans the split and swaps the IPC handles
once, through any all-gather (torch.distributed with NCCL or gloo).
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Sequence

import numpy as np

from .exchange import fixed_limbs  # noqa: F401  (re-export: host mirror of the exchange arithmetic)


@dataclass(frozen=True)
class ShardPlan:
    """Contiguous split of n_total points over n_shards (the first n % k shards get one more)."""

    n_total: int
    n_shards: int

    def __post_init__(self):
        if self.n_shards < 1 or self.n_shards > 8:
            raise ValueError("n_shards must be in [1, 8]")
        if self.n_total < self.n_shards:
            raise ValueError("fewer points than shards")

    def bounds(self, shard: int) -> tuple[int, int]:
        if not 0 <= shard < self.n_shards:
            raise ValueError(f"shard {shard} out of range")
        base, extra = divmod(self.n_total, self.n_shards)
        start = shard * base + min(shard, extra)
        return start, start + base + (1 if shard < extra else 0)

    def all_bounds(self) -> list[tuple[int, int]]:
        return [self.bounds(k) for k in range(self.n_shards)]


def exchange_handles(local: bytes, shard: int, n_shards: int,
                     all_gather: Callable[[object], Sequence[object]]) -> list[bytes]:
    """All-gather every shard's exported handle; return them in shard order."""
    got = list(all_gather((int(shard), bytes(local))))
    if len(got) != n_shards:
        raise RuntimeError(f"expected {n_shards} shard handles, got {len(got)}")
    by_shard = dict(got)
    if sorted(by_shard) != list(range(n_shards)):
        raise RuntimeError(f"shard handles do not cover 0..{n_shards - 1}: {sorted(by_shard)}")
    return [by_shard[k] for k in range(n_shards)]


def torch_all_gather(group=None) -> Callable[[object], list]:
    """all_gather over torch.distributed (NCCL or gloo) for exchange_handles."""
    import torch.distributed as dist

    def gather(obj):
        out = [None] * dist.get_world_size(group)
        dist.all_gather_object(out, obj, group=group)
        return out

    return gather


def init_sharded_state(X_local, max_cuts, y32_local, hp, rng, plan: ShardPlan, shard: int, sigma2: float,
                       all_gather, device: int = 0):
    """This rank's shard of one chain, connected to the other shards.

    `sigma2` must be the chain's initial sigma2 (the same on every shard), e.g.
    float(np.var(y32_full, ddof=1)) as in sampler.init_state; `rng` a DeviceRNG
    with the same seed on every shard."""
    from .sampler import DeviceRNG, SamplerState

    if not isinstance(rng, DeviceRNG):
        raise ValueError("a sharded chain draws its randoms on the device: pass a DeviceRNG (same seed on every shard)")
    start, stop = plan.bounds(shard)
    if X_local.shape[0] != stop - start or y32_local.shape[0] != stop - start:
        raise ValueError(f"shard {shard} holds points [{start}, {stop}); got {X_local.shape[0]}")
    X_local = np.ascontiguousarray(X_local, np.uint8)
    y32_local = np.ascontiguousarray(y32_local, np.float32)
    max_cuts = np.ascontiguousarray(max_cuts, np.int64)
    st = SamplerState(X_local, max_cuts, y32_local, hp, rng, float(sigma2), device,
                      shard=(plan.n_total, shard, plan.n_shards))
    st.shard_connect(exchange_handles(st.shard_export(), shard, plan.n_shards, all_gather))
    return st
