"""Host-side logic of the sweep's exchange and of n-sharding (no GPU).

* the fixed-point limb arithmetic (paper_2410_23244_b200/exchange.py mirrors
  to_limbs / from_limbs in csrc/sweep.cu): totals are independent of the
  order partials arrive in and agree with an exact sum to f64 rounding;
* the shard plan and the IPC-handle all-gather, over torch.distributed gloo
  with world_size 2 (the multi-GPU path's host protocol).
"""

import os
import socket
import sys
from fractions import Fraction

import numpy as np
import pytest

from paper_2410_23244_b200.exchange import exchange_total, fixed_limbs, limbs_total, range_limit, two_level_total
from paper_2410_23244_b200.shard import ShardPlan, exchange_handles


def test_limbs_round_trip_and_signs():
    for x in [0.0, 1.0, -1.0, 0.5, -0.25, 3.0e12, -7.123456789e10, 1e-30, -1e-30, 2.0 ** 44, -(2.0 ** 44)]:
        got = limbs_total(*fixed_limbs(x))
        assert got == pytest.approx(x, abs=2.0 ** -63), x
    with pytest.raises(OverflowError):
        fixed_limbs(2.0 ** 46)


def test_total_is_order_independent_and_exact():
    rng = np.random.default_rng(1)
    parts = list(rng.normal(size=300) * 10.0 ** rng.integers(-6, 6, size=300))
    exact = sum(Fraction(x) for x in parts)
    t = exchange_total(parts)
    for _ in range(5):
        rng.shuffle(parts)
        assert exchange_total(parts) == t  # bit-identical in any arrival order
    assert abs(Fraction(t) - exact) <= abs(exact) * Fraction(2) ** -52 + Fraction(300) * Fraction(2) ** -64


def test_two_level_total_equals_flat():
    """Stage sums per shard, then one forwarded add per shard: the same integers
    as every CTA adding into every shard's words."""
    rng = np.random.default_rng(3)
    parts = list(rng.normal(size=8 * 148) * 10.0 ** rng.integers(-3, 4, size=8 * 148))
    flat = exchange_total(parts)
    for shards in (1, 2, 3, 8):
        cuts = np.sort(rng.choice(np.arange(1, len(parts)), shards - 1, replace=False)) if shards > 1 else []
        split = np.split(np.array(parts), cuts)
        assert two_level_total([list(p) for p in split]) == flat


def test_range_limit_keeps_totals_from_wrapping():
    assert range_limit(1) == 2.0 ** 46 and range_limit(148) == 2.0 ** 38 and range_limit(8 * 148) == 2.0 ** 35
    for ctas in (1, 148, 1184):
        lim = range_limit(ctas)
        x = np.nextafter(lim, 0)
        assert limbs_total(*[ctas * l for l in fixed_limbs(x, lim)]) == pytest.approx(ctas * x, rel=1e-15)
        assert limbs_total(*[ctas * l for l in fixed_limbs(-x, lim)]) == pytest.approx(-ctas * x, rel=1e-15)
        with pytest.raises(OverflowError):
            fixed_limbs(lim, lim)


def test_shard_plan_covers_points_contiguously():
    for n, k in [(10, 3), (1_000_000, 8), (17, 1), (8, 8)]:
        b = ShardPlan(n, k).all_bounds()
        assert b[0][0] == 0 and b[-1][1] == n
        assert all(b[i][1] == b[i + 1][0] for i in range(k - 1))
        assert max(e - s for s, e in b) - min(e - s for s, e in b) <= 1
    with pytest.raises(ValueError):
        ShardPlan(4, 9)


def test_exchange_handles_orders_and_validates():
    handles = {1: b"b" * 8, 0: b"a" * 8}
    got = exchange_handles(b"a" * 8, 0, 2, lambda obj: [(1, handles[1]), obj])
    assert got == [b"a" * 8, b"b" * 8]
    with pytest.raises(RuntimeError):
        exchange_handles(b"a", 0, 2, lambda obj: [obj, obj])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, q):
    import torch.distributed as dist

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from paper_2410_23244_b200.exchange import fixed_limbs, limbs_total
    from paper_2410_23244_b200.shard import ShardPlan, exchange_handles, torch_all_gather

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        plan = ShardPlan(1001, world)
        start, stop = plan.bounds(rank)
        # every shard's partial sums of one slot over its points, as the sweep's CTAs would add them
        rng = np.random.default_rng(7)
        r = rng.normal(size=plan.n_total).astype(np.float32)
        partials = [float(np.sum(r[s:min(s + 100, stop)].astype(np.float64))) for s in range(start, stop, 100)]
        limbs = [0, 0, 0]
        for x in partials:
            for k, lv in enumerate(fixed_limbs(x)):
                limbs[k] += lv
        gathered = torch_all_gather()(limbs)  # stands in for the NVLink adds into every shard's words
        tot = [sum(g[k] for g in gathered) for k in range(3)]
        total = limbs_total(*tot)
        handles = exchange_handles(bytes([rank]) * 16, rank, world, torch_all_gather())
        q.put((rank, total, [h[0] for h in handles], float(np.sum(r.astype(np.float64)))))
    finally:
        dist.destroy_process_group()


def test_two_rank_shard_protocol_gloo():
    import multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, t0, h0, ref), (_, t1, h1, _) = out
    assert t0 == t1  # both shards read the bit-identical total
    assert t0 == pytest.approx(ref, rel=1e-12)
    assert h0 == h1 == [0, 1]  # handles in shard order on every rank
