"""Host mirror of the sweep's cross-CTA / cross-GPU exchange arithmetic.

The sweep (csrc/sweep.cu, to_limbs / from_limbs) turns each CTA's f64 partial
sum into a 111-bit two's-complement fixed-point number with 64 fraction bits,
split into three 37-bit limbs, and every CTA of every shard adds its limbs
(integers) into shared 64-bit words.  Integer addition is associative, so
the total -- and hence every accept decision -- is bit-identical whatever the
order the partials arrive in, on every CTA and every GPU.  This module
restates that arithmetic on the host (same IEEE operations) so the property
can be tested without a GPU.
"""

from __future__ import annotations

import math

LIMB_BITS = 37
LIMB_MASK = (1 << LIMB_BITS) - 1
TOTAL_BITS = 3 * LIMB_BITS  # 111
RANGE = 2.0 ** 45           # single CTA: |partial| must stay below this (the device reports BART_ERANGE)


def range_limit(ctas: int) -> float:
    """The per-CTA bound: 2^46 / (CTAs over all shards, rounded up to a power of
    two), so no total can wrap the 111-bit sum (sweep.cu xrange_limit)."""
    bits = max(0, (int(ctas) - 1).bit_length())
    return 2.0 ** (46 - bits)


def fixed_limbs(x: float, limit: float = RANGE) -> tuple[int, int, int]:
    """to_limbs: hi = floor(x), lo = RN((x - hi) * 2^64); limbs of hi * 2^64 + lo."""
    x = float(x)
    if not abs(x) < limit:
        raise OverflowError(f"partial {x} outside the exchange's fixed-point range")
    hi = math.floor(x)
    rem = x - float(hi)                 # exact
    lo = round(rem * 2.0 ** 64)         # round half to even, like __double2ull_rn
    lo = min(lo, (1 << 64) - 1)         # saturating conversion
    v = (hi << 64) + lo                 # two's complement value
    return v & LIMB_MASK, (v >> LIMB_BITS) & LIMB_MASK, (v >> (2 * LIMB_BITS)) & LIMB_MASK


def limbs_total(t0: int, t1: int, t2: int) -> float:
    """from_limbs: the f64 of (t0 + t1 2^37 + t2 2^74) mod 2^111 / 2^64, same operations as the device."""
    v = (t0 + (t1 << LIMB_BITS) + (t2 << (2 * LIMB_BITS))) % (1 << TOTAL_BITS)
    neg = v >> (TOTAL_BITS - 1)
    if neg:
        v = (1 << TOTAL_BITS) - v
    hi, lo = v >> 64, v & ((1 << 64) - 1)
    mag = float(hi) * 2.0 ** 64 + float(lo)  # two roundings, as __dadd_rn(__dmul_rn(hi, 2^64), lo)
    val = mag * 2.0 ** -64
    return -val if neg else val


def exchange_total(partials) -> float:
    """The total every CTA reads after all `partials` were added (any order)."""
    t = [0, 0, 0]
    for x in partials:
        for k, limb in enumerate(fixed_limbs(x)):
            t[k] += limb
    return limbs_total(*t)


def two_level_total(shard_partials) -> float:
    """The two-level exchange (bart_set_exchange): each shard's CTAs add into
    the shard's stage words; the shard's forwarder adds the stage's limb sums,
    once, into every shard's words.  The final words hold the same integers as
    the flat exchange's, so the total is bit-identical (exchange_total of all
    partials)."""
    t = [0, 0, 0]
    for partials in shard_partials:
        stage = [0, 0, 0]
        for x in partials:
            for k, limb in enumerate(fixed_limbs(x)):
                stage[k] += limb
        for k in range(3):
            t[k] += stage[k]  # the forwarder's one tagged add per word
    return limbs_total(*t)
