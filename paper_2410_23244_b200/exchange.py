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
RANGE = 2.0 ** 45           # |partial| must stay below this (device flags BART error bit 0)


def fixed_limbs(x: float) -> tuple[int, int, int]:
    """to_limbs: hi = floor(x), lo = RN((x - hi) * 2^64); limbs of hi * 2^64 + lo."""
    x = float(x)
    if not abs(x) < RANGE:
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
