"""Correctly rounded fp64 reductions (host side).

Semantics follow ``neurocomm/accum.py:16-49``: every reduction returns the
correctly rounded value of the exact real sum, so it does not depend on the
order of its inputs.  On the host this is ``math.fsum``; on the device the
same numbers come from the exact fixed-point histogram kernel (K5, see
``traffic.aggregate``), and :func:`limbs_to_float` is the single rounding
step that turns its integer accumulators into doubles.
"""

from __future__ import annotations

import math

import numpy as np

__all__ = ["exact_sum", "keyed_sums", "binned_sums", "limbs_to_float"]


def exact_sum(values) -> float:
    """fsum of an iterable (accum.py:16-18)."""
    return math.fsum(values)


def keyed_sums(keys, values):
    """Per-key correctly rounded sums, keys ascending (accum.py:21-41)."""
    keys = np.asarray(keys)
    vals = np.asarray(values, dtype=np.float64)
    if keys.size == 0:
        return keys[:0], vals[:0]
    perm = np.argsort(keys, kind="stable")
    sk = keys[perm]
    sv = vals[perm]
    uniq, first = np.unique(sk, return_index=True)
    bounds = np.append(first, sk.size)
    out = np.fromiter(
        (math.fsum(sv[bounds[n]:bounds[n + 1]]) for n in range(uniq.size)),
        dtype=np.float64,
        count=uniq.size,
    )
    return uniq, out


def binned_sums(keys, values, n_bins: int) -> np.ndarray:
    """Dense per-bin sums for keys in ``[0, n_bins)`` (accum.py:44-49)."""
    dense = np.zeros(n_bins, dtype=np.float64)
    uk, s = keyed_sums(keys, values)
    dense[uk] = s
    return dense


def limbs_to_float(limbs, lsb_exponent: int, digit_bits: int = 32) -> float:
    """Round an exact fixed-point accumulator to the nearest double.

    ``limbs[k]`` holds digit ``k`` (weight ``2**(digit_bits*k)``), each a
    possibly un-normalised non-negative integer.  The represented value is
    ``sum(limbs[k] << digit_bits*k) * 2**lsb_exponent``.  Python's int/int true
    division is correctly rounded (round-half-even), which is exactly the
    rounding ``math.fsum`` applies to the same real number.
    """
    total = 0
    for k, d in enumerate(limbs):
        total += int(d) << (digit_bits * k)
    if total == 0:
        return 0.0
    if lsb_exponent >= 0:
        return float(total << lsb_exponent)
    return total / (1 << (-lsb_exponent))
