"""Capacity-bounded greedy fill shared by neuron placement and GPU grouping.

Drop-in for ``neurocomm/greedy.py``.  The CSR builders are numpy (they run
once per partition); the fill itself is the native K6 routine
``nc_greedy_fill`` (csrc/greedy_fill.cpp), an indexed-heap restatement of
greedy.py:55-117 that picks the same item at every step.  The capacity is
computed here with ``math.fsum`` exactly as greedy.py:70 does, so the C++ side
never has to reproduce a correctly rounded sum.
"""

from __future__ import annotations

import math

import numpy as np

from . import _native

__all__ = ["adjacency_from_edges", "adjacency_from_dense", "greedy_fill"]


def adjacency_from_edges(n_items: int, idx_a, idx_b, values):
    """Symmetric CSR of undirected weighted pairs (greedy.py:32-42).

    Row ``r`` lists first the pairs where ``r`` is ``idx_a`` (in input order),
    then those where it is ``idx_b`` -- the stable-sort order the reference
    produces, which the fill's sequential score adds depend on.
    """
    a = np.asarray(idx_a, dtype=np.int64)
    b = np.asarray(idx_b, dtype=np.int64)
    v = np.asarray(values, dtype=np.float64)
    src = np.concatenate((a, b))
    perm = np.argsort(src, kind="stable")
    counts = np.bincount(src, minlength=n_items)
    indptr = np.zeros(n_items + 1, dtype=np.int64)
    indptr[1:] = np.cumsum(counts)
    return indptr, np.concatenate((b, a))[perm], np.concatenate((v, v))[perm]


def adjacency_from_dense(matrix):
    """CSR over positive off-diagonal cells, row-major (greedy.py:45-52)."""
    m = np.array(matrix, dtype=np.float64)
    np.fill_diagonal(m, 0.0)
    r, c = np.nonzero(m > 0.0)
    indptr = np.zeros(m.shape[0] + 1, dtype=np.int64)
    indptr[1:] = np.cumsum(np.bincount(r, minlength=m.shape[0]))
    return indptr, c.astype(np.int64), m[r, c]


def greedy_fill(weights, indptr, indices, values, n_buckets: int, balance_slack: float = 0.0) -> np.ndarray:
    """Bucket id per item, bit-identical to greedy.py:55-117 (native K6)."""
    w = np.ascontiguousarray(weights, dtype=np.float64)
    m = int(w.size)
    if not 1 <= n_buckets <= m:
        raise ValueError(f"n_buckets must be in [1, {m}], got {n_buckets}")
    if not 0.0 <= balance_slack < 1.0:
        raise ValueError(f"balance_slack must be in [0, 1), got {balance_slack}")
    capacity = (math.fsum(w) / n_buckets) * (1.0 + balance_slack)
    ip = np.ascontiguousarray(indptr, dtype=np.int64)
    ix = np.ascontiguousarray(indices, dtype=np.int64)
    vals = np.ascontiguousarray(values, dtype=np.float64)
    out = np.empty(m, dtype=np.int64)
    rc = _native.lib().nc_greedy_fill(m, _native.ptr(w), _native.ptr(ip), _native.ptr(ix),
                                     _native.ptr(vals), int(n_buckets), float(capacity),
                                     _native.ptr(out))
    _native.check(rc, "greedy_fill")
    return out
