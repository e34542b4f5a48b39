"""GPU-level traffic aggregation (the partitioner's edge-cut matrix) on the GPU.

Drop-in for ``neurocomm/traffic.py``.  ``aggregate`` (traffic.py:66-84) runs
the K5 histogram kernel (csrc/traffic_hist.cu): every contribution
``(p*W_i)*W_j`` is added exactly into fixed-point limbs, and each cell is
rounded once on the host (:func:`.accum.limbs_to_float`), which equals the
reference's per-cell ``math.fsum`` bit for bit.  The N x N reports around it
stay on the host; they touch at most a few hundred numbers.
"""

from __future__ import annotations

import csv
import ctypes as C
import json
import math
from dataclasses import dataclass

import numpy as np

from . import _native
from .accum import limbs_to_float

__all__ = [
    "GpuTrafficGraph", "TrafficReport", "report_from_vector", "aggregate", "per_gpu_send_traffic",
    "peak_reduction", "write_traffic_csv", "read_traffic_csv", "write_traffic_summary",
    "exact_bin_sums", "aggregate_sharded", "aggregate_generated",
]

INT_MAX = 2**31 - 1
INT_MIN = -(2**31)


@dataclass(eq=False)
class GpuTrafficGraph:
    """Symmetric N x N traffic (diagonal = intra-GPU) plus per-GPU weight (traffic.py:27-42)."""

    n_gpus: int
    pg: np.ndarray
    wg: np.ndarray

    def __eq__(self, other) -> bool:
        if not isinstance(other, GpuTrafficGraph):
            return NotImplemented
        return (self.n_gpus == other.n_gpus and np.array_equal(self.pg, other.pg)
                and np.array_equal(self.wg, other.wg))


@dataclass(eq=False)
class TrafficReport:
    """Per-GPU send traffic with max / mean / population std (traffic.py:45-56)."""

    per_gpu_send: np.ndarray
    peak: float
    mean: float
    stddev: float

    @property
    def n_gpus(self) -> int:
        return int(self.per_gpu_send.size)


def report_from_vector(values) -> TrafficReport:
    v = np.asarray(values, dtype=np.float64)
    if v.size == 0:
        return TrafficReport(v, 0.0, 0.0, 0.0)
    return TrafficReport(v, float(np.max(v)), float(np.mean(v)), float(np.std(v)))


def _device():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("traffic aggregation runs on the GPU (K5 histogram); no CUDA device is visible")
    return torch.device("cuda", torch.cuda.current_device())


def _n_digits(lsb: int, msb: int, n_terms: int) -> int:
    bits = (msb - lsb + 1) + max(1, int(n_terms).bit_length()) + 1
    return (bits + 31) // 32 + 2


def _exp_range(x):
    """(floor(log2 min|x|), floor(log2 max|x|)) over the nonzero entries of a device
    float64 tensor, or None if all are zero."""
    import torch
    a = x.abs()
    lo, hi = torch.aminmax(a)
    if float(hi) == 0.0:
        return None
    if float(lo) == 0.0:
        lo = torch.where(a > 0, a, torch.full_like(a, float("inf"))).min()
    return math.frexp(float(lo))[1] - 1, math.frexp(float(hi))[1] - 1


_WINDOWS: dict = {}


def _window(ep, w):
    """contribution_window's (lsb, msb) as a host tuple (cached per tensor pair)."""
    key = (ep.data_ptr(), ep.numel(), w.data_ptr(), w.numel())
    hit = _WINDOWS.get(key)
    if hit is None or hit[0]() is not ep or hit[1]() is not w:
        rp, rw = _exp_range(ep), _exp_range(w)
        if rp is None or rw is None:
            win = (INT_MAX, INT_MIN)
        else:
            win = (max(-1074, rp[0] + 2 * rw[0] - 52), rp[1] + 2 * rw[1] + 4)
        import weakref
        try:
            hit = (weakref.ref(ep), weakref.ref(w), win)
            if len(_WINDOWS) > 64:
                _WINDOWS.clear()
            _WINDOWS[key] = hit
        except TypeError:
            hit = (lambda: ep, lambda: w, win)
    return hit[2]


def contribution_window(ep, w):
    """[lowest mantissa bit, highest bit] exponents bounding every contribution
    (ep * w[i]) * w[j] (device int32[2], the layout nc_traffic_exponents writes).

    From the columns' exponent ranges instead of a pass over the edges: with
    e(x) = floor(log2 |x|), a product of two doubles rounded to nearest has
    e in [e(a) + e(b), e(a) + e(b) + 2], so every nonzero term has its leading
    bit at or below e_max(p) + 2 e_max(w) + 4 and its lowest mantissa bit at or
    above max(-1074, e_min(p) + 2 e_min(w) - 52).  The window only has to
    contain the terms (the sum is exact and rounded once), so a few spare bits
    cost nothing but shared memory.  Cached per (ep, w) tensor pair."""
    import torch
    return torch.tensor(_window(ep, w), dtype=torch.int32, device=ep.device)


def exact_bin_sums(values_dev, keys_dev, n_bins: int, *, pairs=None, stream=None, group=None):
    """Correctly rounded per-bin sums on the device.

    ``pairs=None``: bin ``keys[k]`` receives ``values[k]`` (binned_sums).
    ``pairs=(ei, ej, ep)``: edge mode -- values are the neuron weights, keys
    the assignment, and cell ``min*N+max`` receives ``(ep*w[ei])*w[ej]``.
    Returns a float64 numpy array of ``n_bins`` (or ``n_bins**2``) cells.

    ``group`` (a torch.distributed process group, or ``True`` for the default
    one): every rank passes its own slice of the terms; the exponent range and
    term count are all-reduced so all ranks accumulate on the same fixed-point
    grid, the integer limbs are all-reduced (exact), and every rank rounds the
    same total once -- the SURVEY 8(e) partition-time path.
    """
    import torch
    L = _native.lib()
    st = stream if stream is not None else _native.stream_handle()
    dev = values_dev.device
    mm = torch.tensor([INT_MAX, INT_MIN], dtype=torch.int32, device=dev)
    if pairs is None:
        n = int(values_dev.numel())
        if n:
            _native.check(L.nc_traffic_exponents(None, None, None, values_dev.data_ptr(), n, mm.data_ptr(), st),
                          "weight exponents")
    else:
        ei, ej, ep = pairs
        n = int(ei.numel())
        if n:
            mm = contribution_window(ep, values_dev)
    n_local = n
    n_cells = n_bins * n_bins if pairs is not None else n_bins
    if group is not None:
        import torch.distributed as dist
        grp = None if group is True else group
        mn, mx = mm[0:1].clone(), mm[1:2].clone()
        dist.all_reduce(mn, op=dist.ReduceOp.MIN, group=grp)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX, group=grp)
        mm = torch.cat([mn, mx])
        cnt = torch.tensor([n], dtype=torch.int64, device=dev)
        dist.all_reduce(cnt, group=grp)
        n = int(cnt.item())
    lo, hi = mm.cpu().tolist()
    if n == 0 or lo == INT_MAX:
        return np.zeros(n_cells, dtype=np.float64)
    nd = _n_digits(lo, hi, n)
    limbs = torch.zeros((n_cells, nd), dtype=torch.int64, device=dev)
    if n_local:
        if pairs is None:
            rc = L.nc_weight_histogram(values_dev.data_ptr(), keys_dev.data_ptr(), n_local, n_bins, lo, nd,
                                       limbs.data_ptr(), st)
        elif ei.dtype == torch.int32:
            # one 16-byte record per neuron {weight, gpu}: a single gather per endpoint
            rec = torch.zeros((values_dev.numel(), 4), dtype=torch.int32, device=dev)
            rec[:, :2] = values_dev.to(torch.float64).contiguous().view(torch.int32).view(-1, 2)
            rec[:, 2] = keys_dev.to(torch.int32)
            rc = L.nc_traffic_histogram_packed(ei.data_ptr(), ej.data_ptr(), ep.data_ptr(), rec.data_ptr(), n_local,
                                               n_bins, lo, nd, limbs.data_ptr(), st)
            if rc != 0:   # cells x digits too large for shared memory: the global-limb path
                asg32 = keys_dev.to(torch.int32)
                rc = L.nc_traffic_histogram32(ei.data_ptr(), ej.data_ptr(), ep.data_ptr(), values_dev.data_ptr(),
                                              asg32.data_ptr(), n_local, n_bins, lo, nd, limbs.data_ptr(), st)
        else:
            rc = L.nc_traffic_histogram(ei.data_ptr(), ej.data_ptr(), ep.data_ptr(), values_dev.data_ptr(),
                                        keys_dev.to(torch.int64).data_ptr(), n_local, n_bins, lo, nd,
                                        limbs.data_ptr(), st)
        _native.check(rc, "traffic histogram")
    if group is not None:   # exact: integer limbs (< 2^33 each after the kernel's carry flush)
        import torch.distributed as dist
        dist.all_reduce(limbs, group=None if group is True else group)
    host = limbs.cpu().numpy().view(np.uint64)
    out = np.zeros(n_cells, dtype=np.float64)
    for c in np.flatnonzero(host.any(axis=1)).tolist():
        out[c] = limbs_to_float(host[c].tolist(), lo)
    return out


_DEVICE_GRAPHS: dict = {}


def _device_graph(graph, dev):
    """Edge columns and weights of `graph` on the device, uploaded once per graph object.

    The fifth entry is the common weight when every neuron has the same one
    (generate_synthetic's default weight_low == weight_high), else None.

    Graphs are treated as immutable (SPEC concurrency model); the cache is keyed
    by the object (NeuronGraph defines __eq__, so it is not hashable: keyed by
    id() with a weak reference and a finalizer that evicts the entry) and by the
    identity of its arrays, so replacing an array re-uploads.  Repeated
    aggregation (cross_traffic, the GA fitness, sweep_noise) then only moves
    the assignment.
    """
    import torch
    import weakref
    key = (str(dev), id(graph.weights), id(graph.edge_i), id(graph.edge_j), id(graph.edge_p))
    hit = _DEVICE_GRAPHS.get(id(graph))
    if hit is not None and hit[0]() is graph and hit[1] == key:
        return hit[2]
    up = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(dev)  # noqa: E731
    # int32 ids below 2^31 neurons: K5 streams 16 B per edge instead of 24
    idx = np.int32 if graph.n_neurons < 2**31 else np.int64
    wh = np.asarray(graph.weights, dtype=np.float64)
    w0 = float(wh[0]) if wh.size and bool(np.all(wh == wh[0])) else None
    val = (up(wh, np.float64), up(graph.edge_i, idx), up(graph.edge_j, idx), up(graph.edge_p, np.float64), w0)
    try:
        ref = weakref.ref(graph)
    except TypeError:  # not weak-referenceable: no caching
        return val
    if id(graph) not in _DEVICE_GRAPHS:
        weakref.finalize(graph, _DEVICE_GRAPHS.pop, id(graph), None)
    _DEVICE_GRAPHS[id(graph)] = (ref, key, val)
    return val


def _check_assignment(pm) -> None:
    """The kernels index per-GPU cells by the assignment: refuse values outside [0, n_gpus)
    (where the reference's numpy indexing would raise)."""
    a = np.asarray(pm.assignment)
    if a.size and (int(a.min()) < 0 or int(a.max()) >= int(pm.n_gpus)):
        raise ValueError(f"assignment has GPU indices outside [0, {int(pm.n_gpus)})")


def aggregate(graph, pm) -> GpuTrafficGraph:
    """Collapse neuron traffic onto GPUs (traffic.py:66-84) with the K5 kernel."""
    import torch
    if pm.assignment.size != graph.n_neurons:
        raise ValueError(
            f"partition map covers {pm.assignment.size} neurons, graph has {graph.n_neurons}"
        )
    n = int(pm.n_gpus)
    dev = _device()
    w, ei, ej, ep, w0 = _device_graph(graph, dev)
    if ei.dtype == torch.int32 and 1 <= n <= 256:
        out = _aggregate_fast(pm, w, ei, ej, ep, w0, n)   # range-checks the assignment on the device
        if out is not None:
            return out
    _check_assignment(pm)
    asg = torch.from_numpy(np.ascontiguousarray(pm.assignment, dtype=np.int64)).to(dev)
    cells = exact_bin_sums(w, asg, n, pairs=(ei, ej, ep)).reshape(n, n)
    upper = np.triu(cells)
    pg = upper + np.triu(cells, 1).T
    wg = exact_bin_sums(w, asg, n)
    return GpuTrafficGraph(n, pg, wg)


_RECORDS: dict = {}


def _records(w):
    """One 16-byte record per neuron {double weight; int32 gpu; pad} with the weights
    filled in (the gpu column is written per call), and the weights' fixed-point window
    (lsb, msb) for the per-GPU sums -- cached per weight tensor."""
    import torch
    import weakref
    hit = _RECORDS.get(id(w))
    if hit is not None and hit[0]() is w:
        return hit[1], hit[2]
    rec = torch.zeros((w.numel(), 4), dtype=torch.int32, device=w.device)
    rec[:, :2] = w.contiguous().view(torch.int32).view(-1, 2)
    rw = _exp_range(w)
    win = (INT_MAX, INT_MIN) if rw is None else (max(-1074, rw[0] - 52), rw[1] + 1)
    try:
        if len(_RECORDS) > 16:
            _RECORDS.clear()
        _RECORDS[id(w)] = (weakref.ref(w), rec, win)
    except TypeError:
        pass
    return rec, win


def _aggregate_fast(pm, w, ei, ej, ep, w0, n: int):
    """aggregate() for int32 edge ids and up to 256 GPUs with one host -> device copy
    (the assignment, through a pinned buffer) and one device -> host copy (limbs,
    counts, range flag).  The assignment is narrowed to uint8, counted and
    range-checked on the device (nc_assignment_u8).

    Every weight equal to w0 (generate_synthetic's default): K5 gathers a 1-byte gpu
    id per endpoint (nc_traffic_histogram_uniform), and wg[g] = count_g * w0 in one
    IEEE multiply -- the correctly rounded value of the exact sum math.fsum returns
    (count_g < 2^53 is exact in a double).  Otherwise the packed {weight, gpu}
    records (weights cached per graph) and the exact per-GPU weight histogram.
    None if the cells do not fit in shared memory (the general path then runs)."""
    import torch
    dev = ei.device
    L = _native.lib()
    st = _native.stream_handle()
    a = torch.from_numpy(np.ascontiguousarray(pm.assignment))
    m = int(a.numel())
    n_edges = int(ei.numel())
    lo, hi = _window(ep, w) if n_edges else (INT_MAX, INT_MIN)
    nd = _n_digits(lo, hi, n_edges) if lo != INT_MAX else 3
    n_lim = n * n * nd
    if w0 is None:
        rec, (wlo, whi) = _records(w)
        ndw = _n_digits(wlo, whi, m) if wlo != INT_MAX else 3
    else:
        ndw = 0
    # pg limbs | per-GPU counts | range flag | wg limbs (weighted)
    buf = torch.zeros(n_lim + n + 1 + n * ndw, dtype=torch.int64, device=dev)
    o_cnt, o_bad, o_wg = n_lim, n_lim + n, n_lim + n + 1
    asg8 = torch.empty(max(m, 1), dtype=torch.uint8, device=dev)
    asg = None
    if m:
        pin = torch.empty(m, dtype=torch.int64, pin_memory=True)
        pin.copy_(a)
        asg = pin.to(dev, non_blocking=True)
        _native.check(L.nc_assignment_u8(asg.data_ptr(), m, n, asg8.data_ptr(), buf[o_cnt:].data_ptr(),
                                         buf[o_bad:].data_ptr(), st), "assignment")
    if lo != INT_MAX:
        if w0 is not None:
            rc = L.nc_traffic_histogram_uniform(ei.data_ptr(), ej.data_ptr(), ep.data_ptr(), float(w0),
                                                asg8.data_ptr(), n_edges, n, lo, nd, buf.data_ptr(), st)
        else:
            rec[:, 2].copy_(asg8[:m])
            rc = L.nc_traffic_histogram_packed(ei.data_ptr(), ej.data_ptr(), ep.data_ptr(), rec.data_ptr(), n_edges,
                                               n, lo, nd, buf.data_ptr(), st)
        if rc != 0:
            return None
    if w0 is None and m and wlo != INT_MAX:
        # out-of-range entries are flagged (and raise below) but must not index the cells
        safe = asg8[:m].to(torch.int64)
        _native.check(L.nc_weight_histogram(w.data_ptr(), safe.data_ptr(), m, n, wlo, ndw, buf[o_wg:].data_ptr(), st),
                      "weight histogram")
    host = buf.cpu().numpy()
    if host[o_bad]:
        raise ValueError(f"assignment has GPU indices outside [0, {n})")
    cells = _round_cells(host[:n_lim], n * n, nd, lo).reshape(n, n)
    pg = np.triu(cells) + np.triu(cells, 1).T
    if w0 is not None:
        wg = host[o_cnt:o_cnt + n].astype(np.float64) * float(w0)
    else:
        wg = _round_cells(host[o_wg:], n, ndw, wlo) if ndw and wlo != INT_MAX else np.zeros(n, dtype=np.float64)
    return GpuTrafficGraph(n, pg, wg)


def _round_cells(flat, n_cells: int, nd: int, lsb: int) -> np.ndarray:
    limbs = flat.view(np.uint64).reshape(n_cells, nd)
    out = np.zeros(n_cells, dtype=np.float64)
    for c in np.flatnonzero(limbs.any(axis=1)).tolist():
        out[c] = limbs_to_float(limbs[c].tolist(), lsb)
    return out


def aggregate_sharded(edge_i, edge_j, edge_p, weights, assignment, n_gpus: int, group=True) -> GpuTrafficGraph:
    """aggregate() over an edge list split across ranks: every rank
    passes its own slice of (edge_i, edge_j, edge_p) and the full weights and
    assignment; the K5 limbs are all-reduced over NCCL and rounded once, so every
    rank returns pg / wg bit-identical to the single-GPU aggregate of the whole
    graph (any split, any order: the sums are exact)."""
    import torch
    dev = _device()
    def up(a, dt):
        if isinstance(a, np.ndarray):
            return torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(dev)
        return a.to(device=dev)

    ei, ej = up(edge_i, np.int64), up(edge_j, np.int64)
    ep, w = up(edge_p, np.float64), up(weights, np.float64)
    asg = up(assignment, np.int64)
    n = int(n_gpus)
    cells = exact_bin_sums(w, asg, n, pairs=(ei, ej, ep), group=group).reshape(n, n)
    pg = np.triu(cells) + np.triu(cells, 1).T
    wg = exact_bin_sums(w, asg, n)
    return GpuTrafficGraph(n, pg, wg)


def aggregate_generated(spec, pm, *, weights=None, group=None) -> GpuTrafficGraph:
    """aggregate() (traffic.py:66-84) of a generated network (sim.GeneratorSpec) without
    materialising it: K5 consumes the generator's edges and fp64 p on the fly
    (nc_traffic_histogram_generated), so the reference's traffic matrix of a 1e10-synapse
    network (configs 3-5) costs one pass of the generator.  Bit-identical to
    ``aggregate(spec.host_graph(), pm)`` (weights: None = all 1, else float64 [M]).
    ``group`` (torch.distributed, True = default group): every rank enumerates its slice
    of the rows and the integer limbs are all-reduced before the one rounding."""
    import torch
    m = int(spec.n_neurons)
    if pm.assignment.size != m:
        raise ValueError(f"partition map covers {pm.assignment.size} neurons, graph has {m}")
    _check_assignment(pm)
    n = int(pm.n_gpus)
    dev = _device()
    L = _native.lib()
    st = _native.stream_handle()
    asg32 = torch.from_numpy(np.ascontiguousarray(pm.assignment, dtype=np.int32)).to(dev)
    w_dev = None if weights is None else torch.from_numpy(np.ascontiguousarray(weights, dtype=np.float64)).to(dev)
    # window: every term is p (times two weights) with p in [lo, hi) of the ranges in use
    ranges = []
    if spec.p_in > 0:
        ranges.append(spec.intra_p_range)
    if spec.p_out > 0 and spec.n_communities > 1:
        ranges.append(spec.inter_p_range)
    lo_p = min(r[0] for r in ranges) if ranges else 1.0
    hi_p = max(r[1] for r in ranges) if ranges else 1.0
    if w_dev is None:
        ew = (0, 0)
    else:
        ew = _exp_range(w_dev)
        if ew is None:
            raise ValueError("weights are all zero")
    ep_lo, ep_hi = math.frexp(lo_p)[1] - 1, math.frexp(hi_p)[1] - 1
    lsb = max(-1074, ep_lo + 2 * ew[0] - 52)
    msb = ep_hi + 2 * ew[1] + 4
    n_terms = m * (m - 1) // 2                     # an upper bound on the edge count
    nd = _n_digits(lsb, msb, n_terms)
    limbs = torch.zeros((n * n, nd), dtype=torch.int64, device=dev)
    rank, world = 0, 1
    if group is not None:
        import torch.distributed as dist
        grp = None if group is True else group
        rank, world = dist.get_rank(grp), dist.get_world_size(grp)
    r0, r1 = m * rank // world, m * (rank + 1) // world
    g = spec.to_c()
    _native.check(L.nc_traffic_histogram_generated(C.byref(g), None if w_dev is None else w_dev.data_ptr(),
                                                   asg32.data_ptr(), r0, r1, n, lsb, nd, limbs.data_ptr(), st),
                  "traffic histogram (generated)")
    if group is not None:
        import torch.distributed as dist
        dist.all_reduce(limbs, group=None if group is True else group)
    host = limbs.cpu().numpy().view(np.uint64)
    cells = np.zeros(n * n, dtype=np.float64)
    for c in np.flatnonzero(host.any(axis=1)).tolist():
        cells[c] = limbs_to_float(host[c].tolist(), lsb)
    cells = cells.reshape(n, n)
    pg = np.triu(cells) + np.triu(cells, 1).T
    wsrc = torch.ones(m, dtype=torch.float64, device=dev) if w_dev is None else w_dev
    wg = exact_bin_sums(wsrc, torch.from_numpy(np.ascontiguousarray(pm.assignment, dtype=np.int64)).to(dev), n)
    return GpuTrafficGraph(n, pg, wg)


def per_gpu_send_traffic(gt: GpuTrafficGraph) -> TrafficReport:
    """Off-diagonal row fsums (traffic.py:87-95)."""
    send = np.array([math.fsum(np.delete(gt.pg[a], a)) for a in range(gt.n_gpus)], dtype=np.float64)
    return report_from_vector(send)


def peak_reduction(baseline: TrafficReport, candidate: TrafficReport) -> float:
    """Percent drop of the candidate peak below the baseline peak (traffic.py:98-106)."""
    if baseline.n_gpus != candidate.n_gpus:
        raise ValueError(
            f"reports cover different GPU counts: {baseline.n_gpus} vs {candidate.n_gpus}"
        )
    if baseline.peak == 0.0:
        raise ValueError("baseline peak is zero; reduction is undefined")
    return 100.0 * (baseline.peak - candidate.peak) / baseline.peak


def write_traffic_csv(report: TrafficReport, destination, value_column: str = "send_traffic") -> None:
    with open(destination, "w", newline="") as fh:
        out = csv.writer(fh, lineterminator="\n")
        out.writerow(["gpu", value_column])
        out.writerows([g, repr(v)] for g, v in enumerate(report.per_gpu_send.tolist()))


def read_traffic_csv(source) -> TrafficReport:
    with open(source, newline="") as fh:
        rows = list(csv.reader(fh))
    if not rows or len(rows[0]) != 2 or rows[0][0] != "gpu":
        raise ValueError(f"unexpected traffic CSV header in {source}")
    return report_from_vector([float(r[1]) for r in rows[1:]])


def write_traffic_summary(report: TrafficReport, destination) -> None:
    doc = {"peak": report.peak, "mean": report.mean, "stddev": report.stddev, "n_gpus": report.n_gpus}
    with open(destination, "w", newline="\n") as fh:
        json.dump(doc, fh, indent=2, sort_keys=True)
        fh.write("\n")
