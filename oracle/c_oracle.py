"""ctypes wrapper of oracle/build/libsim_oracle.so -- TEST INFRASTRUCTURE ONLY."""

from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "build" / "libsim_oracle.so"


class OracleLif(C.Structure):
    _fields_ = [(n, C.c_float) for n in ("alpha_v", "alpha_i", "beta", "v_rest", "v_reset", "v_th",
                                         "w_unit", "w_ext", "v_init_span")] + [
        ("ext_threshold", C.c_uint32), ("ext_lanes", C.c_int32), ("t_ref", C.c_int32),
        ("g_inh", C.c_int32), ("inh_every", C.c_int32), ("seed", C.c_uint64)]


_lib = None


def load():
    global _lib
    if _lib is None:
        if not LIB.is_file():
            subprocess.run(["make", "-C", str(HERE)], check=True, capture_output=True)
        _lib = C.CDLL(str(LIB))
        _lib.oracle_simulate.restype = C.c_int
        _lib.oracle_philox.restype = None
    return _lib


def philox(ctr, seed: int):
    c = (C.c_uint32 * 4)(*[int(x) & 0xFFFFFFFF for x in ctr])
    out = (C.c_uint32 * 4)()
    load().oracle_philox(c, C.c_uint64(seed), out)
    return list(out)


def _p(a):
    return C.c_void_p(a.ctypes.data) if a is not None else None


def simulate_csr(rowptr, col, q, owner, n_shards, next_hop, lif: dict, steps: int, *, threads: int = 0,
                 raster=True, counts=True):
    """Run the C oracle on a symmetric gid-space CSR; returns a dict of outputs."""
    M = int(rowptr.size - 1)
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    q = np.ascontiguousarray(q, dtype=np.uint8)
    owner = np.ascontiguousarray(owner, dtype=np.int32)
    nh = np.ascontiguousarray(np.asarray(next_hop).reshape(-1), dtype=np.int32)
    prm = OracleLif(**{k: lif[k] for k, _ in OracleLif._fields_})
    ras = np.zeros((steps, M), dtype=np.uint8) if raster else None
    dl = np.zeros((steps, n_shards, n_shards), dtype=np.int64) if counts else None
    hp = np.zeros((steps, n_shards, n_shards), dtype=np.int64) if counts else None
    v = np.zeros(M, dtype=np.float32)
    i = np.zeros(M, dtype=np.float32)
    rc = load().oracle_simulate(C.c_int64(M), _p(rowptr), _p(col), _p(q), _p(owner), C.c_int32(n_shards),
                                _p(nh), C.byref(prm), C.c_int32(steps), C.c_int32(threads), _p(ras), _p(dl),
                                _p(hp), _p(v), _p(i))
    if rc != 0:
        raise ValueError("oracle: a neuron targets a shard with no next hop in the routing table")
    return {"raster": None if ras is None else ras.astype(bool), "deliv": dl, "hop": hp, "v": v, "i": i}


def symmetric_csr(n, edge_i, edge_j, q_edge):
    """Row = post, cols = pre (both directions of every edge), rows in gid order."""
    rows = np.concatenate([edge_j, edge_i]).astype(np.int64)
    cols = np.concatenate([edge_i, edge_j]).astype(np.int64)
    qq = np.concatenate([q_edge, q_edge]).astype(np.uint8)
    order = np.argsort(rows, kind="stable")
    rowptr = np.zeros(n + 1, dtype=np.int64)
    rowptr[1:] = np.cumsum(np.bincount(rows, minlength=n))
    return rowptr, cols[order].astype(np.int32), qq[order]


def generate_sbm_csr(n, n_comm, p_in, p_out, seed, *, intra=(0.5, 1.0), inter=(0.05, 0.5), threads=0):
    """CPU restatement of the device SBM generator: symmetric gid-space CSR (rowptr, col, q)."""
    lib = load()
    lib.oracle_generate_sbm.restype = C.c_int64
    args = [C.c_int64(n), C.c_int64(n_comm), C.c_double(p_in), C.c_double(p_out), C.c_double(intra[0]),
            C.c_double(intra[1]), C.c_double(inter[0]), C.c_double(inter[1]), C.c_uint64(seed), C.c_int32(threads)]
    rowptr = np.zeros(n + 1, dtype=np.int64)
    nnz = lib.oracle_generate_sbm(*args, _p(rowptr), None, None)
    col = np.empty(nnz, dtype=np.int32)
    q = np.empty(nnz, dtype=np.uint8)
    lib.oracle_generate_sbm(*args, _p(rowptr), _p(col), _p(q))
    return rowptr, col, q


def generate_random_csr(n, degree, seed, *, threads=0):
    return generate_sbm_csr(n, 1, degree / max(n - 1, 1), 0.0, seed, threads=threads)
