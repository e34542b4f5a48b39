"""The C-ABI library loads and exports every symbol include/neurocomm_b200.h declares (no GPU needed)."""

from __future__ import annotations

import ctypes
import re
import subprocess
from pathlib import Path

import numpy as np

from paper_2205_07125_b200 import _native

ROOT = Path(__file__).resolve().parents[1]


def header_symbols() -> set[str]:
    text = (ROOT / "include" / "neurocomm_b200.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return set(re.findall(r"\b(nc_[a-z0-9_]+)\s*\(", text))


def test_library_exports_header():
    lib = _native.lib()
    declared = header_symbols()
    assert declared, "no symbols parsed from the header"
    out = subprocess.run(["nm", "-D", "--defined-only", str(_native.LIB_PATH)], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (nc_[a-z0-9_]+)", out))
    assert declared <= exported, declared - exported
    assert declared <= set(_native.exported_symbols()) | {"nc_abi_version", "nc_last_error"}
    assert lib.nc_abi_version() == _native.ABI_VERSION


def test_struct_layout_matches_header():
    # sizes the C side sees are fixed by the header; ctypes mirrors must agree
    assert ctypes.sizeof(_native.LifParamsC) == 64
    assert ctypes.sizeof(_native.ShardC) % 8 == 0


def test_error_path_host_entry_point():
    lib = _native.lib()
    out = np.zeros(3, dtype=np.int64)
    rc = lib.nc_greedy_fill(3, np.ones(3).ctypes.data, np.zeros(4, dtype=np.int64).ctypes.data, None, None, 5,
                            1.0, out.ctypes.data)
    assert rc == _native.NC_E_ARG
    assert b"n_buckets" in lib.nc_last_error()


def test_struct_field_offsets_match_header(tmp_path):
    """Every ctypes mirror field sits at the offset the C compiler gives it in the header
    (offsetof over a generated translation unit, compiled with gcc here)."""
    structs = {"nc_lif_params_t": _native.LifParamsC, "nc_shard_t": _native.ShardC,
               "nc_graphgen_t": _native.GraphGenC, "nc_xchg_t": _native.XchgC}
    lines = ["#include <stdio.h>", "#include <stddef.h>", '#include "neurocomm_b200.h"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append(f'printf("{cname} size %zu\\n", sizeof({cname}));')
        for f in py._fields_:
            lines.append(f'printf("{cname} {f[0]} %zu\\n", offsetof({cname}, {f[0]}));')
    lines += ["return 0; }"]
    src = tmp_path / "offsets.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "offsets"
    subprocess.run(["gcc", "-std=c11", "-I", str(ROOT / "include"), str(src), "-o", str(exe)], check=True)
    got = {}
    for ln in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.splitlines():
        cname, field, off = ln.split()
        got[(cname, field)] = int(off)
    for cname, py in structs.items():
        assert got[(cname, "size")] == ctypes.sizeof(py), cname
        for f in py._fields_:
            assert got[(cname, f[0])] == getattr(py, f[0]).offset, (cname, f[0])


OPS = ["abi_version", "sim_init", "sim_step_fused", "sim_step_binned", "sim_deliver_push", "sim_deliver_pull",
       "sim_lif_update", "sim_end_step", "exchange_local", "xchg_p2p", "xchg_seal", "xchg_scatter",
       "nccl_exchange", "stamp", "run_persistent"]


def test_torch_extension_registers_the_step_ops():
    """The thin PyTorch extension (csrc/torch_ops.cpp) loads and registers every step-loop
    op; a bad descriptor is refused before anything reaches the GPU (ValueError, as the
    C-ABI path raises for NC_E_ARG)."""
    import pytest
    import torch
    o = _native.ops()
    for name in OPS:
        assert hasattr(o, name), name
    assert int(o.abi_version()) == _native.ABI_VERSION
    shard = _native.as_bytes(_native.ShardC())          # all zero: no step / status buffers
    with pytest.raises(ValueError, match="invalid nc_shard_t"):
        o.sim_end_step(shard, 0)
    with pytest.raises(RuntimeError, match="bytes"):
        o.sim_end_step(torch.zeros(3, dtype=torch.uint8), 0)


def test_edges_narrow_host_pass():
    """nc_edges_narrow (the host half of sim.upload_edges, CPU only): int64 ids -> int32,
    fp64 p -> q_from_p's uint8 weight units, every thread split; out-of-range ids -> NC_E_ARG."""
    import numpy as np
    from paper_2205_07125_b200 import _native, sim as S
    L = _native.lib()
    rng = np.random.default_rng(5)
    for n, threads in ((1, 0), (70_001, 3), (300_000, 0)):
        m = 9_000
        ei = rng.integers(0, m, n).astype(np.int64)
        ej = rng.integers(0, m, n).astype(np.int64)
        p = rng.uniform(0.0, 1.0, n)
        p[: min(n, 6)] = [1e-300, 1 / 32, 0.5, 1.0, 31 / 32, 1 - 1e-16][: min(n, 6)]
        oi, oj, oq = np.empty(n, np.int32), np.empty(n, np.int32), np.empty(n, np.uint8)
        rc = L.nc_edges_narrow(ei.ctypes.data, ej.ctypes.data, p.ctypes.data, n, m, oi.ctypes.data, oj.ctypes.data,
                               oq.ctypes.data, threads)
        assert rc == 0
        np.testing.assert_array_equal(oi, ei)
        np.testing.assert_array_equal(oj, ej)
        np.testing.assert_array_equal(oq, S.q_from_p(p))
        ej[n // 2] = m
        assert L.nc_edges_narrow(ei.ctypes.data, ej.ctypes.data, p.ctypes.data, n, m, oi.ctypes.data,
                                 oj.ctypes.data, oq.ctypes.data, threads) != 0
        ej[n // 2] = 0
        ei[n - 1] = -1
        assert L.nc_edges_narrow(ei.ctypes.data, ej.ctypes.data, p.ctypes.data, n, m, oi.ctypes.data,
                                 oj.ctypes.data, oq.ctypes.data, threads) != 0
