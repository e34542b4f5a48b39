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
