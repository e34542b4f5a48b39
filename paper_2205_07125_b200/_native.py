"""ctypes binding of libneurocomm_b200.so (include/neurocomm_b200.h).

The shared library is the only compute path: there is no Python or CPU
fallback for any entry point.  If the library is missing or was built for a
different ABI, every call raises ``RuntimeError`` naming the build command.
Tensors are passed as raw pointers (``tensor.data_ptr()``) together with the
current CUDA stream handle, so PyTorch only provides memory and streams.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_NAME = "libneurocomm_b200.so"
LIB_PATH = Path(__file__).resolve().parent / LIB_NAME
ABI_VERSION = 4

NC_OK, NC_E_ARG, NC_E_CUDA, NC_E_OVERFLOW, NC_E_TIMEOUT, NC_E_NCCL, NC_E_PARSE, NC_E_IO = range(8)
MAX_SHARDS = 16
INTERNAL_ID_BITS = 26

c_void_p, c_int32, c_int64, c_uint32, c_uint64, c_double, c_float = (
    C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_double, C.c_float)


class LifParamsC(C.Structure):
    _fields_ = [
        ("alpha_v", c_float), ("alpha_i", c_float), ("beta", c_float),
        ("v_rest", c_float), ("v_reset", c_float), ("v_th", c_float),
        ("w_unit", c_float), ("w_ext", c_float), ("v_init_span", c_float),
        ("ext_threshold", c_uint32), ("ext_lanes", c_int32), ("t_ref", c_int32),
        ("g_inh", c_int32), ("pad0", c_int32), ("seed", c_uint64),
    ]


class ShardC(C.Structure):
    _fields_ = [
        ("shard", c_int32), ("n_shards", c_int32), ("n_local", c_int32),
        ("local_base", c_int32), ("n_words", c_int32), ("n_tiles", c_int32), ("tile_words", c_int32),
        ("flags", c_int32),
        ("v", c_void_p), ("i_syn", c_void_p), ("refrac", c_void_p), ("acc", c_void_p),
        ("gid", c_void_p), ("hop_mask", c_void_p),
        ("slice_ptr", c_void_p), ("row_meta", c_void_p), ("syn", c_void_p),
        ("push_rowptr", c_void_p), ("push_syn", c_void_p),
        ("bitmap0", c_void_p), ("bitmap1", c_void_p),
        ("fired_ids", c_void_p), ("fired_count", c_void_p),
        ("bucket_ids", c_void_p), ("bucket_count", c_void_p), ("bucket_cap", c_int64),
        ("status", c_void_p), ("step", c_void_p),
        ("raster", c_void_p), ("record_steps", c_int32), ("local_words", c_int32),
        ("spike_total", c_void_p), ("work", c_void_p),
        ("row_perm", c_void_p), ("cta_groups", c_int32), ("pb_bins", c_int32),
        ("pb_rowptr", c_void_p), ("pb_binoff", c_void_p), ("pb_syn", c_void_p), ("pb_rows", c_int32),
        ("pad3", c_int32), ("spk_ids", c_void_p), ("spk_count", c_void_p), ("spk_cap", c_int64),
        ("kstamp", c_void_p), ("kstamp_steps", c_int32), ("pad4", c_int32),
        ("xsend", c_void_p * MAX_SHARDS), ("xsend_cap", c_int64), ("xsend_on", c_int32), ("xsend_mask", c_int32),
        ("push_winoff", c_void_p), ("push_windows", c_int32), ("push_window_rows", c_int32),
    ]


class GraphGenC(C.Structure):
    _fields_ = [
        ("n_neurons", c_int64), ("n_communities", c_int32), ("shard", c_int32),
        ("p_in", c_double), ("p_out", c_double),
        ("intra_lo", c_double), ("intra_hi", c_double),
        ("inter_lo", c_double), ("inter_hi", c_double),
        ("seed", c_uint64),
        ("owner", c_void_p), ("internal_id", c_void_p),
        ("local_base", c_int32), ("inh_every", c_int32),
        ("n_local", c_int32), ("pad0", c_int32),
    ]


class XchgC(C.Structure):
    _fields_ = [
        ("rank", c_int32), ("n", c_int32), ("cap", c_int32), ("two_level", c_int32),
        ("per_step", c_int32), ("lat_steps", c_int32),
        ("send1_mask", C.c_uint16), ("recv1_mask", C.c_uint16), ("send2_mask", C.c_uint16),
        ("recv2_mask", C.c_uint16),
        ("bucket_cap", c_int64), ("timeout_ns", c_uint64),
        ("step", c_void_p), ("status", c_void_p), ("bitmap0", c_void_p), ("bitmap1", c_void_p),
        ("bucket_ids", c_void_p), ("bucket_count", c_void_p), ("dest_global", c_void_p),
        ("shard_base", c_int64 * (MAX_SHARDS + 1)), ("fwd_row", C.c_uint16 * MAX_SHARDS),
        ("fwd_ids", c_void_p), ("fwd_count", c_void_p), ("hop_ids", c_void_p), ("deliv_ids", c_void_p),
        ("send_hdr", c_void_p), ("send2_hdr", c_void_p), ("recv_hdr", c_void_p), ("recv2_hdr", c_void_p),
        ("recv_ids", c_void_p), ("recv2_ids", c_void_p),
        ("my_inbox", c_void_p), ("my_flags", c_void_p),
        ("peer_inbox", c_void_p * MAX_SHARDS), ("peer_flags", c_void_p * MAX_SHARDS),
        ("done", c_void_p), ("send_done", c_void_p), ("blocks_per_peer", c_int32), ("pad1", c_int32),
        ("barrier", c_void_p), ("lat_start", c_void_p), ("lat_ns", c_void_p),
        ("spk_ids", c_void_p), ("spk_count", c_void_p), ("spk_cap", c_int64), ("dbg", c_void_p),
        ("fused_send", c_int32), ("pad2", c_int32),
    ]


_SIGS = {
    "nc_abi_version": (c_int32, []),
    "nc_last_error": (C.c_char_p, []),
    "nc_greedy_fill": (c_int32, [c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_int32, c_double, c_void_p]),
    "nc_greedy_fill_generated": (c_int32, [C.POINTER(GraphGenC), c_void_p, c_int32, c_double, c_void_p, c_int32]),
    "nc_hostgen_edges": (c_int64, [C.POINTER(GraphGenC), c_void_p, c_void_p, c_void_p, c_int32]),
    "nc_traffic_exponents": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    "nc_traffic_histogram": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int32,
                                       c_int32, c_int32, c_void_p, c_void_p]),
    "nc_traffic_histogram_packed": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int32, c_int32,
                                              c_int32, c_void_p, c_void_p]),
    "nc_traffic_histogram_uniform": (c_int32, [c_void_p, c_void_p, c_void_p, c_double, c_void_p, c_int64, c_int32,
                                               c_int32, c_int32, c_void_p, c_void_p]),
    "nc_edges_narrow": (c_int32, [c_void_p, c_void_p, c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_void_p,
                                  c_int32]),
    "nc_persistent_max_rows": (c_int64, []),
    "nc_assignment_u8": (c_int32, [c_void_p, c_int64, c_int32, c_void_p, c_void_p, c_void_p, c_void_p]),
    "nc_traffic_histogram32": (c_int32, [c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_int32,
                                       c_int32, c_int32, c_void_p, c_void_p]),
    "nc_weight_histogram": (c_int32, [c_void_p, c_void_p, c_int64, c_int32, c_int32, c_int32, c_void_p, c_void_p]),
    "nc_sim_init": (c_int32, [C.POINTER(ShardC), C.POINTER(LifParamsC), c_void_p]),
    "nc_sim_step_fused": (c_int32, [C.POINTER(ShardC), C.POINTER(LifParamsC), c_void_p]),
    "nc_sim_deliver_pull": (c_int32, [C.POINTER(ShardC), c_int32, c_void_p]),
    "nc_sim_deliver_push": (c_int32, [C.POINTER(ShardC), c_int32, c_void_p]),
    "nc_sim_prepare": (c_int32, []),
    "nc_sim_lif_update": (c_int32, [C.POINTER(ShardC), C.POINTER(LifParamsC), c_void_p]),
    "nc_sim_end_step": (c_int32, [C.POINTER(ShardC), c_void_p]),
    "nc_build_push_csr": (c_int32, [C.POINTER(ShardC), c_int32, c_void_p, c_void_p, c_void_p, c_void_p]),
    "nc_exchange_local": (c_int32, [C.POINTER(ShardC), c_int32, c_void_p, c_void_p, c_void_p, c_void_p,
                                    c_int64, c_void_p, c_void_p, c_int32, c_void_p]),
    "nc_graphgen_count": (c_int32, [C.POINTER(GraphGenC), c_int32, c_int32, c_void_p, c_void_p, c_void_p]),
    "nc_graphgen_fill": (c_int32, [C.POINTER(GraphGenC), c_int32, c_int32, c_void_p, c_void_p, c_void_p, c_void_p,
                                   c_void_p, c_void_p]),
    "nc_graphgen_degrees": (c_int32, [C.POINTER(GraphGenC), c_void_p, c_void_p]),
    "nc_graphgen_push": (c_int32, [C.POINTER(GraphGenC), c_int32, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "nc_traffic_histogram_generated": (c_int32, [C.POINTER(GraphGenC), c_void_p, c_void_p, c_int64, c_int64,
                                                 c_int32, c_int32, c_int32, c_void_p, c_void_p]),
    "nc_graphgen_push_windowed": (c_int32, [C.POINTER(GraphGenC), c_int32, c_int32, c_int32, c_void_p, c_void_p,
                                            c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "nc_edges_count": (c_int32, [C.POINTER(GraphGenC), c_void_p, c_void_p, c_int64, c_int32, c_int32, c_void_p,
                                 c_void_p]),
    "nc_edges_fill": (c_int32, [C.POINTER(GraphGenC), c_void_p, c_void_p, c_void_p, c_int64, c_int32, c_int32,
                                c_void_p, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "nc_sell_fill_pads": (c_int32, [c_void_p, c_int64, c_int32, c_int32, c_void_p, c_void_p]),
    "nc_dest_mask_from_csr": (c_int32, [c_void_p, c_void_p, c_void_p, c_int32, c_int32, c_int32, c_void_p, c_int32,
                                        c_void_p, c_int32, c_int32, c_void_p, c_void_p]),
    "nc_repair_balance": (c_int32, [c_int64, c_void_p, c_void_p, c_int32, c_double, c_void_p]),
    "nc_nng_scan": (c_int32, [C.c_char_p, c_void_p, c_void_p, c_void_p]),
    "nc_nng_read": (c_int32, [C.c_char_p, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_void_p, c_void_p]),
    "nc_nng_write": (c_int32, [C.c_char_p, c_int64, c_int64, c_void_p, c_void_p, c_void_p, c_void_p]),
    "nc_pmap_scan": (c_int32, [C.c_char_p, c_void_p, c_void_p, c_void_p]),
    "nc_pmap_read": (c_int32, [C.c_char_p, c_int64, c_int64, c_void_p, c_void_p]),
    "nc_pmap_write": (c_int32, [C.c_char_p, c_int64, c_int64, c_void_p]),
    "nc_build_push_binned": (c_int32, [C.POINTER(ShardC), c_int32, c_void_p, c_void_p, c_void_p, c_void_p,
                                       c_void_p, c_void_p]),
    "nc_sim_step_binned": (c_int32, [C.POINTER(ShardC), C.POINTER(LifParamsC), c_void_p]),
    "nc_sell_pack": (c_int32, [c_void_p, c_int64, c_void_p, c_void_p]),
    "nc_sell_bank_order": (c_int32, [c_void_p, c_void_p, c_int32, c_int32, c_void_p, c_void_p, c_void_p]),
    "nc_sell_repack": (c_int32, [c_void_p, c_void_p, c_void_p, c_int32, c_int32, c_void_p, c_void_p, c_int32,
                                 c_void_p]),
    "nc_xchg_reset": (c_int32, [C.POINTER(XchgC), c_void_p]),
    "nc_xchg_seal": (c_int32, [C.POINTER(XchgC), c_int32, c_void_p]),
    "nc_xchg_scatter": (c_int32, [C.POINTER(XchgC), c_int32, c_void_p]),
    "nc_xchg_p2p": (c_int32, [C.POINTER(XchgC), c_void_p]),
    "nc_nccl_get_unique_id": (c_int32, [c_void_p]),
    "nc_nccl_comm_init": (c_int32, [C.POINTER(c_void_p), c_int32, c_void_p, c_int32]),
    "nc_nccl_comm_destroy": (c_int32, [c_void_p]),
    "nc_nccl_exchange": (c_int32, [c_void_p, C.POINTER(XchgC), c_int32, c_void_p]),
    "nc_ipc_alloc": (c_int32, [C.c_size_t, C.POINTER(c_void_p), c_void_p]),
    "nc_ipc_open": (c_int32, [c_void_p, C.POINTER(c_void_p)]),
    "nc_ipc_close": (c_int32, [c_void_p]),
    "nc_free": (c_int32, [c_void_p]),
    "nc_stamp": (c_int32, [c_void_p, c_void_p, c_int32, c_void_p]),
    "nc_persistent_phase_stamps": (c_int32, [c_void_p]),
    "nc_run_persistent": (c_int32, [C.POINTER(ShardC), C.POINTER(LifParamsC), C.POINTER(XchgC), c_int32, c_int32,
                                    c_void_p, c_void_p, c_void_p, c_int32, c_void_p]),
}

_lib = None


def lib():
    """Load the engine once; raise loudly if it is absent or stale."""
    global _lib
    if _lib is not None:
        return _lib
    path = Path(os.environ.get("NEUROCOMM_B200_LIB", LIB_PATH))
    if not path.is_file():
        raise RuntimeError(
            f"{path} not found: the CUDA engine is required (no CPU fallback). "
            "Build it with `python -c 'import __graft_entry__ as g; g.build()'` or "
            "`make -C paper_2205_07125_b200/csrc`."
        )
    handle = C.CDLL(str(path), mode=C.RTLD_GLOBAL)
    for name, (res, args) in _SIGS.items():
        fn = getattr(handle, name)
        fn.restype = res
        fn.argtypes = args
    got = handle.nc_abi_version()
    if got != ABI_VERSION:
        raise RuntimeError(f"{path} has ABI {got}, expected {ABI_VERSION}; rebuild it")
    _lib = handle
    return _lib


OPS_PATH = Path(__file__).resolve().parent / "libneurocomm_b200_torch.so"
_ops = None


def ops():
    """torch.ops.neurocomm_b200: the thin PyTorch extension (csrc/torch_ops.cpp) through
    which the simulators launch every per-step kernel.  Loaded once; raises loudly if
    it is absent (no fallback)."""
    global _ops
    if _ops is not None:
        return _ops
    import torch
    lib()   # the engine it links against, loaded and ABI-checked first
    # next to the engine (its rpath is $ORIGIN): an engine build elsewhere
    # (NEUROCOMM_B200_LIB, kernel A/Bs) comes with its own extension build
    path = Path(os.environ["NEUROCOMM_B200_LIB"]).with_name(OPS_PATH.name) if "NEUROCOMM_B200_LIB" in os.environ \
        else OPS_PATH
    if not path.is_file():
        raise RuntimeError(f"{path} not found: build it with `make -C paper_2205_07125_b200/csrc` "
                           "(or __graft_entry__.build())")
    torch.ops.load_library(str(path))
    o = torch.ops.neurocomm_b200
    if int(o.abi_version()) != ABI_VERSION:
        raise RuntimeError(f"{path} was built against ABI {int(o.abi_version())}, expected {ABI_VERSION}")
    _ops = o
    return _ops


def as_bytes(obj):
    """A uint8 CPU tensor viewing a ctypes struct / array (no copy: later field writes show)."""
    import torch
    return torch.frombuffer(obj, dtype=torch.uint8)


def exported_symbols() -> list[str]:
    return sorted(_SIGS)


def check(rc: int, what: str, err_line=None) -> None:
    """Translate a non-zero NC_E* code into the reference's exception types
    (NC_E_PARSE -> ParseError(message, line) with the reference's message)."""
    if rc == NC_OK:
        return
    msg = (lib().nc_last_error() or b"").decode(errors="replace")
    if rc == NC_E_PARSE:
        from .errors import ParseError
        raise ParseError(msg, int(err_line.value) if err_line is not None else 0)
    if rc == NC_E_IO:
        raise OSError(msg)
    if rc == NC_E_ARG:
        raise ValueError(f"{what}: {msg}")
    raise RuntimeError(f"{what} failed (code {rc}): {msg}")


def ptr(t) -> int | None:
    """Device/host pointer of a tensor or numpy array (None passes NULL)."""
    if t is None:
        return None
    if hasattr(t, "data_ptr"):
        return t.data_ptr()
    return t.ctypes.data


def stream_handle(device=None) -> int:
    import torch
    return torch.cuda.current_stream(device).cuda_stream
