"""SELL-32 pull-synapse layout (include/neurocomm_b200.h) -- host-side planning.

A slice is one warp's 32 consecutive local post rows.  For every (slice,
bitmap tile) block, lane l owns row 32*slice + l and reads slot u at
``slice_ptr[block] + 32*u + l`` (16-byte words of 4 entries).  Within a row's
part of a block, the excitatory pres fill slots [0, emid), the inhibitory
ones the next ceil(n_I/4) slots (row length len_r); row_meta = emid |
(len_r << 16).  Lanes never load past their own len_r; storage past it (up
to the block's longest row) holds pad entries (q = 0 and the tile's first id).

Tiles: when the spike bitmap is larger than shared memory, it is staged in
tiles of ``tile_words`` words and every block only references pres of its
tile (csrc/sim_kernels.cu, ``k_step_fused<true, *>``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

ID_BITS = 26
ID_MASK = (1 << ID_BITS) - 1
SMEM_BYTES = 227 * 1024            # opt-in dynamic shared memory per CTA on sm_100
SMEM_RESERVE = 1024                # static shared memory + slack


def plan_tiles(n_words: int, n_local: int, n_sms: int) -> tuple[int, int, bool]:
    """(n_tiles, tile_words, partials_in_global) for a shard.

    One tile if the whole bitmap fits in shared memory.  Otherwise the per-row
    partial sums of a CTA's rows share the shared memory with the tile; when
    they would take more than a quarter of it (very large shards) they move to
    the global `acc` array instead (one extra 8-byte read-modify-write per row
    and tile).
    """
    budget_all = SMEM_BYTES - SMEM_RESERVE
    whole = (n_words + 3) // 4 * 4
    if whole * 4 <= budget_all:
        return 1, whole, False
    n_slices = (n_local + 31) // 32
    per = (n_slices + n_sms - 1) // n_sms
    part = per * 32 * 4
    global_part = part > budget_all // 4
    budget = budget_all - (0 if global_part else part)
    tw = budget // 4 // 4 * 4
    return (n_words + tw - 1) // tw, tw, global_part


def device_sms(device=None) -> int:
    import torch
    return torch.cuda.get_device_properties(device).multi_processor_count


@dataclass
class SellCSR:
    """One shard's pull synapses on the device."""

    slice_ptr: object      # torch int64 [n_slices*n_tiles + 1], uint4 units
    row_meta: object       # torch int32 [n_local*n_tiles]: emid | (row slots << 16)
    syn: object            # torch int32 [4*slice_ptr[-1]] packed entries
    n_tiles: int
    tile_words: int
    n_local: int
    n_real: int            # real (non-pad) synapses
    dest: object = None    # torch int32 [n_local]: shards hosting targets of each row
    partials_global: bool = False

    @property
    def n_entries(self) -> int:
        return int(self.syn.numel())


def layout_from_counts(counts, n_local: int, n_tiles: int):
    """slice_ptr, row_meta from per-(row, tile, sign) entry counts (torch or numpy int arrays)."""
    xp = _xp(counts)
    c = counts.reshape(n_local, n_tiles, 2)
    e_slots = (c[:, :, 0] + 3) // 4
    i_slots = (c[:, :, 1] + 3) // 4
    row_slots = e_slots + i_slots
    n_slices = (n_local + 31) // 32
    padded = _zeros(xp, (n_slices * 32, n_tiles), like=row_slots)
    padded[:n_local] = row_slots
    blk = padded.reshape(n_slices, 32, n_tiles).max(1)[0] if xp == "torch" else \
        padded.reshape(n_slices, 32, n_tiles).max(axis=1)
    flat = blk.reshape(-1).astype("int64") if xp == "np" else blk.reshape(-1).to(_torch().int64)
    ptr = _zeros(xp, (n_slices * n_tiles + 1,), like=flat)
    if xp == "torch":
        torch = _torch()
        ptr[1:] = torch.cumsum(flat * 32, 0)
        if row_slots.numel() and int(row_slots.max().item()) > 0x7FFF:
            raise ValueError("row too long for 16-bit slot counts")
        meta = (e_slots.reshape(-1).to(torch.int64) | (row_slots.reshape(-1).to(torch.int64) << 16)).to(torch.int32)
    else:
        ptr[1:] = np.cumsum(flat * 32)
        if row_slots.size and row_slots.max() > 0x7FFF:
            raise ValueError("row too long for 16-bit slot counts")
        meta = (e_slots.reshape(-1).astype(np.uint32) | (row_slots.reshape(-1).astype(np.uint32) << 16))
    return ptr, meta


def host_build(row, pre_internal, q, inh, n_local: int, n_tiles: int, tile_words: int):
    """numpy SELL-32 arrays from a synapse list (row = local post, pre internal id, q, inhibitory)."""
    row = np.asarray(row, dtype=np.int64)
    pre = np.asarray(pre_internal, dtype=np.int64)
    tile = (pre >> 5) // tile_words
    seg = (row * n_tiles + tile) * 2 + np.asarray(inh, dtype=np.int64)
    counts = np.bincount(seg, minlength=n_local * n_tiles * 2).astype(np.int64)
    ptr, meta = layout_from_counts(counts, n_local, n_tiles)
    emid = meta & np.uint32(0xFFFF)
    syn = np.zeros(int(ptr[-1]) * 4, dtype=np.uint32)
    n_blocks = ptr.size - 1
    for b in range(n_tiles if n_tiles > 1 else 0):  # pad = first id of the block's tile
        pad = np.uint32(b * tile_words * 32)
        for blk in range(b, n_blocks, n_tiles):
            syn[ptr[blk] * 4: ptr[blk + 1] * 4] = pad
    order = np.argsort(seg, kind="stable")
    sseg = seg[order]
    first = np.cumsum(counts) - counts
    k = np.arange(sseg.size, dtype=np.int64) - first[sseg]
    r = sseg // 2 // n_tiles
    t = (sseg // 2) % n_tiles
    slot = np.where(sseg % 2 == 1, emid.astype(np.int64)[r * n_tiles + t], 0) + k // 4
    pos = (ptr[(r // 32) * n_tiles + t] + slot * 32 + (r % 32)) * 4 + (k % 4)
    syn[pos] = (np.asarray(q, dtype=np.uint32)[order] << np.uint32(ID_BITS)) | pre[order].astype(np.uint32)
    return ptr, meta, syn


def decode(csr: SellCSR):
    """Every real synapse of a device SellCSR as torch tensors (row_local, pre_internal, q, inh)."""
    import torch
    dev = csr.syn.device
    T = csr.n_tiles
    ptr = csr.slice_ptr
    n_blocks = ptr.numel() - 1
    blen = (ptr[1:] - ptr[:-1]) // 32                                        # slots per block
    total = int(ptr[-1].item())
    # slot index of every uint4 -> (block, slot u, lane)
    blk_of = torch.repeat_interleave(torch.arange(n_blocks, device=dev), blen * 32)
    off = torch.arange(total, device=dev, dtype=torch.int64) - ptr[:-1][blk_of]
    u, lane = off // 32, off % 32
    s, t = blk_of // T, blk_of % T
    row = s * 32 + lane
    ent = csr.syn[: total * 4].view(-1, 4).to(torch.int64) & 0xFFFFFFFF      # [total, 4]
    valid_row = row < csr.n_local
    emid = torch.zeros_like(row)
    emid[valid_row] = (csr.row_meta.to(torch.int64) & 0xFFFF)[row[valid_row] * T + t[valid_row]]
    inh = (u >= emid)
    q = ent >> ID_BITS
    keep = (q > 0) & valid_row[:, None]
    rows4 = row[:, None].expand(-1, 4)[keep]
    inh4 = inh[:, None].expand(-1, 4)[keep]
    return rows4, (ent & ID_MASK)[keep], q[keep], inh4


def _xp(a):
    return "np" if isinstance(a, np.ndarray) else "torch"


def _torch():
    import torch
    return torch


def _zeros(xp, shape, like):
    if xp == "np":
        return np.zeros(shape, dtype=like.dtype)
    return _torch().zeros(shape, dtype=like.dtype, device=like.device)
