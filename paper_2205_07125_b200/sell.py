"""J-SELL-32 pull-synapse layout (include/neurocomm_b200.h) -- host-side planning.

A slice is one warp's 32 consecutive local post rows.  For every (slice,
bitmap tile) block, lane l owns row 32*slice + l, which has len_l 16-byte
slots of 4 entries there: the excitatory pres fill slots [0, emid), the
inhibitory ones the next ceil(n_I/4) slots; row_meta = emid | (len_l << 16).
The block stores slot u of every lane with len > u contiguously, in lane
order (jagged: no padding to the longest row), so below the shortest row of
the block slot u of lane l sits at u*32 + l.  Entries are (q << 26) | id
with the pre id relative to the first id of the block's tile; unused entries
of a row's E/I segments hold the pad entry 0 (id 0, q = 0).

Builders fill the *padded* SELL-32 form first (block = longest row x 32 lanes,
slot u of lane l at padded_ptr + u*32 + l) and convert it (nc_sell_repack on
the device, :func:`jagged_gather` on the host).

Tiles: when the spike bitmap is larger than shared memory, it is staged in
tiles of ``tile_words`` words and every block only references pres of its
tile (csrc/sim_kernels.cu, ``k_step_fused<true, *>``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

ID_BITS = 26                       # unpacked builder entry: (q << 26) | tile-relative id
ID_MASK = (1 << ID_BITS) - 1
SLOT_ENTRIES = 5                   # packed slot: 5 fields of 25 bits, (q << 19) | tile-relative id
FIELD_ID_BITS = 19
BIT_XOR = 31                       # packed id stores 31 - (bit in word) in its low 5 bits
FIELD_MASK = (1 << 25) - 1
MAX_TILE_WORDS = 1 << (FIELD_ID_BITS - 5)   # 16384 words: tile-relative ids fit 19 bits
SMEM_BYTES = 227 * 1024            # opt-in dynamic shared memory per CTA on sm_100
SMEM_RESERVE = 2048                # static shared memory (tile claim counters, mbarriers) + slack


MAX_TILES = 256                    # csrc/sim_kernels.cu kMaxTiles
BALANCE_UNITS = 6                  # tiled kernel: (slice, tile) units per warp at least ...
BALANCE_MAX_TILES = 8              # ... up to this many tiles


SMEM_TILED = 160 * 1024            # tiled step: shared memory left to L1 for the loads in flight


def plan_tiles(n_words: int, n_local: int, n_sms: int) -> tuple[int, int, bool]:
    """(n_tiles, tile_words, partials_in_global) for a shard.

    One tile if the whole bitmap fits in shared memory.  Otherwise the tiled
    kernel double-buffers tiles (two buffers of ``tile_words``), next to the
    per-row partial sums of a CTA's rows; when those would take more than a
    quarter of shared memory (very large shards) they move to the global `acc`
    array instead (one extra integer reduction per row and tile).  The tiled
    kernel keeps its shared memory under SMEM_TILED: the rest of the SM's
    256 KB stays L1, which stages the synapse loads in flight (measured on
    B200 at 2/4 GPUs: 0.92/0.85 of HBM peak at 194 KB against 0.78/0.75 at
    227 KB; with the v5 kernel 152 KB beats 196 KB by 1.4 % at 2 GPUs and ties
    at 4, while every extra tile costs ~1 %).  Tiles are equal-sized.
    """
    budget_all = SMEM_BYTES - SMEM_RESERVE
    whole = (n_words + 3) // 4 * 4
    if whole <= MAX_TILE_WORDS and whole * 4 <= min(budget_all, SMEM_TILED):
        return 1, whole, False
    n_slices = (n_local + 31) // 32
    per = (n_slices + n_sms - 1) // n_sms
    part = per * 32 * 4
    global_part = part > budget_all // 4
    budget = min(budget_all, SMEM_TILED) - (0 if global_part else part)
    tw_max = min(MAX_TILE_WORDS, max(32, budget // 8 // 32 * 32))
    T = (n_words + tw_max - 1) // tw_max
    # small shards (strong scaling): warps claim (slice, tile) units dynamically, so with
    # few units per warp the last round leaves many warps idle.  Below BALANCE_UNITS
    # units per warp the blocks are split in two (block_split) and, if that is still
    # short, the bitmap is cut into more tiles (measured on the config-2 network over
    # 4 GPUs, 250 k rows/GPU: 2 tiles 0.79, split 0.84; 125 k rows/GPU: 2 tiles 0.61,
    # 8 tiles 0.66, 2 tiles split 0.73, 4 tiles split 0.74 of the copy peak)
    if n_slices * T < BALANCE_UNITS * n_sms * 32:
        T = max(T, min(BALANCE_MAX_TILES, -(-BALANCE_UNITS * n_sms * 32 // (2 * max(n_slices, 1)))))
    if T > MAX_TILES:
        raise ValueError(f"spike bitmap of {n_words} words needs {T} tiles (max {MAX_TILES})")
    tw = ((n_words + T - 1) // T + 31) // 32 * 32   # multiple of 32: both buffers start in bank 0
    return T, tw, global_part


def triple_buffer(n_local: int, n_tiles: int, tile_words: int, n_sms: int, partials_global: bool) -> bool:
    """Three tile buffers (nc_shard_t.flags bit 3) when a shard has 3+ tiles and they fit
    next to the partial sums under SMEM_TILED: the small tiles of small strong-scaling
    shards, where warps otherwise wait for the last warp of tile t before t + 2 loads."""
    if n_tiles < 3:
        return False
    per = ((n_local + 31) // 32 + n_sms - 1) // n_sms
    part = 0 if partials_global else per * 32 * 4
    return 3 * tile_words * 4 + part <= SMEM_TILED


def block_split(n_local: int, n_tiles: int, n_sms: int) -> int:
    """log2 of the parts each (slice, tile) block is split into for the warps' claims
    (nc_shard_t.flags bits 1-2; tiled kernel only): 1 below BALANCE_UNITS units per warp."""
    n_slices = (n_local + 31) // 32
    return 1 if n_tiles > 1 and n_slices * n_tiles < BALANCE_UNITS * n_sms * 32 else 0


def device_sms(device=None) -> int:
    import torch
    return torch.cuda.get_device_properties(device).multi_processor_count


@dataclass
class SellCSR:
    """One shard's pull synapses on the device."""

    slice_ptr: object      # torch int64 [n_slices*n_tiles + 1], J-SELL block starts, uint4 units
    row_meta: object       # torch int32 [n_tiles*n_local] by position: emid | (row slots << 16)
    syn: object            # torch int32 [4*slice_ptr[-1]] packed entries
    n_tiles: int
    tile_words: int
    n_local: int
    n_real: int            # real (non-pad) synapses
    dest: object = None    # torch int32 [n_local]: shards hosting targets of each row
    partials_global: bool = False
    row_perm: object = None  # torch int32 [n_tiles*n_local]: CTA-local index of the row at position p of
                             # tile t (None = identity; see include/neurocomm_b200.h)
    cta_groups: int = 1      # CTAs the tiled placement was built for
    has_pull: bool = True    # False: placeholders only (push-only network, event-driven engines)

    @property
    def n_entries(self) -> int:
        return int(self.syn.numel())


def tile_placement(lens, n_local: int, n_tiles: int, cta_groups: int):
    """Per-tile row placement for tiled layouts (include/neurocomm_b200.h).

    ``lens``: [n_local, n_tiles] slots of every row in every tile (numpy or
    torch).  Within the positions CTA c owns (slices s = c mod cta_groups, in
    slice then lane order) the rows of those same slices are placed in
    descending order of their tile-t length.  Returns (perm [n_tiles, n_local]
    position -> row, pos_of [n_local, n_tiles] row -> position), or
    (None, None) for one tile."""
    if n_tiles == 1:
        return None, None
    G = int(cta_groups)
    if _xp(lens) == "np":
        rows = np.arange(n_local, dtype=np.int64)
        cta = (rows >> 5) % G
        perm = np.empty((n_tiles, n_local), dtype=np.int32)
        pos_of = np.empty((n_local, n_tiles), dtype=np.int32)
        order_pos = np.lexsort((rows, cta))
        for t in range(n_tiles):
            order_rows = np.lexsort((rows, -np.asarray(lens[:, t], dtype=np.int64), cta))
            perm[t, order_pos] = order_rows
            pos_of[order_rows, t] = order_pos
        return perm, pos_of
    torch = _torch()
    dev = lens.device
    rows = torch.arange(n_local, dtype=torch.int64, device=dev)
    cta = (rows >> 5) % G
    lens = lens.to(torch.int64)
    span = int(lens.max().item()) + 1 if lens.numel() else 1
    perm = torch.empty((n_tiles, n_local), dtype=torch.int32, device=dev)
    pos_of = torch.empty((n_local, n_tiles), dtype=torch.int32, device=dev)
    order_pos = torch.argsort(cta * n_local + rows)
    for t in range(n_tiles):
        key = (cta * span + (span - 1 - lens[:, t])) * n_local + rows
        order_rows = torch.argsort(key)
        perm[t, order_pos] = order_rows.to(torch.int32)
        pos_of[order_rows, t] = order_pos.to(torch.int32)
    return perm, pos_of


def local_index(perm, cta_groups: int):
    """Placement rows -> CTA-local indices k = 32*(s div G) + row mod 32 (what row_perm stores)."""
    return ((perm >> 5) // cta_groups) * 32 + (perm & 31)


def row_slots(counts, n_local: int, n_tiles: int):
    """[n_local, n_tiles] slots per row and tile from per-(row, tile, sign) entry counts."""
    c = counts.reshape(n_local, n_tiles, 2)
    E = SLOT_ENTRIES
    return (c[:, :, 0] + E - 1) // E + (c[:, :, 1] + E - 1) // E


def layout_from_counts(counts, n_local: int, n_tiles: int, perm=None):
    """Padded SELL-32 block starts and (position-indexed) row_meta from
    per-(row, tile, sign) entry counts (torch or numpy int arrays) and the
    tile placement `perm` (None = identity); jagged_ptr(meta) gives the J-SELL
    starts."""
    xp = _xp(counts)
    c = counts.reshape(n_local, n_tiles, 2)
    if perm is not None:   # to position order: c[p, t] = counts of the row placed at p in tile t
        if xp == "np":
            c = c[np.asarray(perm, dtype=np.int64).T, np.arange(n_tiles)[None, :]]
        else:
            torch = _torch()
            c = c[perm.to(torch.int64).T, torch.arange(n_tiles, device=c.device)[None, :]]
    e_slots = (c[:, :, 0] + SLOT_ENTRIES - 1) // SLOT_ENTRIES
    i_slots = (c[:, :, 1] + SLOT_ENTRIES - 1) // SLOT_ENTRIES
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
        meta = (e_slots.T.reshape(-1).to(torch.int64) | (row_slots.T.reshape(-1).to(torch.int64) << 16)).to(torch.int32)
    else:
        ptr[1:] = np.cumsum(flat * 32)
        if row_slots.size and row_slots.max() > 0x7FFF:
            raise ValueError("row too long for 16-bit slot counts")
        meta = (e_slots.T.reshape(-1).astype(np.uint32) | (row_slots.T.reshape(-1).astype(np.uint32) << 16))
    return ptr, meta


def _block_lens(meta, n_local: int, n_tiles: int):
    """Row slot counts as [n_blocks, 32] (block = slice * n_tiles + tile), numpy or torch."""
    xp = _xp(meta)
    n_slices = (n_local + 31) // 32
    if xp == "np":
        lens = np.zeros((n_slices * 32, n_tiles), dtype=np.int64)
        lens[:n_local] = (np.asarray(meta).view(np.uint32) >> np.uint32(16)).astype(np.int64).reshape(n_tiles,
                                                                                                     n_local).T
        return lens.reshape(n_slices, 32, n_tiles).transpose(0, 2, 1).reshape(-1, 32)
    torch = _torch()
    lens = torch.zeros((n_slices * 32, n_tiles), dtype=torch.int64, device=meta.device)
    lens[:n_local] = ((meta.to(torch.int64) & 0xFFFFFFFF) >> 16).reshape(n_tiles, n_local).T
    return lens.reshape(n_slices, 32, n_tiles).permute(0, 2, 1).reshape(-1, 32)


def jagged_ptr(meta, n_local: int, n_tiles: int):
    """J-SELL block starts (uint4 units, n_blocks + 1) from row_meta."""
    lens = _block_lens(meta, n_local, n_tiles)
    if _xp(meta) == "np":
        out = np.zeros(lens.shape[0] + 1, dtype=np.int64)
        out[1:] = np.cumsum(lens.sum(axis=1))
        return out
    torch = _torch()
    out = torch.zeros(lens.shape[0] + 1, dtype=torch.int64, device=meta.device)
    out[1:] = torch.cumsum(lens.sum(1), 0)
    return out


def padded_ptr(meta, n_local: int, n_tiles: int):
    """Padded SELL-32 block starts (uint4 units): every block = longest row x 32."""
    lens = _block_lens(meta, n_local, n_tiles)
    if _xp(meta) == "np":
        out = np.zeros(lens.shape[0] + 1, dtype=np.int64)
        out[1:] = np.cumsum(lens.max(axis=1) * 32)
        return out
    torch = _torch()
    out = torch.zeros(lens.shape[0] + 1, dtype=torch.int64, device=meta.device)
    out[1:] = torch.cumsum(lens.max(1)[0] * 32, 0)
    return out


def jagged_gather(pptr: np.ndarray, meta: np.ndarray, n_local: int, n_tiles: int) -> np.ndarray:
    """For every J-SELL slot (in storage order), its position in the padded form (uint4 units)."""
    lens = _block_lens(meta, n_local, n_tiles)
    hi = lens.max(axis=1)
    n_pairs = int(hi.sum())
    b_idx = np.repeat(np.arange(lens.shape[0], dtype=np.int64), hi)
    u = np.arange(n_pairs, dtype=np.int64) - np.repeat(np.cumsum(hi) - hi, hi)
    act = lens[b_idx] > u[:, None]                                     # [pairs, 32]
    padded = np.asarray(pptr, dtype=np.int64)[b_idx][:, None] + u[:, None] * 32 + np.arange(32, dtype=np.int64)
    return padded[act]                                                 # row-major = storage order


def host_build(row, pre_internal, q, inh, n_local: int, n_tiles: int, tile_words: int, cta_groups: int = 148):
    """numpy J-SELL-32 arrays (slice_ptr, row_meta, syn, row_perm) from a synapse
    list (row = local post, pre internal id, q, inhibitory).  row_perm is the
    flattened [n_tiles, n_local] tile placement, None for one tile."""
    row = np.asarray(row, dtype=np.int64)
    pre = np.asarray(pre_internal, dtype=np.int64)
    tile = (pre >> 5) // tile_words
    seg = (row * n_tiles + tile) * 2 + np.asarray(inh, dtype=np.int64)
    counts = np.bincount(seg, minlength=n_local * n_tiles * 2).astype(np.int64)
    perm, pos_of = tile_placement(row_slots(counts, n_local, n_tiles), n_local, n_tiles, cta_groups)
    ptr, meta = layout_from_counts(counts, n_local, n_tiles, perm)
    emid = meta & np.uint32(0xFFFF)
    E = SLOT_ENTRIES
    syn = np.zeros(int(ptr[-1]) * E, dtype=np.uint32)   # unpacked, pad entry 0 (q = 0)
    order = np.argsort(seg, kind="stable")
    sseg = seg[order]
    first = np.cumsum(counts) - counts
    k = np.arange(sseg.size, dtype=np.int64) - first[sseg]
    r = sseg // 2 // n_tiles
    t = (sseg // 2) % n_tiles
    p = r if pos_of is None else pos_of[r, t].astype(np.int64)           # position of the row in tile t
    slot = np.where(sseg % 2 == 1, emid.astype(np.int64)[t * n_local + p], 0) + k // E
    pos = (ptr[(p // 32) * n_tiles + t] + slot * 32 + (p % 32)) * E + (k % E)
    rel = pre[order] - (pre[order] >> 5) // tile_words * tile_words * 32     # tile-relative id
    syn[pos] = (np.asarray(q, dtype=np.uint32)[order] << np.uint32(ID_BITS)) | rel.astype(np.uint32)
    packed = pack_slots(syn)
    gather = jagged_gather(ptr, meta, n_local, n_tiles)
    jsyn = packed.reshape(-1, 4)[gather].reshape(-1)
    return (jagged_ptr(meta, n_local, n_tiles), meta, jsyn,
            None if perm is None else local_index(perm, cta_groups).reshape(-1))


def pack_slots(unpacked: np.ndarray) -> np.ndarray:
    """numpy twin of nc_sell_pack: 5 unpacked entries (q << 26 | id) per slot -> 4 uint32 words."""
    e = np.asarray(unpacked, dtype=np.uint64).reshape(-1, SLOT_ENTRIES)
    f = ((e >> np.uint64(ID_BITS)) << np.uint64(FIELD_ID_BITS)) | \
        ((e & np.uint64((1 << FIELD_ID_BITS) - 1)) ^ np.uint64(BIT_XOR))
    lo = f[:, 0] | (f[:, 1] << np.uint64(25)) | ((f[:, 2] & np.uint64((1 << 14) - 1)) << np.uint64(50))
    hi = (f[:, 2] >> np.uint64(14)) | (f[:, 3] << np.uint64(11)) | (f[:, 4] << np.uint64(36))
    out = np.empty((e.shape[0], 4), dtype=np.uint32)
    out[:, 0] = (lo & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    out[:, 1] = (lo >> np.uint64(32)).astype(np.uint32)
    out[:, 2] = (hi & np.uint64(0xFFFFFFFF)).astype(np.uint32)
    out[:, 3] = (hi >> np.uint64(32)).astype(np.uint32)
    return out.reshape(-1)


def field_id(f):
    """Tile-relative pre id of packed fields (the low 5 bits store 31 - bit; jsell.cuh)."""
    return (f & ((1 << FIELD_ID_BITS) - 1)) ^ BIT_XOR


def unpack_slots(words):
    """Packed slots ([n, 4] int64 tensor of uint32 words) -> [n, 5] fields (torch)."""
    x, y, z, w = (words[:, i] for i in range(4))
    f = [x, (x >> 25) | (y << 7), (y >> 18) | (z << 14), (z >> 11) | (w << 21), w >> 4]
    import torch
    return torch.stack(f, 1) & FIELD_MASK


def to_padded(csr: SellCSR):
    """(padded_ptr, padded syn) of a SellCSR; slots past a row's length hold 0 (q = 0)."""
    torch = _torch()
    T, n_local = csr.n_tiles, csr.n_local
    pptr = padded_ptr(csr.row_meta, n_local, T)
    out = torch.zeros(max(int(pptr[-1].item()) * 4, 4), dtype=torch.int32, device=csr.syn.device)
    if csr.syn.is_cuda:
        from . import _native
        _native.check(_native.lib().nc_sell_repack(pptr.data_ptr(), csr.slice_ptr.data_ptr(),
                                                   csr.row_meta.data_ptr(), T, n_local, csr.syn.data_ptr(),
                                                   out.data_ptr(), 0, _native.stream_handle(csr.syn.device)),
                      "sell repack")
    else:
        g = jagged_gather(pptr.numpy(), csr.row_meta.numpy(), n_local, T)
        out.view(-1, 4)[torch.from_numpy(g)] = csr.syn[: g.size * 4].view(-1, 4)
    return pptr, out


def decode(csr: SellCSR):
    """Every real synapse of a SellCSR as torch tensors (row_local, pre_internal, q, inh)."""
    import torch
    ptr, syn = to_padded(csr)
    dev = syn.device
    T = csr.n_tiles
    n_blocks = ptr.numel() - 1
    blen = (ptr[1:] - ptr[:-1]) // 32                                        # slots per block
    total = int(ptr[-1].item())
    # slot index of every uint4 -> (block, slot u, lane)
    blk_of = torch.repeat_interleave(torch.arange(n_blocks, device=dev), blen * 32)
    off = torch.arange(total, device=dev, dtype=torch.int64) - ptr[:-1][blk_of]
    u, lane = off // 32, off % 32
    s, t = blk_of // T, blk_of % T
    pos = s * 32 + lane                                                     # position in its tile
    ent = unpack_slots(syn[: total * 4].view(-1, 4).to(torch.int64) & 0xFFFFFFFF)   # [total, 5] fields
    valid_row = pos < csr.n_local
    emid = torch.zeros_like(pos)
    emid[valid_row] = (csr.row_meta.to(torch.int64) & 0xFFFF)[t[valid_row] * csr.n_local + pos[valid_row]]
    row = pos.clone()
    if csr.row_perm is not None:   # CTA-local index k -> row (include/neurocomm_b200.h)
        G = csr.cta_groups
        k = csr.row_perm.to(torch.int64)[t[valid_row] * csr.n_local + pos[valid_row]]
        c = (pos[valid_row] >> 5) % G
        row[valid_row] = ((c + (k >> 5) * G) << 5) + (k & 31)
    inh = (u >= emid)
    q = ent >> FIELD_ID_BITS
    keep = (q > 0) & valid_row[:, None]
    rows5 = row[:, None].expand(-1, SLOT_ENTRIES)[keep]
    inh5 = inh[:, None].expand(-1, SLOT_ENTRIES)[keep]
    pre = field_id(ent) + (t * (csr.tile_words * 32))[:, None]   # back to internal ids
    return rows5, pre[keep], q[keep], inh5


def _xp(a):
    return "np" if isinstance(a, np.ndarray) else "torch"


def _torch():
    import torch
    return torch


def _zeros(xp, shape, like):
    if xp == "np":
        return np.zeros(shape, dtype=like.dtype)
    return _torch().zeros(shape, dtype=like.dtype, device=like.device)
