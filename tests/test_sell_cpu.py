"""SELL-32 layout (host builder + decoder) on CPU: every synapse lands in its
row's lane, in its tile's block, E before I, pads carry q = 0."""

from __future__ import annotations

import numpy as np
import pytest
import torch

from paper_2205_07125_b200 import sell


@pytest.mark.parametrize("n_local,n_tiles,tile_words", [(70, 1, 64), (100, 3, 8), (33, 2, 4), (5, 4, 4)])
def test_host_build_round_trip(n_local, n_tiles, tile_words):
    rng = np.random.default_rng(n_local)
    n_ids = n_tiles * tile_words * 32
    m = 40 * n_local
    row = rng.integers(0, n_local, m)
    pre = rng.integers(0, n_ids, m)
    q = rng.integers(1, 33, m)
    inh = rng.random(m) < 0.2
    ptr, meta, syn, perm = sell.host_build(row, pre, q, inh, n_local, n_tiles, tile_words, cta_groups=2)
    assert ptr[-1] * 4 == syn.size
    csr = sell.SellCSR(torch.from_numpy(ptr), torch.from_numpy(meta.view(np.int32)),
                       torch.from_numpy(syn.view(np.int32)), n_tiles, tile_words, n_local, m,
                       row_perm=None if perm is None else torch.from_numpy(perm), cta_groups=2)
    r2, p2, q2, i2 = (x.numpy() for x in sell.decode(csr))
    a = np.stack([row, pre, q, inh]).T
    b = np.stack([r2, p2, q2, i2]).T
    a = a[np.lexsort(a.T[::-1])]
    b = b[np.lexsort(b.T[::-1])]
    np.testing.assert_array_equal(a, b)
    # jagged blocks hold exactly their positions' slots; every row's slots hold its
    # E entries, then its I entries, each segment padded to a multiple of 5
    if perm is None:
        perm2 = np.tile(np.arange(n_local), (n_tiles, 1))
    else:   # CTA-local index -> row
        k = perm.reshape(n_tiles, n_local).astype(np.int64)
        c = (np.arange(n_local) >> 5) % 2
        perm2 = ((c + (k >> 5) * 2) << 5) + (k & 31)
    lens = (meta >> np.uint32(16)).astype(np.int64).reshape(n_tiles, n_local).T     # by position
    emid = (meta & np.uint32(0xFFFF)).astype(np.int64).reshape(n_tiles, n_local).T
    pad_rows = np.zeros(((n_local + 31) // 32 * 32, n_tiles), dtype=np.int64)
    pad_rows[:n_local] = lens
    np.testing.assert_array_equal(pad_rows.reshape(-1, 32, n_tiles).sum(axis=1).reshape(-1), np.diff(ptr))
    seg = (row * n_tiles + (pre >> 5) // tile_words) * 2 + inh
    cnt = np.bincount(seg, minlength=n_local * n_tiles * 2).reshape(n_local, n_tiles, 2)
    for t in range(n_tiles):
        r = perm2[t]
        np.testing.assert_array_equal(emid[:, t], (cnt[r, t, 0] + 4) // 5)
        np.testing.assert_array_equal(lens[:, t] - emid[:, t], (cnt[r, t, 1] + 4) // 5)
        # placement: a permutation that keeps every row inside its CTA's slices,
        # in descending tile-t length within each CTA
        assert sorted(r.tolist()) == list(range(n_local))
        np.testing.assert_array_equal((r >> 5) % 2, (np.arange(n_local) >> 5) % 2)
        for c in range(2):
            own = np.nonzero((np.arange(n_local) >> 5) % 2 == c)[0]
            assert (np.diff(lens[own, t]) <= 0).all() or n_tiles == 1
    # fields of a tile block hold ids relative to the tile (they index the staged copy)
    f = sell.unpack_slots(torch.from_numpy(syn.astype(np.int64)).view(-1, 4))
    assert (sell.field_id(f) < tile_words * 32).all()
    assert int((f >> sell.FIELD_ID_BITS > 0).sum()) == m


def test_pack_slots_bit_layout():
    """Field i of a slot sits at bit 25 i of x | y<<32 | z<<64 | w<<96 (include/neurocomm_b200.h)."""
    rng = np.random.default_rng(2)
    q = rng.integers(0, 33, (50, 5))
    ids = rng.integers(0, 1 << 19, (50, 5))
    unpacked = ((q << 26) | ids).astype(np.uint32)
    words = sell.pack_slots(unpacked.reshape(-1)).reshape(-1, 4).astype(object)
    for s_ in range(50):
        v = sum(int(words[s_, i]) << (32 * i) for i in range(4))
        for i in range(5):
            assert (v >> (25 * i)) & ((1 << 25) - 1) == (int(q[s_, i]) << 19) | (int(ids[s_, i]) ^ 31)
    f = sell.unpack_slots(torch.from_numpy(sell.pack_slots(unpacked.reshape(-1)).astype(np.int64)).view(-1, 4))
    np.testing.assert_array_equal(f.numpy(), (q << 19) | (ids ^ 31))
    np.testing.assert_array_equal(sell.field_id(f).numpy(), ids)


def test_jagged_positions_match_the_formula():
    """position(u, l) = sum_{v<u} cnt_v + #{l' < l: len_l' > u} (include/neurocomm_b200.h)."""
    rng = np.random.default_rng(3)
    n_local, T = 70, 2
    lens = rng.integers(0, 9, (n_local, T))
    meta = (lens.T.astype(np.uint32) << np.uint32(16)).reshape(-1)   # tile-major
    pptr = sell.padded_ptr(meta, n_local, T)
    jptr = sell.jagged_ptr(meta, n_local, T)
    g = sell.jagged_gather(pptr, meta, n_local, T)
    assert g.size == jptr[-1] == lens.sum()
    for b in range(jptr.size - 1):
        s, t = divmod(b, T)
        L = np.zeros(32, dtype=np.int64)
        rows = np.arange(s * 32, min(s * 32 + 32, n_local))
        L[: rows.size] = lens[rows, t]
        for u in range(L.max(initial=0)):
            for l in np.nonzero(L > u)[0]:
                pos = sum(int((L > v).sum()) for v in range(u)) + int((L[:l] > u).sum())
                assert g[jptr[b] + pos] == pptr[b] + u * 32 + l


def test_plan_tiles():
    assert sell.plan_tiles(1000, 10_000, 148) == (1, 1000, False)
    T, tw, _ = sell.plan_tiles(31_252, 1_000_000, 148)   # config 2: two tiles (ids fit 19 bits)
    assert T == 2 and tw <= sell.MAX_TILE_WORDS
    T, tw, glob = sell.plan_tiles(312_500 + 1, 1_250_000, 148)    # 10 M neurons, 1.25 M local
    assert T > 1 and tw % 4 == 0 and T * tw >= 312_501 and not glob
    per = (1_250_000 // 32 + 147) // 148
    assert 2 * tw * 4 + per * 128 <= sell.SMEM_TILED
    T, tw, glob = sell.plan_tiles(1_562_500 + 1, 12_500_000, 148)  # 50 M neurons, 12.5 M local
    assert glob and T * tw >= 1_562_501 and 2 * tw * 4 <= sell.SMEM_BYTES - sell.SMEM_RESERVE


def test_triple_buffer_choice():
    # 3 buffers only for 3+ tiles that fit next to the partial sums under SMEM_TILED:
    # config 2 over 8 GPUs (4 tiles of 7 840 words) yes; 1 GPU (2 tiles) and config 3 on
    # one GPU (20 tiles of 15 648 words, 188 KB for three) no
    assert sell.triple_buffer(125_000, 4, 7_840, 148, False)
    assert not sell.triple_buffer(1_000_000, 2, 15_648, 148, False)
    assert not sell.triple_buffer(10_000_000, 20, 15_648, 148, True)
    assert sell.triple_buffer(5_000, 5, 64, 148, False)


def test_small_shard_balance():
    # strong scaling of the config-2 network: 1 / 2 GPUs unchanged, 4 GPUs split blocks,
    # 8 GPUs split blocks over 4 tiles (>= BALANCE_UNITS claim units per warp)
    for n_local, want_T, want_split in ((1_000_000, 2, 0), (500_000, 2, 0), (250_000, 2, 1), (125_000, 4, 1)):
        T, tw, glob = sell.plan_tiles(31_250, n_local, 148)
        assert (T, sell.block_split(n_local, T, 148), glob) == (want_T, want_split, False)
        units = (n_local + 31) // 32 * T << sell.block_split(n_local, T, 148)
        assert units >= sell.BALANCE_UNITS * 148 * 32 or T == sell.BALANCE_MAX_TILES
    assert sell.block_split(1000, 1, 148) == 0   # one-tile kernel: never split


def test_layout_from_counts_torch_matches_numpy():
    rng = np.random.default_rng(1)
    counts = rng.integers(0, 50, (77 * 3 * 2,))
    p1, e1 = sell.layout_from_counts(counts, 77, 3)
    p2, e2 = sell.layout_from_counts(torch.from_numpy(counts), 77, 3)
    np.testing.assert_array_equal(p1, p2.numpy())
    np.testing.assert_array_equal(e1.view(np.int32), e2.numpy())


def test_tile_placement_torch_matches_numpy():
    rng = np.random.default_rng(5)
    lens = rng.integers(0, 40, (301, 3))
    p1, q1 = sell.tile_placement(lens, 301, 3, 4)
    p2, q2 = sell.tile_placement(torch.from_numpy(lens), 301, 3, 4)
    np.testing.assert_array_equal(p1, p2.numpy())
    np.testing.assert_array_equal(q1, q2.numpy())
    for t in range(3):
        np.testing.assert_array_equal(p1[t][q1[:, t]], np.arange(301))   # inverse
