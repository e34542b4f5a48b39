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
    ptr, meta, syn = sell.host_build(row, pre, q, inh, n_local, n_tiles, tile_words)
    assert ptr[-1] * 4 == syn.size and (np.diff(ptr) % 32 == 0).all()
    csr = sell.SellCSR(torch.from_numpy(ptr), torch.from_numpy(meta.view(np.int32)),
                       torch.from_numpy(syn.view(np.int32)), n_tiles, tile_words, n_local, m)
    r2, p2, q2, i2 = (x.numpy() for x in sell.decode(csr))
    a = np.stack([row, pre, q, inh]).T
    b = np.stack([r2, p2, q2, i2]).T
    a = a[np.lexsort(a.T[::-1])]
    b = b[np.lexsort(b.T[::-1])]
    np.testing.assert_array_equal(a, b)
    # row lengths bound the real entries, blocks are as long as their longest row
    lens = (meta >> np.uint32(16)).astype(np.int64).reshape(n_local, n_tiles)
    pad_rows = np.zeros(((n_local + 31) // 32 * 32, n_tiles), dtype=np.int64)
    pad_rows[:n_local] = lens
    np.testing.assert_array_equal(pad_rows.reshape(-1, 32, n_tiles).max(axis=1).reshape(-1) * 32, np.diff(ptr))
    # every entry of block (slice, t) references tile t
    for blk in range(ptr.size - 1):
        t = blk % n_tiles
        ent = syn[ptr[blk] * 4: ptr[blk + 1] * 4]
        ids = ent & np.uint32(sell.ID_MASK)
        assert ((ids >> 5) // tile_words == t).all()


def test_plan_tiles():
    assert sell.plan_tiles(1000, 10_000, 148) == (1, 1000, False)
    T, tw, glob = sell.plan_tiles(312_500 + 1, 1_250_000, 148)    # 10 M neurons, 1.25 M local
    assert T > 1 and tw % 4 == 0 and T * tw >= 312_501 and not glob
    per = (1_250_000 // 32 + 147) // 148
    assert tw * 4 + per * 128 <= sell.SMEM_BYTES - sell.SMEM_RESERVE
    T, tw, glob = sell.plan_tiles(1_562_500 + 1, 12_500_000, 148)  # 50 M neurons, 12.5 M local
    assert glob and T * tw >= 1_562_501 and tw * 4 <= sell.SMEM_BYTES - sell.SMEM_RESERVE


def test_layout_from_counts_torch_matches_numpy():
    rng = np.random.default_rng(1)
    counts = rng.integers(0, 50, (77 * 3 * 2,))
    p1, e1 = sell.layout_from_counts(counts, 77, 3)
    p2, e2 = sell.layout_from_counts(torch.from_numpy(counts), 77, 3)
    np.testing.assert_array_equal(p1, p2.numpy())
    np.testing.assert_array_equal(e1.view(np.int32), e2.numpy())
