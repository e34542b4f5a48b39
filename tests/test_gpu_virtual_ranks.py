"""The multi-GPU exchange on ONE GPU: 2 and 4 DistSimulator ranks in one process
(tests/virtual_ranks.py) run the P2P exchange kernels -- direct and two-level
routing, the fused send of the step kernel, the inbox reset between runs --
against the CPU oracle, bit for bit.  (tests/test_gpu_multirank.py runs the same
code one process per GPU when the box has several.)"""

from __future__ import annotations

import numpy as np
import pytest

import paper_2205_07125_b200 as nc
from paper_2205_07125_b200 import sim as S
from oracle import c_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


_cache: dict = {}


def _setup(world: int, mode: str):
    key = (world, mode)
    if key in _cache:
        return _cache[key]
    g = _cache.get("g")
    if g is None:
        g = _cache["g"] = nc.generate_synthetic(nc.ModelSpec(10_000, 1, 100 / 9_999, 0.0, seed=1))
    pm = nc.partition_greedy(g, world)
    gt = nc.aggregate(g, pm)
    if mode == "direct":
        rt = nc.route_p2p(gt)
    else:
        groups = nc.group_gpus(gt, 2)
        rt = nc.build_routing_table(gt, groups, nc.select_bridges(gt, groups))
        assert (rt.via >= 0).any()
    lay = S.ShardLayout.from_assignment(pm.assignment, world)
    nets = [S.Network.from_graph(g, lay, shards=[r]) for r in range(world)]
    rp, col, q = c_oracle.symmetric_csr(g.n_neurons, g.edge_i, g.edge_j, S.q_from_p(g.edge_p))
    ref = c_oracle.simulate_csr(rp, col, q, pm.assignment, world, rt.next_hop_matrix(), S.LifParams().constants(1),
                                60, threads=8)
    _cache[key] = (nets, rt, ref)
    return _cache[key]


@pytest.mark.parametrize("world,mode,fused", [(2, "direct", False), (2, "direct", True), (4, "direct", False),
                                              (4, "direct", True), (4, "two-level", False),
                                              (4, "two-level", True), (8, "direct", False),
                                              (8, "two-level", False), (8, "two-level", True)])
def test_virtual_ranks_p2p_matches_oracle(world, mode, fused):
    """8 ranks = config 4's real shape: 8 GPUs in 2 groups of 4 (gpurun offers 4 GPUs)."""
    from virtual_ranks import VirtualCluster
    nets, rt, ref = _setup(world, mode)
    if world == 8 and mode == "two-level":
        assert sorted(np.bincount(np.asarray(nc.group_gpus(nc.aggregate(_cache["g"], nc.partition_greedy(
            _cache["g"], 8)), 2).membership))) == [4, 4]
    vc = VirtualCluster(nets, S.LifParams(), 1, rt, transport="p2p", delivery="fused", record_raster_steps=60,
                        per_step_counts=True, fused_send=fused, blocks_per_peer=2 if world <= 4 else 1)
    try:
        assert all(s.fused_send == fused for s in vc.sims)
        for attempt in range(2):     # the second run reuses the inboxes (reset must clear them)
            rep = vc.run(60)
            assert rep.spikes > 0
            np.testing.assert_array_equal(rep.raster, ref["raster"], err_msg=f"run {attempt}")
            np.testing.assert_array_equal(rep.deliv_ids, ref["deliv"])
            np.testing.assert_array_equal(rep.hop_ids, ref["hop"])
            np.testing.assert_array_equal(rep.v.view(np.uint32), ref["v"].view(np.uint32))
            assert np.isfinite(rep.extra["exchange_us"]).all()
    finally:
        vc.close()


def test_eight_rank_strong_scaling_shape_matches_one_gpu():
    """The shard shape of config 2 over 8 GPUs -- the bench's strong scaling at N = 8, which
    gpurun cannot run on 8 real GPUs: 125 k rows per rank, 4 bitmap tiles, blocks claimed
    in halves, three tile buffers -- as 8 virtual ranks, against the same network on one GPU
    (2 tiles, one shard): identical rasters and V after 12 steps."""
    import torch
    from virtual_ranks import VirtualCluster
    from paper_2205_07125_b200 import sell
    n = 1_000_000
    spec = S.GeneratorSpec.random(n, 1000.0, seed=1)
    lif = S.LifParams()
    one = S.Network.generate(spec, S.ShardLayout.blocks(n, 1))
    ref = S.Simulator(one, lif, 1, None, record_raster_steps=12).run(12)
    lay1 = one.layout
    del one
    torch.cuda.empty_cache()
    lay = S.ShardLayout.blocks(n, 8)
    nets = [S.Network.generate(spec, lay, shards=[r]) for r in range(8)]
    csr = nets[0].shards[0]
    sms = sell.device_sms()
    assert csr.n_tiles >= 3 and sell.triple_buffer(csr.n_local, csr.n_tiles, csr.tile_words, csr.cta_groups,
                                                   csr.partials_global)
    assert sell.block_split(csr.n_local, csr.n_tiles, sms) == 1
    vc = VirtualCluster(nets, lif, 1, None, transport="p2p", delivery="fused", record_raster_steps=12,
                        blocks_per_peer=1)
    try:
        rep = vc.run(12)
    finally:
        vc.close()
    assert rep.spikes == ref.spikes > 0
    np.testing.assert_array_equal(rep.raster, ref.raster)
    np.testing.assert_array_equal(rep.v.view(np.uint32), ref.v.view(np.uint32))
    np.testing.assert_array_equal(rep.i_syn.view(np.uint32), ref.i_syn.view(np.uint32))
    assert lay1.n_neurons == lay.n_neurons
