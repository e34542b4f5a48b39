"""Parity on downscaled copies of BASELINE configs 3, 4 and 5 (the real sizes run in
bench_configs.py).  Same generator family, same planner
calls, the engines the real runs use, many bitmap tiles forced where the real sizes have
them -- checked bit for bit against the CPU oracle on the host restatement of the
generated network (GeneratorSpec.host_graph)."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2205_07125_b200 as nc
from paper_2205_07125_b200 import partition as P
from paper_2205_07125_b200 import sim as S
from oracle import c_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _oracle(g, pm, rt, lif, seed, steps):
    rp, col, q = c_oracle.symmetric_csr(g.n_neurons, g.edge_i, g.edge_j, S.q_from_p(g.edge_p))
    nh = rt.next_hop_matrix() if rt is not None else S.ExchangePlan(pm.n_gpus, None).next_hop
    return c_oracle.simulate_csr(rp, col, q, pm.assignment, pm.n_gpus, nh, lif.constants(seed), steps, threads=8)


def _check(rep, ref):
    assert rep.spikes > 0
    np.testing.assert_array_equal(rep.raster, ref["raster"])
    np.testing.assert_array_equal(rep.v.view(np.uint32), ref["v"].view(np.uint32))
    if rep.n_gpus > 1:
        np.testing.assert_array_equal(rep.deliv_ids, ref["deliv"])
        np.testing.assert_array_equal(rep.hop_ids, ref["hop"])


_cache: dict = {}


def _cfg3_family():
    """1/50 of config 3's neurons at 1/10 of its degree, the reference's partition."""
    if "c3" not in _cache:
        spec = S.GeneratorSpec.random(200_000, 100.0, seed=5)
        g = spec.host_graph()
        pm = P.partition_greedy_generated(spec, 4)
        assert np.array_equal(pm.assignment, nc.partition_greedy(g, 4).assignment)
        gt = nc.aggregate(g, pm)
        _cache["c3"] = (spec, g, pm, gt)
    return _cache["c3"]


@pytest.mark.parametrize("delivery", ["fused", "push"])
def test_config3_family_reference_partition(delivery):
    spec, g, pm, gt = _cfg3_family()
    rt = nc.route_p2p(gt)
    lay = S.ShardLayout.from_assignment(pm.assignment, 4)
    net = S.Network.generate(spec, lay, tile_words=256)     # 25 tiles, as config 3 has 20
    assert net.shards[0].n_tiles > 16
    lif = S.LifParams()
    rep = S.Simulator(net, lif, 2, rt, delivery=delivery, record_raster_steps=30, per_step_counts=True).run(30)
    _check(rep, _oracle(g, pm, rt, lif, 2, 30))


@pytest.mark.parametrize("rate", [5.0, 20.0])
def test_config4_family_two_level_vs_direct(rate):
    spec, g, pm, gt = _cfg3_family()
    groups = nc.group_gpus(gt, 2)
    two = nc.build_routing_table(gt, groups, nc.select_bridges(gt, groups))
    assert (two.via >= 0).any()
    lay = S.ShardLayout.from_assignment(pm.assignment, 4)
    net = S.Network.generate(spec, lay)
    lif = S.LifParams.for_rate(rate)
    reps = {}
    for name, rt in (("direct", nc.route_p2p(gt)), ("two-level", two)):
        reps[name] = S.Simulator(net, lif, 3, rt, delivery="push", record_raster_steps=25,
                                 per_step_counts=True).run(25)
        _check(reps[name], _oracle(g, pm, rt, lif, 3, 25))
    # routing changes the path, not the content
    np.testing.assert_array_equal(reps["direct"].raster, reps["two-level"].raster)
    np.testing.assert_array_equal(reps["direct"].deliv_ids, reps["two-level"].deliv_ids)


@pytest.mark.parametrize("n_shards,delivery", [(2, "fused"), (2, "push"), (1, "persistent"), (1, "fused")])
def test_config5_family_regional(n_shards, delivery):
    """64 regions, 90 % of the synapses intra-region, many sparse bitmap tiles."""
    n, c, deg = 128_000, 64, 100.0
    size = n / c
    spec = S.GeneratorSpec(n, c, 0.9 * deg / (size - 1), 0.1 * deg / (n - size), seed=9)
    key = ("c5", n_shards)
    if key not in _cache:
        _cache[key] = spec.host_graph()
    g = _cache[key]
    lay = S.ShardLayout.blocks(n, n_shards)
    pm = nc.PartitionMap(n_shards, lay.owner.astype(np.int64))
    net = S.Network.generate(spec, lay, tile_words=64, pull=(delivery == "fused"), push=(delivery != "fused"))
    lif = S.LifParams()
    rep = S.Simulator(net, lif, 4, None, delivery=delivery, record_raster_steps=30, per_step_counts=True).run(30)
    _check(rep, _oracle(g, pm, None, lif, 4, 30))
