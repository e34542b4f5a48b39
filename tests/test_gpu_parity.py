"""GPU parity: the CUDA engine against the CPU oracle and the reference fixtures.

* K5 aggregate: pg / wg bit-equal to the reference's fsum results.
* simulate(): per-step rasters, per-pair delivered and per-hop id counts and
  the final V / I bit-equal to oracle/sim_oracle.c, for 1, 2 and 4 partitions,
  direct and two-level routing, fused / pull / push delivery.
* the device graph generator: its CSR read back drives the oracle to the same
  rasters, and its edge count matches the SBM expectation.
"""

from __future__ import annotations

import numpy as np
import pytest

import paper_2205_07125_b200 as nc
from paper_2205_07125_b200 import sell
from paper_2205_07125_b200 import sim as S
from oracle import c_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


_graphs: dict = {}


def graph(name, idx=None, **spec):
    key = name
    if key not in _graphs:
        _graphs[key] = nc.generate_synthetic(nc.ModelSpec(**spec))
    return _graphs[key]


def cfg1(seed=1):
    return graph(f"cfg1_{seed}", n_neurons=10_000, n_communities=1, p_in=100 / 9_999, p_out=0.0, seed=seed)


# ------------------------------------------------------------------ K5

def test_aggregate_bit_identical_to_reference(ref_fixtures):
    idx, arr = ref_fixtures
    for case in idx["cases"]:
        g = graph(case["graph"], **idx["graphs"][case["graph"]]["spec"])
        pm = nc.partition_greedy(g, case["n_gpus"], nc.PartitionConfig(balance_slack=case["slack"]))
        gt = nc.aggregate(g, pm)
        np.testing.assert_array_equal(gt.pg.view(np.uint64), arr[f"{case['key']}/pg"].view(np.uint64),
                                      err_msg=case["key"])
        np.testing.assert_array_equal(gt.wg.view(np.uint64), arr[f"{case['key']}/wg"].view(np.uint64))
        rnd = nc.partition_random(g, case["n_gpus"], seed=case["random_seed"])
        np.testing.assert_array_equal(nc.aggregate(g, rnd).pg, arr[f"{case['key']}/pg_random"])
        assert nc.cross_traffic(g, pm).hex() == case["cross_traffic"]


def test_aggregate_uniform_weights_path():
    """Every weight equal (generate_synthetic's default): K5 gathers only a 1-byte gpu id
    per endpoint and wg = count * w0; pg / wg must still be math.fsum per cell, also for
    a GPU without neurons and for one GPU."""
    import math
    rng = np.random.default_rng(11)
    m, e = 3000, 40000
    i = rng.integers(0, m - 1, e)
    j = np.minimum(i + 1 + rng.integers(0, 400, e), m - 1)
    keep = i < j
    key = np.unique(i[keep] * m + j[keep])
    ei, ej = key // m, key % m
    p = rng.uniform(1e-9, 1.0, ei.size)
    for w0, n in ((1.0, 8), (0.3, 5), (3.7e10, 1), (1e-20, 3)):
        w = np.full(m, w0)
        g = nc.NeuronGraph(m, w, ei, ej, p)
        asg = rng.integers(0, n, m)
        if n > 2:
            asg[asg == n - 1] = 0          # one GPU without neurons
        pm = nc.PartitionMap(n, asg)
        gt = nc.aggregate(g, pm)
        a, b = asg[ei], asg[ej]
        c = p * w0 * w0
        for x in range(n):
            assert gt.wg[x] == math.fsum(w[asg == x]), (w0, n, x)
            for y in range(x, n):
                sel = (np.minimum(a, b) == x) & (np.maximum(a, b) == y)
                assert gt.pg[x, y] == math.fsum(c[sel]), (w0, n, x, y)
                assert gt.pg[y, x] == gt.pg[x, y]
    # assignment values outside [0, n) raise on both paths (range-checked on the device
    # on the uniform one), and a valid call afterwards is unaffected
    gw = nc.NeuronGraph(m, rng.uniform(0.5, 2.0, m), ei, ej, p)
    for gr in (g, gw):
        for bad in (-1, 3, 300):
            asg = rng.integers(0, 3, m)
            asg[m // 2] = bad
            with pytest.raises(ValueError, match="outside"):
                nc.aggregate(gr, nc.PartitionMap(3, asg))
    pm = nc.PartitionMap(3, rng.integers(0, 3, m))
    assert nc.aggregate(g, pm).pg[0, 0] == math.fsum(p[(pm.assignment[ei] == 0) & (pm.assignment[ej] == 0)]
                                                      * w0 * w0)


def test_genetic_partition_matches_reference(ref_fixtures):
    """GA baseline: same numpy stream, fitness through the exact GPU aggregate."""
    idx, arr = ref_fixtures
    for case in idx["ga"]:
        g = graph(case["graph"], **idx["graphs"][case["graph"]]["spec"])
        cfg = nc.GaConfig(population_size=case["population_size"], generations=case["generations"],
                          seed=case["seed"])
        pm = nc.partition_genetic(g, case["n_gpus"], cfg)
        np.testing.assert_array_equal(pm.assignment, arr[case["key"]], err_msg=case["key"])


def test_aggregate_order_independent_and_wide_exponents():
    rng = np.random.default_rng(3)
    m, e = 300, 4000
    i = rng.integers(0, m - 1, e)
    j = np.minimum(i + 1 + rng.integers(0, 50, e), m - 1)
    keep = i < j
    key = np.unique(i[keep] * m + j[keep])
    ei, ej = key // m, key % m
    p = rng.uniform(1e-6, 1.0, ei.size)
    w = np.exp(rng.uniform(-30, 30, m))  # ~2^87 dynamic range
    g = nc.NeuronGraph(m, w, ei, ej, p)
    pm = nc.PartitionMap(4, rng.integers(0, 4, m))
    gt = nc.aggregate(g, pm)
    perm = rng.permutation(ei.size)
    gt2 = nc.aggregate(nc.NeuronGraph(m, w, ei[perm], ej[perm], p[perm]), pm)
    np.testing.assert_array_equal(gt.pg, gt2.pg)
    # correctly rounded: equal to fsum per cell
    import math
    a, b = pm.assignment[ei], pm.assignment[ej]
    c = p * w[ei] * w[ej]
    for x in range(4):
        for y in range(x, 4):
            sel = (np.minimum(a, b) == x) & (np.maximum(a, b) == y)
            assert gt.pg[x, y] == math.fsum(c[sel])
    assert all(gt.wg[x] == math.fsum(w[pm.assignment == x]) for x in range(4))


# ------------------------------------------------------------------ simulate

def oracle_run(g, pm, rt, lif, seed, steps):
    q = S.q_from_p(g.edge_p)
    rp, col, qq = c_oracle.symmetric_csr(g.n_neurons, g.edge_i, g.edge_j, q)
    n = pm.n_gpus
    nh = rt.next_hop_matrix() if rt is not None else S.ExchangePlan(n, None).next_hop
    return c_oracle.simulate_csr(rp, col, qq, pm.assignment, n, nh, lif.constants(seed), steps, threads=8)


def assert_same(rep, ref):
    np.testing.assert_array_equal(rep.raster, ref["raster"])
    np.testing.assert_array_equal(rep.v.view(np.uint32), ref["v"].view(np.uint32))
    np.testing.assert_array_equal(rep.i_syn.view(np.uint32), ref["i"].view(np.uint32))
    if rep.n_gpus > 1:
        np.testing.assert_array_equal(rep.deliv_ids, ref["deliv"])
        np.testing.assert_array_equal(rep.hop_ids, ref["hop"])


def routes(g, pm, mode):
    gt = nc.aggregate(g, pm)
    if mode == "direct":
        return nc.route_p2p(gt)
    groups = nc.group_gpus(gt, 2)
    return nc.build_routing_table(gt, groups, nc.select_bridges(gt, groups))


@pytest.mark.parametrize("n_gpus,mode", [(1, "direct"), (2, "direct"), (4, "direct"), (4, "two-level")])
def test_config1_simulate_matches_oracle(n_gpus, mode):
    g = cfg1(1)
    pm = nc.partition_greedy(g, n_gpus)
    rt = routes(g, pm, mode) if n_gpus > 1 else None
    lif = S.LifParams()
    rep = nc.simulate(g, pm, rt, 100, lif, seed=1)
    ref = oracle_run(g, pm, rt, lif, 1, 100)
    assert ref["raster"].sum() > 1000
    assert_same(rep, ref)
    if mode == "two-level":
        assert rep.exchange == "two-level" and rt.bridges == {(0, 1): 0, (1, 0): 2}


@pytest.mark.parametrize("delivery", ["pull", "push"])
def test_delivery_variants_identical(delivery):
    g = cfg1(2)
    pm = nc.partition_greedy(g, 4)
    rt = routes(g, pm, "two-level")
    lif = S.LifParams(ext_rate_hz=240.0)
    a = nc.simulate(g, pm, rt, 60, lif, seed=2, delivery="fused")
    b = nc.simulate(g, pm, rt, 60, lif, seed=2, delivery=delivery)
    np.testing.assert_array_equal(a.raster, b.raster)
    np.testing.assert_array_equal(a.v, b.v)
    np.testing.assert_array_equal(a.hop_ids, b.hop_ids)


def test_persistent_engine_matches_oracle():
    """One cooperative kernel for all steps (push delivery + LIF, grid barriers)."""
    g = cfg1(1)
    pm = nc.partition_greedy(g, 1)
    lif = S.LifParams()
    rep = nc.simulate(g, pm, None, 100, lif, seed=1, delivery="persistent")
    ref = oracle_run(g, pm, None, lif, 1, 100)
    assert_same(rep, ref)


def test_persistent_engine_across_launches():
    """The persistent engine's per-step counters (chunk claims, buckets) are reset at the
    end of every step inside the kernel, so a run split over several launches
    (advance(7), advance(13), advance(20)) gives the one-launch result."""
    import torch
    g = cfg1(2)
    pm = nc.partition_greedy(g, 1)
    lif = S.LifParams()
    net = S.Network.from_graph(g, S.ShardLayout.from_assignment(pm.assignment, 1))
    sim = S.Simulator(net, lif, 3, None, delivery="persistent", record_raster_steps=40, per_step_counts=True)
    whole = sim.run(40)
    assert_same(whole, oracle_run(g, pm, None, lif, 3, 40))
    sim.reset(40)
    for k in (7, 13, 20):
        sim.advance(k)
    torch.cuda.synchronize()
    sim.check_status()
    split = sim.report(40, 0.0)
    np.testing.assert_array_equal(split.raster, whole.raster)
    np.testing.assert_array_equal(split.v.view(np.uint32), whole.v.view(np.uint32))


@pytest.mark.parametrize("tile_words", [None, 64])
def test_binned_push_engine_matches_oracle(tile_words):
    """Event-driven step with binned push: each CTA sums its bin of every spiking
    pre's synapses in shared memory, then updates its rows (one kernel per step)."""
    g = cfg1(1)
    pm = nc.partition_greedy(g, 1)
    lif = S.LifParams()
    lay = S.ShardLayout.from_assignment(pm.assignment, 1)
    net = S.Network.from_graph(g, lay, tile_words=tile_words)
    for use_graph in (True, False):
        rep = S.Simulator(net, lif, 1, None, delivery="binned", record_raster_steps=100, per_step_counts=True,
                          use_graph=use_graph).run(100)
        assert_same(rep, oracle_run(g, pm, None, lif, 1, 100))


def test_binned_push_on_device_generated_network():
    """Device generator + bank placement + binned push agree with the pull kernel."""
    spec = S.GeneratorSpec(20_000, 2, 0.01, 0.002, seed=3)
    lay = S.ShardLayout.blocks(spec.n_neurons, 1)
    net = S.Network.generate(spec, lay, tile_words=160)
    lif = S.LifParams()
    a = S.Simulator(net, lif, 7, None, delivery="fused", record_raster_steps=80).run(80)
    b = S.Simulator(net, lif, 7, None, delivery="binned", record_raster_steps=80).run(80)
    np.testing.assert_array_equal(a.raster, b.raster)
    np.testing.assert_array_equal(a.v.view(np.uint32), b.v.view(np.uint32))


def test_partition_invariance_and_route_independence():
    """Rasters do not depend on how many GPUs or which routes carry the spikes."""
    g = cfg1(3)
    lif = S.LifParams()
    base = nc.simulate(g, nc.partition_greedy(g, 1), None, 80, lif, seed=3)
    for n in (2, 4):
        pm = nc.partition_greedy(g, n)
        for mode in ("direct", "two-level"):
            rep = nc.simulate(g, pm, routes(g, pm, mode), 80, lif, seed=3)
            np.testing.assert_array_equal(rep.raster, base.raster)
            np.testing.assert_array_equal(rep.v, base.v)
    # random placement too
    pm = nc.partition_random(g, 4, seed=9)
    rep = nc.simulate(g, pm, routes(g, pm, "direct"), 80, lif, seed=3)
    np.testing.assert_array_equal(rep.raster, base.raster)


@pytest.mark.parametrize("tile_words,glob,split,buffers", [(64, False, None, None), (100, False, 0, None),
                                                           (96, True, None, None), (96, True, 0, None),
                                                           (64, False, 2, None), (64, False, None, 2),
                                                           (96, True, None, 3)])
def test_tiled_bitmap_matches_oracle(tile_words, glob, split, buffers, monkeypatch):
    """Force the shared-memory tiling of the spike bitmap (used above ~1.8 M neurons),
    with the per-row partial sums in shared memory or (huge shards) in global memory, the
    blocks claimed whole (split 0), in halves (small shards: the default here) or in
    quarters, and two or three tile buffers (the default for these small tiles: three)."""
    if split is not None:
        monkeypatch.setattr(sell, "block_split", lambda *a: split)
    if buffers is not None:
        monkeypatch.setattr(sell, "triple_buffer", lambda *a: buffers == 3)
    g = cfg1(2)
    pm = nc.partition_greedy(g, 2)
    rt = routes(g, pm, "direct")
    lif = S.LifParams()
    lay = S.ShardLayout.from_assignment(pm.assignment, 2)
    net = S.Network.from_graph(g, lay, tile_words=tile_words, partials_global=glob)
    assert all(c.n_tiles > 1 for c in net.shards.values())
    for delivery in ("fused", "pull"):
        rep = S.Simulator(net, lif, 2, rt, delivery=delivery, record_raster_steps=60, per_step_counts=True).run(60)
        assert_same(rep, oracle_run(g, pm, rt, lif, 2, 60))


def test_graph_replay_equals_eager():
    g = cfg1(1)
    pm = nc.partition_greedy(g, 2)
    rt = routes(g, pm, "direct")
    a = nc.simulate(g, pm, rt, 70, seed=5, use_graph=True)
    b = nc.simulate(g, pm, rt, 70, seed=5, use_graph=False)
    np.testing.assert_array_equal(a.raster, b.raster)
    np.testing.assert_array_equal(a.deliv_ids, b.deliv_ids)


def test_edge_cases_empty_and_tiny():
    # no edges at all: only the drive acts
    g = nc.generate_synthetic(nc.ModelSpec(40, 1, 0.0, 0.0, seed=1))
    pm = nc.partition_greedy(g, 3)
    rep = nc.simulate(g, pm, None, 30, S.LifParams(ext_rate_hz=300.0), seed=1)
    ref = oracle_run(g, pm, None, S.LifParams(ext_rate_hz=300.0), 1, 30)
    assert_same(rep, ref)
    # a GPU with a single neuron, ragged shards
    g = nc.generate_synthetic(nc.ModelSpec(33, 2, 0.5, 0.1, 0.5, 3.0, seed=4))
    pm = nc.PartitionMap(3, np.array([0] * 31 + [1] + [2]))
    rt = routes(g, pm, "direct")
    rep = nc.simulate(g, pm, rt, 40, S.LifParams(ext_rate_hz=300.0), seed=2)
    assert_same(rep, oracle_run(g, pm, rt, S.LifParams(ext_rate_hz=300.0), 2, 40))


def test_missing_demand_rejected():
    g = cfg1(1)
    pm = nc.partition_greedy(g, 2)
    gt = nc.GpuTrafficGraph(2, np.zeros((2, 2)), np.ones(2))
    with pytest.raises(ValueError, match="no demand"):
        nc.simulate(g, pm, nc.route_p2p(gt), 5)


# ------------------------------------------------------------------ device generator

def test_device_generator_matches_oracle_and_statistics():
    import torch
    spec = S.GeneratorSpec(12_000, 4, 0.02, 0.002, seed=7)
    lay = S.ShardLayout.blocks(spec.n_neurons, 2)
    net = S.Network.generate(spec, lay)
    tiled = S.Network.generate(spec, lay, tile_words=40)
    banked = S.Network.generate(spec, lay, tile_words=64, bank_order=True)
    # expected undirected edges
    sizes = nc.model.community_sizes(spec.n_neurons, spec.n_communities)
    intra = sum(s * (s - 1) // 2 for s in sizes.tolist()) * spec.p_in
    inter = (spec.n_neurons ** 2 - (sizes ** 2).sum()) / 2 * spec.p_out
    mean = intra + inter
    assert abs(net.n_synapses / 2 - mean) < 4 * np.sqrt(mean)
    # symmetric: every synapse appears in both directions
    posts, pres, qs = [], [], []
    for h in range(2):
        post, pre, q = net.host_csr(h)
        posts.append(post), pres.append(pre), qs.append(q)
    post, pre, q = np.concatenate(posts), np.concatenate(pres), np.concatenate(qs)
    fw = np.stack([post, pre, q]).T
    bw = np.stack([pre, post, q]).T
    fw = fw[np.lexsort(fw.T[::-1])]
    bw = bw[np.lexsort(bw.T[::-1])]
    np.testing.assert_array_equal(fw, bw)
    # the same network through the oracle
    sel = pre > post
    ei, ej, qq = post[sel], pre[sel], q[sel]
    rp, col, qc = c_oracle.symmetric_csr(spec.n_neurons, ei, ej, qq)
    lif = S.LifParams()
    rt_nh = S.ExchangePlan(2, None).next_hop
    ref = c_oracle.simulate_csr(rp, col, qc, lay.owner, 2, rt_nh, lif.constants(4), 50, threads=8)
    for nw in (net, tiled, banked):
        sim = S.Simulator(nw, lif, 4, None, record_raster_steps=50, per_step_counts=True)
        rep = sim.run(50)
        np.testing.assert_array_equal(rep.raster, ref["raster"])
        np.testing.assert_array_equal(rep.deliv_ids, ref["deliv"])
        np.testing.assert_array_equal(rep.v, ref["v"])
    del torch


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_config1_gpu_matches_committed_rasters(seed):
    """BASELINE config 1 (4 partitions, the reference's two-level routes, 100 steps) on the
    GPU against the committed golden rasters of tests/golden/oracle_rasters.json."""
    import hashlib
    import json
    from pathlib import Path
    gold = json.loads((Path(__file__).resolve().parent / "golden" / "oracle_rasters.json").read_text())
    want = gold["seeds"][str(seed)]
    fx = np.load(Path(__file__).resolve().parent / "golden" / "reference_fixtures.npz")
    from paper_2205_07125_b200.routing import RoutingTable
    g = cfg1(seed)
    pm = nc.partition_greedy(g, 4)
    key = f"cfg1_s{seed}/p0"
    rt = RoutingTable(4, 2, fx[f"{key}/rt_src"], fx[f"{key}/rt_dst"], fx[f"{key}/rt_via"], {})
    rep = nc.simulate(g, pm, rt, gold["steps"], S.LifParams(), seed=seed)
    assert hashlib.sha256(np.ascontiguousarray(rep.raster, dtype=np.uint8).tobytes()).hexdigest() == \
        want["raster_sha256"]
    assert rep.raster.sum(axis=1).astype(int).tolist() == want["spikes_per_step"]
    assert rep.deliv_ids.sum(axis=0).astype(int).tolist() == want["deliv_total"]
    assert rep.hop_ids.sum(axis=0).astype(int).tolist() == want["hop_total"]
    assert hashlib.sha256(np.ascontiguousarray(rep.v, dtype=np.float32).view(np.uint32).tobytes()).hexdigest() == \
        want["v_sha256"]


# ------------------------------------------------------------------ the benchmarked network

def _row_hash(rows, cols, q, n):
    """Order-independent per-row digest of (col, q) pairs (int64 wrap-around sums)."""
    import torch
    h = (cols.to(torch.int64) * 0x9E3779B1 + q.to(torch.int64) * 0x85EBCA77 + 0x27D4EB2F) & 0xFFFFFFFF
    h = h * h + cols.to(torch.int64)
    out = torch.zeros(n, dtype=torch.int64, device=cols.device)
    out.index_add_(0, rows, h)
    return out


def test_config2_network_matches_oracle():
    """BASELINE config 2 itself -- 1M neurons x ~1k synapses, the device generator, the
    2-tile bank-ordered packed J-SELL layout bench.py times -- against the oracle's own CPU
    generator and loop: same synapse multiset per row, then 20 steps of rasters, V and I
    bit for bit."""
    import os
    import torch
    spec = S.GeneratorSpec.random(1_000_000, 1000.0, seed=1)
    lay = S.ShardLayout.blocks(spec.n_neurons, 1)
    net = S.Network.generate(spec, lay)
    csr = net.shards[0]
    assert csr.n_tiles == 2 and csr.row_perm is not None
    threads = os.cpu_count() or 1
    rowptr, col, q = c_oracle.generate_random_csr(spec.n_neurons, 1000.0, spec.seed, threads=threads)
    assert int(rowptr[-1]) == net.n_synapses
    dev = csr.syn.device
    # graph: per-row digests of the decoded device layout vs the oracle's CSR
    row, pre, qq, _ = sell.decode(csr)
    lay = net.layout           # generate() reorders each shard's rows by degree
    gid_of_internal = torch.full((lay.n_words * 32,), -1, dtype=torch.int64, device=dev)
    gid_of_internal[: lay.n_local(0)] = torch.from_numpy(lay.members[0]).to(dev)
    post = torch.from_numpy(lay.members[0]).to(dev)[row]
    hd = _row_hash(post, gid_of_internal[pre], qq, spec.n_neurons)
    del row, pre, qq, post, gid_of_internal
    rp = torch.from_numpy(rowptr).to(dev)
    rows = torch.repeat_interleave(torch.arange(spec.n_neurons, device=dev), rp[1:] - rp[:-1])
    ho = _row_hash(rows, torch.from_numpy(col).to(dev), torch.from_numpy(q).to(dev), spec.n_neurons)
    del rows, rp
    assert torch.equal(hd, ho), f"{int((hd != ho).sum())} rows differ between the device and oracle generators"
    del hd, ho
    torch.cuda.empty_cache()
    # dynamics
    steps = 20
    lif = S.LifParams()
    rep = S.Simulator(net, lif, 1, None, record_raster_steps=steps).run(steps)
    ref = c_oracle.simulate_csr(rowptr, col, q, np.zeros(spec.n_neurons, dtype=np.int32), 1, [[-1]],
                                lif.constants(1), steps, threads=threads, counts=False)
    assert rep.spikes > 1000
    np.testing.assert_array_equal(rep.raster.sum(1), ref["raster"].sum(1))
    np.testing.assert_array_equal(rep.raster, ref["raster"])
    np.testing.assert_array_equal(rep.v.view(np.uint32), ref["v"].view(np.uint32))
    np.testing.assert_array_equal(rep.i_syn.view(np.uint32), ref["i"].view(np.uint32))


def test_push_only_generator_matches_oracle():
    """Network.generate(pull=False, push=True): the push CSR and destination masks straight
    from the generator (nc_graphgen_push) drive the event-driven engines to the oracle's
    rasters -- 2 shards with the local exchange (push delivery) and 1 shard (persistent)."""
    spec = S.GeneratorSpec(12_000, 4, 0.02, 0.002, seed=7)
    lif = S.LifParams()
    for n_shards, delivery in ((2, "push"), (1, "persistent"), (1, "push")):
        lay = S.ShardLayout.blocks(spec.n_neurons, n_shards)
        full = S.Network.generate(spec, lay)                         # pull layout (oracle CSR source)
        lean = S.Network.generate(spec, lay, pull=False, push=True)
        assert lean.n_synapses == full.n_synapses
        with pytest.raises(ValueError, match="pull layout"):
            S.Simulator(lean, lif, 4, None, delivery="fused")
        posts, pres, qs = [], [], []
        for h in range(n_shards):
            post, pre, q = full.host_csr(h)
            posts.append(post), pres.append(pre), qs.append(q)
        post, pre, q = np.concatenate(posts), np.concatenate(pres), np.concatenate(qs)
        sel = pre > post
        rp, col, qc = c_oracle.symmetric_csr(spec.n_neurons, post[sel], pre[sel], q[sel])
        nh = S.ExchangePlan(n_shards, None).next_hop
        ref = c_oracle.simulate_csr(rp, col, qc, lay.owner, n_shards, nh, lif.constants(4), 40, threads=8)
        rep = S.Simulator(lean, lif, 4, None, delivery=delivery, record_raster_steps=40,
                          per_step_counts=True).run(40)
        assert rep.spikes > 0
        np.testing.assert_array_equal(rep.raster, ref["raster"])
        np.testing.assert_array_equal(rep.deliv_ids, ref["deliv"])
        np.testing.assert_array_equal(rep.v.view(np.uint32), ref["v"].view(np.uint32))


@pytest.mark.parametrize("tile_words", [None, 64])
def test_device_edge_builder_equals_host_builder(tile_words):
    """Network.from_graph builds the J-SELL layout on the GPU from the uploaded edge list
    (nc_edges_count / nc_edges_fill); the numpy builder (sell.host_build) is the
    independent check: same synapses per shard, same rasters and counters."""
    g = cfg1(2)
    pm = nc.partition_greedy(g, 3)
    lay = S.ShardLayout.from_assignment(pm.assignment, 3)
    dev_net = S.Network.from_graph(g, lay, tile_words=tile_words)
    host_net = S.Network.from_graph(g, lay, tile_words=tile_words, builder="host")
    assert dev_net.source.endswith("(device build)")
    for h in range(3):
        a = np.stack(dev_net.host_csr(h)).T
        b = np.stack(host_net.host_csr(h)).T
        np.testing.assert_array_equal(a[np.lexsort(a.T[::-1])], b[np.lexsort(b.T[::-1])])
    lif = S.LifParams()
    ra = S.Simulator(dev_net, lif, 2, None, record_raster_steps=30, per_step_counts=True).run(30)
    rb = S.Simulator(host_net, lif, 2, None, record_raster_steps=30, per_step_counts=True).run(30)
    np.testing.assert_array_equal(ra.raster, rb.raster)
    np.testing.assert_array_equal(ra.hop_ids, rb.hop_ids)
    np.testing.assert_array_equal(ra.v.view(np.uint32), rb.v.view(np.uint32))


@pytest.mark.parametrize("idtype", [np.int64, np.int32])
def test_upload_edges_pipeline(idtype):
    """sim.upload_edges (pinned staging buffers, copy engine + side-stream narrowing) gives
    the plain conversion for any chunking, including a ragged last chunk; an endpoint
    outside [0, M) raises after the upload."""
    import torch
    rng = np.random.default_rng(4)
    m, e = 5000, 12345
    ei = rng.integers(0, m, e).astype(idtype)
    ej = rng.integers(0, m, e).astype(idtype)
    p = rng.uniform(1e-9, 1.0, e)
    g = nc.NeuronGraph(m, np.ones(m), ei, ej, p)
    dev = torch.device("cuda", 0)
    want_q = np.clip(np.ceil(p * 32), 1, 32).astype(np.uint8)
    for chunk, depth in ((1 << 22, 3), (1000, 2), (777, 3), (e, 1)):
        a, b, q = S.upload_edges(g, dev, chunk=chunk, depth=depth)
        np.testing.assert_array_equal(a.cpu().numpy(), ei.astype(np.int32))
        np.testing.assert_array_equal(b.cpu().numpy(), ej.astype(np.int32))
        np.testing.assert_array_equal(q.cpu().numpy(), want_q)
    for bad in (-1, m):
        ej2 = ej.copy()
        ej2[e - 3] = bad
        with pytest.raises(ValueError, match="outside"):
            S.upload_edges(nc.NeuronGraph(m, np.ones(m), ei, ej2, p), dev, chunk=1000, depth=2)


def graph_from_csr(rowptr, col, q):
    """NeuronGraph of a symmetric CSR (upper triangle), p = q / 32 (so q_from_p(p) == q)."""
    m = rowptr.size - 1
    rows = np.repeat(np.arange(m, dtype=np.int32), np.diff(rowptr))
    up = col > rows
    ei = rows[up].astype(np.int64)
    del rows
    ej = col[up].astype(np.int64)
    ep = q[up].astype(np.float64) / 32.0
    return nc.NeuronGraph(m, np.ones(m), ei, ej, ep)


def test_simulate_api_at_config2_scale():
    """simulate(graph, pm, rt, steps) -- the drop-in API -- on a 1e9-synapse host
    NeuronGraph (BASELINE config 2's network, from the oracle's CPU generator):
    device edge upload + layout build + 10 steps, bit-equal to the oracle."""
    import os
    threads = os.cpu_count() or 1
    rowptr, col, q = c_oracle.generate_random_csr(1_000_000, 1000.0, 1, threads=threads)
    g = graph_from_csr(rowptr, col, q)
    assert 2 * g.n_edges == int(rowptr[-1]) > 9.9e8
    pm = nc.PartitionMap(1, np.zeros(g.n_neurons, dtype=np.int64))
    lif = S.LifParams()
    rep = nc.simulate(g, pm, None, 10, lif, seed=1)
    ref = c_oracle.simulate_csr(rowptr, col, q, np.zeros(g.n_neurons, dtype=np.int32), 1, [[-1]],
                                lif.constants(1), 10, threads=threads, counts=False)
    assert rep.spikes > 100
    np.testing.assert_array_equal(rep.raster, ref["raster"])
    np.testing.assert_array_equal(rep.v.view(np.uint32), ref["v"].view(np.uint32))


def test_host_generator_equals_device_generator():
    """GeneratorSpec.host_graph (csrc/graphgen_host.cpp: the planner's view, what
    partition_greedy_generated partitions) and Network.generate (csrc/graphgen.cu: what
    the GPU simulates) produce the same synapses: (post, pre, q = ceil(32 p))."""
    spec = S.GeneratorSpec(40_000, 5, 0.01, 0.001, seed=11)
    g = spec.host_graph()
    q = S.q_from_p(g.edge_p)
    want = np.concatenate([np.stack([g.edge_j, g.edge_i, q]), np.stack([g.edge_i, g.edge_j, q])], axis=1).T
    net = S.Network.generate(spec, S.ShardLayout.blocks(spec.n_neurons, 2))
    got = np.concatenate([np.stack(net.host_csr(h)).T for h in range(2)]).astype(np.int64)
    want = want.astype(np.int64)
    np.testing.assert_array_equal(got[np.lexsort(got.T[::-1])], want[np.lexsort(want.T[::-1])])


def test_auto_delivery_picks_a_measured_engine_and_matches_oracle():
    """simulate(delivery="auto"): the engines that fit are timed, the fastest runs; the
    result is the oracle's whichever wins."""
    g = cfg1(3)
    pm = nc.partition_greedy(g, 2)
    lay = S.ShardLayout.from_assignment(pm.assignment, 2)
    net = S.Network.from_graph(g, lay)
    best, times = S.choose_delivery(net, S.LifParams(), 3)
    assert set(times) == {"fused", "push"} and best in times and all(t > 0 for t in times.values())
    rep = nc.simulate(g, pm, None, 40, S.LifParams(), seed=3, delivery="auto")
    assert rep.delivery in ("fused", "push")
    rp, col, q = c_oracle.symmetric_csr(g.n_neurons, g.edge_i, g.edge_j, S.q_from_p(g.edge_p))
    ref = c_oracle.simulate_csr(rp, col, q, pm.assignment, 2, S.ExchangePlan(2, None).next_hop,
                                S.LifParams().constants(3), 40, threads=8)
    np.testing.assert_array_equal(rep.raster, ref["raster"])
    np.testing.assert_array_equal(rep.hop_ids, ref["hop"])


@pytest.mark.parametrize("source", ["generator", "transpose"])
def test_windowed_push_matches_oracle(source):
    """Push rows grouped by post-row window (nc_shard_t push_windows; the persistent engine
    delivers one L2-sized window at a time with a grid barrier in between): generated
    straight from the generator or transposed from the pull layout, 3 windows forced on a
    small network -- persistent (1 shard) and per-kernel push (2 shards) match the oracle."""
    spec = S.GeneratorSpec(12_000, 4, 0.02, 0.002, seed=7)
    lif = S.LifParams()
    for n_shards, delivery in ((1, "persistent"), (2, "push")):
        lay = S.ShardLayout.blocks(spec.n_neurons, n_shards)
        full = S.Network.generate(spec, lay)
        if source == "generator":
            net = S.Network.generate(spec, lay, pull=False, push=True, push_windows=3)
        else:
            net = full
        posts, pres, qs = [], [], []
        for h in range(n_shards):
            post, pre, q = full.host_csr(h)
            posts.append(post), pres.append(pre), qs.append(q)
        post, pre, q = np.concatenate(posts), np.concatenate(pres), np.concatenate(qs)
        sel = pre > post
        rp, col, qc = c_oracle.symmetric_csr(spec.n_neurons, post[sel], pre[sel], q[sel])
        nh = S.ExchangePlan(n_shards, None).next_hop
        ref = c_oracle.simulate_csr(rp, col, qc, lay.owner, n_shards, nh, lif.constants(4), 40, threads=8)
        sim = S.Simulator(net, lif, 4, None, delivery=delivery, record_raster_steps=40, per_step_counts=True,
                          push_windows=3)
        assert all(st.c.push_windows == 3 for st in sim.states)
        for attempt in range(2):
            rep = sim.run(40)
            np.testing.assert_array_equal(rep.raster, ref["raster"], err_msg=f"{delivery} run {attempt}")
            np.testing.assert_array_equal(rep.v.view(np.uint32), ref["v"].view(np.uint32))
            np.testing.assert_array_equal(rep.deliv_ids, ref["deliv"])


@pytest.mark.parametrize("spec_args,n_gpus", [((30_000, 1, 60 / 29_999, 0.0, 3), 4),
                                              ((24_000, 6, 0.01, 0.0008, 5), 8)])
def test_aggregate_of_generated_network(spec_args, n_gpus):
    """traffic.aggregate_generated (K5 fed by the generator, no edge list) equals the
    reference-path aggregate of the same network materialised as a NeuronGraph, bit for
    bit -- also with weights and with the reference partition of that network."""
    from paper_2205_07125_b200 import partition as P
    n, c, p_in, p_out, seed = spec_args
    spec = S.GeneratorSpec(n, c, p_in, p_out, seed=seed)
    g = spec.host_graph()
    pm = P.partition_greedy_generated(spec, n_gpus)
    for w in (None, np.random.default_rng(1).uniform(0.5, 2.0, n)):
        gw = g if w is None else nc.NeuronGraph(n, w, g.edge_i, g.edge_j, g.edge_p)
        want = nc.aggregate(gw, pm)
        got = nc.traffic.aggregate_generated(spec, pm, weights=w)
        np.testing.assert_array_equal(got.pg.view(np.uint64), want.pg.view(np.uint64))
        np.testing.assert_array_equal(got.wg.view(np.uint64), want.wg.view(np.uint64))
