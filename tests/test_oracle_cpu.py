"""The CPU oracle pinned: Philox KATs, and C oracle == independent numpy restatement."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2205_07125_b200 as nc
from paper_2205_07125_b200.sim import LifParams, q_from_p
from oracle import c_oracle, sim_numpy

# Random123 known-answer vectors for philox4x32-10 (ctr, key -> out)
KAT = [
    ((0, 0, 0, 0), 0x0, (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((0xFFFFFFFF,) * 4, 0xFFFFFFFFFFFFFFFF, (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), 0x299F31D0A4093822,
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


@pytest.mark.parametrize("ctr,key,out", KAT)
def test_philox_kat(ctr, key, out):
    assert tuple(c_oracle.philox(ctr, key)) == out
    r = sim_numpy.philox4x32_10(*[np.array([c], dtype=np.uint32) for c in ctr], key)
    assert tuple(int(x[0]) for x in r) == out


def _route(graph, pm, two_level, n_groups=2):
    # pg support from the edge set (positive demand where an edge crosses)
    n = pm.n_gpus
    a, b = pm.assignment[graph.edge_i], pm.assignment[graph.edge_j]
    pg = np.zeros((n, n))
    np.add.at(pg, (a, b), 1.0)
    pg = pg + pg.T
    gt = nc.GpuTrafficGraph(n, pg, np.bincount(pm.assignment, minlength=n).astype(float))
    if not two_level:
        return nc.route_p2p(gt)
    groups = nc.group_gpus(gt, n_groups)
    return nc.build_routing_table(gt, groups, nc.select_bridges(gt, groups))


@pytest.mark.parametrize("n_gpus,two_level,seed", [(1, False, 1), (2, False, 2), (4, False, 3), (4, True, 4),
                                                   (5, True, 5)])
def test_c_oracle_matches_numpy(n_gpus, two_level, seed):
    g = nc.generate_synthetic(nc.ModelSpec(600, 3, 0.08, 0.01, seed=seed))
    pm = nc.partition_greedy(g, n_gpus)
    rt = _route(g, pm, two_level) if n_gpus > 1 else None
    nh = rt.next_hop_matrix() if rt is not None else np.full((1, 1), -1)
    lif = LifParams(ext_rate_hz=260.0).constants(seed)
    q = q_from_p(g.edge_p)
    steps = 60
    rs, dl, hp, v, i = sim_numpy.simulate_numpy(g.n_neurons, g.edge_i, g.edge_j, q, pm.assignment, n_gpus, nh,
                                                lif, steps)
    rp, col, qq = c_oracle.symmetric_csr(g.n_neurons, g.edge_i, g.edge_j, q)
    out = c_oracle.simulate_csr(rp, col, qq, pm.assignment, n_gpus, nh, lif, steps, threads=4)
    assert rs.sum() > 0, "network is silent; pick a stronger drive"
    np.testing.assert_array_equal(out["raster"], rs)
    np.testing.assert_array_equal(out["deliv"], dl)
    np.testing.assert_array_equal(out["hop"], hp)
    np.testing.assert_array_equal(out["v"].view(np.uint32), v.view(np.uint32))
    np.testing.assert_array_equal(out["i"].view(np.uint32), i.view(np.uint32))


def test_oracle_thread_count_invariant():
    g = nc.generate_synthetic(nc.ModelSpec(2000, 1, 0.02, 0.0, seed=8))
    q = q_from_p(g.edge_p)
    rp, col, qq = c_oracle.symmetric_csr(g.n_neurons, g.edge_i, g.edge_j, q)
    lif = LifParams().constants(8)
    owner = np.zeros(g.n_neurons, dtype=np.int32)
    a = c_oracle.simulate_csr(rp, col, qq, owner, 1, [[-1]], lif, 50, threads=1)
    b = c_oracle.simulate_csr(rp, col, qq, owner, 1, [[-1]], lif, 50, threads=8)
    np.testing.assert_array_equal(a["raster"], b["raster"])
    np.testing.assert_array_equal(a["v"], b["v"])


def test_two_level_counts_route_independent():
    """Delivered ids per (source, destination) do not depend on the route; hop counts do."""
    g = nc.generate_synthetic(nc.ModelSpec(800, 4, 0.05, 0.01, seed=6))
    pm = nc.partition_greedy(g, 4)
    q = q_from_p(g.edge_p)
    rp, col, qq = c_oracle.symmetric_csr(g.n_neurons, g.edge_i, g.edge_j, q)
    lif = LifParams(ext_rate_hz=260.0).constants(6)
    d = c_oracle.simulate_csr(rp, col, qq, pm.assignment, 4, _route(g, pm, False).next_hop_matrix(), lif, 40)
    t = c_oracle.simulate_csr(rp, col, qq, pm.assignment, 4, _route(g, pm, True).next_hop_matrix(), lif, 40)
    np.testing.assert_array_equal(d["raster"], t["raster"])
    np.testing.assert_array_equal(d["deliv"], t["deliv"])
    # direct: every delivery is one hop
    np.testing.assert_array_equal(d["hop"], d["deliv"])


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_config1_oracle_matches_committed_rasters(seed):
    """The oracle (+ the bit-identical planner feeding it) reproduces the committed
    config-1 golden rasters (tests/golden/make_raster_golden.py)."""
    import json
    import sys
    from pathlib import Path
    here = Path(__file__).resolve().parent / "golden"
    sys.path.insert(0, str(here))
    import make_raster_golden as mk
    gold = json.loads((here / "oracle_rasters.json").read_text())["seeds"][str(seed)]
    assert mk.digest(mk.case(seed)[4]) == gold
