"""Generate reference fixtures by running the reference package itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports ``neurocomm`` from /root/reference/pkg/src (read-only, untouched)
and records, for a fixed set of inputs, the reference's outputs:

* network build: sha256 of generate_synthetic's arrays (config 1, seeds 1-3,
  plus small planted-partition specs) -- pins our bit-identical generator;
* partition: partition_greedy / partition_random assignments;
* aggregate: pg / wg (exact float64 bit patterns) -- pins the K5 histogram;
* routing: group_gpus, select_bridges, build_routing_table, connection_stats,
  level2_traffic; netsim map_flows / step_latency.

Output: tests/golden/reference_fixtures.npz (+ .json index).  The GPU box has
no /root/reference; the tests only read the committed fixtures.
"""

from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent


def graph_hash(g) -> str:
    h = hashlib.sha256()
    for a in (g.weights, g.edge_i, g.edge_j, g.edge_p):
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main() -> int:
    sys.path.insert(0, str(REF))
    import neurocomm as nc  # noqa: E402  (the reference)

    arrays: dict[str, np.ndarray] = {}
    index: dict[str, dict] = {"graphs": {}, "cases": []}

    specs = {
        "cfg1_s1": dict(n_neurons=10_000, n_communities=1, p_in=100 / 9_999, p_out=0.0, seed=1),
        "cfg1_s2": dict(n_neurons=10_000, n_communities=1, p_in=100 / 9_999, p_out=0.0, seed=2),
        "cfg1_s3": dict(n_neurons=10_000, n_communities=1, p_in=100 / 9_999, p_out=0.0, seed=3),
        "sbm_c4": dict(n_neurons=2_000, n_communities=4, p_in=0.05, p_out=0.002, seed=7),
        "sbm_c8_w": dict(n_neurons=3_001, n_communities=8, p_in=0.03, p_out=0.001, weight_low=0.5,
                         weight_high=2.0, seed=11),
        "tiny_c3": dict(n_neurons=37, n_communities=3, p_in=0.6, p_out=0.1, weight_low=0.25,
                        weight_high=3.0, seed=5),
        "dense_pin1": dict(n_neurons=60, n_communities=2, p_in=1.0, p_out=0.3, seed=9),
        "empty": dict(n_neurons=5, n_communities=1, p_in=0.0, p_out=0.0, seed=3),
    }
    partitions = {
        "cfg1_s1": [(4, 0.0, 2), (8, 0.0, 3)],
        "cfg1_s2": [(4, 0.0, 2)],
        "cfg1_s3": [(4, 0.0, 2)],
        "sbm_c4": [(4, 0.0, 2), (4, 0.1, 2), (3, 0.0, 2)],
        "sbm_c8_w": [(8, 0.0, 2), (8, 0.05, 3), (5, 0.0, 2), (16, 0.0, 4)],
        "tiny_c3": [(3, 0.0, 2), (5, 0.2, 2)],
        "dense_pin1": [(2, 0.0, 1), (4, 0.0, 2)],
        "empty": [(2, 0.0, 1)],
    }
    topo = nc.TopologySpec(gpus_per_node=2, nodes_per_switch=2)
    for name, kw in specs.items():
        spec = nc.ModelSpec(**kw)
        g = nc.generate_synthetic(spec)
        index["graphs"][name] = {"spec": kw, "sha256": graph_hash(g), "n_edges": g.n_edges}
        for k, (n_gpus, slack, n_groups) in enumerate(partitions[name]):
            key = f"{name}/p{k}"
            pm = nc.partition_greedy(g, n_gpus, nc.PartitionConfig(balance_slack=slack))
            rnd = nc.partition_random(g, n_gpus, seed=k + 1)
            gt = nc.aggregate(g, pm)
            gt_rnd = nc.aggregate(g, rnd)
            groups = nc.group_gpus(gt, n_groups)
            bridges = nc.select_bridges(gt, groups)
            rt = nc.build_routing_table(gt, groups, bridges)
            p2p = nc.route_p2p(gt)
            cs = nc.connection_stats(rt)
            l2 = nc.level2_traffic(gt, rt)
            rep = nc.step_latency(nc.map_flows(rt, gt, nc.build_topology(topo, n_gpus), 0.3), rt,
                                  nc.build_topology(topo, n_gpus), noise=0.3)
            arrays[f"{key}/greedy"] = pm.assignment
            arrays[f"{key}/random"] = rnd.assignment
            arrays[f"{key}/pg"] = gt.pg
            arrays[f"{key}/wg"] = gt.wg
            arrays[f"{key}/pg_random"] = gt_rnd.pg
            arrays[f"{key}/groups"] = groups.membership
            arrays[f"{key}/rt_src"] = rt.src
            arrays[f"{key}/rt_dst"] = rt.dst
            arrays[f"{key}/rt_via"] = rt.via
            arrays[f"{key}/p2p_src"] = p2p.src
            arrays[f"{key}/out_degree"] = cs.out_degree
            arrays[f"{key}/level2"] = l2
            index["cases"].append({
                "key": key, "graph": name, "n_gpus": n_gpus, "slack": slack, "n_groups": n_groups,
                "random_seed": k + 1,
                "bridges": [[a, b, v] for (a, b), v in sorted(bridges.items())],
                "cross_traffic": nc.cross_traffic(g, pm).hex(),
                "step_time": rep.step_time.hex(), "setup_time": rep.setup_time.hex(),
                "bottleneck": rep.bottleneck_link,
                "topology": {"gpus_per_node": 2, "nodes_per_switch": 2}, "noise": 0.3,
            })
    # GA baseline (partition.py:187-267): small populations, fitness through aggregate
    index["ga"] = []
    for name, n_gpus, pop, gens, seed in (("tiny_c3", 3, 8, 6, 1), ("sbm_c4", 4, 6, 4, 2)):
        g = nc.generate_synthetic(nc.ModelSpec(**specs[name]))
        ga = nc.partition_genetic(g, n_gpus, nc.GaConfig(population_size=pop, generations=gens, seed=seed))
        key = f"ga/{name}/{n_gpus}"
        arrays[key] = ga.assignment
        index["ga"].append({"key": key, "graph": name, "n_gpus": n_gpus, "population_size": pop,
                            "generations": gens, "seed": seed})
    np.savez_compressed(OUT / "reference_fixtures.npz", **arrays)
    (OUT / "reference_fixtures.json").write_text(json.dumps(index, indent=1, sort_keys=True) + "\n")
    print(f"wrote {len(arrays)} arrays, {len(index['cases'])} cases")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
