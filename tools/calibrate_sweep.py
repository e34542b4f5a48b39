"""Fit the reference's analytic netsim model to a measured config-4 sweep.

    python tools/calibrate_sweep.py profiles/r01_cfg4_sweep_4gpu.json [out.json]

Uses the sweep's pg when present, else the uniform pg of the random network
(neurons/N x degree/N synapses per GPU pair, mean q/32 = 0.75).  Output: the
fitted one-NVSwitch-box TopologySpec (microseconds) and model-vs-measured rows.
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main() -> int:
    import paper_2205_07125_b200 as nc
    src = Path(sys.argv[1])
    d = json.loads(src.read_text())
    cfg = d["config"]
    n = cfg["gpus"]
    if "pg" in d:
        pg = np.array(d["pg"], dtype=np.float64)
    else:
        pg = (np.ones((n, n)) - np.eye(n)) * (cfg["neurons"] / n) * (cfg["degree"] / n) * 0.75
    gt = nc.GpuTrafficGraph(n, pg, np.ones(n))
    groups = nc.routing.GroupAssignment(cfg["groups"], np.array(cfg["groups_membership"]))
    bridges = {(a, b): v for a, b, v in cfg["bridges"]}
    tables = {"direct": nc.route_p2p(gt), "two-level": nc.build_routing_table(gt, groups, bridges)}
    samples = [(tables[r["route"]], r["rate_hz"] * 1e-3, r["exchange_us_p50"]) for r in d["rows"]]
    spec, fit = nc.netsim.calibrate_topology(samples, gt, n)
    out = {
        "source": str(src), "unit": "microseconds per step",
        "model": "one NVSwitch box: gpus_per_node=1, every GPU a node on one switch (netsim.py:65-82)",
        "calibrated_topology_spec": {k: getattr(spec, k) for k in (
            "gpus_per_node", "nodes_per_switch", "intra_node_bandwidth", "inter_node_bandwidth",
            "per_hop_latency", "connection_setup_cost")},
        "rows": [{"route": r["route"], "rate_hz": r["rate_hz"], "measured_p50_us": meas,
                  "model_us": round(model, 2)} for r, (_, _, meas, model) in zip(d["rows"], fit)],
    }
    text = json.dumps(out, indent=1) + "\n"
    if len(sys.argv) > 2:
        Path(sys.argv[2]).write_text(text)
    print(text)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
