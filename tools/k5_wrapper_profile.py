"""Host-side cost of traffic.aggregate around the K5 kernel (1e6 neurons, 4.9e7 edges,
8 GPUs): each stage of the wrapper timed with a device synchronize on both sides.

    python tools/k5_wrapper_profile.py"""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    import paper_2205_07125_b200 as nc
    from paper_2205_07125_b200 import traffic as T
    spec = nc.ModelSpec(1_000_000, 8, 90 / (1_000_000 / 8 - 1), 10 / 1_000_000, seed=1)
    g = nc.generate_synthetic(spec)
    pm = nc.partition_random(g, 8, seed=1)
    nc.aggregate(g, pm)
    torch.cuda.synchronize()
    out = {}

    def t(name, f, reps=20):
        ts = []
        r = None
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            r = f()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
        out[name] = round(float(np.median(ts)) * 1e3, 4)
        return r

    dev = torch.device("cuda", 0)
    t("aggregate_ms", lambda: nc.aggregate(g, pm))
    t("check_assignment_ms", lambda: T._check_assignment(pm))
    a8 = t("astype_u8_ms", lambda: np.asarray(pm.assignment).astype(np.uint8))
    t("h2d_u8_ms", lambda: torch.from_numpy(a8).to(dev))
    t("h2d_i64_ms", lambda: torch.from_numpy(pm.assignment).to(dev))
    w, ei, ej, ep, w0 = t("device_graph_ms", lambda: T._device_graph(g, dev))
    t("window_ms", lambda: T._window(ep, w))
    asg8 = torch.from_numpy(a8).to(dev)
    t("zeros_ms", lambda: torch.zeros(8 * 8 * 6 + 8, dtype=torch.int64, device=dev))
    buf = torch.zeros(8 * 8 * 6 + 8, dtype=torch.int64, device=dev)
    t("scatter_counts_ms", lambda: buf[-8:].scatter_add_(0, asg8.long(), torch.ones(1, dtype=torch.int64,
                                                                                     device=dev).expand(a8.size)))
    t("d2h_ms", lambda: buf.cpu())
    t("aggregate_fast_ms", lambda: T._aggregate_fast(pm, w, ei, ej, ep, w0, 8))
    gw = nc.NeuronGraph(g.n_neurons, np.random.default_rng(2).uniform(0.5, 2.0, g.n_neurons), g.edge_i,
                        g.edge_j, g.edge_p)
    nc.aggregate(gw, pm)
    t("aggregate_weighted_ms", lambda: nc.aggregate(gw, pm))
    print(json.dumps(out), flush=True)
    import cProfile
    import pstats
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(20):
        nc.aggregate(g, pm)
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(25)


if __name__ == "__main__":
    main()
