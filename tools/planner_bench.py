"""Planner stages: ours vs the reference's CPU numbers.

    python tools/planner_bench.py [--sizes 10000,100000,1000000]

For ModelSpec(M, C, 100/(M-1) or the regional split, W = 1, seed=1) it times our
generate_synthetic (host, bit-identical PCG64 stream), partition_greedy (native K6
indexed heap) and aggregate (K5 exact histogram on the GPU), and checks that pg is
bit-identical to the host fsum restatement for the cfg-1 size.  The reference's
times for the same sizes (measured in the build container)
are printed next to them.  One JSON line per size.
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

REFERENCE_S = {   # generate / partition / aggregate, single-threaded reference
    10_000: (0.23, 0.77, 0.095),
    100_000: (3.25, 10.5, 1.48),
    1_000_000: (32.7, 500.6, 9.2),
}


def main():
    import numpy as np
    import torch
    import paper_2205_07125_b200 as nc
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="10000,100000,1000000")
    ap.add_argument("--reps", type=int, default=20)
    args = ap.parse_args()
    for m in [int(x) for x in args.sizes.split(",")]:
        c, n = (1, 4) if m <= 10_000 else ((1, 8) if m <= 100_000 else (8, 8))
        spec = nc.ModelSpec(m, c, 100 / (m - 1) if c == 1 else 90 / (m / c - 1), 0.0 if c == 1 else 10 / m,
                            seed=1)
        t = time.time()
        g = nc.generate_synthetic(spec)
        t_gen = time.time() - t
        t = time.time()
        pm = nc.partition_greedy(g, n)
        t_part = time.time() - t
        nc.aggregate(g, pm)                     # warm: device upload + module load
        torch.cuda.synchronize()
        t = time.time()
        gt = nc.aggregate(g, pm)
        torch.cuda.synchronize()
        t_agg = time.time() - t
        # median over repeated calls (the GA's use), uniform weights (the default spec) and
        # with per-neuron weights (the general 16-byte record path)
        def med(gr):
            ts = []
            for _ in range(args.reps):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                nc.aggregate(gr, pm)
                ts.append(time.perf_counter() - t0)
            return float(np.median(ts))
        t_med = med(g)
        gw = nc.NeuronGraph(g.n_neurons, np.random.default_rng(2).uniform(0.5, 2.0, g.n_neurons), g.edge_i,
                            g.edge_j, g.edge_p)
        nc.aggregate(gw, pm)
        t_med_w = med(gw)
        ref = REFERENCE_S.get(m)
        print(json.dumps({
            "neurons": m, "communities": c, "gpus": n, "edges": int(g.n_edges),
            "ours_s": {"generate_synthetic": round(t_gen, 3), "partition_greedy": round(t_part, 3),
                       "aggregate": round(t_agg, 4), "aggregate_median": round(t_med, 5),
                       "aggregate_weighted_median": round(t_med_w, 5)},
            "reference_s": None if ref is None else dict(zip(("generate_synthetic", "partition_greedy", "aggregate"),
                                                            ref)),
            "cross_traffic": float(np.triu(gt.pg, 1).sum()),
        }), flush=True)


if __name__ == "__main__":
    main()
