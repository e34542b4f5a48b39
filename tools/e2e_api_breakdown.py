"""Where simulate(NeuronGraph, ...) spends its time on the config-2 network (1e6 x 1e3,
the bench's e2e_api case): edge upload, device layout build, simulator setup, steps.

    python tools/e2e_api_breakdown.py [--neurons 1000000] [--degree 1000] [--steps 20]

Prints one JSON line (seconds, host wall clock with a device synchronize on each side)."""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    import paper_2205_07125_b200 as nc
    from paper_2205_07125_b200 import sim as S
    ap = argparse.ArgumentParser()
    ap.add_argument("--neurons", type=int, default=1_000_000)
    ap.add_argument("--degree", type=float, default=1000.0)
    ap.add_argument("--steps", type=int, default=20)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    t = time.perf_counter()
    g = S.GeneratorSpec.random(args.neurons, args.degree, seed=1).host_graph()
    t_gen = time.perf_counter() - t
    pm = nc.PartitionMap(1, np.zeros(args.neurons, dtype=np.int64))
    out = {"neurons": args.neurons, "edges": int(g.edge_i.size), "host_graph_s": round(t_gen, 2),
           "host_bytes": int(g.edge_i.nbytes + g.edge_j.nbytes + g.edge_p.nbytes)}

    def timed(f):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = f()
        torch.cuda.synchronize()
        return r, round(time.perf_counter() - t0, 4)

    # the first simulate() call is what the bench's e2e_api measures (after the bench's own run)
    import cProfile
    import io
    import pstats
    pr = cProfile.Profile()
    pr.enable()
    rep, out["simulate_first_s"] = timed(lambda: nc.simulate(g, pm, None, args.steps, seed=1))
    pr.disable()
    prof = io.StringIO()
    pstats.Stats(pr, stream=prof).sort_stats("tottime").print_stats(25)
    out["loop_ms"] = round(rep.elapsed_ms, 3)
    for name, chunk in (("upload_s", 1 << 22), ("upload_chunk_1M_s", 1 << 20), ("upload_chunk_16M_s", 1 << 24)):
        r, out[name] = timed(lambda: S.upload_edges(g, dev, chunk=chunk))
        del r
    torch.cuda.empty_cache()
    _, out["upload_pageable_s"] = timed(lambda: [torch.from_numpy(a).to(dev) for a in (g.edge_i, g.edge_j, g.edge_p)])
    torch.cuda.empty_cache()
    lay = S.ShardLayout.from_assignment(pm.assignment, 1)
    net, out["from_graph_s"] = timed(lambda: S.Network.from_graph(g, lay))
    lif = S.LifParams()
    sim, out["simulator_s"] = timed(lambda: S.Simulator(net, lif, 1, None, record_raster_steps=args.steps,
                                                        per_step_counts=True))
    _, out["run_s"] = timed(lambda: sim.run(args.steps))
    del sim, net
    torch.cuda.empty_cache()
    _, out["simulate_again_s"] = timed(lambda: nc.simulate(g, pm, None, args.steps, seed=1))
    out["threads"] = torch.get_num_threads()
    print(json.dumps(out), flush=True)
    print(prof.getvalue(), file=sys.stderr)


if __name__ == "__main__":
    main()
