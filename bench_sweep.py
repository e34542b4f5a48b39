"""Config-4 sweep: two-level routing vs direct all-to-all over firing rates.

    torchrun --nproc-per-node N bench_sweep.py [--neurons-per-gpu 1250000] [--groups 2]

BASELINE config 4 is 10 M neurons on 8 B200 split into 2 groups x 4 GPUs; this
harness keeps its per-GPU load (1.25 M neurons x ~1 000 synapses per GPU) and
runs at the N GPUs available (gpurun offers up to 4: 2 groups x 2 GPUs).  For
every rate in {1, 2, 5, 10, 20, 50} Hz and both route tables it reports
steps/s, exchange latency p50/p99 (device %globaltimer, see bench.py), ids and
bytes per step on every channel, and the reference's analytic netsim step time
for the same tables (netsim.py:177-246) next to the measurement.

The route tables come from the reference's planner applied to the generated
network: pg[a][b] = sum over synapses between shards a and b of q/32 (the
quantised connection probability), wg = neurons per shard; then group_gpus ->
select_bridges -> build_routing_table (two-level) or route_p2p (direct).
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

RATES = (1, 2, 5, 10, 20, 50)


def traffic_matrix(net, rank, world, dev):
    """pg from the device synapse arrays (exact integer sums of q), all-reduced over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2205_07125_b200 import sell
    lay = net.layout
    row, pre, q, _ = sell.decode(net.shards[rank])
    base = torch.from_numpy(lay.base.astype(np.int64)).to(dev)
    owner = torch.bucketize(pre, base[1:], right=True)
    m = torch.zeros((world, world), dtype=torch.int64, device=dev)
    m[:, rank] = torch.zeros(world, dtype=torch.int64, device=dev).index_add_(0, owner, q)
    dist.all_reduce(m)
    del row, pre, q, owner
    return m.cpu().numpy().astype(np.float64) / 32.0


def main() -> int:
    import torch
    import torch.distributed as dist

    import paper_2205_07125_b200 as nc
    from paper_2205_07125_b200 import sim as S
    from paper_2205_07125_b200.distributed import DistSimulator

    ap = argparse.ArgumentParser()
    ap.add_argument("--neurons-per-gpu", type=int, default=1_250_000)
    ap.add_argument("--degree", type=float, default=1000.0)
    ap.add_argument("--groups", type=int, default=2)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--delivery", default="push", choices=["push", "fused"])
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--blocks-per-peer", type=int, default=None)
    ap.add_argument("--rates", default=",".join(str(r) for r in RATES))
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "sweep.json"))
    args = ap.parse_args()

    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rank, world = dist.get_rank(), dist.get_world_size()
    n = args.neurons_per_gpu * world
    t0 = time.time()
    spec = S.GeneratorSpec.random(n, args.degree, seed=args.seed)
    net = S.Network.generate(spec, S.ShardLayout.blocks(n, world), device=dev, shards=[rank])
    pg = traffic_matrix(net, rank, world, dev)
    gt = nc.GpuTrafficGraph(world, pg, np.array([net.layout.n_local(h) for h in range(world)], dtype=np.float64))
    groups = nc.group_gpus(gt, args.groups)
    tables = {"direct": nc.route_p2p(gt),
              "two-level": nc.build_routing_table(gt, groups, nc.select_bridges(gt, groups))}
    build_s = time.time() - t0
    topo = nc.build_topology(nc.TopologySpec(gpus_per_node=max(1, world // args.groups), nodes_per_switch=8), world)
    rows = []
    for rate in [float(r) for r in args.rates.split(",")]:
        lif = S.LifParams.for_rate(rate)
        for mode, rt in tables.items():
            sim = DistSimulator(net, lif, args.seed, rt, transport="p2p", delivery=args.delivery,
                                latency_steps=args.warmup + args.steps, graph_chunk=50,
                                blocks_per_peer=args.blocks_per_peer)
            sim.reset(1)
            sim.advance(args.warmup)
            torch.cuda.synchronize()
            hop0 = sim.hop_ids.clone()
            sp0 = sim.state.spike_total.clone()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            sim.advance(args.steps)
            e1.record()
            torch.cuda.synchronize()
            ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
            sim.check_status()
            hop = (sim.hop_ids - hop0)[0]
            dist.all_reduce(hop)
            spikes = sim.state.spike_total - sp0
            dist.all_reduce(spikes)
            lat, lat_min = sim.latencies_us(args.warmup + args.steps)   # per step: max, min over ranks
            lat, lat_min = lat[args.warmup:], lat_min[args.warmup:]
            sim.close()
            if rank == 0:
                h = hop.cpu().numpy().astype(np.float64) / args.steps
                model = nc.step_latency(nc.map_flows(rt, gt, topo, min(1.0, rate * 1e-3)), rt, topo,
                                        noise=min(1.0, rate * 1e-3))
                rows.append({
                    "rate_target_hz": rate, "rate_hz": round(int(spikes.item()) / n / (args.steps * 1e-3), 3),
                    "route": mode, "steps_per_s": round(args.steps / (float(ms.item()) * 1e-3), 1),
                    "exchange_us_p50": round(float(np.percentile(lat, 50)), 2),
                    "exchange_us_p99": round(float(np.percentile(lat, 99)), 2),
                    "exchange_us_p50_transfer_only": round(float(np.percentile(lat_min, 50)), 2),
                    "ids_per_step": round(float(h.sum()), 1), "payload_bytes_per_step": round(float(h.sum()) * 4, 1),
                    # P2P low-latency protocol: 8 bytes per id on the wire (tag + id) + an 8-byte header per message
                    "wire_bytes_per_step": round(float(h.sum()) * 8 + 8 * int((h > 0).sum()), 1),
                    "max_channel_payload_bytes_per_step": round(float(h.max()) * 4, 1),
                    "channels": int((h > 0).sum()),
                    "connections_out_degree": nc.connection_stats(rt).out_degree.tolist(),
                    "netsim_step_time_model_units": model.step_time,
                })
                print(json.dumps(rows[-1]), flush=True)
    if rank == 0:
        # calibrate the reference's analytic model on the measured exchange latency
        samples = [(tables[r["route"]], r["rate_hz"] * 1e-3, r["exchange_us_p50"]) for r in rows]
        spec, fit = nc.netsim.calibrate_topology(samples, gt, world)
        for r, (_, _, meas, model) in zip(rows, fit):
            r["netsim_calibrated_us"] = round(model, 2)
        calib = {k: getattr(spec, k) for k in ("gpus_per_node", "nodes_per_switch", "intra_node_bandwidth",
                                               "inter_node_bandwidth", "per_hop_latency",
                                               "connection_setup_cost")}
        doc = {"calibrated_topology_spec_us": calib, "pg": pg.tolist(),
               "config": {"neurons": n, "gpus": world, "groups": args.groups, "degree": args.degree,
                          "delivery": args.delivery, "steps": args.steps, "warmup": args.warmup,
                          "groups_membership": groups.membership.tolist(),
                          "bridges": [[a, b, v] for (a, b), v in sorted(tables["two-level"].bridges.items())],
                          "build_s": round(build_s, 1)},
               "rows": rows}
        Path(args.out).parent.mkdir(parents=True, exist_ok=True)
        Path(args.out).write_text(json.dumps(doc, indent=1) + "\n")
    dist.barrier()
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
