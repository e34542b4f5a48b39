"""BASELINE config 1 on N GPUs (run under torchrun, N = 4 for the reference setup):

    torchrun --nproc-per-node 4 tools/cfg1_bench.py [--steps 2000]

The reference's own pipeline builds the network and the routes --
generate_synthetic(ModelSpec(10_000, 1, 100/9_999, 0, seed=1)), partition_greedy(g, N),
aggregate, group_gpus(gt, 2) + select_bridges + build_routing_table (two-level) or
route_p2p (direct) -- and the simulator runs it with every transport / engine.  Prints one
JSON line per run: steps/s (max over ranks of CUDA-event time), exchange p50/p99 (us) and
ids per step on the wire.  Parity of the same runs is tested in tests/test_gpu_multirank.py.
"""
import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2205_07125_b200 as nc
    from paper_2205_07125_b200 import sim as S
    from paper_2205_07125_b200.distributed import DistSimulator
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=50)
    args = ap.parse_args()
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rank, world = dist.get_rank(), dist.get_world_size()
    g = nc.generate_synthetic(nc.ModelSpec(10_000, 1, 100 / 9_999, 0.0, seed=1))
    pm = nc.partition_greedy(g, world)
    gt = nc.aggregate(g, pm)
    groups = nc.group_gpus(gt, 2)
    tables = {"direct": nc.route_p2p(gt), "two-level": nc.build_routing_table(gt, groups, nc.select_bridges(gt, groups))}
    lay = S.ShardLayout.from_assignment(pm.assignment, world)
    net = S.Network.from_graph(g, lay, device=dev, shards=[rank])
    lif = S.LifParams()
    for mode, rt in tables.items():
        for transport, delivery in (("p2p", "fused"), ("p2p", "persistent"), ("nccl", "fused")):
            sim = DistSimulator(net, lif, 1, rt, transport=transport, delivery=delivery,
                                latency_steps=args.warmup + args.steps)
            sim.reset(1)
            sim.advance(args.warmup)
            torch.cuda.synchronize()
            hop0 = sim.hop_ids.clone()
            dist.barrier()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            dist.all_reduce(torch.zeros(1, device=dev))   # device-aligned start (bench.align_start)
            e0.record()
            sim.advance(args.steps)
            e1.record()
            torch.cuda.synchronize()
            ms = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
            dist.all_reduce(ms, op=dist.ReduceOp.MAX)
            sim.check_status()
            hop = (sim.hop_ids - hop0)[0]
            dist.all_reduce(hop)
            lat, lat_min = sim.latencies_us(args.warmup + args.steps)   # per step: max, min over ranks
            lat, lat_min = lat[args.warmup:], lat_min[args.warmup:]
            sim.close()
            if rank == 0:
                h = hop.cpu().numpy().astype(np.float64) / args.steps
                print(json.dumps({
                    "config": "1: 10k x ~100, partition_greedy(4), G=2", "route": mode, "transport": transport,
                    "engine": delivery, "gpus": world, "steps": args.steps,
                    "steps_per_s": round(args.steps / (float(ms.item()) * 1e-3), 1),
                    "exchange_us_p50": round(float(np.percentile(lat, 50)), 2),
                    "exchange_us_p99": round(float(np.percentile(lat, 99)), 2),
                    "exchange_us_p50_transfer_only": round(float(np.percentile(lat_min, 50)), 2),
                    "ids_per_step": round(float(h.sum()), 1), "channels": int((h > 0).sum()),
                    "out_degree": nc.connection_stats(rt).out_degree.tolist()}), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
