"""Where the persistent engine's exchange latency goes (torchrun, one rank per GPU):
per step and rank the device stamps "buckets ready" (after the LIF grid barrier) and
"all inbound spikes in the bitmap" (after the exchange barrier), gathered on rank 0.

    torchrun --nproc-per-node 4 tools/persist_skew.py [--neurons 10000000] [--steps 1000]

Prints percentiles of: the per-step spread of the ready stamps across ranks (skew: the
globaltimer is one clock per node), the per-rank exchange time, and SURVEY 8(d)'s
latency (per-step max over ranks)."""
import argparse
import json
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    import torch.distributed as dist
    from paper_2205_07125_b200 import sim as S
    from paper_2205_07125_b200.distributed import DistSimulator
    ap = argparse.ArgumentParser()
    ap.add_argument("--neurons", type=int, default=10_000_000)
    ap.add_argument("--degree", type=float, default=1000.0)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--blocks-per-peer", type=int, default=None)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rank, world = dist.get_rank(), dist.get_world_size()
    spec = S.GeneratorSpec.random(args.neurons, args.degree, seed=1)
    net = S.Network.generate(spec, S.ShardLayout.blocks(args.neurons, world), device=dev, shards=[rank],
                             pull=False, push=True)
    n = args.warmup + args.steps
    sim = DistSimulator(net, S.LifParams(), 1, None, transport="p2p", delivery="persistent", latency_steps=n,
                        blocks_per_peer=args.blocks_per_peer)
    sim.reset(1)
    sim.advance(n)
    torch.cuda.synchronize()
    sim.check_status()
    st = sim.lat_stamps[:, args.warmup:n].contiguous()
    parts = [torch.zeros_like(st) for _ in range(world)]
    dist.all_gather(parts, st)
    if rank == 0:
        a = torch.stack(parts).cpu().numpy().astype(np.float64)   # [rank, 2, steps]
        ready, done = a[:, 0], a[:, 1]
        skew = (ready.max(0) - ready.min(0)) / 1e3
        per_rank = (done - ready) / 1e3
        lat = per_rank.max(0)
        pct = lambda x: {p: round(float(np.percentile(x, p)), 2) for p in (50, 90, 99)}  # noqa: E731
        out = {"world": world, "neurons": args.neurons, "steps": args.steps,
               "ready_skew_us": pct(skew), "latency_max_over_ranks_us": pct(lat),
               "latency_min_over_ranks_us": pct(per_rank.min(0)),
               "per_rank_p50_us": [round(float(np.percentile(x, 50)), 2) for x in per_rank],
               "last_ready_rank_histogram": np.bincount(ready.argmax(0), minlength=world).tolist(),
               "step_us_p50": round(float(np.percentile(np.diff(ready.max(0)), 50)) / 1e3, 2)}
        print(json.dumps(out), flush=True)
        if args.out:
            Path(args.out).write_text(json.dumps(out) + "\n")
    sim.close()
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
