"""Per-phase timing of the P2P spike exchange (run under torchrun, one rank per GPU):

    torchrun --nproc-per-node N tools/xchg_stamps.py [--delivery fused|persistent]

Prints, per rank, medians over steps 20..63 of the exchange blocks' globaltimer
stamps: start -> message published -> peer flag seen -> inbound ids scattered.
"""
import argparse
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import torch
    import torch.distributed as dist
    from paper_2205_07125_b200 import sim as S, distributed as D
    ap = argparse.ArgumentParser()
    ap.add_argument("--neurons", type=int, default=1_000_000)
    ap.add_argument("--delivery", default="fused")
    args = ap.parse_args()
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    n = args.neurons * world
    spec = S.GeneratorSpec.random(n, 1000.0, seed=1)
    net = S.Network.generate(spec, S.ShardLayout.blocks(n, world), device=dev, shards=[rank])
    sim = D.DistSimulator(net, S.LifParams(), 1, None, transport="p2p", delivery=args.delivery, latency_steps=80,
                          debug_stamps=True)
    sim.reset(1)
    sim.advance(80)
    torch.cuda.synchronize()
    st = sim.dbg.cpu().numpy().astype(np.float64)       # [64, n*B, 4]
    if rank == 0:
        print("dbg ptr", sim.X.dbg, sim.dbg.data_ptr(), "nonzero", int((st != 0).sum()), "step", int(sim.state.step.item()))
    B = int(sim.X.blocks_per_peer) or 1
    st = st[20:64, : world * B]
    peers = [b for b in range(world) if b != rank]
    rows = []
    for b in peers:
        blk = st[:, b * B:(b + 1) * B]                  # [steps, B, 4]
        t0 = blk[:, :, 0].min(axis=1)
        pub = blk[:, :, 1].max(axis=1) - t0
        seen = blk[:, :, 2].max(axis=1) - t0
        done = blk[:, :, 3].max(axis=1) - t0
        rows.append((b, np.median(pub) / 1e3, np.median(seen) / 1e3, np.median(done) / 1e3))
    lat, lat_max = sim.latencies_us(80)
    msg = " | ".join("peer %d: published %.1f  flag %.1f  scattered %.1f" % r for r in rows)
    out = [None] * world
    dist.all_gather_object(out, f"rank {rank} (us from exchange start, median) {msg}")
    if rank == 0:
        print("\n".join(out))
        print("exchange p50 %.1f us (min over ranks), %.1f incl skew" % (np.median(lat[20:]), np.median(lat_max[20:])))
    sim.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
