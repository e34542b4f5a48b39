"""Multi-rank parity worker (run under torchrun, one rank per GPU).

Every rank simulates its own shard of the config-1 network and exchanges
spikes over NVLink with the selected transport; rank 0 checks the gathered
rasters, per-pair / per-hop counts and final state against the CPU oracle.
Exit code 0 = parity, 1 = mismatch.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))


def main() -> int:
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2205_07125_b200 as nc
    from paper_2205_07125_b200 import sim as S
    from paper_2205_07125_b200.distributed import DistSimulator
    from oracle import c_oracle

    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rank, world = dist.get_rank(), dist.get_world_size()
    steps = int(os.environ.get("NC_STEPS", "100"))
    g = nc.generate_synthetic(nc.ModelSpec(10_000, 1, 100 / 9_999, 0.0, seed=1))
    pm = nc.partition_greedy(g, world)
    gt = nc.aggregate(g, pm)
    lif = S.LifParams()
    ok = True
    for mode in ("direct", "two-level"):
        if mode == "two-level" and world < 3:
            continue
        if mode == "direct":
            rt = nc.route_p2p(gt)
        else:
            groups = nc.group_gpus(gt, 2)
            rt = nc.build_routing_table(gt, groups, nc.select_bridges(gt, groups))
        lay = S.ShardLayout.from_assignment(pm.assignment, world)
        net = S.Network.from_graph(g, lay, device=dev, shards=[rank])
        ref = None
        if rank == 0:
            rp, col, q = c_oracle.symmetric_csr(g.n_neurons, g.edge_i, g.edge_j, S.q_from_p(g.edge_p))
            ref = c_oracle.simulate_csr(rp, col, q, pm.assignment, world, rt.next_hop_matrix(), lif.constants(1),
                                        steps, threads=8)
        runs = [(t, "fused") for t in os.environ.get("NC_TRANSPORTS", "p2p,nccl").split(",")]
        runs += [("p2p", "fused+send"), ("p2p", "persistent"), ("p2p", "binned"), ("nccl", "binned")]
        for transport, delivery in runs:
            # fused+send: the step kernel's own P2P send, forced on (off by default at this size)
            sim = DistSimulator(net, lif, 1, rt, transport=transport, delivery=delivery.split("+")[0],
                                record_raster_steps=steps, per_step_counts=True,
                                fused_send=(delivery == "fused+send"))
            assert sim.fused_send == (delivery == "fused+send")
            rep = sim.run(steps)
            # a second run on the same simulator (reset() must clear the P2P inboxes: tags restart)
            rep2 = sim.run(steps) if transport == "p2p" else rep
            sim.close()
            if rank == 0:
                checks = {
                    "raster": np.array_equal(rep.raster, ref["raster"]),
                    "deliv": np.array_equal(rep.deliv_ids, ref["deliv"]),
                    "hop": np.array_equal(rep.hop_ids, ref["hop"]),
                    "v": np.array_equal(rep.v.view(np.uint32), ref["v"].view(np.uint32)),
                    "rerun": (np.array_equal(rep2.raster, ref["raster"]) and np.array_equal(rep2.hop_ids, ref["hop"])
                              and np.array_equal(rep2.v.view(np.uint32), ref["v"].view(np.uint32))),
                }
                good = all(checks.values())
                ok &= good
                print(f"[{world} ranks] {mode:9s} {transport:4s} {delivery:10s} spikes={rep.spikes} "
                      f"{rep.steps_per_s:.0f} steps/s exchange p50={rep.extra['exchange_p50_us']:.1f}us "
                      f"p99={rep.extra['exchange_p99_us']:.1f}us {'OK' if good else 'MISMATCH ' + str(checks)}",
                      flush=True)
    # engine choice by measurement: every rank must get the same answer
    from paper_2205_07125_b200.distributed import choose_delivery
    best, times = choose_delivery(net, lif, 1, rt, steps=10, warmup=3)
    names = [None] * world
    dist.all_gather_object(names, best)
    good = best in times and len(set(names)) == 1 and set(times) <= {"fused", "persistent"}
    ok &= good
    if rank == 0:
        print(f"[{world} ranks] choose_delivery -> {best} {times} {'OK' if good else 'MISMATCH'}", flush=True)
    flag = torch.tensor([1 if ok else 0], device=dev)
    dist.broadcast(flag, 0)
    dist.destroy_process_group()
    return 0 if int(flag.item()) else 1


if __name__ == "__main__":
    raise SystemExit(main())
