"""Multi-rank K5 worker (torchrun, one rank per GPU): the edge list of a graph is
split across ranks, aggregate_sharded() all-reduces the exact limbs, and every rank
must return pg / wg bit-identical to the single-GPU aggregate().  Exit 0 = equal."""

from __future__ import annotations

import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))


def main() -> int:
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2205_07125_b200 as nc
    from paper_2205_07125_b200.traffic import aggregate_sharded

    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    ok = True
    for spec, n_gpus in ((nc.ModelSpec(10_000, 1, 100 / 9_999, 0.0, seed=1), 4),
                         (nc.ModelSpec(3_001, 8, 0.03, 0.001, weight_low=0.5, weight_high=2.0, seed=11), 8),
                         (nc.ModelSpec(37, 3, 0.6, 0.1, weight_low=0.25, weight_high=3.0, seed=5), 5)):
        g = nc.generate_synthetic(spec)
        pm = nc.partition_greedy(g, n_gpus)
        whole = nc.aggregate(g, pm)
        # uneven, interleaved split (and an empty slice on the last rank for the tiny graph)
        idx = np.arange(g.n_edges)
        mine = idx[(idx * 7 + 3) % world == rank] if g.n_edges > 100 else (idx if rank == 0 else idx[:0])
        part = aggregate_sharded(g.edge_i[mine], g.edge_j[mine], g.edge_p[mine], g.weights, pm.assignment, n_gpus)
        same = (np.array_equal(part.pg.view(np.uint64), whole.pg.view(np.uint64))
                and np.array_equal(part.wg.view(np.uint64), whole.wg.view(np.uint64)))
        ok &= same
        if rank == 0:
            print(f"[{world} ranks] M={g.n_neurons} E={g.n_edges} N={n_gpus}: {'OK' if same else 'MISMATCH'}",
                  flush=True)
    # K5 fed by the generator, rows split over the ranks (traffic.aggregate_generated(group=True))
    from paper_2205_07125_b200 import sim as S
    gspec = S.GeneratorSpec(40_000, 5, 0.01, 0.001, seed=3)
    gpm = nc.PartitionMap(6, (np.arange(gspec.n_neurons) * 5 % 6).astype(np.int64))
    one = nc.traffic.aggregate_generated(gspec, gpm)
    split = nc.traffic.aggregate_generated(gspec, gpm, group=True)
    same = (np.array_equal(one.pg.view(np.uint64), split.pg.view(np.uint64))
            and np.array_equal(one.wg.view(np.uint64), split.wg.view(np.uint64)))
    ok &= same
    if rank == 0:
        print(f"[{world} ranks] aggregate_generated rows split over ranks: {'OK' if same else 'MISMATCH'}", flush=True)
    flag = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    dist.destroy_process_group()
    return 0 if int(flag.item()) else 1


if __name__ == "__main__":
    raise SystemExit(main())
