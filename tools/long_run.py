"""Long-run check (one process per GPU under torchrun, or one GPU): the config-2 network for
`--steps` steps with the P2P exchange (pull engine) and, on one GPU, the persistent engine;
every status word must stay clear (no overflow, no watchdog) and the run must not drift
(spikes per step in the last 1 000 steps vs the first timed 1 000).

    torchrun --nproc-per-node 2 tools/long_run.py --steps 100000"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    import torch.distributed as dist
    from paper_2205_07125_b200 import sim as S
    from paper_2205_07125_b200.distributed import DistSimulator
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=100_000)
    ap.add_argument("--neurons", type=int, default=1_000_000)
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    rank = dist.get_rank() if world > 1 else 0
    spec = S.GeneratorSpec.random(args.neurons, 1000.0, seed=1)
    lay = S.ShardLayout.blocks(args.neurons, world)
    out = {"world": world, "steps": args.steps}
    engines = ["fused"] if world > 1 else ["fused", "persistent"]
    for eng in engines:
        net = S.Network.generate(spec, lay, shards=[rank] if world > 1 else None, push=(eng == "persistent"),
                                 pull=(eng == "fused"))
        if world > 1:
            sim = DistSimulator(net, S.LifParams(), 1, None, transport="p2p", delivery=eng)
        else:
            sim = S.Simulator(net, S.LifParams(), 1, None, delivery=eng)
        sim.reset(1)
        sim.prepare(1000)
        t = time.time()
        counts = []
        done = 0
        while done < args.steps:
            before = sum(int(s.spike_total.item()) for s in sim.states)
            sim.advance(1000)
            torch.cuda.synchronize()
            sim.check_status()
            counts.append(sum(int(s.spike_total.item()) for s in sim.states) - before)
            done += 1000
        out[eng] = {"wall_s": round(time.time() - t, 1), "spikes_first_1k": counts[1], "spikes_last_1k": counts[-1],
                    "steps_per_s_wall": round(args.steps / (time.time() - t), 1)}
        del sim, net
        torch.cuda.empty_cache()
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
