"""Stage-by-stage NCCL transport check (torchrun, 2+ ranks); prints progress."""
import os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[2]))


def log(*a):
    print(f"[rank {os.environ.get('RANK')}] {time.strftime('%H:%M:%S')}", *a, flush=True)


def main():
    import torch
    import torch.distributed as dist
    import paper_2205_07125_b200 as nc
    from paper_2205_07125_b200 import sim as S
    from paper_2205_07125_b200.distributed import DistSimulator
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    rank, world = dist.get_rank(), dist.get_world_size()
    g = nc.generate_synthetic(nc.ModelSpec(10_000, 1, 100 / 9_999, 0.0, seed=1))
    pm = nc.partition_greedy(g, world)
    lay = S.ShardLayout.from_assignment(pm.assignment, world)
    net = S.Network.from_graph(g, lay, device=dev, shards=[rank])
    log("network built")
    sim = DistSimulator(net, S.LifParams(), 1, None, transport="nccl", use_graph=False)
    log("simulator constructed (comm init + warm-up exchange done)")
    sim.reset(1)
    log("reset done")
    sim.advance_eager(1)
    torch.cuda.synchronize()
    log("1 eager step done")
    sim.advance_eager(20)
    torch.cuda.synchronize()
    log("21 eager steps done", int(sim.state.spike_total.item()))
    sim.use_graph = True
    sim.advance(20)
    torch.cuda.synchronize()
    log("20 graph steps done", int(sim.state.spike_total.item()))
    sim.check_status()
    sim.close()
    dist.destroy_process_group()
    log("ok")


if __name__ == "__main__":
    main()
