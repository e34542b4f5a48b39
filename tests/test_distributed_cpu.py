"""Host-side logic of the multi-GPU exchange on CPU: channel sets and the
gloo-backed destination-mask gather (world_size 2)."""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2205_07125_b200 as nc
from paper_2205_07125_b200.sim import ExchangePlan, ShardLayout
from paper_2205_07125_b200.distributed import channel_masks


def _rt_two_level():
    pg = np.array([[0, 5, 1, 1], [5, 0, 1, 1], [1, 1, 0, 5], [1, 1, 5, 0]], float)
    gt = nc.GpuTrafficGraph(4, pg, np.ones(4))
    groups = nc.group_gpus(gt, 2)
    return nc.build_routing_table(gt, groups, nc.select_bridges(gt, groups))


def test_channel_masks_direct_all_to_all():
    m = channel_masks(ExchangePlan(4, None))
    for r in range(4):
        others = sum(1 << p for p in range(4) if p != r)
        assert m[r]["send1"] == others and m[r]["recv1"] == others
        assert m[r]["send2"] == 0 and m[r]["recv2"] == 0


def test_channel_masks_two_level_consistent():
    rt = _rt_two_level()
    assert rt.bridges == {(0, 1): 0, (1, 0): 2}
    plan = ExchangePlan(4, rt)
    m = channel_masks(plan)
    # every send has a matching receive
    for s in range(4):
        for d in range(4):
            assert bool((m[s]["send1"] >> d) & 1) == bool((m[d]["recv1"] >> s) & 1)
            assert bool((m[s]["send2"] >> d) & 1) == bool((m[d]["recv2"] >> s) & 1)
    # GPU 1 reaches group 1 only through bridge 0; bridge 0 forwards to 2 and 3
    assert m[1]["send1"] == 0b0001
    assert m[0]["send2"] == 0b1100 and m[2]["send2"] == 0b0011
    # connection counts agree with the reference's connection_stats
    out_deg = [bin(m[r]["send1"] | m[r]["send2"]).count("1") for r in range(4)]
    assert out_deg == nc.connection_stats(rt).out_degree.tolist()


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _gather_worker(rank, world, port, result):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2205_07125_b200.distributed import gather_dest

    asg = np.array([0, 1, 1, 0, 1, 0, 0, 1, 1])
    lay = ShardLayout.from_assignment(asg, world)

    class FakeCSR:
        pass

    class FakeNet:
        layout = lay
        shards = {}

    csr = FakeCSR()
    csr.dest = torch.tensor([(rank + 1) * 10 + k for k in range(lay.n_local(rank))], dtype=torch.int32)
    FakeNet.shards = {rank: csr}
    g = gather_dest(FakeNet, rank, world, torch.device("cpu"))
    result[rank] = g.to(torch.int32).numpy().tolist()
    dist.destroy_process_group()


def test_gather_dest_gloo_world2():
    mgr = mp.Manager()
    result = mgr.dict()
    port = _free_port()
    mp.spawn(_gather_worker, args=(2, port, result), nprocs=2, join=True)
    asg = np.array([0, 1, 1, 0, 1, 0, 0, 1, 1])
    lay = ShardLayout.from_assignment(asg, 2)
    want = np.zeros(lay.n_words * 32, dtype=np.int64)
    for h in range(2):
        b = int(lay.base[h])
        want[b:b + lay.n_local(h)] = [(h + 1) * 10 + k for k in range(lay.n_local(h))]
    assert result[0] == want.tolist() and result[1] == want.tolist()
