"""Virtual ranks: N DistSimulator ranks in ONE process on ONE GPU (test infrastructure).

The driver's GPU test box has a single GPU, so the one-process-per-GPU tests
(tests/test_gpu_multirank.py) skip there.  This harness runs the same
DistSimulator code -- the P2P exchange kernels k_p2p (direct and two-level),
the fused send of the step kernel, the inbox protocol, reset() -- for 2..4
ranks that share one device:

* bootstrap collectives go through :class:`ThreadGroup` (one Python thread per
  rank, a shared slot array and a barrier) instead of torch.distributed, and
  the P2P inboxes are exchanged as raw device pointers
  (``same_process = True``) instead of CUDA IPC handles;
* stepping is driven from the main thread, per step: every rank's step kernel
  on one stream (so all of them finish before any exchange kernel starts --
  the exchange kernels spin on each other and must not starve a step kernel
  of SMs), then every rank's exchange kernel on its own stream, concurrently
  (they wait for each other's messages exactly as on separate GPUs), then the
  end-of-step kernels.
"""

from __future__ import annotations

import threading


class _Hub:
    def __init__(self, n: int):
        self.n = n
        self.bar = threading.Barrier(n, timeout=300)
        self.slots = [None] * n


class ThreadGroup:
    """The collectives DistSimulator uses (distributed.TorchGroup), for ranks that are threads."""

    same_process = True

    def __init__(self, hub: _Hub, rank: int):
        self.hub = hub
        self.rank = rank
        self.world = hub.n

    def _exchange(self, obj):
        import torch
        torch.cuda.synchronize()
        self.hub.slots[self.rank] = obj
        self.hub.bar.wait()
        out = list(self.hub.slots)
        self.hub.bar.wait()
        return out

    def all_reduce(self, t, op: str = "sum"):
        vals = self._exchange(t.clone())
        acc = vals[0].clone()
        for v in vals[1:]:
            if op == "sum":
                acc += v
            elif op == "max":
                acc = acc.maximum(v)
            else:
                acc = acc.minimum(v)
        t.copy_(acc)

    def all_gather(self, parts, t):
        vals = self._exchange(t.clone())
        for p, v in zip(parts, vals):
            p.copy_(v)

    def all_gather_object(self, out, obj):
        out[:] = self._exchange(obj)

    def broadcast_object_list(self, objs, src: int = 0):
        objs[:] = self._exchange(list(objs))[src]

    def barrier(self):
        import torch
        torch.cuda.synchronize()
        self.hub.bar.wait()


def parallel(n: int, fn):
    """fn(rank) in n threads; re-raises the first failure (a rank that fails leaves the
    others at a barrier, which times out)."""
    out = [None] * n
    err = []

    def run(r):
        try:
            out[r] = fn(r)
        except BaseException as e:   # noqa: BLE001 -- propagated below
            err.append(e)

    ts = [threading.Thread(target=run, args=(r,)) for r in range(n)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    if err:
        raise err[0]
    return out


class VirtualCluster:
    """N ranks of distributed.DistSimulator on the current device."""

    def __init__(self, nets, lif, seed, rt, **kw):
        import torch
        from paper_2205_07125_b200.distributed import DistSimulator
        n = len(nets)
        self.n = n
        self.hub = _Hub(n)
        kw.setdefault("use_graph", False)
        kw.setdefault("blocks_per_peer", 2)
        self.sims = parallel(n, lambda r: DistSimulator(nets[r], lif, seed, rt, group=ThreadGroup(self.hub, r),
                                                        **kw))
        self.s0 = torch.cuda.Stream()
        self.streams = [torch.cuda.Stream() for _ in range(n)]

    def reset(self, counter_steps: int):
        parallel(self.n, lambda r: self.sims[r].reset(counter_steps))

    def step(self, steps: int):
        import torch
        s0 = self.s0
        s0.wait_stream(torch.cuda.current_stream())
        for _ in range(steps):
            for sim in self.sims:
                sim.step_kernels(s0.cuda_stream)
            ready = s0.record_event()
            done = []
            for sim, st in zip(self.sims, self.streams):
                st.wait_event(ready)
                sim.exchange_kernels(st.cuda_stream)
                done.append(st.record_event())
            for ev in done:
                s0.wait_event(ev)
            for sim in self.sims:
                sim.end_kernels(s0.cuda_stream)
        torch.cuda.current_stream().wait_stream(s0)

    def run(self, steps: int):
        """reset + steps; returns rank 0's report (rasters and counters gathered over the ranks)."""
        import torch
        per_step = self.sims[0].per_step_counts
        self.reset(steps if per_step else 1)
        self.step(steps)
        torch.cuda.synchronize()
        for sim in self.sims:
            sim.check_status()
        return parallel(self.n, lambda r: self.sims[r]._report(steps, 0.0))[0]

    def close(self):
        parallel(self.n, lambda r: self.sims[r].close())
