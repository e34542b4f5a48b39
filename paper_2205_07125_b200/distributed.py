"""One process per GPU: the spike exchange over NVLink / NVSwitch.

Rank r owns shard r of the reference's PartitionMap (partition.py:60-65) and
runs the step kernel on its own neurons; spikes move between ranks along the
RoutingTable (routing.py:61-115, 184-231):

* ``transport="nccl"``: per phase one grouped ncclSend/ncclRecv (the engine's
  own communicator, bootstrapped over torch.distributed) of fixed-capacity
  [count | ids] messages, then a scatter kernel;
* ``transport="p2p"``: one device-initiated kernel per step that stores ids
  straight into the peers' IPC-mapped inboxes and signals with system-scope
  release/acquire flags (csrc/exchange_dist.cu).

Two-level routes (``rt.via >= 0``) add the relay phase: a bridge re-buckets the
ids it received from its group by final destination and forwards them (phase
2).  torch.distributed is used only for bootstrap (unique id, IPC handles,
destination masks) and for gathering results; nothing on the step path goes
through it.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native
from .routing import RoutingTable
from .sim import ExchangePlan, LifParams, Network, SimReport, _ShardState, _as_u16

__all__ = ["channel_masks", "gather_dest", "DistSimulator", "TorchGroup", "choose_delivery"]


class TorchGroup:
    """The collectives the exchange needs for bootstrap and result gathering, over
    torch.distributed (one process per GPU).  Nothing on the step path uses them.

    ``same_process`` False: peers' P2P windows are opened with CUDA IPC handles.
    A group whose ranks share one process (and device) sets it True, and the raw
    device pointers are exchanged instead (tests/virtual_ranks.py)."""

    same_process = False

    def __init__(self):
        import torch.distributed as dist
        self._d = dist
        self.rank = dist.get_rank()
        self.world = dist.get_world_size()

    def all_reduce(self, t, op: str = "sum"):
        d = self._d
        d.all_reduce(t, op={"sum": d.ReduceOp.SUM, "max": d.ReduceOp.MAX, "min": d.ReduceOp.MIN}[op])

    def all_gather(self, parts, t):
        self._d.all_gather(parts, t)

    def all_gather_object(self, out, obj):
        self._d.all_gather_object(out, obj)

    def broadcast_object_list(self, objs, src: int = 0):
        self._d.broadcast_object_list(objs, src=src)

    def barrier(self):
        self._d.barrier()


def channel_masks(plan: ExchangePlan) -> list[dict]:
    """Per rank: send1/recv1 (first hops), send2/recv2 (relay hops) as peer bitmasks.

    Derived from the global plan so both ends of every channel agree (NCCL
    needs matched send/recv pairs).
    """
    n = plan.n
    send1 = [0] * n
    for s in range(n):
        for d in range(n):
            h = int(plan.next_hop[s, d])
            if d != s and h >= 0 and h != s:
                send1[s] |= 1 << h
    send2 = [0] * n
    for b in range(n):
        for s in range(n):
            send2[b] |= int(plan.fwd[b, s])
    recv1 = [sum(1 << s for s in range(n) if (send1[s] >> r) & 1) for r in range(n)]
    recv2 = [sum(1 << b for b in range(n) if (send2[b] >> r) & 1) for r in range(n)]
    return [{"send1": send1[r], "recv1": recv1[r], "send2": send2[r], "recv2": recv2[r]} for r in range(n)]


def gather_dest(net: Network, rank: int, world: int, device, group=None):
    """Destination mask of every internal id on every rank (all_gather of the shard masks)."""
    import torch
    grp = group if group is not None else TorchGroup()
    lay = net.layout
    width = max(lay.n_local(h) for h in range(lay.n_shards))
    mine = torch.zeros(max(width, 1), dtype=torch.int32, device=device)
    n_local = lay.n_local(rank)
    if n_local:
        mine[:n_local] = net.shards[rank].dest
    parts = [torch.zeros_like(mine) for _ in range(world)]
    grp.all_gather(parts, mine)
    g = torch.zeros(lay.n_words * 32, dtype=torch.int32, device=device)
    for h in range(world):
        b = int(lay.base[h])
        g[b:b + lay.n_local(h)] = parts[h][: lay.n_local(h)]
    return _as_u16(g)



def choose_delivery(net: Network, lif: LifParams, seed: int, rt: RoutingTable | None = None, *, candidates=None,
                    steps: int = 20, warmup: int = 5, group=None, **kw):
    """sim.choose_delivery for one process per GPU: every engine that fits on EVERY rank
    is timed (max over ranks) and all ranks return the same fastest one."""
    import torch
    from .sim import _timed_steps, delivery_candidates
    grp = group if group is not None else TorchGroup()
    names = ["fused", "persistent"]
    if candidates is None:
        mine = delivery_candidates(net)
        rows = max(net.layout.n_local(h) for h in net.shards)
        fits = rows <= int(_native.lib().nc_persistent_max_rows())   # the persistent engine's LIF masks
        ok = torch.tensor([int(n in mine or (n == "persistent" and "push" in mine and fits)) for n in names],
                          dtype=torch.int32, device=net.device)
        grp.all_reduce(ok, "min")
        candidates = [n for n, f in zip(names, ok.tolist()) if f]
    if not candidates:
        raise ValueError("no delivery engine fits this network on every rank")
    times = {}
    for d in candidates:
        sim = DistSimulator(net, lif, seed, rt, delivery=d, transport="p2p", group=grp, **kw)
        t = torch.tensor([_timed_steps(sim, warmup, steps)], dtype=torch.float64, device=net.device)
        grp.all_reduce(t, "max")
        times[d] = float(t.item())
        sim.close()
    return min(times, key=times.get), times


class DistSimulator:
    """Step loop of this rank's shard with a multi-GPU spike exchange."""

    def __init__(self, net: Network, lif: LifParams = LifParams(), seed: int = 0, rt: RoutingTable | None = None,
                 *, transport: str = "p2p", delivery: str = "fused", msg_cap: int | None = None,
                 record_raster_steps: int = 0, per_step_counts: bool = False, latency_steps: int = 4096,
                 use_graph: bool = True, graph_chunk: int = 64, timeout_s: float = 10.0,
                 blocks_per_peer: int | None = None, fused_send: bool | None = None, group=None,
                 debug_stamps: bool = False, push_windows: int | None = None):
        """``fused_send``: the fused step kernel stores phase-1 spikes straight into the
        peers' inboxes (P2P transport); off by default (see below).  ``group``: collectives
        for bootstrap (default: torch.distributed)."""
        import torch
        if transport not in ("p2p", "nccl"):
            raise ValueError(f"transport must be 'p2p' or 'nccl', got {transport!r}")
        if delivery not in ("fused", "push", "pull", "persistent", "binned"):
            raise ValueError(f"delivery must be 'fused', 'pull', 'push', 'binned' or 'persistent', got {delivery!r}")
        if delivery == "persistent" and transport != "p2p":
            raise ValueError("the persistent engine exchanges spikes with device-initiated P2P stores (transport='p2p')")
        self.g = group if group is not None else TorchGroup()
        self.rank = self.g.rank
        self.world = self.g.world
        from .sim import _check_layouts
        _check_layouts(net, delivery)
        lay = net.layout
        if lay.n_shards != self.world:
            raise ValueError(f"partition has {lay.n_shards} GPUs but {self.world} ranks are running")
        if self.rank not in net.shards:
            raise ValueError(f"rank {self.rank} has no shard in this network")
        self.net = net
        self.lif = lif
        self.c_lif = lif.to_c(seed)
        self.lib = _native.lib()
        self.transport = transport
        self.delivery = delivery
        self.plan = ExchangePlan(self.world, rt)
        self.masks = channel_masks(self.plan)[self.rank]
        self.n = self.world
        self.use_graph = use_graph
        self.graph_chunk = graph_chunk
        self.per_step_counts = per_step_counts
        self.latency_steps = latency_steps
        if blocks_per_peer is None:
            # more blocks per peer = more parallel NVLink stores and scatter; measured at 4 GPUs
            # (config-4 sweep): p50 6.5 -> 4.1 us direct, 23 -> 11 us two-level at 10 Hz for 8 -> 32
            from . import sell
            blocks_per_peer = min(32, max(8, sell.device_sms(net.device) // max(self.n, 1)))
        self.blocks_per_peer = max(1, int(blocks_per_peer))
        dev = net.device
        self.dev = dev

        # global message capacity: the exact per-rank bucket bound, maxed over ranks
        probe = _ShardState(net, self.rank, self.plan, record_steps=0, push=False, bucket_cap=None)
        cap_t = torch.tensor([probe.exact_cap], dtype=torch.int64, device=dev)
        self.g.all_reduce(cap_t, "max")
        cap = int(cap_t.item())
        if msg_cap is not None:
            cap = min(cap, int(msg_cap))
        self.cap = max(cap, 1)
        del probe
        from .sim import push_windows_for
        if push_windows is None:
            push_windows = push_windows_for(lay.n_local(self.rank)) if delivery == "persistent" else 1
        self.state = _ShardState(net, self.rank, self.plan, record_steps=record_raster_steps,
                                 push=(delivery in ("push", "persistent")), binned=(delivery == "binned"),
                                 bucket_cap=None, bucket_stride=self.cap, push_windows=push_windows)
        self.states = [self.state]
        self.record_steps = int(record_raster_steps)
        self.dest_global = gather_dest(net, self.rank, self.world, dev, self.g)

        i32 = dict(dtype=torch.int32, device=dev)
        n, cap = self.n, self.cap
        self.fwd_ids = torch.zeros(n * cap if self.plan.two_level else 1, **i32)
        self.fwd_count = torch.zeros(n, **i32)
        self.hdr = torch.zeros(4, n, **i32)                    # send, send2, recv, recv2
        self.recv_ids = torch.zeros(n * cap if transport == "nccl" else 1, **i32)
        self.recv2_ids = torch.zeros(n * cap if (transport == "nccl" and self.plan.two_level) else 1, **i32)
        self.lat_stamps = torch.zeros((2, max(latency_steps, 1)), dtype=torch.int64, device=dev)
        # P2P: the exchange kernel records its own duration per step (no stamp kernels)
        self.lat_ns = torch.zeros(max(latency_steps, 1), **i32)
        self._gbar = torch.zeros(1, **i32)
        self.hop_ids = None
        self.deliv_ids = None

        X = _native.XchgC()
        X.rank, X.n, X.cap, X.two_level = self.rank, n, cap, int(self.plan.two_level)
        X.per_step, X.lat_steps = int(per_step_counts), 0
        if transport == "p2p":
            X.lat_ns, X.lat_steps = self.lat_ns.data_ptr(), int(latency_steps)
        X.send1_mask, X.recv1_mask = self.masks["send1"], self.masks["recv1"]
        X.send2_mask, X.recv2_mask = self.masks["send2"], self.masks["recv2"]
        X.bucket_cap = self.state.bucket_cap
        X.timeout_ns = int(timeout_s * 1e9)
        st = self.state
        X.step, X.status = st.step.data_ptr(), st.status.data_ptr()
        X.bitmap0, X.bitmap1 = st.bitmaps[0].data_ptr(), st.bitmaps[1].data_ptr()
        X.bucket_ids, X.bucket_count = st.bucket_ids.data_ptr(), st.bucket_count.data_ptr()
        X.dest_global = self.dest_global.data_ptr()
        for h in range(n + 1):
            X.shard_base[h] = int(lay.base[h]) if h < n else int(lay.base[n])
        for s in range(n):
            X.fwd_row[s] = int(self.plan.fwd[self.rank, s])
        X.fwd_ids, X.fwd_count = self.fwd_ids.data_ptr(), self.fwd_count.data_ptr()
        X.send_hdr, X.send2_hdr = self.hdr[0].data_ptr(), self.hdr[1].data_ptr()
        X.recv_hdr, X.recv2_hdr = self.hdr[2].data_ptr(), self.hdr[3].data_ptr()
        X.recv_ids, X.recv2_ids = self.recv_ids.data_ptr(), self.recv2_ids.data_ptr()
        if self.state.spk_ids is not None:   # binned delivery: remote spikes join the step's list
            X.spk_ids, X.spk_count, X.spk_cap = (self.state.spk_ids.data_ptr(), self.state.spk_count.data_ptr(),
                                                 self.state.spk_cap)
        self.dbg = None
        if debug_stamps:   # per-block phase stamps of the first 64 steps (tools/xchg_stamps.py)
            self.dbg = torch.zeros((64, n * self.blocks_per_peer, 4), dtype=torch.int64, device=dev)
            X.dbg = self.dbg.data_ptr()
        self.X = X
        self._comm = None
        self._ipc_own: list[int] = []
        self._ipc_peer: list[int] = []
        if transport == "nccl":
            self._setup_nccl()
        else:
            self._setup_p2p()
        # fused send (P2P exchange after the fused step): the step kernel stores its bucketed
        # spikes straight into the first hops' inboxes and writes the headers; the exchange
        # kernel only receives phase 1 (and runs the relay phase of two-level routing).  It
        # lowers the exposed exchange time (p50, max over ranks, 8.2 -> 7.0 us at 2 GPUs,
        # 9.6 -> 8.8 us at 4) but the extra stores lengthen the step kernel more than that:
        # steps/s 3 548 -> 3 495 and 6 602 -> 6 531 (same box, 1 000 steps,
        # profiles/r02_fused_send_ab/), and on config 1 the last-CTA header pass alone cost
        # 63.6 k vs 66.9 k steps/s.  So it is off unless asked for (fused_send=True).
        self.fused_send = (transport == "p2p" and delivery == "fused" and int(self.state.bucket_cap) <= cap
                           and bool(fused_send))
        if self.fused_send:
            c = self.state.c
            for h in range(n):
                c.xsend[h] = X.peer_inbox[h] if h != self.rank else None
            c.xsend_cap, c.xsend_on, c.xsend_mask = cap, 1, self.masks["send1"]
            X.fused_send = 1
        from .sim import StepGraphs
        self._graphs = StepGraphs(dev, self._one_step, graph_chunk)
        self.ops = _native.ops()
        self.c_lif_t = _native.as_bytes(self.c_lif)
        self.X_t = _native.as_bytes(self.X)
        _native.check(self.lib.nc_sim_prepare(), "prepare")

    # ------------------------------------------------------------ bootstrap
    def _setup_nccl(self):
        if self.g.same_process:
            raise ValueError("the NCCL transport needs one process per GPU")
        uid = C.create_string_buffer(128)
        if self.rank == 0:
            _native.check(self.lib.nc_nccl_get_unique_id(uid), "nccl unique id")
        obj = [bytes(uid.raw) if self.rank == 0 else None]
        self.g.broadcast_object_list(obj, src=0)
        buf = C.create_string_buffer(obj[0], 128)
        comm = C.c_void_p()
        _native.check(self.lib.nc_nccl_comm_init(C.byref(comm), self.world, buf, self.rank), "nccl comm init")
        self._comm = comm
        # NCCL connects peers lazily on first use; do that eagerly (outside any
        # CUDA-graph capture) with one exchange of empty messages per phase.
        import torch
        st = _native.stream_handle(self.dev)
        for phase in ((1, 2) if self.plan.two_level else (1,)):
            _native.check(self.lib.nc_nccl_exchange(self._comm, C.byref(self.X), phase, st), "nccl warm-up")
        torch.cuda.synchronize(self.dev)
        self.hdr.zero_()

    def _setup_p2p(self):
        n, cap = self.n, self.cap
        inbox_words = 4 * n * (cap + 1) * 2    # (phase, parity, src) slots of (cap + 1) tagged 8-byte words
        flag_words = 2 * _native.MAX_SHARDS + 16 + 2 * _native.MAX_SHARDS  # flags, done/barrier/lat, send_done
        handles = []
        ptrs = []
        for words in (inbox_words, flag_words):
            p = C.c_void_p()
            h = C.create_string_buffer(64)
            _native.check(self.lib.nc_ipc_alloc(words * 4, C.byref(p), h), "ipc alloc")
            self._ipc_own.append(p.value)
            handles.append(bytes(h.raw))
            ptrs.append(p.value)
        allh = [None] * self.world
        # one process per GPU: IPC handles; ranks sharing a process: the pointers themselves
        self.g.all_gather_object(allh, ptrs if self.g.same_process else handles)
        X = self.X
        X.my_inbox, X.my_flags = ptrs[0], ptrs[1]
        base = ptrs[1]
        X.done = base + 4 * (2 * _native.MAX_SHARDS)
        X.barrier = base + 4 * (2 * _native.MAX_SHARDS + 1)
        X.lat_start = base + 4 * (2 * _native.MAX_SHARDS + 2)  # 8-byte aligned
        X.send_done = base + 4 * (2 * _native.MAX_SHARDS + 16)
        X.blocks_per_peer = self.blocks_per_peer
        for peer in range(self.world):
            if peer == self.rank:
                X.peer_inbox[peer], X.peer_flags[peer] = ptrs[0], ptrs[1]
                continue
            if self.g.same_process:
                X.peer_inbox[peer], X.peer_flags[peer] = allh[peer]
                continue
            opened = []
            for k in range(2):
                p = C.c_void_p()
                hb = C.create_string_buffer(allh[peer][k], 64)
                _native.check(self.lib.nc_ipc_open(hb, C.byref(p)), "ipc open")
                self._ipc_peer.append(p.value)
                opened.append(p.value)
            X.peer_inbox[peer], X.peer_flags[peer] = opened

    def close(self):
        """Release the communicator and IPC windows (collective: call on every rank)."""
        import torch
        torch.cuda.synchronize(self.dev)
        # captured graphs reference the communicator and the IPC windows
        self._graphs.clear()
        torch.cuda.synchronize(self.dev)
        self.g.barrier()
        for p in self._ipc_peer:
            self.lib.nc_ipc_close(C.c_void_p(p))
        self._ipc_peer = []
        self.g.barrier()
        for p in self._ipc_own:
            self.lib.nc_free(C.c_void_p(p))
        self._ipc_own = []
        if self._comm is not None:
            self.lib.nc_nccl_comm_destroy(self._comm)
            self._comm = None

    # ------------------------------------------------------------ stepping
    def reset(self, counter_steps: int):
        import torch
        st = _native.stream_handle(self.dev)
        s = self.state
        _native.check(self.lib.nc_sim_init(C.byref(s.c), C.byref(self.c_lif), st), "sim init")
        s.raster.zero_()
        rows = counter_steps if self.per_step_counts else 1
        if getattr(self, "hop_ids", None) is not None and self.hop_ids.shape[0] == rows:
            self.hop_ids.zero_()        # same buffers: a captured step graph stays valid
            self.deliv_ids.zero_()
        else:
            self.hop_ids = torch.zeros((rows, self.n, self.n), dtype=torch.int64, device=self.dev)
            self.deliv_ids = torch.zeros((rows, self.n, self.n), dtype=torch.int64, device=self.dev)
            self.X.hop_ids, self.X.deliv_ids = self.hop_ids.data_ptr(), self.deliv_ids.data_ptr()
            self._graphs.clear()
        self.lat_stamps.zero_()
        self.lat_ns.zero_()
        _native.check(self.lib.nc_xchg_reset(C.byref(self.X), st), "xchg reset")
        torch.cuda.synchronize(self.dev)
        self.g.barrier()     # every inbox cleared before any rank's first send

    def _exchange(self, st):
        O, X = self.ops, self.X_t
        if self.transport == "p2p":
            O.xchg_p2p(X, st)
            return
        comm = int(self._comm.value)
        O.xchg_seal(X, 1, st)
        O.nccl_exchange(comm, X, 1, st)
        O.xchg_scatter(X, 1, st)
        if self.plan.two_level:
            O.xchg_seal(X, 2, st)
            O.nccl_exchange(comm, X, 2, st)
            O.xchg_scatter(X, 2, st)

    def _one_step(self, st):
        self.step_kernels(st)
        self.exchange_kernels(st)
        self.end_kernels(st)

    # the per-step launches go through the thin PyTorch extension (torch.ops.neurocomm_b200)
    def step_kernels(self, st):
        """Delivery + LIF + bucketing of this rank's shard (and the fused send)."""
        O = self.ops
        s = self.state
        lif = self.c_lif_t
        if self.delivery == "binned":
            O.sim_step_binned(s.c_t, lif, st)
        elif self.delivery == "fused":
            O.sim_step_fused(s.c_t, lif, st)
        else:
            if self.delivery == "push":
                O.sim_deliver_push(s.c_t, self.c_lif.g_inh, st)
            else:
                O.sim_deliver_pull(s.c_t, self.c_lif.g_inh, st)
            O.sim_lif_update(s.c_t, lif, st)

    def exchange_kernels(self, st):
        s = self.state
        if self.transport == "p2p":
            self._exchange(st)          # stamps its own start (buckets ready) and end
        else:
            self.ops.stamp(self.lat_stamps[0], s.step, self.latency_steps, st)
            self._exchange(st)
            self.ops.stamp(self.lat_stamps[1], s.step, self.latency_steps, st)

    def end_kernels(self, st):
        self.ops.sim_end_step(self.state.c_t, st)

    def launches_per_step(self) -> float:
        if self.delivery == "persistent":
            return 0.0  # one cooperative launch per advance() call
        step = 2 if self.delivery in ("fused", "binned") else 3
        if self.transport == "p2p":
            return step + 1 + (1 if self.plan.two_level else 0)
        ex = 2 * (2 if self.plan.two_level else 1) + (1 if self.plan.two_level else 0)
        return step + ex + 2

    def advance_eager(self, steps: int):
        st = _native.stream_handle(self.dev)
        for _ in range(steps):
            self._one_step(st)

    def advance(self, steps: int):
        if self.delivery == "persistent":
            s = self.state
            st = _native.stream_handle(self.dev)
            self.ops.run_persistent(s.c_t, self.c_lif_t, self.X_t, int(steps), self.blocks_per_peer, self._gbar,
                                    self.lat_stamps[0], self.lat_stamps[1], self.latency_steps, st)
            return
        if not self.use_graph:
            self.advance_eager(steps)
            return
        self._graphs.run(steps)

    def prepare(self, steps: int):
        """Capture every CUDA graph a following advance(steps) replays (no work is run)."""
        if self.use_graph and self.delivery != "persistent":
            self._graphs.prepare(steps)

    def check_status(self):
        flags = self.state.status.cpu().tolist()
        if flags[0]:
            raise RuntimeError(f"rank {self.rank}: spike message overflow (capacity {self.cap}); raise msg_cap")
        if flags[1]:
            raise RuntimeError(f"rank {self.rank}: exchange watchdog expired waiting for a peer")

    def latencies_us(self, steps: int) -> tuple[np.ndarray, np.ndarray]:
        """Per-step exchange time (us) from this rank's buckets-ready stamp to its last inbound
        spike: (max over ranks, min over ranks).  The maximum is SURVEY 8(d)'s exchange
        latency (it includes waiting for the slowest peer's buckets); the minimum is the
        rank that became ready last, i.e. transfer + signalling alone."""
        import torch
        k = min(steps, self.latency_steps)
        if self.transport == "p2p" and self.delivery != "persistent":
            d = self.lat_ns[:k].to(torch.float64)
        else:
            d = (self.lat_stamps[1, :k] - self.lat_stamps[0, :k]).to(torch.float64)
        lo, hi = d.clone(), d.clone()
        self.g.all_reduce(lo, "min")
        self.g.all_reduce(hi, "max")
        return hi.cpu().numpy() / 1e3, lo.cpu().numpy() / 1e3

    def run(self, steps: int) -> SimReport:
        """Run `steps` steps; every rank gets the full report (rasters gathered)."""
        import torch
        self.reset(steps if self.per_step_counts else 1)
        if self.record_steps and self.record_steps < steps:
            raise ValueError("record_raster_steps is smaller than the number of steps")
        self.prepare(steps)
        self.g.barrier()
        torch.cuda.synchronize(self.dev)
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        self.advance(steps)
        t1.record()
        torch.cuda.synchronize(self.dev)
        ms = torch.tensor([t0.elapsed_time(t1)], dtype=torch.float64, device=self.dev)
        self.g.all_reduce(ms, "max")
        self.check_status()
        return self._report(steps, float(ms.item()))

    def _report(self, steps: int, ms: float) -> SimReport:
        import torch
        lay = self.net.layout
        s = self.state
        hop = self.hop_ids.clone()
        deliv = self.deliv_ids.clone()
        self.g.all_reduce(hop)
        self.g.all_reduce(deliv)
        width = max((lay.n_local(h) + 31) // 32 for h in range(lay.n_shards))
        nmax = max(lay.n_local(h) for h in range(lay.n_shards))
        raster = None
        if self.record_steps:
            mine = torch.zeros((steps, max(width, 1)), dtype=torch.int32, device=self.dev)
            mine[:, : s.local_words] = s.raster[:steps, : s.local_words]
            parts = [torch.zeros_like(mine) for _ in range(self.world)]
            self.g.all_gather(parts, mine)
            raster = np.zeros((steps, lay.n_neurons), dtype=bool)
            for h in range(self.world):
                nl = lay.n_local(h)
                if not nl:
                    continue
                words = parts[h].cpu().numpy().view(np.uint32)[:, : (nl + 31) // 32]
                bits = ((words[:, :, None] >> np.arange(32, dtype=np.uint32)) & np.uint32(1)).reshape(steps, -1)
                raster[:, lay.members[h]] = bits[:, :nl].astype(bool)
        vt = torch.zeros((2, max(nmax, 1)), dtype=torch.float32, device=self.dev)
        vt[0, : s.n_local] = s.v[: s.n_local]
        vt[1, : s.n_local] = s.i_syn[: s.n_local]
        parts = [torch.zeros_like(vt) for _ in range(self.world)]
        self.g.all_gather(parts, vt)
        v = np.zeros(lay.n_neurons, dtype=np.float32)
        i = np.zeros(lay.n_neurons, dtype=np.float32)
        for h in range(self.world):
            nl = lay.n_local(h)
            p = parts[h].cpu().numpy()
            v[lay.members[h]] = p[0, :nl]
            i[lay.members[h]] = p[1, :nl]
        sp = s.spike_total.clone()
        self.g.all_reduce(sp)
        lat, lat_min = self.latencies_us(steps)
        mode = "two-level" if self.plan.two_level else "direct"
        return SimReport(steps=steps, n_gpus=self.world, raster=raster, deliv_ids=deliv.cpu().numpy(),
                         hop_ids=hop.cpu().numpy(), spikes=int(sp.item()), v=v, i_syn=i, elapsed_ms=ms,
                         exchange=mode, delivery=self.delivery,
                         extra={"transport": self.transport, "exchange_us": lat, "exchange_transfer_us": lat_min,
                                "exchange_p50_us": float(np.percentile(lat, 50)) if lat.size else None,
                                "exchange_p99_us": float(np.percentile(lat, 99)) if lat.size else None})
