"""simulate(steps): the per-timestep spiking hot loop on B200.

New relative to the reference (neurocomm models one step only analytically,
netsim.py:177-273); it consumes exactly what the reference pipeline produces:
``NeuronGraph`` (model.py:53-92) -> ``PartitionMap`` (partition.py:60-65) ->
``RoutingTable`` (routing.py:61-115).  Semantics are DESIGN.md section 3; the
CPU oracle restating them is oracle/sim_oracle.c.

Per step and shard (one shard per GPU, or several shards on one GPU with the
"local" transport):

  fused  : nc_sim_step_fused   K3 pull delivery + K1 LIF + K2 ballot/bucket
  push   : nc_sim_deliver_push (event driven) then nc_sim_lif_update (K1+K2)
  then the spike exchange (route-table next hops, two-level relay) and
  nc_sim_end_step.  Everything stays on the device; the step counter lives in
  device memory, so a chunk of steps is captured once in a CUDA graph and
  replayed.

PyTorch provides device memory, streams, CUDA graphs and torch.distributed;
every kernel is in libneurocomm_b200.so.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native
from . import sell
from .model import INTER_P_RANGE, INTRA_P_RANGE, ModelSpec, NeuronGraph, community_sizes
from .routing import RoutingTable

__all__ = [
    "LifParams", "ShardLayout", "ExchangePlan", "Network", "Simulator", "SimReport", "simulate",
    "q_from_p", "inhibitory_mask", "ID_BITS", "StepGraphs", "choose_delivery",
]

ID_BITS = sell.ID_BITS  # unpacked builder entry: (q << 26) | tile-relative pre id
ID_MASK = sell.ID_MASK
Q_LEVELS = 32           # synaptic weight units: q = ceil(32 p) in [1, 32]


# ---------------------------------------------------------------- parameters

@dataclass(frozen=True)
class LifParams:
    """Current-based LIF neuron + Poisson drive.

    Constants are computed in fp64 on the host and rounded once to fp32
    (:meth:`constants`); the update then runs entirely in fp32 with explicit
    round-to-nearest operations in a fixed order on both GPU and oracle.
    """

    dt_ms: float = 1.0
    tau_m_ms: float = 20.0
    tau_syn_ms: float = 5.0
    v_rest: float = 0.0
    v_reset: float = 0.0
    v_th: float = 20.0
    t_ref_steps: int = 2
    w_syn: float = 0.32          # synaptic current of one q=32 (p=1) synapse event
    g_inh: int = 4               # inhibitory synapses weigh -g_inh * q
    inh_every: int = 5           # gid % inh_every == inh_every-1 is inhibitory (0 = none)
    ext_rate_hz: float = 215.0   # Poisson rate of each of ext_lanes external inputs (~10 Hz firing)
    ext_lanes: int = 4
    w_ext: float = 4.0           # synaptic current of one external event

    @classmethod
    def for_rate(cls, hz: float, **kw) -> "LifParams":
        """Parameters whose drive gives about `hz` Hz mean firing (degree 100-1000 nets).

        Interpolates RATE_CALIBRATION, measured with the C oracle on a 20k-neuron,
        degree-1000 random network (steps 100-400, default parameters).
        """
        ext, rate = RATE_CALIBRATION[:, 0], RATE_CALIBRATION[:, 1]
        if not rate[0] <= hz <= rate[-1]:
            raise ValueError(f"calibrated for {rate[0]}..{rate[-1]} Hz, got {hz}")
        return cls(ext_rate_hz=float(np.interp(hz, rate, ext)), **kw)

    def constants(self, seed: int) -> dict:
        f32 = lambda x: float(np.float32(x))  # noqa: E731
        if not (self.dt_ms > 0 and self.tau_m_ms > 0 and self.tau_syn_ms > 0):
            raise ValueError("dt_ms, tau_m_ms and tau_syn_ms must be > 0")
        if not 0 <= self.t_ref_steps <= 255:
            raise ValueError("t_ref_steps must be in [0, 255]")
        if not 0 <= self.ext_lanes <= 4:
            raise ValueError("ext_lanes must be in [0, 4]")
        p_lane = self.ext_rate_hz * self.dt_ms * 1e-3
        if not 0.0 <= p_lane < 1.0:
            raise ValueError(f"ext_rate_hz * dt must be a probability < 1, got {p_lane}")
        decay_v = math.exp(-self.dt_ms / self.tau_m_ms)
        return {
            "alpha_v": f32(decay_v),
            "alpha_i": f32(math.exp(-self.dt_ms / self.tau_syn_ms)),
            "beta": f32(1.0 - decay_v),
            "v_rest": f32(self.v_rest), "v_reset": f32(self.v_reset), "v_th": f32(self.v_th),
            "w_unit": f32(self.w_syn / Q_LEVELS),
            "w_ext": f32(self.w_ext),
            "v_init_span": float(np.float32(self.v_th) - np.float32(self.v_reset)),
            "ext_threshold": min(int(round(p_lane * 2.0**32)), 2**32 - 1),
            "ext_lanes": int(self.ext_lanes), "t_ref": int(self.t_ref_steps),
            "g_inh": int(self.g_inh), "inh_every": int(self.inh_every),
            "seed": int(seed) & (2**64 - 1),
        }

    def to_c(self, seed: int) -> _native.LifParamsC:
        k = self.constants(seed)
        return _native.LifParamsC(
            alpha_v=k["alpha_v"], alpha_i=k["alpha_i"], beta=k["beta"], v_rest=k["v_rest"],
            v_reset=k["v_reset"], v_th=k["v_th"], w_unit=k["w_unit"], w_ext=k["w_ext"],
            v_init_span=k["v_init_span"], ext_threshold=k["ext_threshold"], ext_lanes=k["ext_lanes"],
            t_ref=k["t_ref"], g_inh=k["g_inh"], pad0=0, seed=k["seed"])


# (ext_rate_hz per lane, measured firing rate Hz) -- see LifParams.for_rate
RATE_CALIBRATION = np.array([
    (140, 0.068), (160, 0.676), (180, 2.994), (190, 4.91), (200, 7.314), (210, 9.727), (215, 10.968),
    (220, 12.248), (230, 14.867), (240, 17.438), (260, 22.468), (280, 27.036), (300, 31.523),
    (330, 37.63), (360, 43.524), (400, 50.916)])


def q_from_p(p) -> np.ndarray:
    """Synaptic weight units of connection probability p: ceil(32 p) clipped to [1, 32]."""
    return np.clip(np.ceil(np.asarray(p, dtype=np.float64) * Q_LEVELS), 1, Q_LEVELS).astype(np.uint8)


def inhibitory_mask(gid, every: int) -> np.ndarray:
    g = np.asarray(gid, dtype=np.int64)
    if every <= 0:
        return np.zeros(g.shape, dtype=bool)
    return (g % every) == every - 1


# ---------------------------------------------------------------- layout

@dataclass
class ShardLayout:
    """Internal renumbering: shard h owns the 32-aligned id range [base[h], base[h] + count[h])."""

    n_neurons: int
    n_shards: int
    owner: np.ndarray          # int32 [M]
    members: list              # per shard: ascending gids (int64)
    base: np.ndarray           # int64 [n+1], base[n] = end of the last shard's padded range
    internal_id: np.ndarray    # int32 [M]
    n_words: int               # bitmap words incl. a guard word, multiple of 4

    @classmethod
    def from_assignment(cls, assignment, n_shards: int, order_key=None, group_key=None) -> "ShardLayout":
        """Shards from a PartitionMap assignment.  Inside a shard, neurons are in
        ascending gid, or by descending `order_key` (ties: gid) when given --
        the engine passes the degree so the 32 rows of a SELL slice have
        similar lengths (less padding) -- within ascending `group_key` groups
        when given (the engine passes the inhibitory flag: excitatory ids first,
        then inhibitory ones, so most bitmap tiles hold pres of one sign and a
        row's synapses in such a tile need one E/I segment instead of two --
        half the per-(row, tile) segment padding)."""
        owner = np.ascontiguousarray(assignment, dtype=np.int64)
        if owner.size and (owner.min() < 0 or owner.max() >= n_shards):
            raise ValueError("assignment has GPU indices outside [0, n_gpus)")
        if n_shards > _native.MAX_SHARDS:
            raise ValueError(f"at most {_native.MAX_SHARDS} shards are supported, got {n_shards}")
        members = [np.flatnonzero(owner == h) for h in range(n_shards)]
        if order_key is not None:
            key = np.asarray(order_key)
            if group_key is not None:
                grp = np.asarray(group_key)
                members = [m[np.lexsort((m, -key[m], grp[m]))] for m in members]
            else:
                members = [m[np.lexsort((m, -key[m]))] for m in members]
        counts = np.array([m.size for m in members], dtype=np.int64)
        padded = (counts + 31) // 32 * 32
        base = np.zeros(n_shards + 1, dtype=np.int64)
        base[1:] = np.cumsum(padded)
        internal = np.empty(owner.size, dtype=np.int64)
        for h, m in enumerate(members):
            internal[m] = base[h] + np.arange(m.size)
        n_words = (int(base[-1]) // 32 + 1 + 3) // 4 * 4
        if n_words * 32 > (1 << _native.INTERNAL_ID_BITS):
            raise ValueError(f"network too large for {_native.INTERNAL_ID_BITS}-bit neuron ids")
        return cls(int(owner.size), n_shards, owner.astype(np.int32), members, base,
                   internal.astype(np.int32), n_words)

    @classmethod
    def blocks(cls, n_neurons: int, n_shards: int) -> "ShardLayout":
        """Contiguous near-equal blocks (the placement greedy recovers on C = N planted graphs)."""
        sizes = community_sizes(n_neurons, n_shards)
        return cls.from_assignment(np.repeat(np.arange(n_shards), sizes), n_shards)

    def reordered(self, order_key, inh_every: int = 0) -> "ShardLayout":
        """Same shards, rows ordered by descending `order_key` inside each shard, the
        excitatory neurons before the inhibitory ones when `inh_every` > 0."""
        grp = inhibitory_mask(np.arange(self.n_neurons), inh_every).astype(np.int8) if inh_every > 0 else None
        return ShardLayout.from_assignment(self.owner, self.n_shards, order_key, grp)

    @property
    def guard_id(self) -> int:
        return (self.n_words - 1) * 32

    def n_local(self, h: int) -> int:
        return int(self.members[h].size)


# ---------------------------------------------------------------- network

def host_sell(graph: NeuronGraph, layout: ShardLayout, shard: int, inh_every: int, n_tiles: int,
              tile_words: int, cta_groups: int = 148):
    """J-SELL-32 arrays (ptr, meta, syn, row_perm) of one shard from a host NeuronGraph (numpy; see sell.py)."""
    q = q_from_p(graph.edge_p)
    post = np.concatenate([graph.edge_j, graph.edge_i]).astype(np.int64)
    pre = np.concatenate([graph.edge_i, graph.edge_j]).astype(np.int64)
    qq = np.concatenate([q, q])
    keep = layout.owner[post] == shard
    post, pre, qq = post[keep], pre[keep], qq[keep]
    row = layout.internal_id[post].astype(np.int64) - int(layout.base[shard])
    return sell.host_build(row, layout.internal_id[pre], qq, inhibitory_mask(pre, inh_every),
                           layout.n_local(shard), n_tiles, tile_words, cta_groups)


@dataclass
class GeneratorSpec:
    """Device SBM generator spec with the distributions of ModelSpec/generate_synthetic."""

    n_neurons: int
    n_communities: int
    p_in: float
    p_out: float
    seed: int = 0
    intra_p_range: tuple = INTRA_P_RANGE
    inter_p_range: tuple = INTER_P_RANGE

    @classmethod
    def from_model_spec(cls, spec: ModelSpec, **kw) -> "GeneratorSpec":
        return cls(spec.n_neurons, spec.n_communities, spec.p_in, spec.p_out, spec.seed, **kw)

    @classmethod
    def random(cls, n_neurons: int, degree: float, seed: int = 0) -> "GeneratorSpec":
        """C = 1 random network with mean degree `degree` (synapses per neuron)."""
        return cls(n_neurons, 1, degree / max(n_neurons - 1, 1), 0.0, seed)

    def to_c(self) -> "_native.GraphGenC":
        return _native.GraphGenC(
            n_neurons=self.n_neurons, n_communities=self.n_communities, p_in=self.p_in, p_out=self.p_out,
            intra_lo=self.intra_p_range[0], intra_hi=self.intra_p_range[1], inter_lo=self.inter_p_range[0],
            inter_hi=self.inter_p_range[1], seed=int(self.seed) & (2**64 - 1))

    def host_graph(self, threads: int = 0) -> NeuronGraph:
        """The generated network as a host NeuronGraph (model.py:53-92): edges ascending
        (i, j), their fp64 p, unit weights -- what the reference's planner consumes.
        Host restatement of the device generator (csrc/graphgen_host.cpp)."""
        L = _native.lib()
        g = self.to_c()
        n = int(L.nc_hostgen_edges(C.byref(g), None, None, None, int(threads)))
        if n < 0:
            _native.check(-1, "host generator")
        ei = np.empty(n, dtype=np.int64)
        ej = np.empty(n, dtype=np.int64)
        ep = np.empty(n, dtype=np.float64)
        if L.nc_hostgen_edges(C.byref(g), ei.ctypes.data, ej.ctypes.data, ep.ctypes.data, int(threads)) != n:
            raise RuntimeError("host generator: edge count changed between passes")
        return NeuronGraph(self.n_neurons, np.ones(self.n_neurons), ei, ej, ep)


ShardCSR = sell.SellCSR


class Network:
    """Per-shard pull CSRs on the device plus the replicated destination masks."""

    def __init__(self, layout: ShardLayout, shards: dict, device, inh_every: int, *, n_synapses: int,
                 source: str):
        self.layout = layout
        self.shards = shards          # shard index -> ShardCSR (the shards this process owns)
        self.device = device
        self.inh_every = inh_every
        self.n_synapses = n_synapses  # real (unpadded) synapses over the owned shards
        self.source = source

    # ------------------------------------------------------------ builders
    @classmethod
    def from_graph(cls, graph: NeuronGraph, layout: ShardLayout, *, device=None, inh_every: int = 5,
                   shards=None, tile_words: int | None = None, partials_global: bool = False,
                   bank_order: bool = True, builder: str = "device") -> "Network":
        """Pull layouts of a host NeuronGraph (model.py:53-92).  ``builder="device"``:
        the edge columns are uploaded once (int32 ids + uint8 weight units) and the
        J-SELL layout is built on the GPU by the generator's passes (nc_edges_count /
        nc_edges_fill): 1e9 synapses in seconds.  ``"host"``: numpy (sell.host_build),
        kept as an independent builder for the tests."""
        import torch
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        if builder == "device":
            return cls._from_graph_device(graph, layout, dev, inh_every, shards, tile_words, partials_global,
                                          bank_order)
        if builder != "host":
            raise ValueError(f"builder must be 'device' or 'host', got {builder!r}")
        deg = np.bincount(graph.edge_i, minlength=graph.n_neurons) + np.bincount(graph.edge_j,
                                                                               minlength=graph.n_neurons)
        layout = layout.reordered(deg, inh_every)
        own = range(layout.n_shards) if shards is None else shards
        out = {}
        nsyn = 0
        sms = sell.device_sms(dev)
        for h in own:
            n_local = layout.n_local(h)
            T, TW, pglob = _tiles(layout, n_local, sms, tile_words, partials_global)
            ptr, meta, syn, perm = host_sell(graph, layout, h, inh_every, T, TW, sms)
            counts_real = int(np.count_nonzero(layout.owner[np.concatenate([graph.edge_i, graph.edge_j])] == h))
            n_real = int(counts_real)
            csr = ShardCSR(torch.from_numpy(ptr).to(dev), torch.from_numpy(meta.view(np.int32)).to(dev),
                           torch.from_numpy(syn.view(np.int32)).to(dev), T, TW, n_local, n_real,
                           partials_global=pglob,
                           row_perm=None if perm is None else torch.from_numpy(perm).to(dev), cta_groups=sms)
            csr.dest = _dest_masks(csr, layout, h, dev)
            out[h] = csr
            nsyn += n_real
        return cls(layout, out, dev, inh_every, n_synapses=nsyn, source="host graph")

    @classmethod
    def _from_graph_device(cls, graph, layout, dev, inh_every, shards, tile_words, partials_global, bank_order):
        import torch
        if layout.n_neurons != graph.n_neurons:
            raise ValueError("layout and graph disagree on the neuron count")
        L = _native.lib()
        st = _native.stream_handle(dev)
        ei, ej, qd = upload_edges(graph, dev)
        n = int(ei.numel())
        deg = torch.bincount(ei, minlength=graph.n_neurons) + torch.bincount(ej, minlength=graph.n_neurons)
        layout = layout.reordered(deg.cpu().numpy(), inh_every)
        del deg
        owner_d = torch.from_numpy(layout.owner).to(dev)
        internal_d = torch.from_numpy(layout.internal_id).to(dev)
        own = range(layout.n_shards) if shards is None else shards
        sms = sell.device_sms(dev)
        out = {}
        nsyn = 0
        for h in own:
            n_local = layout.n_local(h)
            g = _native.GraphGenC(n_neurons=graph.n_neurons, n_communities=1, shard=h, owner=owner_d.data_ptr(),
                                  internal_id=internal_d.data_ptr(), local_base=int(layout.base[h]),
                                  inh_every=inh_every, n_local=n_local)
            count = lambda T, TW, lo, up, g=g: L.nc_edges_count(C.byref(g), ei.data_ptr(), ej.data_ptr(),  # noqa
                                                               n, T, TW, lo.data_ptr(), st)
            fill = lambda T, TW, ptr, meta, pos, fl, syn, g=g: L.nc_edges_fill(  # noqa: E731
                C.byref(g), ei.data_ptr(), ej.data_ptr(), qd.data_ptr(), n, T, TW, ptr.data_ptr(), meta.data_ptr(),
                None if pos is None else pos.data_ptr(), fl.data_ptr(), syn.data_ptr(), st)
            csr, n_real = _build_pull_shard(layout, h, dev, sms, tile_words, partials_global, bank_order, count,
                                            fill)
            csr.dest = _dest_masks(csr, layout, h, dev)
            out[h] = csr
            nsyn += n_real
        return cls(layout, out, dev, inh_every, n_synapses=nsyn, source="host graph (device build)")

    @classmethod
    def generate(cls, spec: GeneratorSpec, layout: ShardLayout, *, device=None, inh_every: int = 5,
                 shards=None, tile_words: int | None = None, bank_order: bool = True, pull: bool = True,
                 push: bool = False, push_windows: int | None = None, group_inhibitory: bool = True) -> "Network":
        """Counter-based device generator (csrc/graphgen.cu); every shard regenerates the same graph.

        ``pull``: the J-SELL pull layout (fused / pull / binned delivery).  ``push``:
        the push CSR of the event-driven engines, generated directly (without the
        pull layout when ``pull`` is False: 4 B per synapse instead of 3.2 + 4 + the
        build's transient 8), grouped into ``push_windows`` post-row windows (None:
        push_windows_for(rows of the shard), what the persistent engine wants).
        ``group_inhibitory``: excitatory internal ids before inhibitory ones in each
        shard (ShardLayout.from_assignment); results are identical either way."""
        import torch
        if not (pull or push):
            raise ValueError("generate at least one of the pull and push layouts")
        if layout.n_neurons != spec.n_neurons:
            raise ValueError("layout and generator disagree on the neuron count")
        if not 1 <= spec.n_communities <= spec.n_neurons:
            raise ValueError("n_communities must be in [1, n_neurons]")
        if not 0.0 <= spec.p_out <= spec.p_in <= 1.0:
            raise ValueError("edge probabilities must satisfy 0 <= p_out <= p_in <= 1")
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        L = _native.lib()
        st = _native.stream_handle(dev)
        # pass 0: degrees -> rows of each shard ordered by degree (SELL padding)
        g0 = _native.GraphGenC(
            n_neurons=spec.n_neurons, n_communities=spec.n_communities, shard=0, p_in=spec.p_in, p_out=spec.p_out,
            intra_lo=spec.intra_p_range[0], intra_hi=spec.intra_p_range[1], inter_lo=spec.inter_p_range[0],
            inter_hi=spec.inter_p_range[1], seed=int(spec.seed) & (2**64 - 1), owner=None, internal_id=None,
            local_base=0, inh_every=inh_every)
        deg = torch.zeros(spec.n_neurons, dtype=torch.int32, device=dev)
        _native.check(L.nc_graphgen_degrees(C.byref(g0), deg.data_ptr(), st), "graphgen degrees")
        layout = layout.reordered(deg.cpu().numpy(), inh_every if group_inhibitory else 0)
        del deg
        owner_d = torch.from_numpy(layout.owner).to(dev)
        internal_d = torch.from_numpy(layout.internal_id).to(dev)
        own = range(layout.n_shards) if shards is None else shards
        out = {}
        nsyn = 0
        sms = sell.device_sms(dev)
        for h in own:
            n_local = layout.n_local(h)
            if not pull:
                csr = _push_only_csr(layout, h, dev)
                g = _native.GraphGenC(
                    n_neurons=spec.n_neurons, n_communities=spec.n_communities, shard=h, p_in=spec.p_in,
                    p_out=spec.p_out, intra_lo=spec.intra_p_range[0], intra_hi=spec.intra_p_range[1],
                    inter_lo=spec.inter_p_range[0], inter_hi=spec.inter_p_range[1],
                    seed=int(spec.seed) & (2**64 - 1), owner=owner_d.data_ptr(), internal_id=internal_d.data_ptr(),
                    local_base=int(layout.base[h]), inh_every=inh_every, n_local=n_local)
                win = push_windows if push_windows is not None else push_windows_for(n_local)
                csr.dest = _generate_push(g, csr, layout, h, dev, win)
                csr.n_real = int(csr._push_total)
                out[h] = csr
                nsyn += csr.n_real
                continue
            g = _native.GraphGenC(
                n_neurons=spec.n_neurons, n_communities=spec.n_communities, shard=h, p_in=spec.p_in,
                p_out=spec.p_out, intra_lo=spec.intra_p_range[0], intra_hi=spec.intra_p_range[1],
                inter_lo=spec.inter_p_range[0], inter_hi=spec.inter_p_range[1],
                seed=int(spec.seed) & (2**64 - 1), owner=owner_d.data_ptr(), internal_id=internal_d.data_ptr(),
                local_base=int(layout.base[h]), inh_every=inh_every, n_local=n_local)
            count = lambda T, TW, lo, up, g=g: L.nc_graphgen_count(C.byref(g), T, TW, lo.data_ptr(),  # noqa: E731
                                                                  up.data_ptr(), st)
            fill = lambda T, TW, ptr, meta, pos, fl, syn, g=g: L.nc_graphgen_fill(  # noqa: E731
                C.byref(g), T, TW, ptr.data_ptr(), meta.data_ptr(), None if pos is None else pos.data_ptr(),
                fl.data_ptr(), syn.data_ptr(), st)
            csr, n_real = _build_pull_shard(layout, h, dev, sms, tile_words, False, bank_order, count, fill)
            csr.dest = _dest_masks(csr, layout, h, dev)
            if push:
                _generate_push(g, csr, layout, h, dev,
                               push_windows if push_windows is not None else push_windows_for(n_local))
            out[h] = csr
            nsyn += n_real
        return cls(layout, out, dev, inh_every, n_synapses=nsyn, source="device generator")

    # ------------------------------------------------------------ helpers
    def global_dest(self):
        """Destination mask of every internal id (int16 bit patterns), for relays."""
        import torch
        g = torch.zeros(self.layout.n_words * 32, dtype=torch.int32, device=self.device)
        for h, csr in self.shards.items():
            b = int(self.layout.base[h])
            g[b:b + self.layout.n_local(h)] = csr.dest
        return _as_u16(g)

    def host_csr(self, shard: int):
        """(post_gid, pre_gid, q) of every synapse of one shard, for the oracle (test/bench only)."""
        row, pre_int, q, inh = (x.cpu().numpy() for x in sell.decode(self.shards[shard]))
        gid_of_internal = np.full(self.layout.n_words * 32, -1, dtype=np.int64)
        for h, m in enumerate(self.layout.members):
            gid_of_internal[int(self.layout.base[h]) + np.arange(m.size)] = m
        pre = gid_of_internal[pre_int]
        if (inhibitory_mask(pre, self.inh_every) != inh).any():
            raise AssertionError("E/I slot split disagrees with the pre neuron types")
        return self.layout.members[shard][row], pre, q.astype(np.uint8)


def upload_edges(graph: NeuronGraph, dev, chunk: int | None = None, depth: int = 3):
    """Edge columns of a NeuronGraph on the device as int32 ids and uint8 weight units
    q = ceil(32 p) (q_from_p).

    int64 id columns (the reference's): `_upload_edges_narrowed`, narrowed on the host.
    Other integer widths: pipelined through `depth` pinned staging buffers of `chunk` edges: the host copies
    chunk k into a pinned buffer (torch's multi-threaded CPU copy, any integer / float
    dtype widened to int64 / float64) while the copy engine moves chunk k-1 and a side
    stream narrows it on the device; endpoint range checks are reduced on the device and
    read once at the end.  (A pageable .to(device) goes through the driver's single
    staging thread.)"""
    import torch
    m = int(graph.n_neurons)
    if m >= 2**31:
        raise ValueError("at most 2^31 - 1 neurons")
    n = int(graph.edge_i.size)
    ei = torch.empty(n, dtype=torch.int32, device=dev)
    ej = torch.empty(n, dtype=torch.int32, device=dev)
    qd = torch.empty(max(n, 1), dtype=torch.uint8, device=dev)
    if n == 0:
        return ei, ej, qd[:0]
    cols = [np.ascontiguousarray(a) for a in (graph.edge_i, graph.edge_j)]
    pcol = np.ascontiguousarray(graph.edge_p, dtype=np.float64)
    if all(c.dtype == np.int64 for c in cols):
        return _upload_edges_narrowed(cols[0], cols[1], pcol, m, ei, ej, qd, dev, chunk or (1 << 23), depth)
    src = [torch.from_numpy(a) for a in cols]
    src_p = torch.from_numpy(pcol)
    c = min(chunk or (1 << 21), n)
    k_buf = min(depth, (n + c - 1) // c)
    host = [torch.empty((3, c), dtype=torch.int64, pin_memory=True) for _ in range(k_buf)]
    devb = [torch.empty((3, c), dtype=torch.int64, device=dev) for _ in range(k_buf)]
    done = [None] * k_buf
    lo = torch.full((1,), 0, dtype=torch.int64, device=dev)
    hi = torch.full((1,), 0, dtype=torch.int64, device=dev)
    side = torch.cuda.Stream(dev)
    side.wait_stream(torch.cuda.current_stream(dev))
    for idx, a in enumerate(range(0, n, c)):
        b = min(n, a + c)
        k, w = idx % k_buf, b - a
        if done[k] is not None:
            done[k].synchronize()          # the copy engine has drained this staging buffer
        h = host[k]
        h[0, :w].copy_(src[0][a:b])
        h[1, :w].copy_(src[1][a:b])
        h[2, :w].view(torch.float64).copy_(src_p[a:b])
        with torch.cuda.stream(side):
            d = devb[k]
            d[:, :w].copy_(h[:, :w], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(side)
            done[k] = ev
            ids = d[:2, :w]
            torch.minimum(lo, ids.min().view(1), out=lo)
            torch.maximum(hi, ids.max().view(1), out=hi)
            ei[a:b].copy_(d[0, :w])
            ej[a:b].copy_(d[1, :w])
            qd[a:b] = torch.ceil(d[2, :w].view(torch.float64) * Q_LEVELS).clamp_(1, Q_LEVELS).to(torch.uint8)
    torch.cuda.current_stream(dev).wait_stream(side)
    for t in (ei, ej, qd, lo, hi):
        t.record_stream(side)
    if int(lo.item()) < 0 or int(hi.item()) >= m:
        raise ValueError(f"edge endpoints outside [0, {m})")
    return ei, ej, qd[:n]


def _upload_edges_narrowed(ci, cj, cp, m: int, ei, ej, qd, dev, chunk: int, depth: int):
    """upload_edges for int64 / fp64 columns (what generate_synthetic and load_graph give):
    the host narrows each chunk into pinned staging buffers -- int32 ids, uint8 weight units,
    endpoint range check -- in one multi-threaded native pass (nc_edges_narrow, the GIL
    released), so the copy engine moves 9 instead of 24 bytes per edge and the device does
    no conversion; the pass over chunk k overlaps the copy of chunk k - 1."""
    import torch
    n = int(ci.size)
    L = _native.lib()
    c = min(chunk, n)
    k_buf = min(depth, (n + c - 1) // c)
    host = [torch.empty(9 * c, dtype=torch.uint8, pin_memory=True) for _ in range(k_buf)]
    done = [None] * k_buf
    side = torch.cuda.Stream(dev)
    side.wait_stream(torch.cuda.current_stream(dev))
    for idx, a in enumerate(range(0, n, c)):
        b = min(n, a + c)
        k, w = idx % k_buf, b - a
        if done[k] is not None:
            done[k].synchronize()
        h = host[k]
        hi, hj, hq = h[: 4 * c].view(torch.int32), h[4 * c: 8 * c].view(torch.int32), h[8 * c:]
        _native.check(L.nc_edges_narrow(ci.ctypes.data + 8 * a, cj.ctypes.data + 8 * a, cp.ctypes.data + 8 * a, w, m,
                                        hi.data_ptr(), hj.data_ptr(), hq.data_ptr(), 0), "edge upload")
        with torch.cuda.stream(side):
            ei[a:b].copy_(hi[:w], non_blocking=True)
            ej[a:b].copy_(hj[:w], non_blocking=True)
            qd[a:b].copy_(hq[:w], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(side)
            done[k] = ev
    torch.cuda.current_stream(dev).wait_stream(side)
    for t in (ei, ej, qd):
        t.record_stream(side)
    return ei, ej, qd[:n]


def _build_pull_shard(layout: ShardLayout, h: int, dev, sms: int, tile_words, partials_global: bool,
                      bank_order: bool, count, fill):
    """J-SELL-32 pull layout of shard h on the device from an edge source (the
    generator or an uploaded edge list): count entries per (row, tile, sign)
    segment -> tile placement and block starts -> fill the unpacked padded SELL
    -> bank order -> pack 5 fields per 16-byte slot -> drop the padding (J-SELL)."""
    import torch
    L = _native.lib()
    st = _native.stream_handle(dev)
    n_local = layout.n_local(h)
    T, TW, pglob = _tiles(layout, n_local, sms, tile_words, partials_global)
    n_seg = max(n_local * T * 2, 1)
    lower = torch.zeros(n_seg, dtype=torch.int32, device=dev)
    upper = torch.zeros(n_seg, dtype=torch.int32, device=dev)
    _native.check(count(T, TW, lower, upper), "pull layout count")
    counts = (lower + upper)[: n_local * T * 2].to(torch.int64)
    perm, pos_of = sell.tile_placement(sell.row_slots(counts, n_local, T), n_local, T, sms)
    ptr, meta = sell.layout_from_counts(counts, n_local, T, perm)
    total = int(ptr[-1].item())
    syn = torch.zeros(max(total * sell.SLOT_ENTRIES, 4), dtype=torch.int32, device=dev)   # unpacked
    _native.check(L.nc_sell_fill_pads(ptr.data_ptr(), ptr.numel() - 1, T, TW, syn.data_ptr(), st), "sell pads")
    lower.zero_()
    pos_of = None if pos_of is None else pos_of.contiguous()
    _native.check(fill(T, TW, ptr, meta, pos_of, lower, syn), "pull layout fill")
    n_real = int(counts.sum().item())
    del upper, counts, lower
    if bank_order:   # spread each lookup instruction's 32 lanes over the 32 banks (config 2,
        # packed slots: shared wavefronts 110 M -> 60 M, kernel 1.3 % faster)
        src = syn.clone()
        _native.check(L.nc_sell_bank_order(ptr.data_ptr(), meta.data_ptr(), T, n_local, src.data_ptr(),
                                           syn.data_ptr(), st), "bank order")
        torch.cuda.synchronize(dev)
        del src
    # 5 entries per slot -> 16-byte slots of 25-bit fields
    packed = torch.empty(max(total * 4, 4), dtype=torch.int32, device=dev)
    _native.check(L.nc_sell_pack(syn.data_ptr(), total, packed.data_ptr(), st), "sell pack")
    torch.cuda.synchronize(dev)
    del syn
    syn = packed
    # padded SELL-32 -> J-SELL-32 (drops the padding of every block to its longest row)
    jptr = sell.jagged_ptr(meta, n_local, T)
    jsyn = torch.empty(max(int(jptr[-1].item()) * 4, 4), dtype=torch.int32, device=dev)
    _native.check(L.nc_sell_repack(ptr.data_ptr(), jptr.data_ptr(), meta.data_ptr(), T, n_local,
                                   syn.data_ptr(), jsyn.data_ptr(), 1, st), "sell repack")
    torch.cuda.synchronize(dev)
    del syn, ptr, pos_of
    csr = ShardCSR(jptr, meta, jsyn, T, TW, n_local, n_real, partials_global=pglob,
                   row_perm=None if perm is None else sell.local_index(perm, sms).reshape(-1).contiguous(),
                   cta_groups=sms)
    return csr, n_real


def _push_only_csr(layout: ShardLayout, h: int, dev) -> ShardCSR:
    """A shard without the pull layout (event-driven engines only): one-tile
    placeholders keep the descriptor valid; has_pull is False."""
    import torch
    csr = ShardCSR(torch.zeros(2, dtype=torch.int64, device=dev), torch.zeros(1, dtype=torch.int32, device=dev),
                   torch.zeros(4, dtype=torch.int32, device=dev), 1, layout.n_words, layout.n_local(h), 0)
    csr.has_pull = False
    return csr


def _generate_push(g, csr: ShardCSR, layout: ShardLayout, h: int, dev, windows: int = 1):
    """Push CSR of shard h straight from the generator (nc_graphgen_push, or
    nc_graphgen_push_windowed for windows > 1), cached on the SellCSR like the
    transposes (push_arrays); returns the destination masks (int32 [n_local])."""
    import torch
    L = _native.lib()
    st = _native.stream_handle(dev)
    n_pre = layout.n_words * 32
    n_local = layout.n_local(h)
    if windows > 1:
        rows = max(32, ((n_local + 31) // 32 + windows - 1) // windows * 32)
        dest16 = torch.zeros(n_local + 2, dtype=torch.int16, device=dev)
        counts = torch.zeros(n_pre * windows, dtype=torch.int32, device=dev)
        _native.check(L.nc_graphgen_push_windowed(C.byref(g), 0, windows, rows, counts.data_ptr(), None, None, None,
                                                  None, dest16.data_ptr(), st), "graphgen windowed push count")
        run = torch.cumsum(counts.view(n_pre, windows), 1, dtype=torch.int64)
        row_len = run[:, -1]
        if n_pre and int(row_len.max().item()) >= 1 << 16:
            raise ValueError("windowed push: a pre neuron has >= 65536 local synapses (16-bit offsets)")
        winoff = torch.zeros((n_pre, windows + 1), dtype=torch.int32, device=dev)
        winoff[:, 1:] = run.to(torch.int32)
        winoff16 = winoff.to(torch.int16)
        rowptr = torch.zeros(n_pre + 1, dtype=torch.int64, device=dev)
        rowptr[1:] = torch.cumsum(row_len, 0)
        del run, winoff, row_len
        total = int(rowptr[-1].item())
        ent = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
        counts.zero_()
        _native.check(L.nc_graphgen_push_windowed(C.byref(g), 1, windows, rows, None, rowptr.data_ptr(),
                                                  winoff16.data_ptr(), counts.data_ptr(), ent.data_ptr(), None, st),
                      "graphgen windowed push fill")
        torch.cuda.synchronize(dev)
        del counts
        csr.__dict__.setdefault("_push_arrays", {})[windows] = {
            "rowptr": rowptr, "syn": ent, "winoff": winoff16, "windows": windows, "rows": rows}
        csr._push_total = total
        return dest16[:n_local].to(torch.int32) & 0xFFFF
    rowptr = torch.zeros(n_pre + 1, dtype=torch.int64, device=dev)
    dest16 = torch.zeros(n_local + 2, dtype=torch.int16, device=dev)
    _native.check(L.nc_graphgen_push(C.byref(g), 0, rowptr.data_ptr(), None, None, dest16.data_ptr(), st),
                  "graphgen push count")
    torch.cumsum(rowptr, 0, out=rowptr)
    total = int(rowptr[-1].item())
    ent = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
    fill = torch.zeros(n_pre, dtype=torch.int32, device=dev)
    _native.check(L.nc_graphgen_push(C.byref(g), 1, rowptr.data_ptr(), fill.data_ptr(), ent.data_ptr(), None, st),
                  "graphgen push fill")
    torch.cuda.synchronize(dev)
    del fill
    csr._push_cache = (rowptr, ent)
    csr.__dict__.setdefault("_push_arrays", {})[1] = {"rowptr": rowptr, "syn": ent, "winoff": None, "windows": 1,
                                                      "rows": 0}
    csr._push_total = total
    return dest16[:n_local].to(torch.int32) & 0xFFFF


def _tiles(layout: ShardLayout, n_local: int, sms: int, tile_words: int | None, partials_global: bool = False):
    """Bitmap tiling (n_tiles, tile_words, partials_in_global): planned from shared
    memory, or forced (tests) with `tile_words` / `partials_global`."""
    if tile_words is None:
        return sell.plan_tiles(layout.n_words, n_local, sms)
    tw = max(4, int(tile_words) // 4 * 4)
    return (layout.n_words + tw - 1) // tw, tw, bool(partials_global)


def _as_u16(t32):
    import torch
    t = t32.to(torch.int32) & 0xFFFF
    return torch.where(t >= 0x8000, t - 0x10000, t).to(torch.int16)


def _dest_masks(csr: ShardCSR, layout: ShardLayout, h: int, dev):
    import torch
    n_local = layout.n_local(h)
    bases = torch.from_numpy(layout.base.astype(np.int32)).to(dev)
    out16 = torch.zeros(n_local + 2, dtype=torch.int16, device=dev)   # OR-ed through aligned 32-bit words
    L = _native.lib()
    _native.check(L.nc_dest_mask_from_csr(csr.slice_ptr.data_ptr(), csr.row_meta.data_ptr(),
                                          None if csr.row_perm is None else csr.row_perm.data_ptr(),
                                          csr.cta_groups, csr.n_tiles,
                                          csr.tile_words, csr.syn.data_ptr(), n_local,
                                          bases.data_ptr(),
                                          layout.n_shards, h, out16.data_ptr(), _native.stream_handle(dev)),
                  "dest mask")
    return out16[:n_local].to(torch.int32) & 0xFFFF


# ---------------------------------------------------------------- exchange plan

class ExchangePlan:
    """Next hops and relay sets from a RoutingTable (routing.py:61-115).

    ``next_hop[s, d]``: first hop of demand (s, d), -1 if there is no demand.
    ``fwd[b, s]``: bitmask of destinations d whose path is (s, b, d) -- the
    shards relay b forwards spikes from s to (two-level routing).
    """

    def __init__(self, n_shards: int, rt: RoutingTable | None):
        n = n_shards
        if rt is None:
            nh = np.full((n, n), -1, dtype=np.int64)
            off = ~np.eye(n, dtype=bool)
            nh[off] = np.tile(np.arange(n), (n, 1))[off]
            via = np.full((n, n), -1, dtype=np.int64)
        else:
            if rt.n_gpus != n:
                raise ValueError(f"routing table covers {rt.n_gpus} GPUs, partition has {n}")
            nh = rt.next_hop_matrix()
            via = np.full((n, n), -1, dtype=np.int64)
            via[rt.src, rt.dst] = rt.via
        fwd = np.zeros((n, n), dtype=np.int64)
        for s in range(n):
            for d in range(n):
                if via[s, d] >= 0:
                    fwd[via[s, d], s] |= 1 << d
        self.n = n
        self.next_hop = nh
        self.fwd = fwd
        self.two_level = bool((via >= 0).any())

    def hop_masks(self, dest, shard: int):
        """Per-neuron next-hop bitmask (int16) from its destination mask."""
        import torch
        hm = torch.zeros_like(dest)
        for d in range(self.n):
            if d == shard:
                continue
            bit = (dest >> d) & 1
            h = int(self.next_hop[shard, d])
            if h < 0:
                if bool(bit.any()):
                    raise ValueError(
                        f"neurons on GPU {shard} target GPU {d} but the routing table has no demand ({shard}, {d})"
                    )
                continue
            hm |= bit << h
        return _as_u16(hm)

    def fwd_table_u16(self) -> np.ndarray:
        return np.ascontiguousarray(self.fwd.astype(np.uint16).reshape(-1))


# ---------------------------------------------------------------- simulator

@dataclass
class SimReport:
    """Outputs of :func:`simulate` (host numpy unless noted)."""

    steps: int
    n_gpus: int
    raster: np.ndarray | None          # bool [recorded steps, M] in global neuron ids
    deliv_ids: np.ndarray              # int64 [steps or 1, N, N]: ids of s delivered to d
    hop_ids: np.ndarray                # int64 [steps or 1, N, N]: ids on channel u->v
    spikes: int                        # total spikes
    v: np.ndarray | None               # final membrane voltage per gid
    i_syn: np.ndarray | None
    elapsed_ms: float                  # device time of the step loop (CUDA events)
    exchange: str = "none"
    delivery: str = "fused"
    extra: dict = field(default_factory=dict)

    @property
    def steps_per_s(self) -> float:
        return self.steps / (self.elapsed_ms * 1e-3) if self.elapsed_ms > 0 else float("inf")

    def spike_ids(self, t: int) -> np.ndarray:
        return np.flatnonzero(self.raster[t])

    def rate_hz(self, dt_ms: float = 1.0) -> float:
        m = self.v.size if self.v is not None else 0
        return self.spikes / max(m, 1) / (self.steps * dt_ms * 1e-3) if m else float("nan")


class _ShardState:
    """Device buffers and the C descriptor of one shard."""

    def __init__(self, net: Network, h: int, plan: ExchangePlan, *, record_steps: int, push: bool,
                 bucket_cap: int | None, bucket_stride: int | None = None, binned: bool = False,
                 push_windows: int = 1):
        import torch
        lay = net.layout
        dev = net.device
        n_local = lay.n_local(h)
        nl = max(n_local, 1)
        self.h = h
        self.n_local = n_local
        self.local_words = (n_local + 31) // 32
        csr = net.shards[h]
        self.csr = csr
        self.v = torch.zeros(nl, dtype=torch.float32, device=dev)
        self.i_syn = torch.zeros(nl, dtype=torch.float32, device=dev)
        self.refrac = torch.zeros(nl, dtype=torch.uint8, device=dev)
        self.acc = torch.zeros(nl, dtype=torch.int32, device=dev)
        self.gid = torch.from_numpy(lay.members[h].astype(np.int32)).to(dev) if n_local else \
            torch.zeros(1, dtype=torch.int32, device=dev)
        self.hop_mask = plan.hop_masks(csr.dest, h) if (lay.n_shards > 1 and n_local) else \
            torch.zeros(nl, dtype=torch.int16, device=dev)
        self.bitmaps = torch.zeros((2, lay.n_words), dtype=torch.int32, device=dev)
        n = lay.n_shards
        if n > 1 and n_local:
            hm = self.hop_mask.to(torch.int32) & 0xFFFF
            per_hop = torch.stack([((hm >> k) & 1).sum() for k in range(n)]).cpu().numpy()
            cap = int(per_hop.max()) if per_hop.size else 1
        else:
            cap = 1
        if bucket_cap is not None:
            cap = min(cap, int(bucket_cap))
        self.exact_cap = cap
        self.bucket_cap = max(cap, 1) if bucket_stride is None else int(bucket_stride)
        self.bucket_ids = torch.zeros(n * self.bucket_cap, dtype=torch.int32, device=dev)
        self.bucket_count = torch.zeros(n, dtype=torch.int32, device=dev)
        self.status = torch.zeros(2, dtype=torch.int32, device=dev)
        self.step = torch.zeros(1, dtype=torch.int32, device=dev)
        self.record_steps = int(record_steps)
        self.raster = torch.zeros((max(self.record_steps, 1), max(self.local_words, 1)), dtype=torch.int32,
                                  device=dev)
        self.spike_total = torch.zeros(1, dtype=torch.int64, device=dev)
        self.work = torch.zeros(4 + 32, dtype=torch.int32, device=dev)   # + per-window push claims
        self.push_rowptr = self.push_syn = None
        self.push = None
        if push:
            self.push = push_arrays(csr, lay, h, dev, push_windows)
            self.push_rowptr, self.push_syn = self.push["rowptr"], self.push["syn"]
        self.pb = None
        self.spk_ids = self.spk_count = None
        if binned:
            self.pb = _push_binned(csr, lay, h, dev)
        if binned:
            # spike lists by step parity (local fired ids from the LIF phase, remote ones
            # appended by the exchange); every internal id fires at most once per step
            self.spk_cap = lay.n_words * 32
            self.spk_ids = torch.zeros(2 * self.spk_cap, dtype=torch.int32, device=dev)
            self.spk_count = torch.zeros(2, dtype=torch.int32, device=dev)
        self.c = _native.ShardC(
            shard=h, n_shards=n, n_local=n_local, local_base=int(lay.base[h]), n_words=lay.n_words,
            n_tiles=csr.n_tiles, tile_words=csr.tile_words,
            flags=(1 if csr.partials_global else 0) | (sell.block_split(n_local, csr.n_tiles, csr.cta_groups) << 1)
            | (8 if sell.triple_buffer(n_local, csr.n_tiles, csr.tile_words, csr.cta_groups, csr.partials_global)
               else 0),
            v=self.v.data_ptr(), i_syn=self.i_syn.data_ptr(), refrac=self.refrac.data_ptr(),
            acc=self.acc.data_ptr(), gid=self.gid.data_ptr(), hop_mask=self.hop_mask.data_ptr(),
            slice_ptr=csr.slice_ptr.data_ptr(), row_meta=csr.row_meta.data_ptr(), syn=csr.syn.data_ptr(),
            push_rowptr=None if self.push_rowptr is None else self.push_rowptr.data_ptr(),
            push_syn=None if self.push_syn is None else self.push_syn.data_ptr(),
            bitmap0=self.bitmaps[0].data_ptr(), bitmap1=self.bitmaps[1].data_ptr(),
            fired_ids=None, fired_count=None,
            bucket_ids=self.bucket_ids.data_ptr(), bucket_count=self.bucket_count.data_ptr(),
            bucket_cap=self.bucket_cap, status=self.status.data_ptr(), step=self.step.data_ptr(),
            raster=self.raster.data_ptr() if self.record_steps > 0 else None,
            record_steps=self.record_steps, local_words=self.local_words,
            spike_total=self.spike_total.data_ptr(), work=self.work.data_ptr(),
            row_perm=None if csr.row_perm is None else csr.row_perm.data_ptr(), cta_groups=csr.cta_groups)
        self.c_t = _native.as_bytes(self.c)   # the descriptor as the torch ops take it (a view)
        if self.push is not None and self.push["windows"] > 1:
            self.c.push_winoff = self.push["winoff"].data_ptr()
            self.c.push_windows, self.c.push_window_rows = self.push["windows"], self.push["rows"]
        if self.pb is not None:
            self.c.pb_bins, self.c.pb_rows = self.pb["bins"], self.pb["rows"]
            self.c.pb_rowptr = self.pb["rowptr"].data_ptr()
            self.c.pb_binoff = self.pb["binoff"].data_ptr()
            self.c.pb_syn = self.pb["syn"].data_ptr()
        if self.spk_ids is not None:
            self.c.spk_ids, self.c.spk_count, self.c.spk_cap = (self.spk_ids.data_ptr(), self.spk_count.data_ptr(),
                                                                self.spk_cap)


def _push_binned(csr: ShardCSR, lay: ShardLayout, h: int, dev, bins: int | None = None):
    """Binned push synapses of one shard (include/neurocomm_b200.h, nc_shard_t pb_*):
    rows = internal pre ids, entries grouped by the bin that owns their post row;
    built on the device by nc_build_push_binned.  bins = the SM count for
    k_step_binned (a CTA per bin), or a few L2-sized windows for the persistent
    engine (nc_shard_t push_windows: the same format).  Cached on the SellCSR."""
    import torch
    L = _native.lib()
    st = _native.stream_handle(dev)
    n_local = lay.n_local(h)
    bins = sell.device_sms(dev) if bins is None else int(bins)
    cache = csr.__dict__.setdefault("_binned_cache", {})
    if bins in cache:
        return cache[bins]
    rows = max(32, ((n_local + 31) // 32 + bins - 1) // bins * 32)
    n_pre = lay.n_words * 32
    scratch = torch.zeros(8, dtype=torch.int32, device=dev)
    c = _native.ShardC(shard=h, n_shards=lay.n_shards, n_local=n_local, local_base=int(lay.base[h]),
                       n_words=lay.n_words, n_tiles=csr.n_tiles, tile_words=csr.tile_words, flags=0,
                       slice_ptr=csr.slice_ptr.data_ptr(), row_meta=csr.row_meta.data_ptr(), syn=csr.syn.data_ptr(),
                       bitmap0=scratch.data_ptr(), bitmap1=scratch.data_ptr(), status=scratch.data_ptr(),
                       step=scratch.data_ptr(),
                       row_perm=None if csr.row_perm is None else csr.row_perm.data_ptr(),
                       cta_groups=csr.cta_groups, pb_bins=bins, pb_rows=rows)
    counts = torch.zeros(n_pre * bins, dtype=torch.int32, device=dev)
    _native.check(L.nc_build_push_binned(C.byref(c), 0, counts.data_ptr(), None, None, None, None, st),
                  "binned push count")
    per_bin = counts.view(n_pre, bins)
    run = torch.cumsum(per_bin, 1, dtype=torch.int64)
    row_len = run[:, -1]
    if n_pre and int(row_len.max().item()) >= 1 << 16:
        raise ValueError("binned push: a pre neuron has >= 65536 local synapses (16-bit bin offsets)")
    binoff = torch.zeros((n_pre, bins + 1), dtype=torch.int32, device=dev)
    binoff[:, 1:] = run.to(torch.int32)
    binoff16 = binoff.to(torch.int16)   # values < 2^16 (two's complement view of uint16)
    rowptr = torch.zeros(n_pre + 1, dtype=torch.int64, device=dev)
    rowptr[1:] = torch.cumsum(row_len, 0)
    total = int(rowptr[-1].item())
    del run, binoff, per_bin
    counts.zero_()
    syn = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
    _native.check(L.nc_build_push_binned(C.byref(c), 1, None, rowptr.data_ptr(), binoff16.data_ptr(),
                                         counts.data_ptr(), syn.data_ptr(), st), "binned push fill")
    torch.cuda.synchronize(dev)
    del counts, scratch
    out = {"bins": bins, "rows": rows, "rowptr": rowptr, "binoff": binoff16, "syn": syn}
    cache[bins] = out
    return out


PUSH_WINDOW_BYTES = 64 << 20   # int32 accumulators per push window (config 3 on 1 GPU, 40 MB: 1 window is fastest)


def push_windows_for(n_local: int) -> int:
    """Windows of the persistent engine's push delivery for a shard (nc_shard_t
    push_windows): 1 while the shard's accumulators (4 B per post row) fit in
    PUSH_WINDOW_BYTES, else enough windows of at most that size (config 5 over 2
    GPUs: 25 M rows -> 2 windows)."""
    return int(min(32, max(1, -(-int(n_local) * 4 // PUSH_WINDOW_BYTES))))


def push_arrays(csr: ShardCSR, lay: ShardLayout, h: int, dev, windows: int = 1) -> dict:
    """Push synapses of one shard for the event-driven engines: {"rowptr", "syn",
    "winoff", "windows", "rows"}; windows > 1 groups every row by post-row window
    (entries relative to the window start).  Generated directly by Network.generate
    (push=True) or transposed from the pull layout here; cached on the SellCSR."""
    cache = csr.__dict__.setdefault("_push_arrays", {})
    if windows in cache:
        return cache[windows]
    if not getattr(csr, "has_pull", True):
        if not cache:
            raise ValueError("this shard has neither a pull layout nor push synapses")
        return next(iter(cache.values()))   # push-only network: the windows it was generated with
    if windows <= 1:
        rowptr, ent = _push_csr(csr, lay, h, dev)
        out = {"rowptr": rowptr, "syn": ent, "winoff": None, "windows": 1, "rows": 0}
    else:
        pb = _push_binned(csr, lay, h, dev, bins=windows)
        out = {"rowptr": pb["rowptr"], "syn": pb["syn"], "winoff": pb["binoff"], "windows": windows,
               "rows": pb["rows"]}
    cache[windows] = out
    return out


def _push_csr(csr: ShardCSR, lay: ShardLayout, h: int, dev):
    """Transpose of the pull synapses (rows = internal pre ids), entries
    (inhibitory << 31) | ((q - 1) << 26) | post_local, built on the device by
    the counting-sort kernel nc_build_push_csr.  Cached on the SellCSR."""
    import torch
    cached = getattr(csr, "_push_cache", None)
    if cached is not None:
        return cached
    L = _native.lib()
    st = _native.stream_handle(dev)
    n_rows = lay.n_words * 32
    scratch = torch.zeros(8, dtype=torch.int32, device=dev)
    c = _native.ShardC(shard=h, n_shards=lay.n_shards, n_local=lay.n_local(h), local_base=int(lay.base[h]),
                       n_words=lay.n_words, n_tiles=csr.n_tiles, tile_words=csr.tile_words, flags=0,
                       slice_ptr=csr.slice_ptr.data_ptr(), row_meta=csr.row_meta.data_ptr(), syn=csr.syn.data_ptr(),
                       bitmap0=scratch.data_ptr(), bitmap1=scratch.data_ptr(), status=scratch.data_ptr(),
                       step=scratch.data_ptr(),
                       row_perm=None if csr.row_perm is None else csr.row_perm.data_ptr(),
                       cta_groups=csr.cta_groups)
    rowptr = torch.zeros(n_rows + 1, dtype=torch.int64, device=dev)
    _native.check(L.nc_build_push_csr(C.byref(c), 0, rowptr.data_ptr(), None, None, st), "push csr count")
    torch.cumsum(rowptr, 0, out=rowptr)
    total = int(rowptr[-1].item())
    ent = torch.empty(max(total, 1), dtype=torch.int32, device=dev)
    fill = torch.zeros(n_rows, dtype=torch.int32, device=dev)
    _native.check(L.nc_build_push_csr(C.byref(c), 1, rowptr.data_ptr(), fill.data_ptr(), ent.data_ptr(), st),
                  "push csr fill")
    del fill, scratch
    csr._push_cache = (rowptr, ent)
    return rowptr, ent


def _check_layouts(net: Network, delivery: str):
    if delivery in ("fused", "pull", "binned") and not all(getattr(c, "has_pull", True)
                                                           for c in net.shards.values()):
        raise ValueError(f"delivery {delivery!r} needs the pull layout: Network.generate(..., pull=True)")


_LIBCUDA = None


def _upload_graph(g, device) -> None:
    """cuGraphUpload of a captured graph: its first replay (often inside a timed region)
    then does not pay the upload of the executable graph (~1 ms for a 20-step graph at 4
    GPUs, where it also stalled the peers' exchange)."""
    import ctypes
    global _LIBCUDA
    if _LIBCUDA is None:
        _LIBCUDA = ctypes.CDLL("libcuda.so.1")
        _LIBCUDA.cuGraphUpload.argtypes = [ctypes.c_void_p, ctypes.c_void_p]
        _LIBCUDA.cuGraphUpload.restype = ctypes.c_int
    rc = _LIBCUDA.cuGraphUpload(ctypes.c_void_p(int(g.raw_cuda_graph_exec())),
                                ctypes.c_void_p(_native.stream_handle(device)))
    if rc != 0:
        raise RuntimeError(f"cuGraphUpload failed ({rc})")


class StepGraphs:
    """CUDA graphs of k consecutive steps, one per chunk length k, captured once.

    Capturing does not run anything, so :meth:`prepare` can capture every chunk
    length a loop of `steps` will replay before a timed region starts."""

    def __init__(self, device, one_step, chunk: int):
        self.device = device
        self.one_step = one_step          # one_step(stream_handle) enqueues one step
        self.chunk = max(1, int(chunk))
        self.graphs: dict = {}

    def clear(self):
        self.graphs.clear()

    def _chunks(self, steps: int):
        done = 0
        while done < steps:
            k = min(self.chunk, steps - done)
            yield k
            done += k

    def get(self, k: int):
        import torch
        g = self.graphs.get(k)
        if g is None:
            g = torch.cuda.CUDAGraph()
            side = torch.cuda.Stream(self.device)
            side.wait_stream(torch.cuda.current_stream(self.device))
            with torch.cuda.stream(side):
                g.capture_begin()
                cst = _native.stream_handle(self.device)
                for _ in range(k):
                    self.one_step(cst)
                g.capture_end()
            torch.cuda.current_stream(self.device).wait_stream(side)
            _upload_graph(g, self.device)
            self.graphs[k] = g
        return g

    def prepare(self, steps: int):
        for k in set(self._chunks(steps)):
            self.get(k)

    def run(self, steps: int):
        for k in self._chunks(steps):
            self.get(k).replay()


class Simulator:
    """Runs the step loop for the shards this process owns (all of them, on one device)."""

    def __init__(self, net: Network, lif: LifParams = LifParams(), seed: int = 0, rt: RoutingTable | None = None,
                 *, delivery: str = "fused", record_raster_steps: int = 0, per_step_counts: bool = False,
                 bucket_cap: int | None = None, use_graph: bool = True, graph_chunk: int = 64,
                 push_windows: int | None = None):
        import torch
        if delivery not in ("fused", "push", "pull", "persistent", "binned"):
            raise ValueError(f"delivery must be 'fused', 'pull', 'push', 'binned' or 'persistent', got {delivery!r}")
        if delivery in ("persistent", "binned") and net.layout.n_shards != 1:
            raise ValueError(f"the {delivery} engine runs one shard per GPU; use distributed.DistSimulator")
        if set(net.shards) != set(range(net.layout.n_shards)):
            raise ValueError("the single-process simulator needs every shard of the layout")
        _check_layouts(net, delivery)
        self.net = net
        self.lif = lif
        self.seed = seed
        self.delivery = delivery
        self.plan = ExchangePlan(net.layout.n_shards, rt)
        self.c_lif = lif.to_c(seed)
        self.lib = _native.lib()
        self.n = net.layout.n_shards
        self.per_step_counts = per_step_counts
        self.use_graph = use_graph
        self.graph_chunk = graph_chunk
        self.record_steps = int(record_raster_steps)
        self.states = [
            _ShardState(net, h, self.plan, record_steps=self.record_steps, push=(delivery in ("push", "persistent")),
                        bucket_cap=bucket_cap, binned=(delivery == "binned"),
                        push_windows=(push_windows if push_windows is not None else
                                      push_windows_for(net.layout.n_local(h)) if delivery == "persistent" else 1))
            for h in range(self.n)
        ]
        dev = net.device
        self.dest_global = net.global_dest() if self.n > 1 else torch.zeros(1, dtype=torch.int16, device=dev)
        self.fwd_table = self.plan.fwd_table_u16()
        self.fwd_cap = max(s.bucket_cap for s in self.states) * (self.n if self.plan.two_level else 1)
        self.fwd_ids = torch.zeros(self.n * self.n * self.fwd_cap if self.plan.two_level else 1, dtype=torch.int32,
                                   device=dev)
        self.fwd_count = torch.zeros(self.n * self.n, dtype=torch.int32, device=dev)
        self.shard_array = (_native.ShardC * self.n)(*[s.c for s in self.states])
        self.ops = _native.ops()
        self.c_lif_t = _native.as_bytes(self.c_lif)
        self.shard_array_t = _native.as_bytes(self.shard_array)
        self.fwd_table_t = torch.from_numpy(self.fwd_table)
        self._counter_steps = 0
        self._gbar = torch.zeros(1, dtype=torch.int32, device=dev)
        self.hop_ids = None
        self.deliv_ids = None
        self._graphs = StepGraphs(dev, self._one_step, graph_chunk)
        self._check(self.lib.nc_sim_prepare(), "prepare")

    def _check(self, rc, what):
        _native.check(rc, what)

    def reset(self, counter_steps: int):
        """Initial state and zeroed counters sized for `counter_steps` recorded steps."""
        import torch
        st = _native.stream_handle(self.net.device)
        for s in self.states:
            self._check(self.lib.nc_sim_init(C.byref(s.c), C.byref(self.c_lif), st), "sim init")
            s.raster.zero_()
        rows = counter_steps if self.per_step_counts else 1
        self._counter_steps = rows
        self.hop_ids = torch.zeros((rows, self.n, self.n), dtype=torch.int64, device=self.net.device)
        self.deliv_ids = torch.zeros((rows, self.n, self.n), dtype=torch.int64, device=self.net.device)
        self.fwd_count.zero_()
        if self.n > 1:   # the exchange launches capture the counter buffers reallocated above
            self._graphs.clear()

    def _one_step(self, st):
        """One step's launches, through the thin PyTorch extension (torch.ops.neurocomm_b200)."""
        O = self.ops
        lif = self.c_lif_t
        if self.delivery == "fused":
            for s in self.states:
                O.sim_step_fused(s.c_t, lif, st)
        elif self.delivery == "binned":
            for s in self.states:
                O.sim_step_binned(s.c_t, lif, st)
        else:
            for s in self.states:
                if self.delivery == "push":
                    O.sim_deliver_push(s.c_t, self.c_lif.g_inh, st)
                else:
                    O.sim_deliver_pull(s.c_t, self.c_lif.g_inh, st)
                O.sim_lif_update(s.c_t, lif, st)
        if self.n > 1:
            O.exchange_local(self.shard_array_t, self.n, self.dest_global, self.fwd_table_t, self.fwd_ids,
                             self.fwd_count, self.fwd_cap, self.hop_ids, self.deliv_ids,
                             1 if self.per_step_counts else 0, st)
        for s in self.states:
            O.sim_end_step(s.c_t, st)

    def launches_per_step(self) -> float:
        if self.delivery == "persistent":
            return 0.0  # one launch per advance() call, whatever the step count
        per_shard = 2 if self.delivery in ("fused", "binned") else 3
        ex = 0
        if self.n > 1:
            ex = 3 if self.plan.two_level else 1
        return per_shard * self.n + ex

    def advance_eager(self, steps: int):
        """Enqueue `steps` steps as plain launches on the current stream."""
        st = _native.stream_handle(self.net.device)
        for _ in range(steps):
            self._one_step(st)

    def advance(self, steps: int):
        """Enqueue `steps` steps on the current stream (graph-replayed in chunks)."""
        if self.delivery == "persistent":
            s = self.states[0]
            st = _native.stream_handle(self.net.device)
            self.ops.run_persistent(s.c_t, self.c_lif_t, None, int(steps), 1, self._gbar, None, None, 0, st)
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
        for s in self.states:
            flags = s.status.cpu().tolist()
            if flags[0]:
                raise RuntimeError(f"spike bucket overflow on shard {s.h}: raise bucket_cap")
            if flags[1]:
                raise RuntimeError(f"exchange watchdog expired on shard {s.h}")

    def run(self, steps: int) -> SimReport:
        import torch
        if steps < 0:
            raise ValueError("steps must be >= 0")
        self.reset(steps if self.per_step_counts else 1)
        if self.record_steps and self.record_steps < steps:
            raise ValueError("record_raster_steps is smaller than the number of steps")
        self.prepare(steps)
        torch.cuda.synchronize(self.net.device)
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        self.advance(steps)
        t1.record()
        torch.cuda.synchronize(self.net.device)
        self.check_status()
        return self.report(steps, t0.elapsed_time(t1))

    def report(self, steps: int, elapsed_ms: float) -> SimReport:
        lay = self.net.layout
        raster = None
        if self.record_steps:
            raster = _raster_to_host(self.states, lay, steps, self.net.device)
        v = np.zeros(lay.n_neurons, dtype=np.float32)
        i = np.zeros(lay.n_neurons, dtype=np.float32)
        spikes = 0
        for s in self.states:
            if s.n_local:
                v[lay.members[s.h]] = s.v[: s.n_local].cpu().numpy()
                i[lay.members[s.h]] = s.i_syn[: s.n_local].cpu().numpy()
            spikes += int(s.spike_total.item())
        hop = self.hop_ids.cpu().numpy()
        deliv = self.deliv_ids.cpu().numpy()
        if not self.per_step_counts:
            hop, deliv = hop[:1], deliv[:1]
        mode = "none" if self.n == 1 else ("two-level" if self.plan.two_level else "direct")
        return SimReport(steps=steps, n_gpus=self.n, raster=raster, deliv_ids=deliv, hop_ids=hop, spikes=spikes,
                         v=v, i_syn=i, elapsed_ms=elapsed_ms, exchange=mode, delivery=self.delivery)


def _raster_to_host(states, lay, steps: int, dev, chunk_bytes: int = 256 << 20) -> np.ndarray:
    """bool [steps, M] in gid order from the shards' recorded bitmap rows: bits unpacked
    and scattered to gid order on the device (a step chunk at a time), one copy back."""
    import torch
    raster = np.zeros((steps, lay.n_neurons), dtype=bool)
    if steps == 0 or lay.n_neurons == 0:
        return raster
    shifts = torch.arange(32, dtype=torch.int32, device=dev)
    members = {s.h: torch.from_numpy(np.asarray(lay.members[s.h], dtype=np.int64)).to(dev) for s in states if s.n_local}
    rows = max(1, chunk_bytes // lay.n_neurons)
    for a in range(0, steps, rows):
        b = min(steps, a + rows)
        out = torch.zeros((b - a, lay.n_neurons), dtype=torch.bool, device=dev)
        for s in states:
            if not s.n_local:
                continue
            words = s.raster[a:b, : s.local_words]
            bits = ((words.unsqueeze(-1) >> shifts) & 1).reshape(b - a, -1)[:, : s.n_local]
            out[:, members[s.h]] = bits.bool()
        raster[a:b] = out.cpu().numpy()
    return raster


# ---------------------------------------------------------------- engine choice

def _timed_steps(sim, warm: int, steps: int) -> float:
    """ms per step of `steps` steps after `warm` (CUDA events on the current stream)."""
    import torch
    sim.reset(1)
    sim.prepare(warm)
    sim.prepare(steps)
    sim.advance(warm)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    sim.advance(steps)
    e1.record()
    torch.cuda.synchronize()
    sim.check_status()
    return e0.elapsed_time(e1) / max(steps, 1)


def delivery_candidates(net: Network) -> list:
    """Engines that can run `net` here: the pull kernel if the layout has it, the
    event-driven engines if the push CSR fits next to it (4 B per synapse)."""
    import torch
    out = []
    if all(getattr(c, "has_pull", True) for c in net.shards.values()):
        out.append("fused")
    cached = all(getattr(c, "_push_arrays", None) for c in net.shards.values())
    free = torch.cuda.mem_get_info(net.device)[0]
    if cached or 4.4 * net.n_synapses + 2e9 < free:
        rows = max(net.layout.n_local(h) for h in net.shards)
        one = net.layout.n_shards == 1
        out.append("persistent" if one and rows <= int(_native.lib().nc_persistent_max_rows()) else "push")
    return out


def choose_delivery(net: Network, lif: LifParams, seed: int, rt: RoutingTable | None = None, *,
                    candidates=None, steps: int = 20, warmup: int = 5):
    """The fastest delivery engine for this network and drive, measured (every engine gives
    bit-identical results, tests/test_gpu_parity.py): (name, {name: ms per step}).  The pull
    kernel streams every synapse each step; the event-driven engines do work proportional
    to spikes x degree, so which one wins depends on rate, size and bitmap tiling."""
    cands = list(candidates) if candidates else delivery_candidates(net)
    if not cands:
        raise ValueError("no delivery engine fits this network on this device")
    times = {}
    for d in cands:
        sim = Simulator(net, lif, seed, rt, delivery=d)
        times[d] = _timed_steps(sim, warmup, steps)
        del sim
    best = min(times, key=times.get)
    return best, times


# ---------------------------------------------------------------- public API

def simulate(graph: NeuronGraph, pm, rt: RoutingTable | None, steps: int, lif: LifParams = LifParams(),
             seed: int = 0, *, delivery: str = "fused", record: tuple = ("raster", "counts"),
             use_graph: bool = True, device=None) -> SimReport:
    """Simulate `steps` 1-ms steps of the LIF network on the reference's partition and routes.

    ``graph``/``pm``/``rt`` are the reference pipeline's outputs
    (generate_synthetic -> partition_greedy -> build_routing_table or route_p2p).
    ``rt=None`` means direct routing.  All partitions run on the current CUDA
    device with the local exchange transport; use :mod:`.distributed` for one
    process per GPU.  ``delivery="auto"`` times the engines that fit
    (:func:`choose_delivery`) and runs the fastest.
    """
    if steps < 0:
        raise ValueError(f"steps must be >= 0, got {steps}")
    if pm.assignment.size != graph.n_neurons:
        raise ValueError(f"partition map covers {pm.assignment.size} neurons, graph has {graph.n_neurons}")
    layout = ShardLayout.from_assignment(pm.assignment, pm.n_gpus)
    net = Network.from_graph(graph, layout, device=device, inh_every=lif.inh_every)
    if delivery == "auto":   # measure the engines that fit, keep the fastest (identical results)
        delivery, _ = choose_delivery(net, lif, seed, rt)
    sim = Simulator(net, lif, seed, rt, delivery=delivery,
                    record_raster_steps=steps if "raster" in record else 0,
                    per_step_counts="counts" in record, use_graph=use_graph)
    return sim.run(steps)
