"""Benchmark: simulated 1-ms steps per second of the spiking hot loop.

Default (N=1): BASELINE config 2 -- 1M LIF neurons x ~1k synapses (random, C=1,
device-generated with the generate_synthetic distributions), single B200,
update + delivery kernels, 1000 timed steps.  N>1 (torchrun): strong scaling of the
same network (block partition over the N GPUs, direct P2P spike exchange); `--scaling
weak` grows the network to 1M neurons per GPU instead.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints one JSON line (rank 0).  See DESIGN.md section 6 for every field.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "simulated steps/sec at 1/2/4/8 B200; p50/p99 spike-exchange µs/step"
UNIT = "steps/s"


def load_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.is_file():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured"}
    return {"hbm_gbs": 6650.0, "source": "fallback"}


class ClockSampler:
    """SM clock and throttle reasons sampled every few ms DURING the timed region
    (NVML in a background thread; nvidia-smi polling if NVML is unavailable), so
    even a 10-ms timed region carries a clock record."""

    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap", "hw_power_brake"]

    def __init__(self, index: int, period_s: float = 0.002):
        self.index = index
        self.period = period_s
        self.sm: list[float] = []
        self.max_mhz = None
        self.reasons: set[str] = set()
        self.source = None
        self._stop = threading.Event()
        self._t = None
        self._proc = None

    def _handle(self, nv):
        try:
            import torch
            pr = torch.cuda.get_device_properties(self.index)
            bus = "%08x:%02x:%02x.0" % (pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id)
            return nv.nvmlDeviceGetHandleByPciBusId(bus.encode())
        except Exception:
            return nv.nvmlDeviceGetHandleByIndex(self.index)

    def _nvml_loop(self, nv, h):
        bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap,
                nv.nvmlClocksEventReasonHwPowerBrakeSlowdown]
        while not self._stop.is_set():
            try:
                self.sm.append(float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
                for name, b in zip(self.NAMES, bits):
                    if r & b:
                        self.reasons.add(name)
            except Exception:
                pass
            self._stop.wait(self.period)

    def _smi_loop(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        self._proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                       "--format=csv,noheader,nounits", "-lms", "20"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        for line in self._proc.stdout:
            f = [x.strip() for x in line.split(",")]
            try:
                self.sm.append(float(f[0]))
                self.max_mhz = float(f[1])
            except (ValueError, IndexError):
                continue
            for name, val in zip(self.NAMES, f[2:6]):
                if val.lower() == "active":
                    self.reasons.add(name)

    def __enter__(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            h = self._handle(nv)
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self.source = "nvml, %.0f ms period" % (self.period * 1e3)
            self._t = threading.Thread(target=self._nvml_loop, args=(nv, h), daemon=True)
        except Exception:
            self.source = "nvidia-smi -lms 20"
            self._t = threading.Thread(target=self._smi_loop, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._proc is not None:
            self._proc.terminate()
        if self._t is not None:
            self._t.join(timeout=5)
        return False

    def summary(self) -> dict:
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.sm), "source": self.source}


def total_neurons(args, world: int) -> int:
    return args.neurons * world if args.scaling == "weak" else args.neurons


def workload_name(args, world: int) -> str:
    n = total_neurons(args, world)
    if args.communities > 1:
        return (f"regional (config 5 family): {n} neurons in {args.communities} regions, "
                f"{args.intra_frac:.0%} of ~{args.degree:.0f} synapses intra-region, {world} GPU(s), block partition")
    if world == 1 and n == 1_000_000:
        return "config 2: 1M LIF neurons x 1k synapses, single B200, update + delivery kernels"
    if args.scaling == "weak":
        return (f"weak scaling: {args.neurons} neurons/GPU x {args.degree:.0f} synapses, {world} GPU(s), "
                f"block partition, direct exchange ({args.transport})")
    return (f"strong scaling: {n} neurons x {args.degree:.0f} synapses"
            f"{' (the config-2 network)' if n == 1_000_000 else ''} over {world} GPU(s), block partition, "
            f"direct exchange ({args.transport})")


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# --------------------------------------------------------------------------- ours

def make_sim(net, lif, args, delivery, world, record_raster_steps: int = 0):
    from paper_2205_07125_b200 import sim as S
    if world > 1:
        from paper_2205_07125_b200 import distributed as D
        cap = args.msg_cap if args.msg_cap is not None else (65536 if args.transport == "nccl" else None)
        fs = args.fused_send == "on"
        return D.DistSimulator(net, lif, args.seed, None, transport=args.transport, delivery=delivery,
                               msg_cap=cap, latency_steps=args.warmup + args.steps, graph_chunk=args.chunk,
                               record_raster_steps=record_raster_steps, fused_send=fs)
    return S.Simulator(net, lif, args.seed, None, delivery=delivery, graph_chunk=args.chunk)


def enable_kernel_stamps(sim, n_steps: int) -> None:
    """Device %globaltimer stamps of the fused step kernel for every step (first CTA start,
    last CTA end; nc_shard_t.kstamp): the kernel's duration inside the timed loop.
    Set before the step graph is captured."""
    import torch
    for s in sim.states:
        s.kstamp_buf = torch.zeros(2 * n_steps, dtype=torch.int64, device=s.v.device)
        s.c.kstamp = s.kstamp_buf.data_ptr()
        s.c.kstamp_steps = n_steps


def live_kernel_ms(sim, first: int, n: int, world: int, dev):
    """Mean in-loop duration of the fused step kernel over steps [first, first + n):
    (max over ranks, [per rank]) -- the per-rank spread is the step skew every
    exchange waits for."""
    import torch
    import torch.distributed as dist
    buf = getattr(sim.states[0], "kstamp_buf", None)
    if buf is None:
        return None, None
    st = buf.view(-1, 2)[first:first + n]
    d = (st[:, 1] - st[:, 0]).to(torch.float64)
    t = (d.mean() / 1e6).reshape(1).to(dev)
    per = [float(t.item())]
    if world > 1:
        parts = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        per = [float(x.item()) for x in parts]
    return max(per), per


def align_start(world: int, dev) -> None:
    """N>1: a one-element NCCL all-reduce enqueued right before the start event.  Every
    rank's stream passes it only once the last rank has enqueued it, so the timed region
    starts together on all GPUs -- not at each host's own moment after the barrier, where a
    rank whose host returned a few ms late would be charged to every other rank's exchange
    (which waits for its spikes): 20 steps at 4 GPUs read 1 934 steps/s that way, against
    6 988 over 300 steps."""
    if world > 1:
        import torch
        import torch.distributed as dist
        dist.all_reduce(torch.zeros(1, device=dev))


def time_steps(sim, args, world, dev, clocks=None):
    """W warm-up steps, then exactly K timed steps between barrier + synchronize;
    CUDA events on the launching stream, max over ranks.  Returns (ms, spikes, lat, lat_min)."""
    import torch
    import torch.distributed as dist

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    sim.reset(1)
    for s in sim.states:
        if getattr(s, "kstamp_buf", None) is not None:
            s.kstamp_buf.view(-1, 2)[:, 0] = -1     # start: atomicMin from ~0
            s.kstamp_buf.view(-1, 2)[:, 1] = 0      # end: atomicMax from 0
    # every CUDA graph the warm-up and the timed loop replay is captured here, outside both
    sim.prepare(args.warmup)
    sim.prepare(args.steps)
    sim.advance(args.warmup)
    barrier()
    spikes0 = sum(int(s.spike_total.item()) for s in sim.states)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    ctx = clocks if clocks is not None else _Null()
    with ctx:   # the sampler starts (nvmlInit: ms, varying per host) before the aligned start
        align_start(world, dev)
        e0.record()
        sim.advance(args.steps)
        e1.record()
        torch.cuda.synchronize()
    barrier()
    ms = e0.elapsed_time(e1)
    spikes = sum(int(s.spike_total.item()) for s in sim.states) - spikes0
    sim.check_status()
    lat = lat_min = None
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        sp = torch.tensor([spikes], device=dev, dtype=torch.int64)
        dist.all_reduce(sp)
        spikes = int(sp.item())
        lat, lat_min = sim.latencies_us(args.warmup + args.steps)     # per step: max, min over ranks
        lat, lat_min = lat[args.warmup:], lat_min[args.warmup:]
        # ids this rank put on each channel, over warm-up + timed steps (hop counters of rank 0's row)
        row = sim.hop_ids.sum(0)[rank_of(sim)].to(torch.float64) / max(args.warmup + args.steps, 1)
        mx, tot = row.max().reshape(1), row.sum().reshape(1)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(tot)
        lat = (lat, float(mx.item()), float(tot.item()) / world)
    return ms, spikes, lat, lat_min


class _Null:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def kernel_ms(sim, which: str, reps: int = 50) -> float:
    """Average duration of one kernel, timed alone with CUDA events on its stream."""
    import torch
    from paper_2205_07125_b200 import _native
    st = sim.states[0]
    stream = torch.cuda.current_stream()
    k0 = torch.cuda.Event(enable_timing=True)
    k1 = torch.cuda.Event(enable_timing=True)
    O = _native.ops()
    lif = _native.as_bytes(sim.c_lif)

    def run(kind):
        torch.cuda.synchronize()
        k0.record(stream)
        s = stream.cuda_stream
        for _ in range(reps):
            if kind == "fused":
                O.sim_step_fused(st.c_t, lif, s)
            elif kind == "push":  # + the claim-counter reset a real step does
                O.sim_deliver_push(st.c_t, sim.c_lif.g_inh, s)
                O.sim_end_step(st.c_t, s)
            elif kind == "lif":  # with the bucket reset a real step does after the exchange
                O.sim_lif_update(st.c_t, lif, s)
                O.sim_end_step(st.c_t, s)
            else:
                O.sim_end_step(st.c_t, s)
        k1.record(stream)
        torch.cuda.synchronize()
        return k0.elapsed_time(k1) / reps

    if which in ("lif", "push"):
        return max(run(which) - run("end"), 0.0)
    return run(which)


def rank_of(sim) -> int:
    return int(getattr(sim, "rank", 0))


def lat_summary(lat, lat_min, transport, nccl_msg_bytes=None):
    """Exchange latency per SURVEY 8(d): device %globaltimer per rank and step from
    buckets ready to the last inbound spike in the bitmap; p50/p99 over the timed
    steps of the per-step MAX over ranks.  The per-step MIN over ranks (the rank whose
    buckets were ready last: transfer + signalling alone) is reported beside it.
    Wire bytes: P2P moves 8 bytes per id (tag + id) + an 8-byte header per message;
    NCCL moves every message at its full capacity, (cap + 1) x 4 bytes, whatever the
    spike count (`nccl_msg_bytes` per rank and step)."""
    if lat is None:
        return None
    lat, max_channel_ids, ids_per_rank = lat
    p50 = float(np.percentile(lat, 50))
    p50_min = float(np.percentile(lat_min, 50))
    if transport == "p2p":
        bytes_rank = ids_per_rank * 8
        wire = 8
    else:
        bytes_rank = float(nccl_msg_bytes) if nccl_msg_bytes is not None else ids_per_rank * 4
        wire = 4
    return {"p50": round(p50, 2), "p99": round(float(np.percentile(lat, 99)), 2),
            "p50_transfer_only": round(p50_min, 2),
            "p99_transfer_only": round(float(np.percentile(lat_min, 99)), 2),
            "bytes_per_step_per_rank": round(bytes_rank, 1),
            "max_channel_bytes_per_step": round(max_channel_ids * wire, 1),
            "nvlink_gbs_at_transfer_p50": round(bytes_rank / (p50_min * 1e-6) / 1e9, 2) if p50_min > 0 else None,
            "nvlink_peak_gbs": 900.0,
            "bytes_note": "bytes each rank puts on the wire per step (P2P: 8 B per id; NCCL: every message at "
                          "its full capacity); GB/s = that over the p50 transfer-only time, against 900 GB/s "
                          "per direction per GPU (latency bound)",
            "transport": transport,
            "what": "device %globaltimer per step and rank from buckets ready (the exchange kernel's first block, "
                    "which starts after the step kernel) to the last inbound spike ORed into the bitmap; p50/p99 over "
                    "timed steps of the per-step max over ranks (SURVEY 8(d); includes waiting for the slowest "
                    "rank's step kernel); *_transfer_only: of the per-step min over ranks"}


def common_config(args, world: int) -> dict:
    """The `config` both arms print (identical by construction)."""
    return {"workload": workload_name(args, world), "neurons": total_neurons(args, world),
            "mean_degree": args.degree, "communities": args.communities,
            "intra_frac": args.intra_frac if args.communities > 1 else None,
            "generator_seed": args.seed, "lif": "LifParams() defaults (DESIGN.md section 3)",
            "partition": "blocks" if world > 1 else None,
            "exchange": "direct" if world > 1 else "none",
            "l2": ("inputs larger than L2 (the whole synapse array, ~%.1f GB, is streamed every step)"
                   % (3.2 * args.degree * total_neurons(args, world) / 1e9 / world)
                   if 3.2 * args.degree * total_neurons(args, world) / world > 126e6 else
                   "synapse array fits in L2 (126 MB): no flush between steps")}


def run_ours(args) -> dict | None:
    import torch
    import torch.distributed as dist

    from paper_2205_07125_b200 import sell
    from paper_2205_07125_b200 import sim as S

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    n_neurons = total_neurons(args, world)
    spec = generator_spec(args, n_neurons)
    lay = S.ShardLayout.blocks(n_neurons, world)
    t_build = time.time()
    net = S.Network.generate(spec, lay, device=dev, shards=[rank], tile_words=args.tile_words,
                             bank_order=args.bank_order)
    torch.cuda.synchronize()
    t_build = time.time() - t_build
    lif = S.LifParams()

    # ---- headline: the delivery asked for (default: fused pull, the north-star K3 path)
    sim = make_sim(net, lif, args, args.delivery, world)
    if args.delivery == "fused":
        enable_kernel_stamps(sim, args.warmup + args.steps)
    clocks = ClockSampler(local)
    ms, spikes, lat, lat_min = time_steps(sim, args, world, dev, clocks)
    value = args.steps / (ms * 1e-3)
    main_kernel = {"fused": "fused", "push": "push"}.get(args.delivery, "step")
    # fused: the kernel's mean duration inside the timed loop (device stamps); the same
    # kernel timed alone afterwards (50 back-to-back launches, CUDA events) is reported beside
    # it.  binned / persistent engines: one kernel (or one launch) per step, timed as the step
    kms_live, kms_ranks = (live_kernel_ms(sim, args.warmup, args.steps, world, dev) if args.delivery == "fused"
                           else (None, None))
    kms_alone = kernel_ms(sim, main_kernel) if main_kernel != "step" else ms / args.steps
    kms = kms_live if kms_live is not None else kms_alone
    n_local = lay.n_local(rank)
    csr = net.shards[rank]
    # algorithmic bytes of one fused step: 3.2 B per synapse (16-byte slots of 5)
    # + per neuron row_meta 4/tile, V r/w 8, I r/w 8, refrac r/w 2, gid 4, the slice
    # pointers, + the previous spike bitmap read and the new one written
    syn_bytes = int(net.n_synapses) * 16 // 5
    neuron_bytes = n_local * (4 * csr.n_tiles + 8 + 8 + 2 + 4) + csr.slice_ptr.numel() * 8 + 2 * (lay.n_words * 4)
    alg_bytes = syn_bytes + neuron_bytes
    # SURVEY 8(d)'s pull formula (8 B per synapse: 4 B pre id + 4 B weight, 8 B rowptr and 4 B input
    # per neuron, the bitmap) for the same step -- what an unpacked CSR would have to move
    pull_bytes = int(net.n_synapses) * 8 + (n_local + 1) * 8 + n_local * 4 + lay.n_neurons // 8
    layout_bytes = (csr.n_entries * 4 + csr.row_meta.numel() * 4 + csr.slice_ptr.numel() * 8
                    + (csr.row_perm.numel() * 4 if csr.row_perm is not None else 0) + n_local * 22
                    + 2 * lay.n_words * 4)
    peaks = load_peaks()
    if main_kernel != "fused":
        fired_syn = spikes / max(args.steps, 1) * args.degree / max(world, 1)
        if args.delivery == "binned":
            # per spike and bin a 32-byte sector of bin offsets, 4 B per delivered synapse,
            # + LIF state r/w 22 B per neuron
            alg_bytes = spikes / max(args.steps, 1) * sell.device_sms(dev) * 32 + fired_syn * 4 + n_local * 22
        else:
            # the push kernel moves 12 B per delivered synapse
            alg_bytes = fired_syn * 12
    achieved = alg_bytes / (kms * 1e-3) / 1e9
    traffic = None
    prof = ROOT / "profiles" / "ncu_step_fused.json"
    if prof.is_file() and main_kernel == "fused" and world == 1:
        traffic = json.loads(prof.read_text()).get("dram_bytes_per_launch")
    fused_send = getattr(sim, "fused_send", None)
    nccl_bytes = None
    if world > 1 and args.transport == "nccl":   # fixed-capacity messages to every phase-1 peer
        nccl_bytes = bin(sim.masks["send1"]).count("1") * (sim.cap + 1) * 4
    e2e = e2e_measure(sim, net, args, world, rank, lif)
    launches = max(1, int(round(args.steps * sim.launches_per_step())))
    if world > 1:
        sim.close()
    del sim

    # ---- the event-driven alternative on the same network (bit-identical results)
    event = None
    if args.with_push and args.delivery == "fused":
        psim = make_sim(net, lif, args, args.event, world)
        pms, pspikes, plat, plat_min = time_steps(psim, args, world, dev)
        fired_syn = pspikes / max(args.steps, 1) * args.degree / max(world, 1)
        event = {"engine": args.event, "value": round(args.steps / (pms * 1e-3), 2),
                 "ms_per_step": round(pms / args.steps, 5),
                 "delivered_synapses_per_step": round(fired_syn, 1),
                 "exchange_us": lat_summary(plat, plat_min, args.transport),
                 "gpu_launches": max(1, int(round(args.steps * psim.launches_per_step())))}
        if args.event in ("push", "persistent"):
            push_ms = kernel_ms(psim, "push")
            lif_ms = kernel_ms(psim, "lif")
            push_bytes = fired_syn * 12          # 4 B entry read + 4 B read + 4 B write per reduction
            event.update({"push_kernel_ms": round(push_ms, 5), "lif_kernel_ms": round(lif_ms, 5),
                          "push_bound": "L2 atomics: %.3g reductions/s" % (fired_syn / (push_ms * 1e-3)),
                          "push_achieved_gbs": round(push_bytes / (push_ms * 1e-3) / 1e9, 1)})
        if world > 1:
            psim.close()
        del psim

    result = None
    parity = None
    cpu = None
    e2e_api = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu, parity, e2e_api = cpu_baseline_and_parity(net, lay, lif, args, spec)
    if rank == 0:
        result = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 5), "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "fp32 state / int32 synaptic sums",
            "data": "synthetic (device SBM generator, generate_synthetic distributions)",
            "config": common_config(args, world),
            "details": {
                "synapses": int(net.n_synapses) * world, "delivery": args.delivery,
                "firing_rate_hz": round(spikes / n_neurons / (args.steps * 1e-3), 3),
                "synapse_array_gb": round(csr.n_entries * 4 / 1e9, 3),
                "sell_padding": round(csr.n_entries * 4 / max(csr.n_real * 3.2, 1) - 1.0, 4),
                "bitmap_tiles": csr.n_tiles, "graph_build_s": round(t_build, 2),
                "fused_send": fused_send,
            },
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                         "frac": round(achieved / peaks["hbm_gbs"], 4), "traffic": traffic,
                         "kernel": {"fused": "k_step_fused", "push": "k_deliver_push",
                                    "binned": "k_step_binned (whole step)"}.get(args.delivery,
                                                                                 "k_persistent (whole step)"),
                         "kernel_ms": round(kms, 5), "algorithmic_bytes": int(alg_bytes),
                         "bytes_formula": "packed J-SELL: 3.2 B/synapse + 26 B/neuron + bitmaps (DESIGN.md section 5)",
                         "pull_formula_bytes": int(pull_bytes),
                         "layout_bytes": int(layout_bytes),
                         "layout_note": "bytes the layout actually streams per step (J-SELL array incl. its per-"
                                        "(row, tile) segment padding, row_meta, row_perm, block starts, neuron state)",
                         "pull_formula_note": "SURVEY 8(d) pull formula (8 B/synapse unpacked CSR) for the same step; "
                                              "its GB/s over kernel_ms would read %.2fx the copy peak -- the packing, "
                                              "not skipped work (ncu DRAM bytes = traffic)"
                                              % (pull_bytes / (kms * 1e-3) / 1e9 / peaks["hbm_gbs"]),
                         "kernel_ms_source": ("device %globaltimer stamps of every timed step's kernel "
                                              "(first CTA start to last CTA end), mean, max over ranks")
                         if kms_live is not None else "CUDA events, the kernel launched alone",
                         "kernel_ms_per_rank": [round(x, 5) for x in kms_ranks] if kms_ranks else None,
                         "kernel_ms_alone": round(kms_alone, 5),
                         "peak_source": peaks["source"], "spec_peak_gbs": 8000.0,
                         "frac_of_spec": round(achieved / 8000.0, 4)},
            "parity": parity,
            "event_driven": event,
            "exchange_us": lat_summary(lat, lat_min, args.transport, nccl_bytes),
            "cpu_baseline": cpu,
            "e2e": e2e,
            "e2e_api": e2e_api,
            "gpu_launches": launches,
            "clocks": clocks.summary(),
        }
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return result


def generator_spec(args, n_neurons: int):
    from paper_2205_07125_b200 import sim as S
    if args.communities > 1:
        # regional model (config 5): `intra_frac` of each neuron's ~degree synapses inside its region
        c = args.communities
        size = n_neurons / c
        p_in = args.intra_frac * args.degree / max(size - 1, 1)
        p_out = (1 - args.intra_frac) * args.degree / max(n_neurons - size, 1)
        return S.GeneratorSpec(n_neurons, c, min(p_in, 1.0), min(p_out, p_in), seed=args.seed)
    return S.GeneratorSpec.random(n_neurons, args.degree, seed=args.seed)


def oracle_csr(spec, threads: int):
    """The oracle's own CPU restatement of the device generator (oracle/sim_oracle.c):
    the symmetric gid-space CSR of the same network, built without the GPU."""
    from oracle import c_oracle
    return c_oracle.generate_sbm_csr(spec.n_neurons, spec.n_communities, spec.p_in, spec.p_out, spec.seed,
                                     intra=spec.intra_p_range, inter=spec.inter_p_range, threads=threads)


def cpu_baseline_and_parity(net, lay, lif, args, spec):
    """(cpu_baseline, parity) on the benchmarked network, rank 0, N = 1.

    The oracle builds the network itself (its CPU generator), then
    * parity: runs `parity_steps` full steps with the raster on and compares every
      step's raster, the per-step spike counts and the final V / I bit for bit with
      a fresh GPU run of the same steps on the benchmarked device layout;
    * cpu_baseline: times `cpu_steps` more full steps (OpenMP, every host core).
    """
    import hashlib
    from oracle import c_oracle
    from paper_2205_07125_b200 import sim as S
    threads = os.cpu_count() or 1
    t = time.time()
    rowptr, col, q = oracle_csr(spec, threads)
    t_gen = time.time() - t
    owner = np.zeros(lay.n_neurons, dtype=np.int32)
    k = args.parity_steps
    parity = None
    if k > 0:
        gsim = S.Simulator(net, lif, args.seed, None, delivery="fused", record_raster_steps=k, graph_chunk=args.chunk)
        rep = gsim.run(k)
        del gsim
        ref = c_oracle.simulate_csr(rowptr, col, q, owner, 1, [[-1]], lif.constants(args.seed), k, threads=threads,
                                    raster=True, counts=False)
        same_graph = int(rowptr[-1]) == int(net.n_synapses)
        sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()[:16]  # noqa: E731
        parity = {"steps": k, "network": "the benchmarked one: device-generated J-SELL layout (%d tiles, bank "
                                         "order %s) vs the oracle's own CPU generator" % (
                                             net.shards[0].n_tiles, "on" if args.bank_order else "off"),
                  "synapses_equal": same_graph,
                  "raster_equal": bool(np.array_equal(rep.raster, ref["raster"])),
                  "spikes_per_step_equal": bool(np.array_equal(rep.raster.sum(1), ref["raster"].sum(1))),
                  "v_equal": bool(np.array_equal(rep.v.view(np.uint32), ref["v"].view(np.uint32))),
                  "i_equal": bool(np.array_equal(rep.i_syn.view(np.uint32), ref["i"].view(np.uint32))),
                  "spikes": int(rep.raster.sum()), "raster_sha256_16": sha(ref["raster"]),
                  "v_sha256_16": sha(ref["v"])}
    e2e_api = simulate_api_e2e(rowptr, col, q, lif, args) if args.e2e_api else None
    steps = args.cpu_steps
    run = lambda n: c_oracle.simulate_csr(rowptr, col, q, owner, 1, [[-1]], lif.constants(args.seed), n,  # noqa
                                          threads=threads, raster=False, counts=False)
    t = time.time()
    run(0)                                   # setup only (initial state, destination sets)
    setup = time.time() - t
    t = time.time()
    run(steps)
    dt = max(time.time() - t - setup, 1e-9)
    cpu = {"value": round(steps / dt, 4), "unit": UNIT, "cores": threads, "kind": "port",
           "sample": f"{steps} full steps of the same {lay.n_neurons}-neuron network (oracle/sim_oracle.c, "
                     f"OpenMP {threads} threads), {dt:.1f} s excluding {setup:.1f} s setup and the "
                     f"{t_gen:.1f} s CPU network build"}
    return cpu, parity, e2e_api


def simulate_api_e2e(rowptr, col, q, lif, args) -> dict:
    """The drop-in API end to end: simulate(graph, pm, rt, steps) on the benchmarked network
    as a host NeuronGraph (model.py:53-92; built from the oracle's CSR outside the timed
    region, p = q / 32 so the weight units are the same), timed on the host clock around
    the call: edge upload, the device layout build, `steps` steps, raster / V / I read-back."""
    import torch
    import paper_2205_07125_b200 as nc
    m = rowptr.size - 1
    rows = np.repeat(np.arange(m, dtype=np.int32), np.diff(rowptr))
    up = col > rows
    g = nc.NeuronGraph(m, np.ones(m), rows[up].astype(np.int64), col[up].astype(np.int64),
                       q[up].astype(np.float64) / 32.0)
    del rows, up
    pm = nc.PartitionMap(1, np.zeros(m, dtype=np.int64))
    torch.cuda.synchronize()
    t = time.perf_counter()
    rep = nc.simulate(g, pm, None, args.steps, lif, seed=args.seed)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    h2d = g.edge_i.size * (8 + 8 + 8)          # int64 ids + fp64 p uploaded (converted on the device)
    return {"value": round(args.steps / dt, 2), "unit": UNIT, "wall_s": round(dt, 3),
            "steps": args.steps, "loop_ms": round(rep.elapsed_ms, 3), "spikes": int(rep.spikes),
            "h2d_bytes_per_step": int(h2d // max(args.steps, 1)),
            "d2h_bytes_per_step": int(rep.raster[0].size + 8 * m // max(args.steps, 1)) if rep.raster is not None
            else None,
            "note": "simulate(NeuronGraph, PartitionMap, None, steps): host edge columns -> device (int32 ids, "
                    "q from p), J-SELL build on the GPU, the step loop, rasters + final V/I to the host; one "
                    "call, host wall clock"}


def e2e_measure(sim, net, args, world: int, rank: int, lif) -> dict | None:
    """Public API with host buffers: every rank's shard of the network (pull slots, block
    starts, row_meta, tile placement) uploaded from pinned host memory inside the timed
    region (amortised per step), the step loop graph-replayed in chunks with every step's
    spike raster row recorded on the device and read back to pinned host memory after each
    chunk.  N>1: DistSimulator (P2P exchange), barrier before, max over ranks."""
    import torch
    from paper_2205_07125_b200 import sim as S
    csr = net.shards[rank]
    steps = args.steps
    if world > 1:
        import torch.distributed as dist
        esim = make_sim(net, lif, args, "fused", world, record_raster_steps=steps)
        st = esim.state
    else:
        esim = S.Simulator(net, lif, args.seed, None, delivery="fused", record_raster_steps=steps,
                           graph_chunk=args.chunk)
        st = esim.states[0]
    words = st.local_words
    parts = [csr.syn, csr.slice_ptr, csr.row_meta] + ([csr.row_perm] if csr.row_perm is not None else [])
    hosts = []
    for t in parts:
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t)
        hosts.append(h)
    raster_host = torch.empty((steps, words), dtype=torch.int32, pin_memory=True)
    esim.reset(1)
    for k in set(min(args.chunk, steps - d) for d in range(0, steps, args.chunk)):
        esim.prepare(k)                           # graph capture outside the timed region
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
        torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    align_start(world, torch.device("cuda", torch.cuda.current_device()))
    e0.record()
    for t, h in zip(parts, hosts):
        t.copy_(h, non_blocking=True)
    done = 0
    while done < steps:
        k = min(args.chunk, steps - done)
        esim.advance(k)
        raster_host[done:done + k].copy_(st.raster[done:done + k, :words], non_blocking=True)
        done += k
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    h2d = sum(h.numel() * h.element_size() for h in hosts)
    d2h = words * 4
    if world > 1:
        esim.check_status()
        v = torch.tensor([ms, float(h2d), float(d2h)], dtype=torch.float64, device=csr.syn.device)
        mx = v.clone()
        dist.all_reduce(mx[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(v[1:], op=dist.ReduceOp.SUM)
        ms, h2d, d2h = float(mx[0].item()), float(v[1].item()), float(v[2].item())
        esim.close()
    del esim
    if rank != 0:
        return None
    return {"value": round(steps / (ms * 1e-3), 2), "unit": UNIT, "h2d_bytes_per_step": int(h2d // steps),
            "d2h_bytes_per_step": int(d2h),
            "note": "network H2D from pinned memory once per call (amortised), every step's spike raster "
                    "row D2H (per graph chunk)" + ("; bytes summed over ranks, time = max over ranks"
                                                   if world > 1 else "")}


# --------------------------------------------------------------------------- reference arm

def run_reference(args) -> dict | None:
    """CPU oracle port of the same workload on every host core (rank 0 only).

    The oracle builds the same network with its CPU generator (oracle/sim_oracle.c,
    the restatement of csrc/graphgen.cu), runs W warm-up steps and then times K
    full steps of the whole network, K capped so the run stays within about a
    minute (the sample is stated in the output).
    """
    rank, world, _ = dist_env()
    if rank != 0:
        return None
    from oracle import c_oracle
    from paper_2205_07125_b200.sim import LifParams
    # bounded sample: at most ~2.5e9 synapses in host memory (the CPU cost of a step is
    # linear in the synapse count, so an n-neuron slice is timed and scaled by n / total)
    total = total_neurons(args, world)
    threads = os.cpu_count() or 1
    spec = generator_spec(args, total)
    sliced = total * args.degree > 2.5e9
    if sliced:
        n = max(1, int(2.5e9 // args.degree))
        spec.n_neurons = n
        if args.communities > 1:
            spec.n_communities = max(1, args.communities * n // total)
        else:
            spec.p_in = args.degree / max(n - 1, 1)
    n = spec.n_neurons
    t = time.time()
    rowptr, col, q = oracle_csr(spec, threads)
    t_build = time.time() - t
    owner = np.zeros(n, dtype=np.int32)
    lif = LifParams().constants(args.seed)
    run = lambda k: c_oracle.simulate_csr(rowptr, col, q, owner, 1, [[-1]], lif, k, threads=threads,  # noqa: E731
                                          raster=False, counts=False)
    t = time.time()
    run(0)                                   # setup only (initial state, destination sets)
    setup = time.time() - t
    warm = args.warmup
    t = time.time()
    run(warm)
    one = max(time.time() - t - setup, 1e-6) / max(warm, 1)
    steps = int(max(3, min(args.steps, 60.0 // one)))
    t = time.time()
    run(warm + steps)                        # the oracle restarts from step 0: warm-up steps, then the timed ones
    dt = max(time.time() - t - setup - one * warm, 1e-9)
    v = steps / dt * n / total
    return {
        "metric": METRIC, "value": round(v, 4), "unit": UNIT, "n_gpus": world, "steps": steps,
        "warmup": warm, "ms_per_step": round(1e3 / v, 3), "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "fp32 state / int32 synaptic sums",
        "data": "synthetic (oracle CPU generator: the same network as the device generator)", "impl": "reference",
        "config": common_config(args, world),
        "details": {"synapses_simulated": int(rowptr[-1]), "graph_build_s": round(t_build, 2),
                    "engine": "oracle/sim_oracle.c (CPU port of the loop semantics; the reference has no loop)"},
        "cpu_baseline": {"value": round(v, 4), "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{steps} full steps after {warm} warm-up steps of a {n}-neuron network"
                                   + (f" (a {n}/{total} slice; steps/s scaled by that fraction)" if sliced else "")
                                   + f" (oracle/sim_oracle.c, OpenMP {threads} threads; requested --steps "
                                   f"{args.steps}, capped at ~60 s; {setup:.1f} s one-time setup excluded)"},
        "e2e": {"value": round(v, 4), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main() -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--neurons", type=int, default=1_000_000,
                    help="network neurons (strong scaling) or neurons per GPU (--scaling weak)")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="N>1: the same network over N GPUs (strong) or N x --neurons (weak)")
    ap.add_argument("--degree", type=float, default=1000.0)
    ap.add_argument("--communities", type=int, default=1, help=">1: regional SBM (config 5 family)")
    ap.add_argument("--intra-frac", type=float, default=0.9, help="regional: fraction of synapses inside a region")
    ap.add_argument("--delivery", default="fused", choices=["fused", "push", "persistent", "binned"])
    ap.add_argument("--engine", dest="event", default="persistent", choices=["push", "persistent", "binned"],
                    help="event-driven variant reported beside the headline")
    ap.add_argument("--transport", default="p2p", choices=["nccl", "p2p"])
    ap.add_argument("--msg-cap", type=int, default=None,
                    help="ids per exchange message (default: exact bound for p2p, 65536 for nccl, which sends all)")
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--tile-words", type=int, default=None, help="force a bitmap tile size (words; tuning)")
    ap.add_argument("--no-bank-order", dest="bank_order", action="store_false",
                    help="skip the shared-memory bank placement of the synapse entries (tuning)")
    ap.add_argument("--chunk", type=int, default=100)
    ap.add_argument("--cpu-steps", type=int, default=200, help="CPU-baseline sample (~10 s of OpenMP oracle work at config 2)")
    ap.add_argument("--parity-steps", type=int, default=20,
                    help="steps of the benchmarked network checked bit for bit against the oracle (N=1; 0 = off)")
    ap.add_argument("--no-e2e-api", dest="e2e_api", action="store_false",
                    help="skip the simulate() end-to-end measurement (N=1)")
    ap.add_argument("--fused-send", default="off", choices=["on", "off"],
                    help="N>1, P2P: the step kernel stores its spikes into the peers' inboxes (A/B: "
                         "profiles/r02_fused_send_ab/)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-push", dest="with_push", action="store_false",
                    help="skip the event-driven (push) measurement reported beside the headline")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    # stdout carries exactly the one JSON line: anything a library writes to fd 1 while we
    # run (NCCL's "NCCL version ..." banner on rank 0, for one) goes to stderr instead
    sys.stdout.flush()
    json_out = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    res = run_reference(args) if args.impl == "reference" else run_ours(args)
    if res is not None:
        print(json.dumps(res), file=json_out, flush=True)
    json_out.close()
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
