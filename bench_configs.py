"""BASELINE configs 3, 4 and 5 at their real sizes (one process per GPU, torchrun).

    torchrun --nproc-per-node N bench_configs.py --config 3|4|5 [--engines fused,persistent]

* config 3: 10 M neurons x ~1 000 synapses (random, C = 1), direct exchange;
  run at N = 1, 2, 4 (strong scaling of the same network).
* config 4: the config-3 network over N GPUs in 2 groups, direct vs two-level
  routing (the reference's group_gpus -> select_bridges -> build_routing_table
  on the measured traffic matrix) at realised rates 1 / 2 / 5 / 10 / 20 / 50 Hz,
  ids and bytes per hop from the int64 channel counters.
* config 5: 50 M neurons in 64 regions, ~90 % of ~1 000 synapses intra-region,
  two-level routing where N >= 4; memory per GPU reported.

Every engine in --engines that fits the GPU runs on the same network: "fused"
(the pull kernel K3+K1+K2 on the J-SELL layout, 3.2 B/synapse + an 8 B/synapse
transient while building) and "persistent" (the event-driven whole-step
kernel on the push CSR, 4 B/synapse).  Results are bit-identical between
engines (tests/test_gpu_parity.py), so the faster one is the config's number.
Exchange latency is SURVEY 8(d)'s: p50/p99 over steps of the per-step max over
ranks (device %globaltimer), transfer-only (min over ranks) beside it.

Prints one JSON line per (engine, route, rate) point on rank 0 and appends it
to --out.
"""

from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

import bench as B  # noqa: E402  (timing, clocks, latency helpers)

CONFIGS = {
    3: dict(neurons=10_000_000, degree=1000.0, communities=1, intra_frac=None, rates=(None,)),
    4: dict(neurons=10_000_000, degree=1000.0, communities=1, intra_frac=None, rates=(1, 2, 5, 10, 20, 50)),
    5: dict(neurons=50_000_000, degree=1000.0, communities=64, intra_frac=0.9, rates=(None,)),
}
GB = 1e9


def spec_for(cfg: dict, seed: int):
    from paper_2205_07125_b200 import sim as S
    n, c = cfg["neurons"], cfg["communities"]
    if c == 1:
        return S.GeneratorSpec.random(n, cfg["degree"], seed=seed)
    size = n / c
    p_in = cfg["intra_frac"] * cfg["degree"] / (size - 1)
    p_out = (1 - cfg["intra_frac"]) * cfg["degree"] / (n - size)
    return S.GeneratorSpec(n, c, min(p_in, 1.0), min(p_out, p_in), seed=seed)


def main() -> int:
    import torch
    import torch.distributed as dist

    import paper_2205_07125_b200 as nc
    from paper_2205_07125_b200 import sim as S
    from paper_2205_07125_b200.distributed import DistSimulator

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, required=True, choices=sorted(CONFIGS))
    ap.add_argument("--engines", default="fused,persistent")
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--groups", type=int, default=2)
    ap.add_argument("--rates", default=None, help="comma list of target rates (Hz); default per config")
    ap.add_argument("--routes", default=None, help="direct,two-level (default: per config)")
    ap.add_argument("--neurons", type=int, default=None, help="override the config's neuron count (tests)")
    ap.add_argument("--communities", type=int, default=None,
                    help="regional variant (SURVEY 8(d) config 3 'C = 8 (regional)'): C contiguous communities, "
                         "90 %% of each neuron's synapses inside its own")
    ap.add_argument("--chunk", type=int, default=100)
    ap.add_argument("--no-ei-group", dest="ei_group", action="store_false",
                    help="layout A/B: do not put each shard's inhibitory ids after its excitatory ones")
    ap.add_argument("--push-windows", type=int, default=None,
                    help="post-row windows of the push CSR (default: sim.push_windows_for per shard)")
    ap.add_argument("--partition", default="blocks",
                    help="blocks | greedy[:file.npz]: the reference's partition_greedy of the generated network "
                         "(partition_greedy_generated; loaded from the .npz tools/k6_config3.py writes when given, "
                         "else computed here on the host)")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    cfg = dict(CONFIGS[args.config])
    if args.neurons:
        cfg["neurons"] = args.neurons
    if args.communities and args.communities > 1:
        cfg["communities"] = args.communities
        cfg["intra_frac"] = cfg["intra_frac"] or 0.9

    rank, world, local = B.dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    engines = args.engines.split(",")
    spec = spec_for(cfg, args.seed)
    syn_per_gpu = cfg["neurons"] * cfg["degree"] / world
    free = torch.cuda.mem_get_info(dev)[0]
    want_pull = "fused" in engines and syn_per_gpu * 8.0 + 4 * GB < free
    want_push = any(e in ("persistent", "push") for e in engines)
    skipped = {}
    if "fused" in engines and not want_pull:
        skipped["fused"] = ("pull layout build needs ~8 B/synapse transient (%.0f GB) on a GPU with %.0f GB free"
                            % (syn_per_gpu * 8 / GB, free / GB))
    part_s = None
    if args.partition == "blocks":
        lay = S.ShardLayout.blocks(cfg["neurons"], world)
    elif args.partition.startswith("greedy"):
        path = args.partition.split(":", 1)[1] if ":" in args.partition else None
        t0 = time.time()
        if path:
            z = np.load(path)
            meta = json.loads(str(z["meta"]))
            want = {"n_neurons": spec.n_neurons, "n_communities": spec.n_communities, "p_in": spec.p_in,
                    "p_out": spec.p_out, "seed": spec.seed}
            if meta["spec"] != want or meta["n_gpus"] != world:
                raise SystemExit(f"{path}: partition of {meta['spec']} over {meta['n_gpus']} GPUs, need {want} "
                                 f"over {world}")
            asg = z["assignment"].astype(np.int64)
            part_s = meta["seconds"]
        else:
            from paper_2205_07125_b200.partition import partition_greedy_generated
            asg = partition_greedy_generated(spec, world).assignment
            part_s = round(time.time() - t0, 1)
        lay = S.ShardLayout.from_assignment(asg, world)
    else:
        raise SystemExit(f"unknown --partition {args.partition!r}")
    torch.cuda.reset_peak_memory_stats(dev)
    t0 = time.time()
    net = S.Network.generate(spec, lay, device=dev, shards=[rank], pull=want_pull, push=want_push,
                             push_windows=args.push_windows, group_inhibitory=args.ei_group)
    torch.cuda.synchronize()
    build_s = time.time() - t0
    csr = net.shards[rank]
    mem = {"after_build_gb": round(torch.cuda.memory_allocated(dev) / GB, 2),
           "build_peak_gb": round(torch.cuda.max_memory_allocated(dev) / GB, 2),
           "pull_layout_gb": round(csr.n_entries * 4 / GB, 2) if want_pull else None,
           "push_csr_gb": round(next(iter(csr._push_arrays.values()))["syn"].numel() * 4 / GB, 2)
           if want_push else None,
           "push_windows": next(iter(csr._push_arrays.values()))["windows"] if want_push else None,
           "gpu_total_gb": round(torch.cuda.get_device_properties(dev).total_memory / GB, 1)}
    nsyn = torch.tensor([net.n_synapses], dtype=torch.int64, device=dev)
    if world > 1:
        dist.all_reduce(nsyn)

    # routes from the reference planner on the generated network's traffic
    tables = {"direct": None}
    planner = None
    routes = args.routes.split(",") if args.routes else (["direct", "two-level"] if args.config == 4 or (
        args.config == 5 and world >= 4) else ["direct"])
    if "two-level" in routes and world >= 3:
        # the reference's traffic matrix of this network and partition (aggregate, traffic.py:66-84),
        # K5 fed by the generator with the rows split over the ranks (limbs all-reduced)
        t_agg = time.time()
        gt = nc.traffic.aggregate_generated(spec, nc.PartitionMap(world, lay.owner.astype(np.int64)),
                                            group=True if world > 1 else None)
        agg_s = time.time() - t_agg
        groups = nc.group_gpus(gt, args.groups)
        tables["two-level"] = nc.build_routing_table(gt, groups, nc.select_bridges(gt, groups))
        tables["direct"] = nc.route_p2p(gt)
        planner = {"groups": groups.membership.tolist(),
                   "bridges": [[a, b, v] for (a, b), v in sorted(tables["two-level"].bridges.items())],
                   "pg": gt.pg.tolist(), "aggregate_s": round(agg_s, 2),
                   "aggregate": "traffic.aggregate_generated (exact fsum of p per GPU pair, the reference's "
                                "aggregate of the generated network)"}
    tables = {k: v for k, v in tables.items() if k in routes}

    rates = [float(r) for r in args.rates.split(",")] if args.rates else list(cfg["rates"])
    out_path = Path(args.out) if args.out else None
    model_rows = []   # config 4: (route table, nu, measured exchange p50) for the netsim calibration
    digests = {}      # rate -> {engine/route: state digest}

    class A:   # the timing helpers' argument bundle
        steps, warmup, chunk, transport, msg_cap, seed, fused_send = (args.steps, args.warmup, args.chunk, "p2p",
                                                                      None, args.seed, "off")

    for rate in rates:
        lif = S.LifParams() if rate is None else S.LifParams.for_rate(rate)
        for mode, rt in tables.items():
            for eng in engines:
                if eng in skipped or (eng == "fused" and not want_pull) or (eng != "fused" and not want_push):
                    continue
                t_case = time.time()
                pw = args.push_windows if eng == "persistent" else None
                if world > 1:
                    sim = DistSimulator(net, lif, args.seed, rt, transport="p2p", delivery=eng,
                                        latency_steps=args.warmup + args.steps, graph_chunk=args.chunk,
                                        push_windows=pw)
                else:
                    sim = S.Simulator(net, lif, args.seed, rt, delivery=eng, graph_chunk=args.chunk, push_windows=pw)
                if eng == "fused":
                    B.enable_kernel_stamps(sim, args.warmup + args.steps)
                clocks = B.ClockSampler(local)
                ms, spikes, lat, lat_min = B.time_steps(sim, A, world, dev, clocks)
                kms, kms_ranks = (B.live_kernel_ms(sim, args.warmup, args.steps, world, dev) if eng == "fused"
                                  else (None, None))
                hop = sim.hop_ids.sum(0).clone()
                if world > 1:
                    dist.all_reduce(hop)
                # the state after warm-up + timed steps: every engine and route of one rate runs
                # the same dynamics from the same seed, so the digests must agree (bit-exact
                # cross-engine check at real size, where the CPU oracle cannot follow)
                digest = hashlib.sha256()
                for st_ in sim.states:
                    digest.update(st_.v[: st_.n_local].cpu().numpy().tobytes())
                    digest.update(st_.i_syn[: st_.n_local].cpu().numpy().tobytes())
                digest = digest.hexdigest()
                if world > 1:
                    parts = [None] * world
                    dist.all_gather_object(parts, digest)
                    digest = hashlib.sha256("".join(parts).encode()).hexdigest()
                state_sha = digest[:16]
                fused_send = getattr(sim, "fused_send", None)
                sim_windows = sim.states[0].c.push_windows if eng != "fused" else None
                if world > 1:
                    sim.close()
                del sim
                if rank != 0:
                    continue
                n = cfg["neurons"]
                h = hop.cpu().numpy().astype(np.float64) / (args.warmup + args.steps)
                row = {
                    "config": args.config, "n_gpus": world, "engine": eng, "route": mode,
                    "rate_target_hz": rate, "rate_hz": round(spikes / n / (args.steps * 1e-3), 3),
                    "steps_per_s": round(args.steps / (ms * 1e-3), 2), "ms_per_step": round(ms / args.steps, 4),
                    "steps": args.steps, "warmup": args.warmup,
                    "exchange_us": B.lat_summary(lat, lat_min, "p2p"),
                    "kernel_ms": round(kms, 4) if kms else None,
                    "kernel_ms_per_rank": [round(x, 4) for x in kms_ranks] if kms_ranks else None,
                    "ids_per_step": round(float(h.sum()), 1),
                    "wire_bytes_per_step": round(float(h.sum()) * 8 + 8 * int((h > 0).sum()), 1),
                    "channel_ids_per_step": np.round(h, 1).tolist(),
                    "neurons": n, "synapses": int(nsyn.item()), "communities": cfg["communities"],
                    "intra_frac": cfg["intra_frac"], "partition": args.partition.split(":")[0], "partition_s": part_s, "bitmap_tiles": csr.n_tiles if want_pull else None,
                    "fused_send": fused_send, "memory_per_gpu": mem,
                    "push_windows": sim_windows, "ei_group": args.ei_group,
                    "pull_layout_bytes_per_synapse": round(csr.n_entries * 4 / max(net.n_synapses, 1), 4)
                    if want_pull else None, "build_s": round(build_s, 1),
                    "planner": planner, "clocks": clocks.summary(), "case_s": round(time.time() - t_case, 1),
                    "skipped_engines": skipped or None,
                    "state_sha256_16": state_sha,
                }
                if planner is not None and rt is not None:
                    # the reference's analytic per-step model (netsim.py:177-246) for the same table,
                    # activity nu = realised rate x 1 ms, in its own units (calibrated below)
                    nu = min(1.0, row["rate_hz"] * 1e-3)
                    topo = nc.build_topology(nc.TopologySpec(gpus_per_node=max(1, world // args.groups),
                                                             nodes_per_switch=8), world)
                    row["netsim_step_time_model_units"] = nc.step_latency(
                        nc.map_flows(rt, gt, topo, nu), rt, topo, noise=nu).step_time
                    row["connections_out_degree"] = nc.connection_stats(rt).out_degree.tolist()
                    if eng == "persistent" and row["exchange_us"]:
                        model_rows.append((rt, nu, row["exchange_us"]["p50"], row))
                if eng == "fused" and kms:
                    alg = net.n_synapses * 16 / 5 + lay.n_local(rank) * (4 * csr.n_tiles + 22)
                    peak = B.load_peaks()["hbm_gbs"] * GB
                    row["roofline_frac_rank0"] = round(alg / (kms_ranks[0] * 1e-3) / peak, 3)
                    # the bytes the layout actually streams: the J-SELL array with its per-(row, tile)
                    # segment padding, row_meta and row_perm per (row, tile), block starts, state
                    lay_bytes = (csr.n_entries * 4 + csr.row_meta.numel() * 4 + csr.slice_ptr.numel() * 8
                                 + (csr.row_perm.numel() * 4 if csr.row_perm is not None else 0)
                                 + lay.n_local(rank) * 22)
                    row["layout_bytes_rank0"] = int(lay_bytes)
                    row["layout_frac_rank0"] = round(lay_bytes / (kms_ranks[0] * 1e-3) / peak, 3)
                digests.setdefault(str(rate), {})[f"{eng}/{mode}"] = state_sha
                print(json.dumps(row), flush=True)
                if out_path:
                    with out_path.open("a") as f:
                        f.write(json.dumps(row) + "\n")
    if rank == 0 and any(len(d) > 1 for d in digests.values()):
        agree = {"cross_engine_state_agreement": {r: len(set(d.values())) == 1 for r, d in digests.items()},
                 "state_sha256_16": digests,
                 "what": "V and I of every neuron after warm-up + timed steps, per rate: every engine (pull / "
                         "event-driven) and route (direct / two-level) must reach the same bits"}
        print(json.dumps(agree), flush=True)
        if out_path:
            with out_path.open("a") as f:
                f.write(json.dumps(agree) + "\n")
    if rank == 0 and len(model_rows) >= 4:
        # calibrate the reference's TopologySpec on the measured exchange latency
        spec_fit, fit = nc.netsim.calibrate_topology([(rt, nu, t) for rt, nu, t, _ in model_rows], gt, world)
        calib = {k: getattr(spec_fit, k) for k in ("per_hop_latency", "intra_node_bandwidth",
                                                  "inter_node_bandwidth", "connection_setup_cost")}
        summary = {"calibration": calib, "model_vs_measured_us": [
            {"route": r["route"], "rate_hz": r["rate_hz"], "measured_p50": t, "model": round(m, 2)}
            for (_, _, t, r), (_, _, _, m) in zip(model_rows, fit)]}
        print(json.dumps(summary), flush=True)
        if out_path:
            with out_path.open("a") as f:
                f.write(json.dumps(summary) + "\n")
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
