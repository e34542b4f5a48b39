"""Per-GPU pull-kernel time of config-2 strong scaling at N = 1/2/4/8 on ONE GPU: N virtual
ranks (tests/virtual_ranks.py) each own shard r of the block layout, and every step their
step kernels run one after another on one stream -- each alone on the GPU, as on its own
B200 -- with the device %globaltimer stamps of every launch (nc_shard_t.kstamp).  The
exchange between the virtual ranks runs too (on concurrent streams) but its timing says
nothing about NVLink; only the kernel times are reported.

    python tools/vr_kernel.py [--worlds 1,2,4,8] [--steps 200] [--warmup 20]

One JSON line per N: per-rank kernel ms, max, the ideal (N = 1 time / N) and the
algorithmic-bytes roofline fraction of the slowest rank."""
import argparse
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def main():
    import torch
    from paper_2205_07125_b200 import sim as S
    from virtual_ranks import VirtualCluster
    ap = argparse.ArgumentParser()
    ap.add_argument("--worlds", default="1,2,4,8")
    ap.add_argument("--neurons", type=int, default=1_000_000)
    ap.add_argument("--degree", type=float, default=1000.0)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--tile-words", type=int, default=None, help="force the bitmap tile size (A/B)")
    ap.add_argument("--split", type=int, default=None, help="force log2 of the block split (A/B, 0-3)")
    ap.add_argument("--buffers", type=int, default=None, choices=(2, 3), help="force the tile buffer count (A/B)")
    args = ap.parse_args()
    if args.buffers is not None:
        from paper_2205_07125_b200 import sell
        sell.triple_buffer = lambda *a: args.buffers == 3
    if args.split is not None:
        from paper_2205_07125_b200 import sell
        sell.block_split = lambda n_local, n_tiles, n_sms: args.split if n_tiles > 1 else 0
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() \
        else 6544.0
    spec = S.GeneratorSpec.random(args.neurons, args.degree, seed=1)
    t1 = None
    for world in [int(x) for x in args.worlds.split(",")]:
        lay = S.ShardLayout.blocks(args.neurons, world)
        nets = [S.Network.generate(spec, lay, shards=[r], tile_words=args.tile_words) for r in range(world)]
        n = args.warmup + args.steps
        vc = VirtualCluster(nets, S.LifParams(), 1, None, transport="p2p", delivery="fused")
        bufs = []
        for sim in vc.sims:
            s = sim.state
            buf = torch.zeros(2 * n, dtype=torch.int64, device=s.v.device)
            buf.view(-1, 2)[:, 0] = -1
            s.kstamp_buf = buf
            s.c.kstamp = buf.data_ptr()
            s.c.kstamp_steps = n
            bufs.append(buf)
        vc.reset(1)
        vc.step(n)
        torch.cuda.synchronize()
        for sim in vc.sims:
            sim.check_status()
        per = []
        for buf in bufs:
            st = buf.view(-1, 2)[args.warmup:n]
            per.append(float(((st[:, 1] - st[:, 0]).to(torch.float64).mean() / 1e6).item()))
        # algorithmic bytes per rank: packed slots + row_meta / placement + 26 B per neuron + bitmap
        alg = []
        for r, net in enumerate(nets):
            csr = net.shards[r]
            b = csr.syn.numel() * 4 + csr.row_meta.numel() * 4 + csr.slice_ptr.numel() * 8
            b += (csr.row_perm.numel() * 4 if csr.row_perm is not None else 0) + 26 * csr.n_local + lay.n_words * 4
            alg.append(b)
        worst = max(range(world), key=lambda r: per[r])
        if world == 1:
            t1 = per[0]
        out = {"world": world, "neurons": args.neurons, "kernel_ms_per_rank": [round(x, 5) for x in per],
               "kernel_ms_max": round(max(per), 5), "ideal_ms": round(t1 / world, 5) if t1 else None,
               "kernel_efficiency": round(t1 / world / max(per), 3) if t1 else None,
               "tiles": nets[0].shards[0].n_tiles, "split": args.split, "buffers": args.buffers, "tile_words": nets[0].shards[0].tile_words, "rows_per_rank": nets[0].shards[0].n_local,
               "frac_slowest": round(alg[worst] / (per[worst] * 1e-3) / 1e9 / peak, 3)}
        print(json.dumps(out), flush=True)
        vc.close()
        del vc, nets
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
