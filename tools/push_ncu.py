"""The event-driven engine's two per-step kernels (k_deliver_push, k_lif_update) at
config 3 on one GPU (1e7 neurons x 1e3 synapses, push CSR only, ~11 Hz), for an ncu
capture of what bounds them:

    ncu --set full -k regex:"k_deliver_push|k_lif_update" -s 400 -c 2 python tools/push_ncu.py

Without ncu it prints the per-step time of the two-kernel loop."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    from paper_2205_07125_b200 import sim as S
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 300
    spec = S.GeneratorSpec.random(n, 1000.0, seed=1)
    net = S.Network.generate(spec, S.ShardLayout.blocks(n, 1), pull=False, push=True)
    sim = S.Simulator(net, S.LifParams(), 1, None, delivery="push", use_graph=False)
    sim.reset(1)
    sim.prepare(steps)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    spikes = []
    t = time.perf_counter()
    ev[0].record()
    for k in range(steps):
        sim.advance(1)
        ev[k + 1].record()
    torch.cuda.synchronize()
    ms = [ev[k].elapsed_time(ev[k + 1]) for k in range(steps)]
    sim.check_status()
    tail = ms[steps // 2:]
    print(json.dumps({"neurons": n, "synapses": int(net.n_synapses), "steps": steps,
                      "ms_first_10": [round(x, 3) for x in ms[:10]],
                      "ms_per_step_second_half": round(sum(tail) / len(tail), 4),
                      "spikes_total": int(sim.states[0].spike_total.item()),
                      "wall_s": round(time.perf_counter() - t, 2)}))


if __name__ == "__main__":
    main()
