"""The per-kernel event-driven engine's kernels timed alone at config 3 (or N neurons):
k_deliver_push, k_lif_update and k_end_step, each launched back to back with CUDA events
(bench.kernel_ms), after 100 steps of the network.

    python tools/lif_time.py [n_neurons]"""
import sys, torch
sys.path.insert(0, '.')
import bench as B
from paper_2205_07125_b200 import sim as S
n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
spec = S.GeneratorSpec.random(n, 1000.0, seed=1)
net = S.Network.generate(spec, S.ShardLayout.blocks(n, 1), pull=False, push=True)
sim = S.Simulator(net, S.LifParams(), 1, None, delivery="push")
sim.reset(1); sim.prepare(100); sim.advance(100); torch.cuda.synchronize()
print("push_ms", B.kernel_ms(sim, "push", 20), "lif_ms", B.kernel_ms(sim, "lif", 20), "end_ms", B.kernel_ms(sim, "end", 20))
