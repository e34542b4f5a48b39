import sys, torch
sys.path.insert(0, '.')
from paper_2205_07125_b200 import sim as S
n = int(sys.argv[1]); steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
spec = S.GeneratorSpec.random(n, 1000.0, seed=1)
net = S.Network.generate(spec, S.ShardLayout.blocks(n, 1), pull=False, push=True)
sim = S.Simulator(net, S.LifParams(), 1, None, delivery="persistent")
st = sim.states[0]
print("n_local", st.n_local, "spk_cap", st.spk_cap, "push windows", st.c.push_windows, "rowptr", st.push_rowptr.numel(), flush=True)
sim.reset(1)
for k in range(steps):
    sim.advance(1)
    torch.cuda.synchronize()
    if k % 10 == 0:
        print(k, int(st.spk_count[0].item()), int(st.spk_count[1].item()), int(st.spike_total.item()), flush=True)
print("ok")
