"""Per-phase timing of the persistent engine on config 2 (one GPU): push, LIF, exchange."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import numpy as np
    import torch
    from paper_2205_07125_b200 import sim as S, _native
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
    spec = S.GeneratorSpec.random(n, 1000.0, seed=1)
    net = S.Network.generate(spec, S.ShardLayout.blocks(n, 1))
    out = {}
    for mode in ("push", "persistent"):
        sim = S.Simulator(net, S.LifParams(), 1, None, delivery=mode)
        st = torch.zeros((64, 4), dtype=torch.int64, device="cuda")
        _native.lib().nc_persistent_phase_stamps(st.data_ptr() if mode.startswith("persistent") else None)
        sim.reset(1)
        sim.advance(20)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        sim.advance(200)
        e1.record()
        torch.cuda.synchronize()
        out[mode] = 200 / (e0.elapsed_time(e1) * 1e-3)
        if mode.startswith("persistent"):
            a = st.cpu().numpy().astype(np.float64)
            d = np.diff(a, axis=1) / 1e3
            print(mode, "phases (us, median over 64 steps): push %.1f  lif %.1f  exchange %.1f  step %.1f" % (
                np.median(d[:, 0]), np.median(d[:, 1]), np.median(d[:, 2]),
                np.median(np.diff(a[:, 0])) / 1e3))
    print({k: round(v, 1) for k, v in out.items()})


if __name__ == "__main__":
    main()
