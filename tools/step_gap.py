"""Per-step overhead outside the step kernel (config 2, one GPU): CUDA-graph replays of
100 x (step kernel + end-of-step kernel) against 100 x the step kernel alone."""
import ctypes as C
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    from paper_2205_07125_b200 import sim as S, _native
    n = 1_000_000
    net = S.Network.generate(S.GeneratorSpec.random(n, 1000.0, seed=1), S.ShardLayout.blocks(n, 1))
    sim = S.Simulator(net, S.LifParams(), 1, None)
    sim.reset(1)
    sim.advance(50)
    torch.cuda.synchronize()
    L = _native.lib()
    st = sim.states[0]

    def graph(with_end):
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            g.capture_begin()
            for _ in range(100):
                L.nc_sim_step_fused(C.byref(st.c), C.byref(sim.c_lif), s.cuda_stream)
                if with_end:
                    L.nc_sim_end_step(C.byref(st.c), s.cuda_stream)
            g.capture_end()
        torch.cuda.current_stream().wait_stream(s)
        return g

    out = {}
    for name, we in (("step+end", True), ("step", False), ("step+end", True), ("step", False)):
        g = graph(we)
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        out.setdefault(name, []).append(round(e0.elapsed_time(e1) / 500 * 1e3, 2))
    print("us per step:", out)


if __name__ == "__main__":
    main()
