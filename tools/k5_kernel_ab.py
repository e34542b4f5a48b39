"""K5 kernel time alone (uniform-weight and packed paths), CUDA events, median of 30
launches, for kernel A/Bs (NEUROCOMM_B200_LIB=variant).  1e6 neurons, 4.9e7 edges, 8 GPUs.

    python tools/k5_kernel_ab.py"""
import json
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))


def main():
    import torch
    import paper_2205_07125_b200 as nc
    from paper_2205_07125_b200 import _native, traffic as T
    spec = nc.ModelSpec(1_000_000, 8, 90 / (1_000_000 / 8 - 1), 10 / 1_000_000, seed=1)
    g = nc.generate_synthetic(spec)
    pm = nc.partition_random(g, 8, seed=1)
    dev = torch.device("cuda", 0)
    w, ei, ej, ep, w0 = T._device_graph(g, dev)
    n = 8
    lo, hi = T._window(ep, w)
    nd = T._n_digits(lo, hi, ei.numel())
    asg8 = torch.from_numpy(pm.assignment.astype(np.uint8)).to(dev)
    rec, _ = T._records(w)
    rec[:, 2] = asg8.to(torch.int32)
    L = _native.lib()
    st = _native.stream_handle()
    out = {}
    for name, call in (("uniform", lambda b: L.nc_traffic_histogram_uniform(
            ei.data_ptr(), ej.data_ptr(), ep.data_ptr(), 1.0, asg8.data_ptr(), ei.numel(), n, lo, nd, b.data_ptr(), st)),
                       ("packed", lambda b: L.nc_traffic_histogram_packed(
            ei.data_ptr(), ej.data_ptr(), ep.data_ptr(), rec.data_ptr(), ei.numel(), n, lo, nd, b.data_ptr(), st))):
        buf = torch.zeros(n * n * nd, dtype=torch.int64, device=dev)
        ts = []
        for _ in range(33):
            buf.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            _native.check(call(buf), name)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = float(np.median(ts[3:]))
        out[name] = {"ms": round(ms, 4), "stream_gbs": round(16 * ei.numel() / (ms * 1e-3) / 1e9, 1)}
    print(json.dumps({"edges": int(ei.numel()), **out}), flush=True)


if __name__ == "__main__":
    main()
