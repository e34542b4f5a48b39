"""The reference's partition_greedy of BASELINE config 3's network (10 M neurons x ~1 000
synapses, C = 1, W = 1, the device generator's seed-1 network) over 8 GPUs, straight off
the generator (partition.partition_greedy_generated; the NeuronGraph would be 120 GB).
Writes the assignment (uint8) + its spec to an .npz for bench_configs.py --partition greedy.

    python tools/k6_config3.py [n_gpus] [out.npz] [communities]   (C > 1: the regional
    variant of SURVEY 8(d), 90 % of each neuron's synapses inside its community, the
    same spec bench_configs.py --communities C builds)"""
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2205_07125_b200 import partition as P, sim as S  # noqa: E402


def main():
    n_gpus = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    out = Path(sys.argv[2]) if len(sys.argv) > 2 else ROOT / "profiles" / f"r02_k6_config3_greedy{n_gpus}.npz"
    comm = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    import bench_configs as BC
    spec = BC.spec_for(dict(BC.CONFIGS[3], communities=comm, intra_frac=0.9 if comm > 1 else None), 1)
    t = time.time()
    pm = P.partition_greedy_generated(spec, n_gpus)
    dt = time.time() - t
    meta = {"spec": {"n_neurons": spec.n_neurons, "n_communities": spec.n_communities, "p_in": spec.p_in,
                     "p_out": spec.p_out, "seed": spec.seed}, "n_gpus": n_gpus, "seconds": round(dt, 1),
            "counts": np.bincount(pm.assignment, minlength=n_gpus).tolist()}
    np.savez_compressed(out, assignment=pm.assignment.astype(np.uint8), meta=json.dumps(meta))
    print(json.dumps(meta), flush=True)


if __name__ == "__main__":
    main()
