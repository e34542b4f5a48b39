"""Golden vectors for the native NNG / PMAP text I/O, produced by the reference itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_io_golden.py

For a set of well-formed and malformed inputs it records what the reference's
load_graph / load_partition_map return (the parsed arrays) or raise
(ParseError message and line), and the exact bytes its save_graph /
save_partition_map write.  Output: tests/golden/reference_io.json.
"""

from __future__ import annotations

import json
import sys
import tempfile
from pathlib import Path

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent

NNG_CASES = {
    "ok_small": "NNG 1 3 2\n1.0\n0.5\n2.25\n0 1 0.5\n1 2 1.0\n",
    "ok_crlf_ws": "NNG 1 2 1\r\n 1.5 \r\n2e0\r\n0  1\t0.75\r\n",
    "ok_underscore": "NNG 1 2 1\n1_0.5\n1.0\n0 1 1e-05\n",
    "ok_no_final_newline": "NNG 1 2 1\n1.0\n1.0\n0 1 0.125",
    "ok_plus_sign": "NNG 1 2 1\n+1.0\n1.0\n+0 +1 .5\n",
    "empty": "",
    "blank_header": "\n",
    "bad_magic": "NNX 1 2 1\n1.0\n1.0\n0 1 0.5\n",
    "bad_version": "NNG 2 2 1\n1.0\n1.0\n0 1 0.5\n",
    "bad_counts_text": "NNG 1 two 1\n",
    "bad_counts_value": "NNG 1 0 0\n",
    "short": "NNG 1 3 2\n1.0\n1.0\n1.0\n0 1 0.5\n",
    "trailing": "NNG 1 2 1\n1.0\n1.0\n0 1 0.5\nextra\n",
    "bad_weight": "NNG 1 2 1\n1.0x\n1.0\n0 1 0.5\n",
    "quote_weight": "NNG 1 2 1\nit's\n1.0\n0 1 0.5\n",
    "neg_weight": "NNG 1 2 1\n-2.5\n1.0\n0 1 0.5\n",
    "nan_weight": "NNG 1 2 1\nnan\n1.0\n0 1 0.5\n",
    "inf_weight": "NNG 1 2 1\ninf\n1.0\n0 1 0.5\n",
    "bad_edge_fields": "NNG 1 2 1\n1.0\n1.0\n0 1\n",
    "bad_edge_token": "NNG 1 2 1\n1.0\n1.0\n0 b 0.5\n",
    "edge_range": "NNG 1 2 1\n1.0\n1.0\n1 0 0.5\n",
    "edge_range_hi": "NNG 1 2 1\n1.0\n1.0\n0 2 0.5\n",
    "edge_p_zero": "NNG 1 2 1\n1.0\n1.0\n0 1 0.0\n",
    "edge_p_big": "NNG 1 2 1\n1.0\n1.0\n0 1 1.5e300\n",
    "edge_dup": "NNG 1 3 2\n1.0\n1.0\n1.0\n0 1 0.5\n0 1 0.25\n",
    "edge_order": "NNG 1 3 2\n1.0\n1.0\n1.0\n1 2 0.5\n0 1 0.25\n",
    "tab_in_line": "NNG 1 2 1\n1.0\n\t1.0\x07\n0 1 0.5\n",
}
PMAP_CASES = {
    "ok": "PMAP 1 4 2\n0\n0\n1\n1\n",
    "ok_ws": "PMAP 1 2 3\n 2 \r\n1_0\n",
    "empty": "",
    "bad_header": "PMAP 2 4 2\n0\n",
    "bad_counts": "PMAP 1 0 2\n",
    "short": "PMAP 1 3 2\n0\n1\n",
    "trailing": "PMAP 1 1 2\n0\n1\n",
    "bad_index": "PMAP 1 2 2\n0\nx1\n",
    "range": "PMAP 1 2 2\n0\n2\n",
}


def main() -> int:
    sys.path.insert(0, str(REF))
    import numpy as np
    import neurocomm as nc  # noqa: E402  (the reference)
    from neurocomm.partition import load_partition_map, save_partition_map

    out = {"nng": {}, "pmap": {}, "nng_write": {}, "pmap_write": {}}
    with tempfile.TemporaryDirectory() as d:
        p = Path(d) / "f"
        for name, text in NNG_CASES.items():
            p.write_bytes(text.encode())
            try:
                g = nc.load_graph(p)
                out["nng"][name] = {"text": text, "ok": True, "weights": [x.hex() for x in g.weights.tolist()],
                                    "edges": [[int(i), int(j), float(q).hex()] for i, j, q in
                                              zip(g.edge_i, g.edge_j, g.edge_p)]}
            except nc.ParseError as e:
                out["nng"][name] = {"text": text, "ok": False, "message": str(e.args[0]), "line": e.line}
        for name, text in PMAP_CASES.items():
            p.write_bytes(text.encode())
            try:
                pm = load_partition_map(p)
                out["pmap"][name] = {"text": text, "ok": True, "n_gpus": pm.n_gpus,
                                     "assignment": pm.assignment.tolist()}
            except nc.ParseError as e:
                out["pmap"][name] = {"text": text, "ok": False, "message": str(e.args[0]), "line": e.line}
        specs = {"sbm": dict(n_neurons=40, n_communities=3, p_in=0.3, p_out=0.05, weight_low=0.1,
                             weight_high=1e5, seed=2),
                 "tiny": dict(n_neurons=7, n_communities=1, p_in=0.9, p_out=0.0, weight_low=1e-7,
                              weight_high=3e-5, seed=8)}
        for name, kw in specs.items():
            g = nc.generate_synthetic(nc.ModelSpec(**kw))
            nc.save_graph(g, p)
            out["nng_write"][name] = {"spec": kw, "text": p.read_text()}
            pm = nc.partition_greedy(g, 3)
            save_partition_map(pm, p)
            out["pmap_write"][name] = {"spec": kw, "text": p.read_text()}
    (OUT / "reference_io.json").write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
    print("wrote", sum(len(v) for v in out.values()), "cases")
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
