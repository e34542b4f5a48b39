"""Alias shim: the reference's own test suite runs against this package.

``conformance/ref_tests/`` holds verbatim copies of the reference's tests
(/root/reference/pkg/tests: conftest, test_model, test_netsim, test_partition,
test_routing, test_traffic -- not test_cli / test_acceptance, which exercise the
reference's CLI, out of scope per SURVEY section 2).  They import ``neurocomm``;
this conftest, loaded by pytest before theirs, maps ``neurocomm`` and its
submodules onto ``paper_2205_07125_b200`` so every test calls the drop-in.
Run by tests/test_ref_conformance.py (GPU box: aggregate is the K5 kernel).
"""

import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

import paper_2205_07125_b200 as _pkg  # noqa: E402
from paper_2205_07125_b200 import accum, errors, greedy, model, netsim, partition, routing, traffic  # noqa: E402

sys.modules["neurocomm"] = _pkg
for _name, _mod in {"accum": accum, "errors": errors, "greedy": greedy, "model": model, "netsim": netsim,
                    "partition": partition, "routing": routing, "traffic": traffic}.items():
    sys.modules["neurocomm." + _name] = _mod
