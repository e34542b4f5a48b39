"""CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this package, and only as the checker or the
timed CPU baseline; the product package never imports it.

* sim_oracle.c / c_oracle.py -- C restatement of simulate(steps) (OpenMP).
  Parity UNPINNED against the reference (which has no spike loop); pinned by
  Philox known-answer vectors, the independent numpy restatement
  (sim_numpy.py) and committed golden rasters (tests/golden/).
* The planner stages are checked against outputs of the reference itself, not a
  restatement: tests/golden/make_golden.py runs the reference (in the build container) and
  commits its results (reference_fixtures.*, reference_io.json); the reference's own test
  suite runs against the drop-in through conformance/.
"""
