"""The reference's own test suite against the drop-in (conformance/: verbatim copies of
/root/reference/pkg/tests + a neurocomm -> paper_2205_07125_b200 alias shim).

GPU: every copied test must pass (aggregate is the K5 kernel).  CPU: everything but the
tests that reach aggregate must pass, and those must fail only for the missing device
(no silent CPU fallback exists for K5)."""

from __future__ import annotations

import re
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
SUITE = ROOT / "conformance" / "ref_tests"


def _run(*extra):
    cmd = [sys.executable, "-m", "pytest", str(SUITE), "-q", "-p", "no:cacheprovider", "-rf",
           "--rootdir", str(ROOT / "conformance"), *extra]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=1800, cwd=str(ROOT / "conformance"))
    tail = out.stdout[-6000:]
    m = re.search(r"(?:(\d+) failed, )?(\d+) passed", out.stdout)
    failed = int(m.group(1) or 0) if m else -1
    passed = int(m.group(2)) if m else -1
    return out, tail, passed, failed


@pytest.mark.gpu
def test_reference_suite_passes_on_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out, tail, passed, failed = _run()
    print(tail)
    assert out.returncode == 0 and failed == 0 and passed >= 141, tail


def test_reference_suite_on_cpu_fails_only_for_the_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present: see test_reference_suite_passes_on_gpu")
    out, tail, passed, failed = _run("--tb=line")
    assert passed >= 112, tail
    # every failure is the K5 kernel refusing to run without a device
    # --tb=line: one "<file>:<line>: <Error>: <message>" line per failure
    reasons = [ln for ln in out.stdout.splitlines() if re.match(r"^/\S+:\d+: \w+", ln)]
    assert len(reasons) == failed, tail
    other = [ln for ln in reasons if "no CUDA device" not in ln]
    assert not other, "\n".join(other[:20])
