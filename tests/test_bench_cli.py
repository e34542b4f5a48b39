"""bench.py contract on CPU: the reference arm prints exactly one JSON line on stdout.

The GPU arm shares the same stdout handling (library output on fd 1 is moved to stderr),
so this also guards the line the driver parses.
"""

from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_one_json_line():
    cmd = [sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "3", "--warmup", "3",
           "--neurons", "5000", "--degree", "100"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = out.stdout.splitlines()
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference"
    assert d["steps"] == 3 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["higher_is_better"] is True and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1


def test_warmup_below_three_rejected():
    cmd = [sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--warmup", "2"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=120, cwd=ROOT)
    assert out.returncode != 0
    assert out.stdout == ""


def test_reference_arm_config_matches_ours():
    """Both arms print the same `config` dict (bench.common_config), so the driver can
    compare them; the reference arm honours --warmup."""
    sys.path.insert(0, str(ROOT))
    import argparse
    import bench
    args = argparse.Namespace(neurons=1_000_000, degree=1000.0, communities=1, intra_frac=0.9, seed=1,
                              scaling="strong", transport="p2p")
    c1 = bench.common_config(args, 1)
    assert c1["workload"].startswith("config 2") and c1["neurons"] == 1_000_000
    cmd = [sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "3", "--warmup", "4",
           "--neurons", "5000", "--degree", "100"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=300, cwd=ROOT)
    d = json.loads(out.stdout.splitlines()[0])
    args.neurons, args.degree = 5000, 100.0
    assert d["config"] == json.loads(json.dumps(bench.common_config(args, 1)))
    assert d["warmup"] == 4


def test_bench_configs_specs_match_baseline():
    """bench_configs.py's configs 3-5 are BASELINE.json's: 1e7 x 1k random, and 5e7 neurons in
    64 regions with ~90 % of ~1 000 synapses intra-region."""
    sys.path.insert(0, str(ROOT))
    import bench_configs as BC
    base = json.loads((ROOT / "BASELINE.json").read_text())["configs"]
    assert "10M neurons" in base[2] and "50M" in base[4]
    s3 = BC.spec_for(BC.CONFIGS[3], 1)
    assert s3.n_neurons == 10_000_000 and s3.n_communities == 1
    assert abs(s3.p_in * (s3.n_neurons - 1) - 1000.0) < 1e-6
    s5 = BC.spec_for(BC.CONFIGS[5], 1)
    size = s5.n_neurons / s5.n_communities
    intra = s5.p_in * (size - 1)
    inter = s5.p_out * (s5.n_neurons - size)
    assert s5.n_neurons == 50_000_000 and s5.n_communities == 64
    assert abs(intra - 900.0) < 1e-6 and abs(inter - 100.0) < 1e-6
    assert BC.CONFIGS[4]["rates"] == (1, 2, 5, 10, 20, 50)
