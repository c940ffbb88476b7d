"""bench.py contract pieces that run without a GPU: the reference arm's JSON
line (rank 0 prints, other ranks exit silently), the e2e copy fields, the
traffic lookup keyed by build, and the FP64 roofline fields."""

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _bench(*args, env=None, timeout=600):
    e = dict(os.environ)
    e.update(env or {})
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                          env=e, timeout=timeout)


def test_reference_arm_non_zero_rank_prints_nothing():
    p = _bench("--impl", "reference", "--steps", "1", "--warmup", "0",
               env={"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert p.returncode == 0, p.stderr
    assert p.stdout.strip() == ""


def test_reference_arm_line_contract():
    from oracle import ref_c

    if not ref_c.available("hh_subset"):
        pytest.skip("oracle/_ref not built")
    import bench

    ref = bench.reference_arm("hh1m", K=2, W=1, budget_s=2.0)
    assert ref["kind"] == "reference" and ref["cores"] >= 1 and ref["value"] > 0
    assert "hh_subset" in ref["sample"]
    p = _bench("--impl", "reference", "--workload", "hh1m", "--steps", "2", "--warmup", "1")
    assert p.returncode == 0, p.stderr
    line = json.loads(p.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "higher_is_better", "config", "cpu_baseline",
              "e2e"):
        assert k in line, k
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0
    assert line["config"]["workload"] == "hh1m"


def test_e2e_fields_are_per_timestep_with_per_call_beside():
    import bench

    e = bench._e2e_line(1e9, 1000 * 8, 500 * 8, 1000, 2, "call")
    assert e["h2d_bytes_per_step"] == 8 and e["d2h_bytes_per_step"] == 4
    assert e["h2d_bytes_per_call"] == 8000 and e["timesteps_per_call"] == 1000


def test_traffic_lookup_requires_every_build(monkeypatch):
    import bench

    monkeypatch.setattr(bench, "_traffic_record",
                        lambda: {"by_build": {"a-1": {"dram_bytes": 10.0, "capture": "x"},
                                              "b-2": {"dram_bytes": 5.0, "capture": "y"}}})
    assert bench._traffic(["a-1", "b-2"])[0] == 15.0
    t, note = bench._traffic(["a-1", "c-3"])
    assert t is None and "c-3" in note


def test_roofline_object_has_hbm_and_fp64_fractions(monkeypatch):
    import bench

    monkeypatch.setattr(bench, "_traffic_record", lambda: {})
    r = bench._roofline("k", 1e9, (1e9, "census"), 1.0, ["x"], 1965.0)
    assert r["unit"] == "GB/s" and abs(r["achieved"] - 1000.0) < 1e-6
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-12
    assert r["fp64"]["frac"] > 0 and r["bound"] in ("hbm", "fp64")
    assert r["traffic"] is None
