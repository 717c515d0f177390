"""Bench smoke (SURVEY §4 tier 4): tiny sizes through bench.py and a check of
the JSON line the driver reads (the contract in bench.py's docstring)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def _run(args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT, capture_output=True,
                         text=True, timeout=timeout)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    return json.loads(lines[0])


def test_reference_arm_schema():
    """--impl reference: the CPU oracle on a tiny C2-shaped workload."""
    d = _run(["--impl", "reference", "--count", "4099", "--steps", "2", "--warmup", "1"])
    assert BASE_KEYS <= d.keys()
    assert d["impl"] == "reference" and d["unit"] == "GB/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["steps"] == 2 and d["warmup"] == 1
    assert d["config"]["workload"] and d["config"]["count_per_rank"] == 4099
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


@pytest.mark.gpu
def test_hfr_arm_schema_tiny():
    """The product arm at N=1 on a small count: every key the driver reads."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    d = _run(["--count", str((1 << 20) + 3), "--steps", "3", "--warmup", "3", "--no-cpu", "--soak", "0",
              "--e2e-chunks", "2"])
    assert BASE_KEYS <= d.keys() and "impl" not in d
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["scaling"] == "weak"
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] <= 1.2 and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] >= 3
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= d["clocks"].keys()


@pytest.mark.parametrize("algo,n,esz,want", [
    # SURVEY §8(d) "algorithmic bytes": worst rank's NVLink bytes per direction, in units of S
    ("dbt", 8, 4, 2.0), ("dbt", 4, 4, 2.0), ("dbt", 2, 4, 1.0),
    ("pair_dbt", 8, 4, 2.0), ("pair_dbt", 4, 4, 1.5),
    ("nvls", 8, 4, 1.125), ("nvls", 4, 2, 1.25), ("nvls", 2, 4, 1.5),
])
def test_variant_bytes_match_survey(algo, n, esz, want):
    """bench.variant_dir_bytes (the roofline numerator of the tree/NVLS
    variants) reproduces SURVEY §8(d)'s per-direction byte counts, computed
    from the library's own trees (hfr_tree_query, host-only)."""
    sys.path.insert(0, ROOT)
    import bench
    import paper_2408_14158_b200 as hfr
    S = 1 << 20
    assert bench.variant_dir_bytes(hfr, algo, n, S, esz) == pytest.approx(want * S)


def test_variant_bytes_bf16_dbt_between_2_and_3():
    """bf16 DBT: fp32 partials up (16-bit leaves send raw values), bf16 finals
    down — SURVEY's 3S is the all-fp32-partials upper bound."""
    sys.path.insert(0, ROOT)
    import bench
    import paper_2408_14158_b200 as hfr
    S = 1 << 20
    v = bench.variant_dir_bytes(hfr, "dbt", 8, S, 2) / S
    assert 2.0 <= v <= 3.0


def test_variant_bytes_fp8_dbt_leaves_raw():
    """FP8 DBT leaves send 1-byte raw values, not 4-byte fp32 partials."""
    sys.path.insert(0, ROOT)
    import bench
    import paper_2408_14158_b200 as hfr
    S = 1 << 20
    assert bench.variant_dir_bytes(hfr, "dbt", 2, S, 1) == pytest.approx(S * (1 + 1) / 2)  # n=2: raw up + final down
