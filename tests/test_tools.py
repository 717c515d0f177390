"""CPU tests of the measurement tools' host logic (parsers and summaries):
the ncu CSV parser behind profiles/traffic.json (tools/traffic_record.py),
the launch-list share (tools/ncu_summary.py) and the tree-trace analysis
(tools/tree_trace.py).  Fixtures: tests/golden/ncu_metrics_*.csv, in ncu's
--csv metric-list format (the first rows of profiles/r02w_launches.txt's
capture, and hand-written DRAM / NVLink rows with unit scaling)."""
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "tools"))
GOLD = os.path.join(ROOT, "tests", "golden")


def test_traffic_csv_parser_units():
    import traffic_record as tr
    m = tr.metrics_from_csv(os.path.join(GOLD, "ncu_metrics_single_fixture.csv"))
    assert m["dram__bytes_read.sum"] == pytest.approx(1.56e9)
    assert m["dram__bytes_write.sum"] == pytest.approx(1.502e9)   # "1,502.00" Mbyte
    assert m["nvltx__bytes.sum"] == 195035136


def test_traffic_record_merges_same_hash(tmp_path, monkeypatch):
    import traffic_record as tr
    monkeypatch.setattr(tr, "ROOT", str(tmp_path))
    (tmp_path / "profiles").mkdir()
    fx = os.path.join(GOLD, "ncu_metrics_single_fixture.csv")
    monkeypatch.setattr(sys, "argv", ["traffic_record.py", "k", "abc", fx])
    tr.main()
    rec = json.load(open(tmp_path / "profiles" / "traffic.json"))["k"]
    assert rec["source_sha"] == "abc" and rec["dram_bytes"] == pytest.approx(3.062e9)
    assert rec["nvltx_bytes"] == 195035136
    # a new hash replaces the record instead of merging into it
    monkeypatch.setattr(sys, "argv", ["traffic_record.py", "k", "def", os.path.join(GOLD, "ncu_metrics_fixture.csv")])
    tr.main()
    rec = json.load(open(tmp_path / "profiles" / "traffic.json"))["k"]
    assert rec["source_sha"] == "def" and "dram_bytes" not in rec and rec["duration_s"] > 0


def test_bench_traffic_lookup_requires_matching_hash(tmp_path, monkeypatch):
    sys.path.insert(0, ROOT)
    import bench
    monkeypatch.setattr(bench, "ROOT", str(tmp_path))
    (tmp_path / "profiles").mkdir()
    json.dump({"k": {"source_sha": "nope", "dram_bytes": 1.0, "source": "x"}},
              open(tmp_path / "profiles" / "traffic.json", "w"))
    rec, prov = bench.committed_traffic("k")
    assert rec is None and prov["stale"] == "x"
    json.dump({"k": {"source_sha": bench.source_sha(), "dram_bytes": 1.0, "source": "x"}},
              open(tmp_path / "profiles" / "traffic.json", "w"))
    rec, prov = bench.committed_traffic("k")
    assert rec["dram_bytes"] == 1.0 and prov["source_sha"] == bench.source_sha()


def test_tree_trace_analysis_splits_roles(tmp_path):
    import tree_trace as tt
    tr = np.zeros((4, 3, 8), dtype=np.uint64)
    for cta in range(4):
        for ev in range(3):
            t0 = 1000 + 100 * ev
            # even CTAs (tree 0) wait 10 ns, odd ones 40 ns; work 50 ns
            w = 10 if cta % 2 == 0 else 40
            tr[cta, ev] = [(1 << 60) | ev, t0, t0 + w, t0 + w + 20, t0 + w + 50, 0, 0, 0]
    np.save(tmp_path / "rank0.npy", tr)
    rep = tt.analyze(str(tmp_path))[0]
    assert rep["up_tree0"]["n"] == 6 and rep["up_tree1"]["n"] == 6
    assert rep["up_tree0"]["wait_us_sum"] == pytest.approx(6 * 10 / 1e3)
    assert rep["up_tree1"]["wait_us_sum"] == pytest.approx(6 * 40 / 1e3)
    assert rep["up_tree0"]["work_us_mean"] == pytest.approx(0.05)
