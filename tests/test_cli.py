"""(f2) The in-package CLI (paper_2503_02354_b200/cli.py), compatible with the reference's
``coesim`` commands (cli.py:383-476): documents round-trip, ``simulate`` reproduces the
reference-made golden metrics / trace byte for byte, ``compare`` prints the reference's table
columns, and exit codes follow cli.py:36-38.  CPU only (``--execute`` is GPU-only)."""

import json
import os
import subprocess
import sys

import golden_cases

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _cli(*args, cwd):
    env = dict(os.environ, PYTHONPATH=ROOT)
    return subprocess.run([sys.executable, "-m", "paper_2503_02354_b200.cli", *args], cwd=cwd, env=env,
                          capture_output=True, text=True, timeout=600)


def test_simulate_matches_reference_golden(tmp_path):
    for case_name, policy in (("c3_1k", "coserve"), ("c3_1k_samba_lru", "samba_lru")):
        case = golden_cases.load(case_name)
        p = _cli("simulate", "--config", "c3", "--requests", "1000", "--policy", policy, "--out", "m.json",
                 "--trace", "t.jsonl", cwd=tmp_path)
        assert p.returncode == 0, p.stderr
        assert (tmp_path / "m.json").read_text() == case["metrics_json"]
        assert golden_cases.trace_matches(case, (tmp_path / "t.jsonl").read_text())


def test_documents_round_trip(tmp_path):
    p = _cli("gen-workload", "--config", "c3", "--out-dir", "docs", cwd=tmp_path)
    assert p.returncode == 0, p.stderr
    a = _cli("simulate", "--config", "c3", "--policy", "coserve", "--out", "a.json", cwd=tmp_path)
    b = _cli("simulate", "--registry", "docs/registry.json", "--stream", "docs/stream.json", "--device",
             "docs/device.json", "--gpu-executors", "1", "--cpu-executors", "0", "--contention-factor", "1.0",
             "--alloc", "gpu=59", "--no-search", "--policy", "coserve", "--out", "b.json", cwd=tmp_path)
    assert a.returncode == 0 and b.returncode == 0, a.stderr + b.stderr
    assert (tmp_path / "a.json").read_text() == (tmp_path / "b.json").read_text()


def test_compare_table_and_json(tmp_path):
    p = _cli("compare", "--config", "c3", "--ablation", "--out-json", "c.json", "--out-csv", "c.csv", cwd=tmp_path)
    assert p.returncode == 0, p.stderr
    header = p.stdout.splitlines()[0].split()
    assert header == ["policy", "execs", "thpt", "stdev", "makespan", "switches", "evict", "xLRU", "sw-red", "ovh"]
    rows = {r["policy"]: r for r in json.loads((tmp_path / "c.json").read_text())["rows"]}
    assert rows["coserve"]["throughput_x_vs_samba_lru"] > 1.0
    assert rows["coserve"]["switch_reduction_vs_samba_lru"] > 0.0
    assert rows["samba_lru"]["throughput_x_vs_samba_lru"] is None
    # the ablation ladder is monotone (reference criterion C7, test_acceptance.py:384-401)
    ladder = [rows[p]["throughput_mean"] for p in ("coserve", "coserve_em_ra", "coserve_em", "coserve_none")]
    assert ladder == sorted(ladder, reverse=True)


def test_profile_and_search_write_documents(tmp_path):
    p = _cli("profile", "--config", "c3", "--out-dir", ".", cwd=tmp_path)
    assert p.returncode == 0, p.stderr
    doc = json.loads((tmp_path / "perf_profile.json").read_text())
    assert doc["schema_version"] == 1 and doc["entries"]
    p = _cli("search-memory", "--config", "c3", "--sample-requests", "200", "--out", "w.json", cwd=tmp_path)
    assert p.returncode == 0, p.stderr
    w = json.loads((tmp_path / "w.json").read_text())
    assert w["lower"] <= w["chosen"] <= w["upper"]


def test_exit_codes(tmp_path):
    assert _cli("simulate", "--policy", "coserve", cwd=tmp_path).returncode == 2  # no workload
    assert _cli("simulate", "--registry", "nope.json", "--stream", "nope.json", "--policy", "coserve",
                cwd=tmp_path).returncode == 2
    (tmp_path / "bad.json").write_text("{not json")
    assert _cli("simulate", "--registry", "bad.json", "--stream", "bad.json", "--policy", "coserve",
                cwd=tmp_path).returncode == 2
    assert _cli("compare", "--config", "c3", "--policies", "coserve,nope", cwd=tmp_path).returncode == 2
