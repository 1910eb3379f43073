"""bench.py's reference arm on CPU: the oracle port serves a bounded sample and prints the
contract's JSON line (impl, metric, unit, cpu_baseline, e2e with zero transfer bytes); under
torchrun only rank 0 prints."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(env_extra):
    env = dict(os.environ, **env_extra)
    proc = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--config", "c1", "--requests", "1000",
                           "--cpu-budget", "0.5", "--requests", "1000", "--steps", "1", "--warmup", "0"],
                          cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert proc.returncode == 0, proc.stderr[-2000:]
    return proc.stdout.strip().splitlines()


def test_reference_arm_prints_one_contract_line():
    lines = _run({})
    d = json.loads(lines[-1])
    assert d["impl"] == "reference" and d["unit"] == "requests/s" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["steps"] == 1 and d["warmup"] == 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "requests/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_other_ranks_exit_quietly():
    assert _run({"RANK": "1", "WORLD_SIZE": "2"}) == []
