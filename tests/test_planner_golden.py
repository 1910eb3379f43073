"""The native planner reproduces the unmodified reference bit-for-bit:
metrics document and event trace (engine.py:832-838) on every golden case
(the five BASELINE configs, all seven policies, numa/uma, window search)."""

import pytest

import golden_cases
from paper_2503_02354_b200 import engine

CASES = golden_cases.names()


@pytest.mark.parametrize("name", CASES)
def test_planner_matches_reference(name):
    case = golden_cases.load(name)
    metrics, trace = engine.run(golden_cases.run_config(case))
    assert engine.metrics_json(metrics) == case["metrics_json"]
    assert golden_cases.trace_matches(case, engine.trace_jsonl(trace))


def test_golden_set_covers_every_config_and_policy():
    assert {"c1_1k", "c2_1k", "c3_1k", "c4_1k_g2", "c4_1k_g4", "c4_1k_g8", "c5_1k_g8", "c3_10k"} <= set(CASES)
    policies = {golden_cases.load(n)["inputs"]["run"].get("policy") for n in CASES}
    assert policies == set(engine.POLICIES)
