"""Pin the oracle: its restatement of the reference engine must reproduce the
reference's own golden traces and metrics byte-for-byte."""

import pytest

import golden_cases
from oracle import des

FAST = [n for n in golden_cases.names() if not n.endswith("10k")]


def _simulate(case):
    reg, dev, stream, routes, run = golden_cases.docs(case)
    return des.simulate(reg, dev, stream, routes=routes, trace=True, **run)


@pytest.mark.parametrize("name", FAST)
def test_oracle_matches_reference(name):
    case = golden_cases.load(name)
    out = _simulate(case)
    assert des.metrics_json(out["metrics"]) == case["metrics_json"]
    assert golden_cases.trace_matches(case, des.trace_jsonl(out["trace"]))


@pytest.mark.slow
@pytest.mark.parametrize("name", [n for n in golden_cases.names() if n.endswith("10k")])
def test_oracle_matches_reference_10k(name):
    case = golden_cases.load(name)
    out = _simulate(case)
    assert des.metrics_json(out["metrics"]) == case["metrics_json"]
    assert golden_cases.trace_matches(case, des.trace_jsonl(out["trace"]))
