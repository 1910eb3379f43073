"""Load the golden fixtures (tests/golden/*.json.gz) and rebuild their inputs
for the product planner (RunConfig) and for the oracle (plain documents)."""

from __future__ import annotations

import glob
import gzip
import hashlib
import json
import os

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")


def names():
    return sorted(os.path.basename(p)[: -len(".json.gz")] for p in glob.glob(os.path.join(GOLDEN, "*.json.gz")))


def load(name):
    with gzip.open(os.path.join(GOLDEN, f"{name}.json.gz"), "rt") as fh:
        return json.load(fh)


def docs(case):
    """(registry_doc, device_doc, stream_doc, routes_doc, run_kwargs)"""
    from paper_2503_02354_b200 import configs

    inp = case["inputs"]
    if "config" in inp:
        base = os.path.join(configs.CONFIG_DIR, inp["config"])
        reg = configs._read(os.path.join(base, "registry.json"))
        dev = configs._read(os.path.join(base, "device.json"))
        stream = configs._read(os.path.join(base, f"stream_{inp['requests']}.json.gz"))
        rp = os.path.join(base, "routes.json")
        routes = configs._read(rp) if os.path.exists(rp) else None
    else:
        reg, dev, stream, routes = inp["registry"], inp["device"], inp["stream"], None
    return reg, dev, stream, routes, dict(inp["run"])


def run_config(case):
    from paper_2503_02354_b200.engine import RunConfig
    from paper_2503_02354_b200.routing import RoutePlan
    from paper_2503_02354_b200.types import DeviceProfile, ModelRegistry, Request

    reg, dev, stream, routes, run = docs(case)
    reqs = [Request(request_id=int(r["request_id"]), component_type=r["component_type"],
                    arrival_time_s=float(r["arrival_time_s"]), detect_u=float(r["detect_u"]))
            for r in stream["requests"]]
    plans = {c: RoutePlan(tuple(v["experts"]), float(v["branch_prob"])) for c, v in routes.items()} if routes else None
    return RunConfig(registry=ModelRegistry.from_doc(reg), device=DeviceProfile.from_doc(dev), stream=reqs,
                     routes=plans, trace=True, **run)


def trace_matches(case, trace_text):
    if "trace_jsonl" in case:
        return trace_text == case["trace_jsonl"]
    return hashlib.sha256(trace_text.encode()).hexdigest() == case["trace_sha256"]
