"""The pooled expert allocator's placement policy against fragmentation (CPU).

tools/pool_sim.py replays the runtime's allocator (csrc/runtime.cu issue_copy: best fit, large
experts at the top of their run, small ones at the bottom; slack of three largest experts)
over config 5's plans.  With sparse arrivals the plain lowest-address best fit ran out of
contiguous units on the B200 (the C5 rate sweep); the policy must not, for any arrival gap.
"""
import dataclasses
import importlib.util
import os

import pytest

from paper_2503_02354_b200 import configs, engine

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sim():
    spec = importlib.util.spec_from_file_location("pool_sim", os.path.join(ROOT, "tools", "pool_sim.py"))
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


@pytest.mark.slow
@pytest.mark.parametrize("gap", [1e-6, 1e-4, 3e-4, 1e-3])
def test_c5_pool_never_fragments(gap):
    sim = _sim()
    base = configs.load("c5", 10000)
    stream = [dataclasses.replace(r, arrival_time_s=i * gap) for i, r in enumerate(base.stream)]
    w = dataclasses.replace(base, stream=stream)
    p = engine.plan(configs.run_config(w, trace=False, alloc_override={"gpu": 201}, search_enabled=False))
    budget = p.resolved.executors[0][1]
    largest = max(e.param_bytes for e in p.resolved.config.registry.experts.values())
    pool = int(budget) + 3 * largest + 300 * sim.UNIT
    assert sim.sim(p, pool, "split") == "ok"
