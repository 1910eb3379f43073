"""Cross-check, call by call, the two copies of the decision logic (CPU).

The product path decides in the native planner (``csrc/planner.cpp``); the package's
Python API mirrors the reference's pure functions (``expert_pool.TwoStageEvictor.select``,
``scheduler.batch_cap``) for drop-in users.  Each copy is pinned to the reference on its own
(planner: byte-identical goldens; mirrors: the reference's own test suite).  Here every
eviction and batch cap the planner made in a run is replayed through the Python mirror with
the pool / queue state of that moment (rebuilt from the planner's trace and op log), and the
two must agree exactly -- expert_pool.py:96-148, scheduler.py:111-118, engine.py:643-716.
"""

import collections

import pytest

import golden_cases
from paper_2503_02354_b200 import _native, engine, scheduler
from paper_2503_02354_b200.expert_pool import ModelPool, TwoStageEvictor

CASES = ["c3_1k", "c4_1k_g2", "c4_1k_g4", "numa_a80_coserve", "c3_10k_g2_pergpu", "c4_1k_g2_peer"]


def _replay(name):
    case = golden_cases.load(name)
    cfg = golden_cases.run_config(case)
    p = engine.plan(cfg)
    res = p.resolved
    assert res.policy.evict == "two_stage"
    ids = res.expert_ids
    reg = cfg.registry
    pools = []
    for x, placed in enumerate(p.initial_residency()):
        pool = ModelPool(x, res.executors[x][1])
        for e in placed:
            pool.add(ids[e], reg.experts[ids[e]].param_bytes)
        pools.append(pool)
    ops, args = p.ops(), p.op_args()
    loads = collections.defaultdict(collections.deque)
    batches = collections.defaultdict(collections.deque)
    for o in ops:
        (loads if o["kind"] == _native.OP_LOAD else batches)[int(o["executor"])].append(o)
    evictor = TwoStageEvictor(reg)
    pending = [collections.Counter() for _ in pools]  # queued, not in-flight entries per expert
    request_expert = {}
    checked_loads = checked_caps = 0
    for ev in p.trace():
        x, kind = ev["executor"], ev["event"]
        if kind == "assign":
            pending[x][ev["expert_id"]] += 1
            request_expert[(x, ev["request_id"])] = ev["expert_id"]
        elif kind == "load":
            op = loads[x].popleft()
            expert = ids[int(op["expert"])]
            assert expert == ev["expert_id"]
            want = [ids[v] for v in args[int(op["offset"]):int(op["offset"]) + int(op["count"])]]
            got = evictor.select(pools[x], reg.experts[expert].param_bytes, +pending[x])
            assert got == want, f"{name}: load of {expert} on executor {x}: mirror {got} != planner {want}"
            for v in got:
                pools[x].remove(v)
            pools[x].add(expert, reg.experts[expert].param_bytes)
            checked_loads += 1
        elif kind == "batch_start":
            op = batches[x].popleft()
            expert = ids[int(op["expert"])]
            members = args[int(op["offset"]):int(op["offset"]) + 2 * int(op["count"])].reshape(-1, 2)
            queued = pending[x][expert]
            arch = reg.experts[expert].arch
            perf = res.perf.entry(arch, res.executors[x][0])
            cap = scheduler.batch_cap(perf.max_batch, res.executors[x][2],
                                      lambda n: res.cost.inference_memory(arch, res.executors[x][0], n))
            # arrange keeps an expert's queued entries in one run, so the head run is all of them
            assert len(members) == min(cap, queued), f"{name}: batch of {len(members)} on {expert}, cap {cap}"
            pending[x][expert] -= len(members)
            checked_caps += 1
    assert checked_loads == sum(1 for o in ops if o["kind"] == _native.OP_LOAD)
    return checked_loads, checked_caps


@pytest.mark.parametrize("name", CASES)
def test_planner_evictions_equal_python_mirror(name):
    loads, caps = _replay(name)
    assert caps > 0
    if name != "c4_1k_g4":
        assert loads > 0
