"""Invariants of the native planner's physical op log (CPU).

The op log is what the GPU executes, so it must agree with the bit-exact
decision trace: every admission lands in exactly one batch of its executor,
batches are single runs in run-rank order (what K1/K2 reproduce on the GPU),
loads equal the reference's switches, hops follow the admission order.
"""

import collections

import numpy as np
import pytest

import golden_cases
from paper_2503_02354_b200 import _native, configs, engine, runtime
from paper_2503_02354_b200.types import ConfigurationError, MemoryStarvationError

CASES = [n for n in golden_cases.names() if not n.endswith("10k")]


@pytest.mark.parametrize("name", CASES)
def test_op_log_matches_trace_and_admissions(name):
    case = golden_cases.load(name)
    cfg = golden_cases.run_config(case)
    p = engine.plan(cfg)
    metrics = engine.metrics_from_plan(p)
    ops, args, adm = p.ops(), p.op_args(), p.admissions()
    assert len(adm) == sum(len(c) for c in p.resolved.chains)
    loads = [o for o in ops if o["kind"] == _native.OP_LOAD]
    assert len(loads) == metrics.expert_switches
    assert sum(int(o["count"]) for o in loads) == metrics.evictions
    # every (request, stage) admitted once and batched once, on the same executor
    admitted = {(int(a["request"]), int(a["stage"])): int(a["executor"]) for a in adm}
    assert len(admitted) == len(adm)
    batched = {}
    for o in ops:
        if o["kind"] != _native.OP_BATCH:
            continue
        pairs = args[int(o["offset"]):int(o["offset"]) + 2 * int(o["count"])].reshape(-1, 2)
        for r, s in pairs:
            assert (int(r), int(s)) not in batched
            batched[(int(r), int(s))] = int(o["executor"])
    assert batched == admitted
    # per executor: execution order == stable sort of admissions by run rank
    for x in range(len(p.resolved.executors)):
        mine = adm[adm["executor"] == x]
        order = np.argsort(mine["run_rank"], kind="stable")
        sorted_pairs = [(int(mine["request"][i]), int(mine["stage"][i])) for i in order]
        executed = [pair for _e, members in runtime.batches_from_plan(p, executor=x) for pair in members]
        assert executed == sorted_pairs
        ranks = {(int(a["request"]), int(a["stage"])): int(a["run_rank"]) for a in mine}
        for _e, members in runtime.batches_from_plan(p, executor=x):
            assert len({ranks[m] for m in members}) == 1  # one run per batch


@pytest.mark.parametrize("name", ["c4_1k_g2", "c4_1k_g4", "c4_1k_g8", "c5_1k_g8"])
def test_hops_follow_admission_order(name):
    case = golden_cases.load(name)
    p = engine.plan(golden_cases.run_config(case))
    hops = runtime.hops_from_plan(p)
    assert [h[0] for h in hops] == list(range(len(hops)))
    where = {}
    for a in p.admissions():
        where[(int(a["request"]), int(a["stage"]))] = int(a["executor"])
    moved = collections.Counter()
    for _i, src, dst, r, s in hops:
        assert src != dst
        assert where[(r, s)] == src and where[(r, s + 1)] == dst
        moved[(r, s)] += 1
    assert max(moved.values(), default=1) == 1
    # every cross-executor follow-up is a hop
    cross = sum(1 for (r, s), x in where.items() if s > 0 and where[(r, s - 1)] != x)
    assert cross == len(hops)


def test_native_errors_map_to_reference_types():
    w = configs.load("c3", 1000)
    with pytest.raises(ConfigurationError):
        engine.run(configs.run_config(w, policy="nope"))
    with pytest.raises(ConfigurationError):
        engine.run(configs.run_config(w, stream=[]))
    tight = configs.run_config(w, alloc_override={"gpu": 1})  # one expert's worth of budget
    m, _ = engine.run(tight)
    assert m.completed_requests == 1000 and m.expert_switches > 200  # one slot: a switch per run


def test_single_request_and_duplicate_ids():
    w = configs.load("c1", 1000)
    m, trace = engine.run(configs.run_config(w, stream=w.stream[:1], trace=True))
    assert m.completed_requests == 1
    dup = [w.stream[0], w.stream[1], w.stream[0]]
    m2, _ = engine.run(configs.run_config(w, stream=dup))
    assert m2.completed_requests == 2  # reference dict semantics: ids are unique keys


def test_multi_gpu_configs_give_each_gpu_its_own_budget():
    """configs.load(..., gpu_executors=N): one executor per B200, so the reference's
    alloc_override (an expert count for all lanes of ONE device) scales with N and every
    executor gets the single-GPU 12 GB regime (59 x 201 MB), capped by the registry."""
    from paper_2503_02354_b200 import configs, engine

    one = engine.resolve(configs.run_config(configs.load("c3", 1000)))
    b1 = one.alloc["gpu"]["expert_budget_bytes"]
    for n in (2, 4):
        r = engine.resolve(configs.run_config(configs.load("c3", 1000, gpu_executors=n)))
        assert len(r.executors) == n
        assert r.alloc["gpu"]["expert_budget_bytes"] == b1
    r8 = engine.resolve(configs.run_config(configs.load("c3", 1000, gpu_executors=8)))
    total = sum(s.param_bytes for s in r8.config.registry.experts.values())
    assert r8.alloc["gpu"]["expert_budget_bytes"] == total / 8  # all 300 experts fit: full residency


PEER_CASES = [n for n in golden_cases.names() if n.endswith("_peer")]


@pytest.mark.parametrize("name", PEER_CASES)
def test_peer_tier_loads_match_oracle(name):
    """(f3) every LOAD's source tier and source executor equal the oracle's (reference + peer tier)."""
    from oracle import des

    case = golden_cases.load(name)
    reg, dev, stream, routes, run = golden_cases.docs(case)
    ref = des.simulate(reg, dev, stream, routes=routes, trace=False, **run)
    p = engine.plan(golden_cases.run_config(case))
    ids = p.resolved.expert_ids
    tiers = {_native.TIER_HOST: "host", _native.TIER_SSD: "ssd", _native.TIER_PEER: "peer"}
    ours = [(int(o["executor"]), ids[int(o["expert"])], tiers[int(o["tier"])],
             int(o["seq"]) if int(o["tier"]) == _native.TIER_PEER else None)
            for o in p.ops() if o["kind"] == _native.OP_LOAD]
    theirs = [(x, e, tier, src) for (x, e, _v, tier), src in zip(ref["loads"], ref["load_src"])]
    assert ours == theirs
    peer = [o for o in ours if o[2] == "peer"]
    assert peer, "the case exercises no peer load"
    for x, _e, _t, src in peer:
        assert src != x and 0 <= src < len(p.resolved.executors)


def test_peer_tier_rejects_bad_bandwidth():
    case = golden_cases.load("c4_1k_g2_peer")
    cfg = golden_cases.run_config(case)
    cfg.peer_tier = {"read_bandwidth_bytes_per_s": 0.0, "fixed_load_overhead_s": 0.0}
    with pytest.raises(ConfigurationError):
        engine.plan(cfg)
