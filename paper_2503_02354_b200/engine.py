"""Serving runtime entry point: ``run(RunConfig) -> (Metrics, trace)``.

Drop-in mirror of ``coesim.engine`` (``/root/reference/pkg/src/coesim/engine.py``).
``run`` resolves the configuration exactly as the reference does -- policy
table (engine.py:59-76), memory partition (:192-224), perf profile (:374-376),
expert/activation allocation incl. the decay-window search (:412-495),
executor layout (:497-519) -- and hands the decision loop to the native
planner (``csrc/planner.cpp``, ``include/coe_planner.h``), which replays the
admission -> step -> load -> batch -> follow-up cycle bit-exactly and returns
metrics, the trace and the physical op log.

``serve`` (below) is the B200 path: the same plan, executed on the GPU by
``runtime.B200Runtime`` -- GPU grouping (K1/K2), tcgen05 grouped expert MLPs
(K3), copy-engine swap-ins (K4).

Extension over the reference: ``RunConfig.routes`` may supply N-stage chain
templates (``routing.RoutePlan``) per component type for the 3- and 5-stage
configurations; the tail is taken iff ``detect_u < branch_prob``, the
reference's own rule (engine.py:720-727).
"""

from __future__ import annotations

import ctypes
import itertools
import json
from dataclasses import dataclass, field, replace

import numpy as np

from . import _native
from . import profiler as profiler_mod
from . import routing
from .costmodel import CostModel
from .profiler import ALLOC_WINDOW_SEARCH, PerfProfile, WindowSearchResult, build_perf_profile, \
    decay_window_search, decide_allocation_mode
from .seeding import subseed
from .types import SCHEMA_VERSION, ConfigurationError, MemoryStarvationError


@dataclass(frozen=True)
class PolicySpec:
    assign: str      # "makespan" | "round_robin"
    arrange: bool
    evict: str       # "two_stage" | "lru" | "fifo"
    single_gpu: bool
    host_mode: str   # host-cache victim order: "prob" | "lru" | "fifo"


POLICIES = {
    "coserve": PolicySpec("makespan", True, "two_stage", False, "prob"),
    "coserve_em_ra": PolicySpec("round_robin", True, "two_stage", False, "prob"),
    "coserve_em": PolicySpec("round_robin", False, "two_stage", False, "prob"),
    "coserve_none": PolicySpec("round_robin", False, "fifo", False, "fifo"),
    "samba_lru": PolicySpec("round_robin", False, "lru", True, "lru"),
    "samba_fifo": PolicySpec("round_robin", False, "fifo", True, "fifo"),
    "samba_parallel": PolicySpec("round_robin", False, "lru", False, "lru"),
}

_EVICT_CODE = {"two_stage": 0, "lru": 1, "fifo": 2}
_HOST_CODE = {"prob": 0, "lru": 1, "fifo": 2}
_PROCS = ("gpu", "cpu")


@dataclass
class RunConfig:
    """Everything a run depends on (engine.py:79-103), plus ``routes``."""

    registry: object
    device: object
    policy: str
    stream: list
    seed: int = 0
    gpu_executors: int = 3
    cpu_executors: int = 1
    contention_factor: float = 1.15
    cpu_mem_fraction: float = 0.4
    alloc_override: dict | None = None
    alloc_threshold: float = profiler_mod.DEFAULT_ALLOC_THRESHOLD
    plateau_threshold: float = profiler_mod.DEFAULT_PLATEAU_THRESHOLD
    initial_window: int = profiler_mod.DEFAULT_INITIAL_WINDOW
    error_margin: float = profiler_mod.DEFAULT_ERROR_MARGIN
    fit_points: int = profiler_mod.DEFAULT_FIT_POINTS
    search_enabled: bool = True
    search_sample_requests: int = 400
    window_choose: str = "random"
    samba_gpu_only: bool = True
    perf: PerfProfile | None = None
    trace: bool = False
    routes: dict | None = None  # component -> RoutePlan (N-stage extension)
    # (f3) peer-GPU swap-in tier: {"read_bandwidth_bytes_per_s", "fixed_load_overhead_s"}; a LOAD
    # of an expert another GPU executor holds copies it over NVLink (planner.cpp peer_source)
    peer_tier: dict | None = None


@dataclass
class Metrics:
    """Aggregate outcome; wall-clock fields stay out of ``to_doc`` (engine.py:106-160)."""

    policy: str
    seed: int
    completed_requests: int
    follow_ups: int
    makespan_s: float
    throughput_rps: float
    expert_switches: int
    evictions: int
    stale_predictions: int
    per_executor: list
    alloc: dict
    busy_s_total: float = 0.0
    sched_wall_s: float = 0.0
    sched_calls: int = 0

    def mean_service_time_s(self) -> float:
        return self.busy_s_total / self.completed_requests if self.completed_requests else 0.0

    def sched_wall_per_request_s(self) -> float:
        return self.sched_wall_s / self.sched_calls if self.sched_calls else 0.0

    def sched_overhead_ratio(self) -> float:
        service = self.mean_service_time_s()
        return self.sched_wall_per_request_s() / service if service != 0.0 else 0.0

    def to_doc(self) -> dict:
        return {
            "schema_version": SCHEMA_VERSION,
            "policy": self.policy,
            "seed": self.seed,
            "completed_requests": self.completed_requests,
            "follow_ups": self.follow_ups,
            "makespan_s": self.makespan_s,
            "throughput_rps": self.throughput_rps,
            "expert_switches": self.expert_switches,
            "evictions": self.evictions,
            "stale_predictions": self.stale_predictions,
            "busy_s_total": self.busy_s_total,
            "per_executor": self.per_executor,
            "alloc": {proc: self.alloc[proc] for proc in sorted(self.alloc)},
        }


def partition_memory(device, gpu_count: int, cpu_count: int, cpu_mem_fraction: float = 0.4):
    """Per-executor memory by processor and the host-cache budget (engine.py:192-224)."""
    if gpu_count < 0 or cpu_count < 0 or gpu_count + cpu_count < 1:
        raise ConfigurationError(f"need at least one executor, got gpu={gpu_count} cpu={cpu_count}")
    per_exec: dict = {}
    if device.architecture != "numa":
        share = device.tier("device").capacity_bytes / (gpu_count + cpu_count)
        for proc, n in (("gpu", gpu_count), ("cpu", cpu_count)):
            if n:
                per_exec[proc] = share
        return per_exec, 0.0
    if gpu_count:
        per_exec["gpu"] = device.tier("device").capacity_bytes / gpu_count
    host_cap = device.tier("host").capacity_bytes
    cpu_total = host_cap * cpu_mem_fraction if cpu_count else 0.0
    if cpu_count:
        per_exec["cpu"] = cpu_total / cpu_count
    return per_exec, host_cap - cpu_total


def _min_inference(cost: CostModel, arches, proc: str):
    return max(cost.inference_memory(a, proc, 1) for a in arches)


def max_useful_expert_count(registry, device, proc: str, gpu_executors: int, cpu_executors: int,
                            cpu_mem_fraction: float = 0.4) -> int:
    """Largest resident-expert count worth sampling (engine.py:163-189)."""
    per_exec, _ = partition_memory(device, gpu_executors, cpu_executors, cpu_mem_fraction)
    if proc not in per_exec:
        raise ConfigurationError(f"no {proc} executors in this layout")
    arches = sorted({spec.arch for spec in registry.experts.values()})
    lanes = gpu_executors if proc == "gpu" else cpu_executors
    cap_bytes = (per_exec[proc] - _min_inference(CostModel(device), arches, proc)) * lanes
    running = 0
    for n, spec in enumerate(registry.experts_by_descending_prob(), start=1):
        running += spec.param_bytes
        if running >= cap_bytes:
            return n
    return len(registry.experts)


# ---------------------------------------------------------------------------
# configuration resolution (engine.py:357-548)


@dataclass
class ResolvedRun:
    """A fully resolved configuration, ready for the native planner."""

    config: RunConfig
    policy: PolicySpec
    cost: CostModel
    perf: PerfProfile
    alloc: dict
    window_results: dict
    executors: list          # [(proc, expert_budget, inference_budget, k_scale)]
    host_cache_budget: float
    expert_ids: list         # dense index -> expert id (lexicographic)
    arch_ids: list
    request_ids: list
    chains: list             # per request: list of dense expert indices
    arrivals: list


def _executor_counts(config: RunConfig, policy: PolicySpec):
    if policy.single_gpu and config.samba_gpu_only:
        return 1, 0
    return config.gpu_executors, config.cpu_executors


def _resolve_allocation(config, cost, perf, per_exec_mem, gpu_count, cpu_count, window_results) -> dict:
    registry = config.registry
    desc = registry.experts_by_descending_prob()
    prefix = [0]
    for spec in desc:
        prefix.append(prefix[-1] + spec.param_bytes)
    largest = max(spec.param_bytes for spec in desc)
    arches = sorted({spec.arch for spec in registry.experts.values()})
    lanes = {"gpu": gpu_count, "cpu": cpu_count}
    overrides = dict(config.alloc_override or {})
    alloc = {}
    for proc in sorted(per_exec_mem):
        mem = per_exec_mem[proc]
        min_inf = _min_inference(cost, arches, proc)
        if mem < largest + min_inf:
            raise MemoryStarvationError(
                f"{proc} executor memory {mem:.0f} cannot hold the largest expert ({largest} bytes) plus "
                f"a single-item batch ({min_inf:.0f} bytes); reduce the executor count")
        chosen = None
        if proc in overrides:
            chosen = max(1, min(int(overrides[proc]), len(desc)))
            budget = prefix[chosen] / lanes[proc]
        else:
            modes = {decide_allocation_mode(cost, perf, a, proc, mem, config.alloc_threshold) for a in arches}
            if ALLOC_WINDOW_SEARCH in modes and config.search_enabled:
                result = _window_search(config, perf, proc, gpu_count, cpu_count)
                window_results[proc] = result
                chosen = max(1, min(result.chosen, len(desc)))
                budget = prefix[chosen] / lanes[proc]
            else:
                budget = mem - max(cost.inference_memory(a, proc, perf.entry(a, proc).max_batch) for a in arches)
        # python min/max keep the int/float type of the winner (engine.py:453-454)
        budget = min(max(budget, largest), mem - min_inf)
        alloc[proc] = {"expert_budget_bytes": budget, "inference_budget_bytes": mem - budget,
                       "experts_chosen": chosen}
    return alloc


def _window_search(config, perf, proc, gpu_count, cpu_count) -> WindowSearchResult:
    sample = config.stream[: min(config.search_sample_requests, len(config.stream))]
    overrides = dict(config.alloc_override or {})

    def throughput_at(expert_count: int) -> float:
        probe = replace(config, stream=sample, seed=subseed(config.seed, "alloc-sample"),
                        alloc_override={**overrides, proc: expert_count}, search_enabled=False, perf=perf,
                        trace=False)
        return run(probe)[0].throughput_rps

    return decay_window_search(
        throughput_at,
        max_count=max_useful_expert_count(config.registry, config.device, proc, gpu_count, cpu_count,
                                          config.cpu_mem_fraction),
        initial_window=config.initial_window, error_margin=config.error_margin,
        fit_points=config.fit_points, seed=subseed(config.seed, "alloc", proc), choose=config.window_choose,
    )


def resolve(config: RunConfig) -> ResolvedRun:
    if config.policy not in POLICIES:
        raise ConfigurationError(f"unknown policy {config.policy!r}, available: {sorted(POLICIES)}")
    if not config.stream:
        raise ConfigurationError("request stream is empty")
    if config.contention_factor < 1.0:
        raise ConfigurationError("contention_factor must be >= 1")
    policy = POLICIES[config.policy]
    registry = config.registry
    cost = CostModel(config.device)
    gpu_count, cpu_count = _executor_counts(config, policy)
    per_exec_mem, host_budget = partition_memory(config.device, gpu_count, cpu_count, config.cpu_mem_fraction)
    perf = config.perf or build_perf_profile(registry, cost, per_exec_mem, config.plateau_threshold)
    window_results: dict = {}
    alloc = _resolve_allocation(config, cost, perf, per_exec_mem, gpu_count, cpu_count, window_results)
    executors = []
    for proc, n in (("gpu", gpu_count), ("cpu", cpu_count)):
        if n == 0:
            continue
        k_scale = config.contention_factor ** (n - 1)
        executors += [(proc, alloc[proc]["expert_budget_bytes"], alloc[proc]["inference_budget_bytes"], k_scale)] * n

    plans = {c: routing.route(c, registry.rules) for c in registry.rules}
    if config.routes:
        plans.update(config.routes)
    expert_ids = sorted(registry.experts)
    index = {eid: i for i, eid in enumerate(expert_ids)}
    # dict semantics of engine.py:385-387: first-occurrence order, last value wins
    by_id: dict = {}
    for req in config.stream:
        by_id[req.request_id] = req
    # per component type: the two concrete chains routing.resolve_chain can return (shared,
    # read-only lists), then one comparison per request (engine.py:721-725)
    forms = {}
    for comp, plan in plans.items():
        short = [index[eid] for eid in routing.resolve_chain(plan, float("inf"))]
        full = [index[eid] for eid in plan.experts] if len(plan.experts) > 1 else short
        forms[comp] = (full, short, plan.branch_prob, len(plan.experts) > 1)
    chains, arrivals = [], []
    for req in by_id.values():
        try:
            full, short, prob, branches = forms[req.component_type]
        except KeyError:
            raise KeyError(req.component_type) from None
        chains.append(full if (branches and req.detect_u < prob) else short)
        arrivals.append(req.arrival_time_s)
    return ResolvedRun(
        config=config, policy=policy, cost=cost, perf=perf, alloc=alloc, window_results=window_results,
        executors=executors, host_cache_budget=host_budget, expert_ids=expert_ids,
        arch_ids=sorted(registry.arch_classes), request_ids=list(by_id), chains=chains, arrivals=arrivals,
    )


# ---------------------------------------------------------------------------
# native planner


def _ptr(arr: np.ndarray, ctype):
    return arr.ctypes.data_as(ctypes.POINTER(ctype))


class Plan:
    """Owner of one native planner run and its outputs."""

    def __init__(self, resolved: ResolvedRun, record_trace: bool, record_ops: bool):
        self.resolved = resolved
        cfg = resolved.config
        registry = cfg.registry
        ids = resolved.expert_ids
        index = {eid: i for i, eid in enumerate(ids)}
        arch_index = {a: i for i, a in enumerate(resolved.arch_ids)}
        specs = [registry.experts[eid] for eid in ids]
        keep = {}  # arrays must outlive the create call
        keep["bytes"] = np.array([s.param_bytes for s in specs], dtype=np.int64)
        keep["usage"] = np.array([s.usage_prob for s in specs], dtype=np.float64)
        keep["arch"] = np.array([arch_index[s.arch] for s in specs], dtype=np.int32)
        ups = [sorted(index[u] for u in s.upstream) for s in specs]
        keep["up_off"] = np.cumsum([0] + [len(u) for u in ups]).astype(np.int32)
        keep["up_idx"] = np.array([u for lst in ups for u in lst] or [0], dtype=np.int32)
        keep["desc"] = np.array([index[s.expert_id] for s in registry.experts_by_descending_prob()], dtype=np.int32)
        na = len(resolved.arch_ids)
        pv = np.zeros(na * 2, np.uint8); pmb = np.zeros(na * 2, np.int32)
        pk = np.zeros(na * 2); pb = np.zeros(na * 2)
        cv = np.zeros(na * 2, np.uint8); ck = np.zeros(na * 2); cb = np.zeros(na * 2)
        cn = np.ones(na * 2, np.int64); cg = np.ones(na * 2); cbase = np.zeros(na * 2, np.int64)
        citem = np.zeros(na * 2, np.int64)
        for a, arch in enumerate(resolved.arch_ids):
            for p, proc in enumerate(_PROCS):
                i = a * 2 + p
                entry = resolved.perf.entries.get((arch, proc))
                if entry is not None:
                    pv[i], pmb[i], pk[i], pb[i] = 1, entry.max_batch, entry.k_s, entry.b_s
                c = cfg.device.exec_constants.get((arch, proc))
                if c is not None:
                    cv[i], ck[i], cb[i], cn[i], cg[i] = 1, c.k_s, c.b_s, c.n_sat, c.gamma
                    cbase[i], citem[i] = c.intermediate_base_bytes, c.intermediate_per_item_bytes
        keep.update(pv=pv, pmb=pmb, pk=pk, pb=pb, cv=cv, ck=ck, cb=cb, cn=cn, cg=cg, cbase=cbase, citem=citem)
        ex = resolved.executors
        keep["ex_proc"] = np.array([_PROCS.index(e[0]) for e in ex], np.int32)
        keep["ex_eb"] = np.array([float(e[1]) for e in ex], np.float64)
        keep["ex_ib"] = np.array([float(e[2]) for e in ex], np.float64)
        keep["ex_ks"] = np.array([float(e[3]) for e in ex], np.float64)
        keep["req"] = np.array(resolved.request_ids, np.int64)
        keep["arr"] = np.array(resolved.arrivals, np.float64)
        lens = np.fromiter(map(len, resolved.chains), np.int32, len(resolved.chains))
        keep["ch_off"] = np.concatenate([[0], np.cumsum(lens)]).astype(np.int32)
        keep["ch_exp"] = np.fromiter(itertools.chain.from_iterable(resolved.chains), np.int32, int(lens.sum()))

        device = cfg.device
        numa = device.architecture == "numa"
        host = device.tier("host") if numa else None
        ssd = device.tier("ssd")
        c = _native.PlanConfig()
        c.num_experts = len(ids)
        c.expert_bytes = _ptr(keep["bytes"], ctypes.c_int64)
        c.usage_prob = _ptr(keep["usage"], ctypes.c_double)
        c.expert_arch = _ptr(keep["arch"], ctypes.c_int32)
        c.upstream_offsets = _ptr(keep["up_off"], ctypes.c_int32)
        c.upstream_index = _ptr(keep["up_idx"], ctypes.c_int32)
        c.desc_order = _ptr(keep["desc"], ctypes.c_int32)
        c.num_arches = na
        c.perf_valid = _ptr(pv, ctypes.c_uint8)
        c.perf_max_batch = _ptr(pmb, ctypes.c_int32)
        c.perf_k = _ptr(pk, ctypes.c_double)
        c.perf_b = _ptr(pb, ctypes.c_double)
        c.cost_valid = _ptr(cv, ctypes.c_uint8)
        c.cost_k = _ptr(ck, ctypes.c_double)
        c.cost_b = _ptr(cb, ctypes.c_double)
        c.cost_n_sat = _ptr(cn, ctypes.c_int64)
        c.cost_gamma = _ptr(cg, ctypes.c_double)
        c.cost_base_bytes = _ptr(cbase, ctypes.c_int64)
        c.cost_per_item_bytes = _ptr(citem, ctypes.c_int64)
        c.numa = 1 if numa else 0
        c.host_bw = host.read_bandwidth_bytes_per_s if host else 1.0
        c.host_overhead = host.fixed_load_overhead_s if host else 0.0
        c.ssd_bw = ssd.read_bandwidth_bytes_per_s
        c.ssd_overhead = ssd.fixed_load_overhead_s
        c.host_mode = _HOST_CODE[resolved.policy.host_mode] if numa else -1
        c.host_cache_budget = float(resolved.host_cache_budget)
        c.num_executors = len(ex)
        c.exec_proc = _ptr(keep["ex_proc"], ctypes.c_int32)
        c.exec_expert_budget = _ptr(keep["ex_eb"], ctypes.c_double)
        c.exec_inference_budget = _ptr(keep["ex_ib"], ctypes.c_double)
        c.exec_k_scale = _ptr(keep["ex_ks"], ctypes.c_double)
        c.assign_makespan = 1 if resolved.policy.assign == "makespan" else 0
        c.arrange = 1 if resolved.policy.arrange else 0
        c.evict = _EVICT_CODE[resolved.policy.evict]
        c.num_requests = len(resolved.request_ids)
        c.request_id = _ptr(keep["req"], ctypes.c_int64)
        c.arrival_s = _ptr(keep["arr"], ctypes.c_double)
        c.chain_offsets = _ptr(keep["ch_off"], ctypes.c_int32)
        c.chain_experts = _ptr(keep["ch_exp"], ctypes.c_int32)
        c.record_trace = 1 if record_trace else 0
        c.record_ops = 1 if record_ops else 0
        peer = cfg.peer_tier
        if peer is not None:
            bw, ovh = float(peer["read_bandwidth_bytes_per_s"]), float(peer["fixed_load_overhead_s"])
            if not bw > 0 or ovh < 0:
                raise ConfigurationError("peer_tier needs a positive bandwidth and a non-negative overhead")
            c.peer_enabled, c.peer_bw, c.peer_overhead = 1, bw, ovh

        self.lib = _native.planner_lib()
        self.handle = ctypes.c_void_p()
        _check(self.lib, self.lib.coe_plan_create(ctypes.byref(c), ctypes.byref(self.handle)))

    def run(self) -> "Plan":
        _check(self.lib, self.lib.coe_plan_run(self.handle))
        return self

    def __del__(self):
        handle = getattr(self, "handle", None)
        if handle:
            self.lib.coe_plan_destroy(handle)
            self.handle = None

    # -- outputs ----------------------------------------------------------
    def raw_metrics(self) -> _native.PlanMetrics:
        m = _native.PlanMetrics()
        self.lib.coe_plan_metrics_get(self.handle, ctypes.byref(m))
        return m

    def executor_stats(self):
        n = len(self.resolved.executors)
        busy = (ctypes.c_double * n)()
        switches = (ctypes.c_int64 * n)()
        self.lib.coe_plan_executor_stats(self.handle, busy, switches)
        return list(busy), list(switches)

    def trace_arrays(self):
        n = self.lib.coe_plan_trace_len(self.handle)
        t = np.empty(n, np.float64); ex = np.empty(n, np.int32); ev = np.empty(n, np.int32)
        exp = np.empty(n, np.int32); req = np.empty(n, np.int64)
        if n:
            self.lib.coe_plan_trace(self.handle, t.ctypes.data, ex.ctypes.data, ev.ctypes.data,
                                    exp.ctypes.data, req.ctypes.data)
        return t, ex, ev, exp, req

    def trace(self) -> list:
        t, ex, ev, exp, req = self.trace_arrays()
        ids = self.resolved.expert_ids
        names = _native.EVENT_NAMES
        out = []
        for i in range(len(t)):
            x, e, r = int(ex[i]), int(exp[i]), int(req[i])
            out.append({"time_s": float(t[i]), "executor": None if x < 0 else x, "event": names[ev[i]],
                        "expert_id": None if e < 0 else ids[e], "request_id": None if r < 0 else r})
        return out

    def initial_residency(self) -> list:
        n = len(self.resolved.executors)
        off = np.zeros(n + 1, np.int32)
        exp = np.zeros(max(1, len(self.resolved.expert_ids) * n), np.int32)
        _check(self.lib, self.lib.coe_plan_initial_residency(self.handle, off.ctypes.data, exp.ctypes.data))
        return [exp[off[i]:off[i + 1]].tolist() for i in range(n)]

    def ops(self) -> np.ndarray:
        n = self.lib.coe_plan_num_ops(self.handle)
        if n == 0:
            return np.zeros(0, dtype=_OP_DTYPE)
        buf = ctypes.cast(self.lib.coe_plan_ops(self.handle), ctypes.POINTER(ctypes.c_byte * (n * _OP_DTYPE.itemsize)))
        return np.frombuffer(bytes(buf.contents), dtype=_OP_DTYPE)

    def op_args(self) -> np.ndarray:
        n = self.lib.coe_plan_num_op_args(self.handle)
        if n == 0:
            return np.zeros(0, np.int32)
        return np.ctypeslib.as_array(self.lib.coe_plan_op_args(self.handle), shape=(n,)).copy()

    def admissions(self) -> np.ndarray:
        n = self.lib.coe_plan_num_admissions(self.handle)
        if n == 0:
            return np.zeros(0, dtype=_ADM_DTYPE)
        buf = ctypes.cast(self.lib.coe_plan_admissions(self.handle),
                          ctypes.POINTER(ctypes.c_byte * (n * _ADM_DTYPE.itemsize)))
        return np.frombuffer(bytes(buf.contents), dtype=_ADM_DTYPE)


_OP_DTYPE = np.dtype([("executor", np.int32), ("kind", np.int32), ("expert", np.int32), ("count", np.int32),
                      ("offset", np.int64), ("time_s", np.float64), ("tier", np.int32), ("seq", np.int32)])
_ADM_DTYPE = np.dtype([("executor", np.int32), ("run_rank", np.int32), ("request", np.int32),
                       ("stage", np.int32)])
assert _OP_DTYPE.itemsize == ctypes.sizeof(_native.Op)
assert _ADM_DTYPE.itemsize == ctypes.sizeof(_native.Admission)


def _check(lib, code: int) -> None:
    if code == _native.COE_OK:
        return
    message = lib.coe_plan_last_error().decode("utf-8", "replace")
    if code == _native.COE_ERR_CONFIG:
        raise ConfigurationError(message)
    if code == _native.COE_ERR_STARVATION:
        raise MemoryStarvationError(message)
    if code == _native.COE_ERR_VALUE:
        raise ValueError(message)
    raise RuntimeError(message)


def metrics_from_plan(plan: Plan) -> Metrics:
    resolved = plan.resolved
    raw = plan.raw_metrics()
    busy, switches = plan.executor_stats()
    makespan = raw.makespan_s
    completed = int(raw.completed)
    per_executor = [
        {"executor": i, "proc": proc, "busy_s": busy[i],
         "busy_fraction": busy[i] / makespan if makespan > 0 else 0.0, "switches": int(switches[i])}
        for i, (proc, *_rest) in enumerate(resolved.executors)
    ]
    return Metrics(
        policy=resolved.config.policy, seed=resolved.config.seed, completed_requests=completed,
        follow_ups=int(raw.follow_ups), makespan_s=makespan,
        throughput_rps=completed / makespan if makespan > 0 else 0.0,
        expert_switches=sum(int(s) for s in switches), evictions=int(raw.evictions),
        stale_predictions=int(raw.stale_predictions), per_executor=per_executor, alloc=resolved.alloc,
        busy_s_total=sum(busy), sched_wall_s=raw.sched_wall_s, sched_calls=int(raw.sched_calls),
    )


def plan(config: RunConfig, record_ops: bool = True) -> Plan:
    """Resolve ``config`` and run the native planner; the result carries the op log."""
    return Plan(resolve(config), record_trace=config.trace, record_ops=record_ops).run()


def run(config: RunConfig):
    """Plan one configuration to completion: ``(Metrics, trace)`` (engine.py:827-829)."""
    p = Plan(resolve(config), record_trace=config.trace, record_ops=False).run()
    return metrics_from_plan(p), (p.trace() if config.trace else [])


def metrics_json(metrics: Metrics) -> str:
    return json.dumps(metrics.to_doc(), sort_keys=True, indent=2) + "\n"


def trace_jsonl(trace: list) -> str:
    lines = [json.dumps(rec, sort_keys=True, separators=(",", ":")) for rec in trace]
    return "".join(line + "\n" for line in lines)
