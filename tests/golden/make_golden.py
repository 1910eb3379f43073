"""Generate golden traces / metrics by running the UNMODIFIED reference.

Run in the build container (needs ``/root/reference``):

    python tests/golden/make_golden.py

For every case it imports ``coesim`` from ``/root/reference/pkg/src``, runs
``engine.Simulation`` on the committed documents and freezes
``metrics_json`` and ``trace_jsonl`` (engine.py:832-838).  N-stage cases
(configs 2 and 5) use a one-method subclass overriding ``_on_arrival``
(engine.py:720-727) so the tail of a route template is taken iff
``detect_u < branch_prob`` -- SURVEY §0.5.  Large runs store the SHA-256 of
the trace instead of the full text.  Output: ``tests/golden/<case>.json.gz``.
"""

from __future__ import annotations

import gzip
import hashlib
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")

from coesim import engine, workload  # noqa: E402
from coesim.costmodel import CostModel, load_device_preset  # noqa: E402
from coesim.types import DeviceProfile, ModelRegistry  # noqa: E402

CONFIGS = os.path.join(ROOT, "paper_2503_02354_b200", "data", "configs")
FULL_TRACE_LIMIT = 12000
# nominal NVLink 5 peer copy: 900 GB/s per direction, ~80 % as copy-engine payload, 10 us setup
PEER_TIER = {"read_bandwidth_bytes_per_s": 720e9, "fixed_load_overhead_s": 1e-5}


def read(path):
    opener = gzip.open if path.endswith(".gz") else open
    with opener(path, "rt") as fh:
        return json.load(fh)


class NStage(engine.Simulation):
    """Reference engine with N-stage chain templates (only _on_arrival differs)."""

    routes_doc: dict = {}

    def _on_arrival(self, t, req):
        route = self.routes_doc.get(req.component_type)
        if route is None:
            return super()._on_arrival(t, req)
        experts = list(route["experts"])
        req.chain = experts if (len(experts) > 1 and req.detect_u < route["branch_prob"]) else experts[:1]
        self._record(t, None, "arrival", None, req.request_id)
        self._admit(t, req, follow_up=False)


class PeerCost(CostModel):
    """The reference cost model plus a 'peer' tier (an NVLink copy from another GPU's HBM)."""

    peer = (1.0, 0.0)  # (read_bandwidth_bytes_per_s, fixed_load_overhead_s)

    def load_latency_from(self, tier_name, nbytes):
        if tier_name == "peer":
            if nbytes <= 0:
                raise ValueError(f"load size must be positive, got {nbytes}")
            return nbytes / self.peer[0] + self.peer[1]
        return super().load_latency_from(tier_name, nbytes)


class PeerTier(NStage):
    """Reference engine with a peer-GPU swap-in tier.

    Extension semantics (the repo's RunConfig.peer_tier): a LOAD of an expert that some GPU
    executor holds in its pool -- and is not loading right now -- copies it over NVLink from the
    lowest-id such executor instead of from the host/ssd tier (engine.py:643-677 picks the source
    at load start, :579-586).  The scheduler's switch-cost predictions (_load_latency, used by
    _admit and _invalidate_prediction, engine.py:583-586) keep the reference's host/ssd tier: a
    peer copy is an opportunistic fast path.  (Quoting the peer latency to assign() as well makes
    the makespan rule replicate experts across GPUs and evict others: -6 % to -59 % throughput
    on these cases -- DESIGN.md §6b.)  Everything else is the unmodified reference.
    """

    def __init__(self, config):
        super().__init__(config)
        self.cost = PeerCost(config.device)
        self._loading = {}

    def _peer_source(self, expert_id):
        for ex in self.executors:
            if ex.proc == "gpu" and ex.pool.has(expert_id) and self._loading.get(ex.id) != expert_id:
                return ex.id
        return None

    def _source_tier(self, expert_id):
        if self._peer_source(expert_id) is not None:
            return "peer"
        return super()._source_tier(expert_id)

    def _load_latency(self, expert_id):
        spec = self.registry.experts[expert_id]
        return self.cost.load_latency_from(super()._source_tier(expert_id), spec.param_bytes)

    def _start_load(self, t, ex, run_entries, spec):
        super()._start_load(t, ex, run_entries, spec)
        self._loading[ex.id] = spec.expert_id

    def _on_load_done(self, t, ex):
        self._loading.pop(ex.id, None)
        super()._on_load_done(t, ex)


def run_case(registry_doc, device_doc, stream_doc, routes_doc, run):
    registry = ModelRegistry.from_doc(registry_doc)
    device = DeviceProfile.from_doc(device_doc)
    stream = workload.stream_from_doc(stream_doc)
    run = dict(run)
    peer = run.pop("peer_tier", None)
    cfg = engine.RunConfig(registry=registry, device=device, stream=stream, trace=True, **run)
    sim_cls = NStage if routes_doc else engine.Simulation
    if peer is not None:
        sim_cls = PeerTier
        PeerCost.peer = (float(peer["read_bandwidth_bytes_per_s"]), float(peer["fixed_load_overhead_s"]))
    NStage.routes_doc = routes_doc or {}
    metrics, trace = sim_cls(cfg).run()
    return engine.metrics_json(metrics), engine.trace_jsonl(trace)


def config_case(name, requests, **run_overrides):
    base = os.path.join(CONFIGS, name)
    cfg = read(os.path.join(base, "config.json"))
    routes_path = os.path.join(base, "routes.json")
    routes = read(routes_path) if os.path.exists(routes_path) else None
    run = dict(cfg["run"])
    run.update(run_overrides)
    if run.get("alloc_override") is None:
        run.pop("alloc_override", None)
    inputs = {"config": name, "requests": requests, "run": run}
    docs = (read(os.path.join(base, "registry.json")), read(os.path.join(base, "device.json")),
            read(os.path.join(base, f"stream_{requests}.json.gz")), routes)
    return inputs, docs


def inline_case(device_name, components, requests, interarrival, gen_seed, **run):
    reg = workload.generate_registry(num_components=components, seed=gen_seed)
    stream = workload.generate_stream(reg, requests, interarrival_s=interarrival, seed=gen_seed)
    docs = (reg.to_doc(), load_device_preset(device_name).to_doc(), workload.stream_to_doc(stream), None)
    inputs = {"registry": docs[0], "device": docs[1], "stream": docs[2], "run": dict(run)}
    return inputs, docs


def cases():
    out = {}
    out["c1_1k"] = config_case("c1", 1000)
    out["c2_1k"] = config_case("c2", 1000)
    out["c3_1k"] = config_case("c3", 1000)
    out["c3_1k_samba_lru"] = config_case("c3", 1000, policy="samba_lru")
    out["c3_1k_samba_fifo"] = config_case("c3", 1000, policy="samba_fifo")
    out["c4_1k_g2"] = config_case("c4", 1000, gpu_executors=2)
    out["c4_1k_g4"] = config_case("c4", 1000, gpu_executors=4)
    out["c4_1k_g8"] = config_case("c4", 1000, gpu_executors=8)
    out["c5_1k_g8"] = config_case("c5", 1000, gpu_executors=8)
    out["c2_10k"] = config_case("c2", 10000)
    out["c3_10k"] = config_case("c3", 10000)
    out["c1_10k"] = config_case("c1", 10000)
    out["c4_10k_g2"] = config_case("c4", 10000, gpu_executors=2)
    out["c4_10k_g8"] = config_case("c4", 10000, gpu_executors=8)
    # the multi-GPU configurations as benched: 12 GB per GPU (override scales with the GPU count)
    for n in (2, 4, 8):
        out[f"c4_10k_g{n}_pergpu"] = config_case("c4", 10000, gpu_executors=n, alloc_override={"gpu": 59 * n})
        out[f"c3_10k_g{n}_pergpu"] = config_case("c3", 10000, gpu_executors=n, alloc_override={"gpu": 59 * n})
    out["c5_10k_g8"] = config_case("c5", 10000, gpu_executors=8)
    # (f3) peer-GPU swap-in tier: NVLink 5 copies from another GPU's HBM (PEER_TIER, nominal)
    for n in (2, 4):
        out[f"c3_10k_g{n}_pergpu_peer"] = config_case("c3", 10000, gpu_executors=n, alloc_override={"gpu": 59 * n},
                                                       peer_tier=PEER_TIER)
        out[f"c4_10k_g{n}_pergpu_peer"] = config_case("c4", 10000, gpu_executors=n, alloc_override={"gpu": 59 * n},
                                                       peer_tier=PEER_TIER)
    out["c4_1k_g2_peer"] = config_case("c4", 1000, gpu_executors=2, peer_tier=PEER_TIER)
    out["c5_1k_g8_peer"] = config_case("c5", 1000, gpu_executors=8, peer_tier=PEER_TIER)
    for policy in ("coserve", "coserve_em_ra", "coserve_em", "coserve_none", "samba_lru", "samba_fifo",
                   "samba_parallel"):
        out[f"numa_a80_{policy}"] = inline_case("numa-3080ti", 80, 300, 0.004, 3, policy=policy, seed=3,
                                                gpu_executors=3, cpu_executors=1, search_enabled=False)
    out["numa_a80_coserve_search"] = inline_case("numa-3080ti", 80, 300, 0.004, 4, policy="coserve", seed=4,
                                                 gpu_executors=2, cpu_executors=1, search_enabled=True,
                                                 search_sample_requests=150)
    out["uma_a40_coserve"] = inline_case("uma-m2", 40, 200, 0.004, 7, policy="coserve", seed=7,
                                         gpu_executors=2, cpu_executors=1, search_enabled=False)
    out["uma_a40_samba_fifo"] = inline_case("uma-m2", 40, 200, 0.004, 7, policy="samba_fifo", seed=7,
                                            gpu_executors=2, cpu_executors=1, search_enabled=False)
    return out


def main(only=None):
    for name, (inputs, docs) in cases().items():
        if only and name not in only:
            continue
        metrics_text, trace_text = run_case(*docs, inputs["run"])
        doc = {"name": name, "inputs": inputs, "metrics_json": metrics_text,
               "trace_sha256": hashlib.sha256(trace_text.encode()).hexdigest(),
               "trace_lines": trace_text.count("\n")}
        if doc["trace_lines"] <= FULL_TRACE_LIMIT:
            doc["trace_jsonl"] = trace_text
        path = os.path.join(HERE, f"{name}.json.gz")
        with open(path, "wb") as raw, gzip.GzipFile(fileobj=raw, mode="wb", compresslevel=9, mtime=0) as fh:
            fh.write(json.dumps(doc, sort_keys=True).encode("utf-8"))
        print(f"{name}: {doc['trace_lines']} trace lines, {os.path.getsize(path) / 1024:.0f} KiB")


if __name__ == "__main__":
    main(sys.argv[1:] or None)
