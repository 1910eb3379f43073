"""Generate the five BASELINE.json configurations as committed documents.

Run HERE (build container): the registry/stream generators of the reference
(``coesim.workload``, out of scope per SURVEY §2 -- "use its documents as-is")
are imported from ``/root/reference/pkg/src``; N-stage and heterogeneous
registries (configs 2 and 5) are built by this script.  Output goes to
``paper_2503_02354_b200/data/configs/<name>/`` and travels with the repo, so
the GPU box never needs the reference.

    python tools/make_configs.py

Device documents use the B200 constants in ``data/b200_exec.json`` (written
by ``tools/hwprofile.py`` from measured K3 timings; roofline estimates until
then).
"""

from __future__ import annotations

import gzip
import json
import math
import os
import random
import sys

REF = "/root/reference/pkg/src"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "paper_2503_02354_b200", "data", "configs")
sys.path.insert(0, REF)

from coesim import workload  # noqa: E402  (reference generator, input producer only)
from coesim.types import ArchClass, ExpertSpec, ModelRegistry, RoutingRule  # noqa: E402

sys.path.insert(0, ROOT)
from paper_2503_02354_b200 import configs as cfgmod  # noqa: E402


def write(path, doc, gz=False):
    os.makedirs(os.path.dirname(path), exist_ok=True)
    text = json.dumps(doc, sort_keys=True, separators=(",", ":") if gz else None, indent=None if gz else 1)
    if gz:
        with open(path, "wb") as raw, gzip.GzipFile(fileobj=raw, mode="wb", compresslevel=9, mtime=0) as fh:
            fh.write(text.encode("utf-8"))
    else:
        with open(path, "w") as fh:
            fh.write(text + "\n")


def stage_chain_registry(stage_sizes, arch_of, bytes_of, seed, arch_kinds):
    """N-stage DAG: stage-k expert -> one stage-(k+1) 'next' expert; every
    stage-(k+1) expert gets >= 1 upstream.  Components map 1:1 to stage-0
    experts with a uniform mix; chains follow the next pointers."""
    rng = random.Random(seed)
    stages = []
    for k, size in enumerate(stage_sizes):
        stages.append([f"s{k}-{i:03d}" for i in range(size)])
    nxt = {}
    for k in range(len(stages) - 1):
        src, dst = stages[k], list(stages[k + 1])
        rng.shuffle(dst)
        for i, eid in enumerate(src):
            nxt[eid] = dst[i % len(dst)] if i < len(dst) else rng.choice(dst)
    ups = {}
    for a, b in nxt.items():
        ups.setdefault(b, set()).add(a)
    comps = [f"c{i:03d}" for i in range(len(stages[0]))]
    mix = {c: 1.0 / len(comps) for c in comps}
    routes, invocations = {}, {}
    per_request = 0.0
    for c, first in zip(comps, stages[0]):
        chain = [first]
        while chain[-1] in nxt:
            chain.append(nxt[chain[-1]])
        routes[c] = {"experts": chain, "branch_prob": 1.0}
        for e in chain:
            invocations[e] = invocations.get(e, 0.0) + mix[c]
            per_request += mix[c]
    experts = {}
    for k, ids in enumerate(stages):
        for eid in ids:
            if k > 0 and eid not in ups:
                continue  # never routed to
            experts[eid] = ExpertSpec(expert_id=eid, arch=arch_of(eid), param_bytes=bytes_of(eid),
                                      upstream=frozenset(ups.get(eid, ())),
                                      usage_prob=invocations.get(eid, 0.0) / per_request)
    rules = {}
    for c, first in zip(comps, stages[0]):
        chain = routes[c]["experts"]
        rules[c] = RoutingRule(component_type=c, classification_expert_id=first,
                               detection_expert_id=chain[1] if len(chain) > 1 else None,
                               detection_prob=1.0 if len(chain) > 1 else 0.0)
    arches = {a: ArchClass(id=a, kind=kind) for a, kind in arch_kinds.items()}
    reg = ModelRegistry(arch_classes=arches, experts=experts, rules=rules, component_mix=mix)
    reg.validate()
    return reg, routes


def main():
    exec_table = cfgmod.load_exec_table()
    made = {}

    # C1: 16 small MLP experts, 2-stage
    shapes = {"cls-r101": (1024, 4096, 64), "det-y5": (1024, 4096, 64)}
    reg = workload.generate_registry(num_components=12, num_detection_experts=4, detection_coverage=1.0,
                                     zipf_s=1.0, expert_bytes=cfgmod.expert_bytes(1024, 4096), seed=0)
    made["c1"] = (reg, None, shapes, {"alloc_override": None}, "16 MLP experts d=1024 h=4096, 2-stage, resident")

    # C2: 64 experts, 3-stage chains, uniform, all resident
    d, h = 2048, 8192
    reg, routes = stage_chain_registry([22, 21, 21], lambda e: "mlp-2048x8192", lambda e: cfgmod.expert_bytes(d, h),
                                       seed=2, arch_kinds={"mlp-2048x8192": "classification"})
    made["c2"] = (reg, routes, {"mlp-2048x8192": (d, h, 128)}, {"alloc_override": None},
                  "64 MLP experts d=2048 h=8192, 3-stage chains, uniform, resident")

    # C3: 300-expert board-shaped CoE, 60 GB, 12 GB HBM expert budget
    d, h = 4096, 12288
    shapes = {"cls-r101": (d, h, 256), "det-y5": (d, h, 256)}
    reg = workload.generate_registry(num_components=280, num_detection_experts=20, detection_coverage=0.5,
                                     zipf_s=0.6, expert_bytes=cfgmod.expert_bytes(d, h), seed=0)
    made["c3"] = (reg, None, shapes, {"alloc_override": {"gpu": 59}},
                  "300 MLP experts d=4096 h=12288 (60.4 GB), 12 GB expert budget (59 resident), zipf 0.6")

    # C4: C3 with Zipf 1.0 routing across 1/2/4/8 GPUs, 12 GB per GPU
    reg = workload.generate_registry(num_components=280, num_detection_experts=20, detection_coverage=0.5,
                                     zipf_s=1.0, expert_bytes=cfgmod.expert_bytes(d, h), seed=0)
    made["c4"] = (reg, None, shapes, {"alloc_override": {"gpu": 59}},
                  "C3 with zipf 1.0 routing; 12 GB expert budget per GPU; 1/2/4/8 GPUs")

    # C5: heterogeneous 8M-1B params, 5-stage chains, full residency.  A request's activation
    # width d is constant along its chain (each chain draws d, each expert draws h = {4,8,16}*d,
    # capped at 61440), so stages hand T x d activations to each other without re-projection.
    rng = random.Random(5)
    d_choices, d_weights = (1024, 2048, 4096, 8192), (0.3, 0.3, 0.25, 0.15)
    sizes = [60, 60, 60, 60, 60]
    chain_d = [rng.choices(d_choices, weights=d_weights)[0] for _ in range(sizes[0])]
    # next pointers are a permutation per stage (stage_chain_registry, seed 55), so derive each
    # expert's chain from the routes after building, then assign shapes
    reg, routes = stage_chain_registry(sizes, lambda e: "tmp", lambda e: 1, seed=55,
                                       arch_kinds={"tmp": "classification"})
    arch_of_expert, bytes_of = {}, {}
    for comp, route in sorted(routes.items()):
        d = chain_d[int(comp[1:])]
        for eid in route["experts"]:
            h = min(rng.choice((4, 8, 16)) * d, 61440)
            arch_of_expert[eid] = f"mlp-{d}x{h}"
            bytes_of[eid] = cfgmod.expert_bytes(d, h)
    arch_kinds = {a: "classification" for a in set(arch_of_expert.values())}
    reg, routes = stage_chain_registry(sizes, lambda e: arch_of_expert[e], lambda e: bytes_of[e], seed=55,
                                       arch_kinds=arch_kinds)
    shape_of = {a: (int(a[4:].split("x")[0]), int(a.split("x")[1]), 64) for a in arch_kinds}
    made["c5"] = (reg, routes, shape_of, {"alloc_override": None},
                  "300 heterogeneous MLP experts (8M-1B params, 11 shapes, d constant per chain), "
                  "5-stage chains, full residency")

    for name, (reg, routes, shapes, run, desc) in made.items():
        base = os.path.join(OUT, name)
        write(os.path.join(base, "registry.json"), reg.to_doc())
        for n in (1000, 10000):
            stream = workload.generate_stream(reg, n, interarrival_s=1e-6, seed=0)
            write(os.path.join(base, f"stream_{n}.json.gz"), workload.stream_to_doc(stream), gz=True)
        if routes:
            write(os.path.join(base, "routes.json"), routes)
        write(os.path.join(base, "config.json"), {
            "name": name, "description": desc,
            "shapes": {a: {"d": s[0], "h": s[1], "T": s[2]} for a, s in sorted(shapes.items())},
            "run": dict({"policy": "coserve", "gpu_executors": 1, "cpu_executors": 0, "contention_factor": 1.0,
                         "search_enabled": False}, **run),
        })
        write(os.path.join(base, "device.json"), cfgmod.device_doc(shapes, exec_table))
        print(name, len(reg.experts), "experts", sum(s.param_bytes for s in reg.experts.values()) / 1e9, "GB")


if __name__ == "__main__":
    main()
