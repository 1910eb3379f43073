"""The five BASELINE.json configurations and the shared B200 device document.

Each configuration lives in ``data/configs/<name>/`` (generated once by
``tools/make_configs.py`` and committed): ``registry.json``,
``stream_<n>.json.gz``, optional N-stage ``routes.json``, ``device.json`` (the
device document *both* the planner and the oracle read -- SURVEY §7 step 7)
and ``config.json`` (expert MLP shapes per arch and the RunConfig knobs).

Shapes: an expert of arch ``a`` is a 2-layer MLP ``Y = gelu(X W1^T) W2^T``
with ``W1: [h, d]``, ``W2: [d, h]`` bf16; a request carries ``T`` rows of
``d`` features.  ``param_bytes = 2*d*h*2``.
"""

from __future__ import annotations

import gzip
import json
import os
from dataclasses import dataclass

from .routing import RoutePlan
from .types import DeviceProfile, ModelRegistry, Request

DATA = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data")
CONFIG_DIR = os.path.join(DATA, "configs")
EXEC_TABLE = os.path.join(DATA, "b200_exec.json")
NAMES = ("c1", "c2", "c3", "c4", "c5")


# B200 memory tiers (measured on the pool: pinned H2D 55.6 GB/s, gpurun_out/probe_box.json);
# the host tier holds every expert, so swap-ins are always host-tier DMA.
TIERS = (
    {"tier": "device", "capacity_bytes": 180_000_000_000, "read_bandwidth_bytes_per_s": 6.5e12,
     "fixed_load_overhead_s": 0.0},
    {"tier": "host", "capacity_bytes": 160_000_000_000, "read_bandwidth_bytes_per_s": 55.5e9,
     "fixed_load_overhead_s": 2e-5},
    {"tier": "ssd", "capacity_bytes": 0, "read_bandwidth_bytes_per_s": 7e9, "fixed_load_overhead_s": 1e-4},
)


def expert_bytes(d: int, h: int) -> int:
    return 2 * d * h * 2


def shape_key(d: int, h: int, T: int) -> str:
    return f"{d}x{h}x{T}"


def estimate_exec(d: int, h: int, T: int) -> dict:
    """Roofline estimate (1.2 PFLOP/s per row block, weights at 5.5 TB/s + 8 us launch)."""
    return {"k_s": 4.0 * T * d * h / 1.2e15, "b_s": 4.0 * d * h / 5.5e12 + 8e-6, "source": "estimate"}


def load_exec_table() -> dict:
    """Measured per-shape constants (tools/hwprofile.py on a B200), keyed by shape."""
    if os.path.exists(EXEC_TABLE):
        with open(EXEC_TABLE) as fh:
            return json.load(fh)
    return {}


def tiers(table: dict) -> list:
    """Memory tiers; the host tier's bandwidth/overhead are measured when available."""
    out = [dict(t) for t in TIERS]
    host = table.get("host_tier")
    if host:
        out[1]["read_bandwidth_bytes_per_s"] = float(host["read_bandwidth_bytes_per_s"])
        out[1]["fixed_load_overhead_s"] = float(host["fixed_load_overhead_s"])
    return out


def device_doc(shapes: dict, table: dict) -> dict:
    """Device document with one gpu exec-constant entry per arch (shape)."""
    consts = []
    measured = table.get("shapes", {})
    for arch, (d, h, T) in sorted(shapes.items()):
        entry = measured.get(shape_key(d, h, T)) or estimate_exec(d, h, T)
        consts.append({
            "arch": arch, "proc": "gpu", "k_s": float(entry["k_s"]), "b_s": float(entry["b_s"]),
            "n_sat": 1_000_000, "gamma": 1.0, "intermediate_base_bytes": 0,
            "intermediate_per_item_bytes": T * (d + h) * 2,
        })
    return {"schema_version": 1, "name": "b200-hgx", "architecture": "numa", "tiers": tiers(table),
            "exec_constants": consts}


def _read(path: str):
    opener = gzip.open if path.endswith(".gz") else open
    with opener(path, "rt", encoding="utf-8") as fh:
        return json.load(fh)


@dataclass
class Workload:
    """A configuration's documents, decoded."""

    name: str
    registry: ModelRegistry
    device: DeviceProfile
    stream: list
    routes: dict | None
    shapes: dict          # arch -> (d, h, T)
    run: dict             # RunConfig keyword arguments
    docs: dict            # raw documents (for the oracle)
    description: str


def load(name: str, requests: int = 1000, gpu_executors: int | None = None) -> Workload:
    base = os.path.join(CONFIG_DIR, name)
    cfg = _read(os.path.join(base, "config.json"))
    reg_doc = _read(os.path.join(base, "registry.json"))
    dev_doc = _read(os.path.join(base, "device.json"))
    stream_doc = _read(os.path.join(base, f"stream_{requests}.json.gz"))
    routes_path = os.path.join(base, "routes.json")
    routes_doc = _read(routes_path) if os.path.exists(routes_path) else None
    stream = [Request(request_id=int(r["request_id"]), component_type=r["component_type"],
                      arrival_time_s=float(r["arrival_time_s"]), detect_u=float(r["detect_u"]))
              for r in stream_doc["requests"]]
    routes = None
    if routes_doc:
        routes = {c: RoutePlan(tuple(v["experts"]), float(v["branch_prob"])) for c, v in routes_doc.items()}
    run = dict(cfg["run"])
    if gpu_executors is not None:
        run["gpu_executors"] = gpu_executors
        # The reference's alloc_override counts experts for ALL gpu lanes of one device (its
        # lanes share that device's memory: budget = bytes of the top-k experts / lanes,
        # engine.py:436).  Here each executor is its own B200, so "12 GB per GPU" at N GPUs
        # is an override of N x the single-GPU count.
        ov = run.get("alloc_override")
        if ov and "gpu" in ov and gpu_executors > 1:
            run["alloc_override"] = dict(ov, gpu=int(ov["gpu"]) * gpu_executors)
    if run.get("alloc_override") is None:
        run.pop("alloc_override", None)
    return Workload(
        name=name, registry=ModelRegistry.from_doc(reg_doc), device=DeviceProfile.from_doc(dev_doc), stream=stream,
        routes=routes, shapes={a: (s["d"], s["h"], s["T"]) for a, s in cfg["shapes"].items()}, run=run,
        docs={"registry": reg_doc, "device": dev_doc, "stream": stream_doc, "routes": routes_doc},
        description=cfg["description"],
    )


def run_config(w: Workload, **overrides):
    """A ``RunConfig`` for this workload (planner-ready)."""
    from .engine import RunConfig

    kwargs = dict(registry=w.registry, device=w.device, stream=w.stream, routes=w.routes)
    kwargs.update(w.run)
    kwargs.update(overrides)
    return RunConfig(**kwargs)
