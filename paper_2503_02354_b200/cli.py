"""Command-line driver, compatible with the reference's ``coesim`` CLI (cli.py:383-476).

    python -m paper_2503_02354_b200.cli <command> ...

Commands (same names, document formats and exit codes as the reference -- 0 ok, 2
configuration / schema / file problems, 3 a run that fails, cli.py:36-38):

* ``gen-workload``  -- write a committed configuration's registry / stream / device (and
  N-stage routes) documents (the generator itself is the reference's: the
  documents under data/configs were made with it);
* ``profile``       -- ``perf_profile.json`` for a device document (profiler.py:177-216);
  ``--measure`` first re-measures the B200 exec / swap constants on this GPU
  (``profiler.measure_b200_device``) and writes the device document they imply;
* ``search-memory`` -- the decay-window allocation search (profiler.py:281-419) on the
  virtual clock, or ``--measured`` on real B200 serving probes;
* ``simulate``      -- one policy: metrics JSON (and a JSONL trace) byte-identical to the
  reference's; ``--execute`` also serves the plan on the GPU and adds the measured
  requests/s (device-timed) under ``"b200"`` on stderr-free stdout;
* ``compare``       -- several policies with the reference's table (xLRU, sw-red, ovh
  columns, cli.py:306-380); ``--execute`` adds measured B200 requests/s per policy.

Workloads come from ``--config c1..c5`` (committed documents, ``--requests`` 1000 or
10000) or from ``--registry``/``--stream``/``--device`` files.
"""

from __future__ import annotations

import argparse
import csv
import gzip
import json
import statistics
import sys
from pathlib import Path

from . import configs, engine, profiler
from .costmodel import PRESET_NAMES, CostModel, load_device_preset
from .engine import POLICIES
from .routing import RoutePlan
from .types import (ConfigurationError, DeviceProfile, MemoryStarvationError, ModelRegistry, Request,
                    SchemaError)

EXIT_OK, EXIT_CONFIG, EXIT_SIM = 0, 2, 3
DEFAULT_POLICIES = ["coserve", "samba_parallel", "samba_lru", "samba_fifo"]
ABLATION_POLICIES = ["coserve", "coserve_em_ra", "coserve_em", "coserve_none", "samba_lru"]


def _read_json(path) -> dict:
    path = Path(path)
    if not path.exists():
        raise ConfigurationError(f"{path} does not exist")
    opener = gzip.open if str(path).endswith(".gz") else open
    try:
        with opener(path, "rt") as fh:
            return json.load(fh)
    except json.JSONDecodeError as exc:
        raise SchemaError(f"{path} is not valid JSON: {exc}") from exc


def _write_json(path, doc: dict) -> None:
    Path(path).write_text(json.dumps(doc, sort_keys=True, indent=2) + "\n")


def _load_device(name_or_path: str) -> DeviceProfile:
    if name_or_path in PRESET_NAMES:
        return load_device_preset(name_or_path)
    return DeviceProfile.from_doc(_read_json(name_or_path))


def _stream_from_doc(doc: dict) -> list:
    if doc.get("schema_version") != 1 or "requests" not in doc:
        raise SchemaError("stream document needs schema_version 1 and requests")
    return [Request(request_id=int(r["request_id"]), component_type=r["component_type"],
                    arrival_time_s=float(r["arrival_time_s"]), detect_u=float(r["detect_u"]))
            for r in doc["requests"]]


class _Work:
    """A workload from --config or from document files."""

    def __init__(self, args):
        self.shapes = None
        self.name = None
        if getattr(args, "config", None):
            w = configs.load(args.config, args.requests, gpu_executors=args.gpu_executors)
            self.name, self.registry, self.device, self.stream = w.name, w.registry, w.device, w.stream
            self.routes, self.shapes, self.run, self.docs = w.routes, w.shapes, dict(w.run), w.docs
            if getattr(args, "device", None):
                self.device = _load_device(args.device)
            return
        if not (args.registry and args.stream):
            raise ConfigurationError("give --config, or both --registry and --stream")
        self.registry = ModelRegistry.from_doc(_read_json(args.registry))
        self.stream = _stream_from_doc(_read_json(args.stream))
        self.device = _load_device(args.device or "numa-3080ti")
        self.routes = None
        if getattr(args, "routes", None):
            self.routes = {c: RoutePlan(tuple(v["experts"]), float(v["branch_prob"]))
                           for c, v in _read_json(args.routes).items()}
        self.run = {"gpu_executors": args.gpu_executors if args.gpu_executors is not None else 3,
                    "cpu_executors": args.cpu_executors, "contention_factor": args.contention_factor,
                    "cpu_mem_fraction": args.cpu_mem_fraction}

    def config(self, policy: str, seed: int, **over) -> engine.RunConfig:
        kw = dict(self.run)
        kw.pop("policy", None)
        kw.update(over)
        return engine.RunConfig(registry=self.registry, device=self.device, policy=policy, stream=self.stream,
                                seed=seed, routes=self.routes, **kw)


def _parse_alloc(text: str | None) -> dict | None:
    if not text:
        return None
    out = {}
    for part in text.split(","):
        proc, _, count = part.partition("=")
        if proc not in ("gpu", "cpu") or not count.isdigit():
            raise ConfigurationError(f"bad --alloc entry {part!r} (want gpu=N or cpu=N)")
        out[proc] = int(count)
    return out


def _execute(work: _Work, cfg: engine.RunConfig, steps: int = 2) -> dict:
    """Serve the plan on the GPU (runtime.B200Runtime): device-timed requests/s over ``steps``
    steps after one warm-up, plus what moved."""
    from . import runtime

    if work.shapes is None:
        raise ConfigurationError("--execute needs --config (expert shapes)")
    plan = engine.plan(cfg)
    if len(plan.resolved.executors) != 1 or plan.resolved.executors[0][0] != "gpu":
        raise ConfigurationError("--execute serves one gpu executor (use bench.py under torchrun for N GPUs)")
    rt = runtime.B200Runtime.for_plan(plan, runtime.shape_of(_FakeW(work.shapes)), profile=True)
    try:
        n = len(plan.resolved.request_ids)
        rt.fill_inputs(n)
        ms = []
        for i in range(steps + 1):
            st = rt.step(plan)
            rt.synchronize()
            if i:
                ms.append(rt.timing()["total_ms"])
        runs, violations = rt.check()
        if violations:
            raise RuntimeError(f"GPU grouping found {violations} batches straddling two runs")
        return {"requests_per_s": n / (statistics.fmean(ms) / 1e3), "ms_per_step": statistics.fmean(ms),
                "loads": st["loads"], "load_bytes": st["load_bytes"], "waves": st["waves"], "runs": runs}
    finally:
        rt.close()


class _FakeW:
    def __init__(self, shapes):
        self.shapes = shapes


def cmd_gen_workload(args) -> int:
    w = configs.load(args.config, args.requests)
    out = Path(args.out_dir)
    out.mkdir(parents=True, exist_ok=True)
    for name in ("registry", "stream", "device", "routes"):
        if w.docs.get(name) is not None:
            _write_json(out / f"{name}.json", w.docs[name])
            print(f"wrote {out / (name + '.json')}")
    return EXIT_OK


def cmd_profile(args) -> int:
    work = _Work(args)
    device = work.device
    if args.measure:
        shapes = sorted(set(work.shapes.values())) if work.shapes else []
        if not shapes:
            raise ConfigurationError("--measure needs --config (expert shapes)")
        doc = profiler.measure_b200_device(shapes)
        device = DeviceProfile.from_doc(configs.device_doc(work.shapes, doc["shapes"]))
        _write_json(Path(args.out_dir) / "device.json", device.to_doc())
        print(f"wrote {Path(args.out_dir) / 'device.json'} (measured on {doc['gpu']})")
    cost = CostModel(device)
    mem, _host = engine.partition_memory(device, work.run.get("gpu_executors", 3), work.run.get("cpu_executors", 1),
                                         work.run.get("cpu_mem_fraction", 0.4))
    perf = profiler.build_perf_profile(work.registry, cost, mem, args.plateau_threshold)
    path = Path(args.out_dir) / "perf_profile.json"
    _write_json(path, perf.to_doc())
    print(f"wrote {path}")
    return EXIT_OK


def cmd_search_memory(args) -> int:
    work = _Work(args)
    if args.measured:
        from . import runtime

        cfg = work.config(args.policy, args.seed)
        res = profiler.search_memory_allocation_measured(
            cfg, runtime.shape_of(_FakeW(work.shapes)), proc=args.proc, sample_requests=args.sample_requests,
            seed=args.seed, initial_window=args.initial_window, error_margin=args.error_margin,
            fit_points=args.fit_points, choose=args.choose)
    else:
        res = profiler.search_memory_allocation(
            work.registry, work.device, args.proc, work.stream[:args.sample_requests], seed=args.seed,
            policy=args.policy, gpu_executors=work.run.get("gpu_executors", 3),
            cpu_executors=work.run.get("cpu_executors", 1), initial_window=args.initial_window,
            error_margin=args.error_margin, fit_points=args.fit_points, choose=args.choose)
    _write_json(args.out, res.to_doc())
    print(f"window [{res.lower}, {res.upper}] chosen {res.chosen} -> {args.out}")
    return EXIT_OK


def cmd_simulate(args) -> int:
    work = _Work(args)
    over = {"trace": bool(args.trace)}
    alloc = _parse_alloc(args.alloc)
    if alloc:
        over["alloc_override"] = alloc
    if args.no_search:
        over["search_enabled"] = False
    cfg = work.config(args.policy, args.seed, **over)
    metrics, trace = engine.run(cfg)
    text = engine.metrics_json(metrics)
    if args.out:
        Path(args.out).write_text(text)
    else:
        sys.stdout.write(text)
    if args.trace:
        Path(args.trace).write_text(engine.trace_jsonl(trace))
    if args.execute:
        b200 = _execute(work, work.config(args.policy, args.seed, **dict(over, trace=False)))
        print(json.dumps({"b200": b200}, sort_keys=True))
    return EXIT_OK


def _aggregate(policy: str, runs: list, measured: list) -> dict:
    thpts = [m.throughput_rps for m in runs]
    row = {
        "policy": policy, "executors": f"{runs[0].per_executor[-1]['executor'] + 1}x",
        "throughput_mean": statistics.fmean(thpts),
        "throughput_stdev": statistics.stdev(thpts) if len(thpts) > 1 else 0.0,
        "makespan_mean": statistics.fmean(m.makespan_s for m in runs),
        "switches_mean": statistics.fmean(m.expert_switches for m in runs),
        "evictions_mean": statistics.fmean(m.evictions for m in runs),
        "stale_mean": statistics.fmean(m.stale_predictions for m in runs),
        "sched_overhead_mean": statistics.fmean(m.sched_overhead_ratio() for m in runs),
        "runs": [{"seed": m.seed, "throughput_rps": m.throughput_rps, "makespan_s": m.makespan_s,
                  "expert_switches": m.expert_switches, "evictions": m.evictions,
                  "stale_predictions": m.stale_predictions} for m in runs],
    }
    if measured:
        row["b200_requests_per_s"] = statistics.fmean(x["requests_per_s"] for x in measured)
    return row


def cmd_compare(args) -> int:
    if args.ablation:
        policies = list(ABLATION_POLICIES)
    elif args.policies:
        policies = [p.strip() for p in args.policies.split(",") if p.strip()]
    else:
        policies = list(DEFAULT_POLICIES)
    unknown = [p for p in policies if p not in POLICIES]
    if unknown:
        raise ConfigurationError(f"unknown policies: {unknown}, available: {sorted(POLICIES)}")
    work = _Work(args)
    rows = []
    for policy in policies:
        runs, measured = [], []
        for i in range(args.seeds):
            cfg = work.config(policy, args.base_seed + i)
            runs.append(engine.run(cfg)[0])
            if args.execute:
                measured.append(_execute(work, cfg))
        rows.append(_aggregate(policy, runs, measured))
    baseline = next((r for r in rows if r["policy"] == "samba_lru"), None)
    for row in rows:
        if baseline is None or row is baseline:
            row["throughput_x_vs_samba_lru"] = row["switch_reduction_vs_samba_lru"] = None
            continue
        row["throughput_x_vs_samba_lru"] = (row["throughput_mean"] / baseline["throughput_mean"]
                                            if baseline["throughput_mean"] else None)
        row["switch_reduction_vs_samba_lru"] = (1.0 - row["switches_mean"] / baseline["switches_mean"]
                                                if baseline["switches_mean"] else None)
        if "b200_requests_per_s" in row and "b200_requests_per_s" in baseline:
            row["b200_x_vs_samba_lru"] = row["b200_requests_per_s"] / baseline["b200_requests_per_s"]
    header = (f"{'policy':<15} {'execs':>5} {'thpt':>9} {'stdev':>8} {'makespan':>9} "
              f"{'switches':>9} {'evict':>8} {'xLRU':>6} {'sw-red':>7} {'ovh':>9}")
    if args.execute:
        header += f" {'B200 req/s':>11} {'B200 xLRU':>9}"
    print(header)
    print("-" * len(header))
    for row in rows:
        x = f"{row['throughput_x_vs_samba_lru']:.2f}" if row["throughput_x_vs_samba_lru"] else "-"
        red = (f"{100 * row['switch_reduction_vs_samba_lru']:.1f}%"
               if row["switch_reduction_vs_samba_lru"] is not None else "-")
        line = (f"{row['policy']:<15} {row['executors']:>5} {row['throughput_mean']:>9.2f} "
                f"{row['throughput_stdev']:>8.2f} {row['makespan_mean']:>9.3f} {row['switches_mean']:>9.1f} "
                f"{row['evictions_mean']:>8.1f} {x:>6} {red:>7} {row['sched_overhead_mean']:>9.2e}")
        if args.execute:
            bx = row.get("b200_x_vs_samba_lru")
            line += f" {row['b200_requests_per_s']:>11.1f} {(f'{bx:.2f}' if bx else '-'):>9}"
        print(line)
    if args.out_json:
        _write_json(args.out_json, {"schema_version": 1, "workload": work.name or args.registry,
                                    "device": work.device.name,
                                    "seeds": [args.base_seed + i for i in range(args.seeds)], "rows": rows})
        print(f"wrote {args.out_json}")
    if args.out_csv:
        fields = ["policy", "executors", "throughput_mean", "throughput_stdev", "makespan_mean", "switches_mean",
                  "evictions_mean", "stale_mean", "sched_overhead_mean", "throughput_x_vs_samba_lru",
                  "switch_reduction_vs_samba_lru", "b200_requests_per_s", "b200_x_vs_samba_lru"]
        with open(args.out_csv, "w", newline="") as fh:
            writer = csv.DictWriter(fh, fieldnames=fields, extrasaction="ignore")
            writer.writeheader()
            writer.writerows(rows)
        print(f"wrote {args.out_csv}")
    return EXIT_OK


def _workload_args(sub) -> None:
    sub.add_argument("--config", choices=configs.NAMES, help="committed configuration (data/configs)")
    sub.add_argument("--requests", type=int, default=1000, choices=(1000, 10000))
    sub.add_argument("--registry", help="registry JSON file (alternative to --config)")
    sub.add_argument("--stream", help="request stream JSON file (alternative to --config)")
    sub.add_argument("--routes", help="N-stage routes JSON file (optional, with --registry)")
    sub.add_argument("--device", help="device preset or JSON file (default: the config's / numa-3080ti)")
    sub.add_argument("--gpu-executors", type=int, default=None)
    sub.add_argument("--cpu-executors", type=int, default=1)
    sub.add_argument("--cpu-mem-fraction", type=float, default=0.4)
    sub.add_argument("--contention-factor", type=float, default=1.15)


def build_parser() -> argparse.ArgumentParser:
    ap = argparse.ArgumentParser(prog="paper_2503_02354_b200.cli", description=__doc__.split("\n\n")[0])
    subs = ap.add_subparsers(dest="cmd", required=True)
    gen = subs.add_parser("gen-workload", help="write a configuration's documents")
    gen.add_argument("--config", choices=configs.NAMES, required=True)
    gen.add_argument("--requests", type=int, default=1000, choices=(1000, 10000))
    gen.add_argument("--out-dir", default=".")
    prof = subs.add_parser("profile", help="build perf_profile.json for a device")
    _workload_args(prof)
    prof.add_argument("--measure", action="store_true", help="re-measure the B200 constants on this GPU first")
    prof.add_argument("--plateau-threshold", type=float, default=profiler.DEFAULT_PLATEAU_THRESHOLD)
    prof.add_argument("--out-dir", default=".")
    search = subs.add_parser("search-memory", help="decay-window allocation search")
    _workload_args(search)
    search.add_argument("--proc", choices=("gpu", "cpu"), default="gpu")
    search.add_argument("--policy", choices=sorted(POLICIES), default="coserve")
    search.add_argument("--seed", type=int, default=0)
    search.add_argument("--sample-requests", type=int, default=400)
    search.add_argument("--initial-window", type=int, default=profiler.DEFAULT_INITIAL_WINDOW)
    search.add_argument("--error-margin", type=float, default=profiler.DEFAULT_ERROR_MARGIN)
    search.add_argument("--fit-points", type=int, default=profiler.DEFAULT_FIT_POINTS)
    search.add_argument("--choose", choices=("random", "midpoint"), default="random")
    search.add_argument("--measured", action="store_true", help="throughput probes served on the GPU")
    search.add_argument("--out", default="window_search.json")
    sim = subs.add_parser("simulate", help="run one policy on one workload")
    _workload_args(sim)
    sim.add_argument("--policy", choices=sorted(POLICIES), required=True)
    sim.add_argument("--seed", type=int, default=0)
    sim.add_argument("--alloc", help="pin resident expert counts, e.g. gpu=35 or gpu=35,cpu=10")
    sim.add_argument("--no-search", action="store_true", help="disable the allocation search")
    sim.add_argument("--out", help="metrics JSON path (stdout when omitted)")
    sim.add_argument("--trace", help="write a JSONL event trace to this path")
    sim.add_argument("--execute", action="store_true", help="also serve the plan on the GPU")
    comp = subs.add_parser("compare", help="run several policies across seeds")
    _workload_args(comp)
    comp.add_argument("--seeds", type=int, default=1)
    comp.add_argument("--base-seed", type=int, default=0)
    comp.add_argument("--policies", help="comma-separated list; default " + ",".join(DEFAULT_POLICIES))
    comp.add_argument("--ablation", action="store_true", help="compare the coserve ablation ladder")
    comp.add_argument("--execute", action="store_true", help="also serve every plan on the GPU")
    comp.add_argument("--out-csv")
    comp.add_argument("--out-json")
    return ap


COMMANDS = {"gen-workload": cmd_gen_workload, "profile": cmd_profile, "search-memory": cmd_search_memory,
            "simulate": cmd_simulate, "compare": cmd_compare}


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return COMMANDS[args.cmd](args)
    except (ConfigurationError, SchemaError, OSError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_CONFIG
    except (MemoryStarvationError, RuntimeError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_SIM


if __name__ == "__main__":
    sys.exit(main())
