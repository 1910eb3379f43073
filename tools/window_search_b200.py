"""Decay-window allocation search on B200: measured vs virtual-clock throughput.

    python tools/window_search_b200.py [config] [sample_requests]
Writes gpurun_out/window_search_<config>.json with both curves and the chosen windows.
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_02354_b200 import configs, engine, profiler, runtime
from paper_2503_02354_b200.seeding import subseed

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 400
w = configs.load(name, 1000)
cfg = configs.run_config(w, trace=False)
measured = profiler.search_memory_allocation_measured(cfg, runtime.shape_of(w), sample_requests=n, steps=2,
                                                      seed=subseed(0, "alloc", "gpu"))
virtual = profiler.search_memory_allocation(w.registry, w.device, "gpu", cfg.stream[:n], seed=subseed(0, "alloc", "gpu"),
                                            policy=cfg.policy, gpu_executors=1, cpu_executors=0)
from dataclasses import replace
base = replace(cfg, stream=cfg.stream[:n], search_enabled=False, trace=False)
gx, cx = engine._executor_counts(base, engine.resolve(base).policy)
out = {"config": name, "sample_requests": n, "measured": measured.to_doc(), "virtual": virtual.to_doc(),
       "search": {"max_count": engine.max_useful_expert_count(base.registry, base.device, "gpu", gx, cx,
                                                              base.cpu_mem_fraction),
                  "initial_window": profiler.DEFAULT_INITIAL_WINDOW, "error_margin": profiler.DEFAULT_ERROR_MARGIN,
                  "fit_points": profiler.DEFAULT_FIT_POINTS, "choose": "random", "seed": subseed(0, "alloc", "gpu")}}
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open(f"gpurun_out/window_search_{name}.json", "w"), indent=1)
print(json.dumps({k: (v["lower"], v["upper"], v["chosen"]) for k, v in out.items() if isinstance(v, dict)}))
print("measured samples", measured.throughput_samples)
print("virtual samples", virtual.throughput_samples)
