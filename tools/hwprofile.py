"""B200 hardware profiler: measured device constants for the virtual clock.

Runs on the GPU box.  For every expert shape of the committed configs it times
the real K3 grouped MLP (one batch of n requests, n = 1..16, CUDA events,
median of repeats) and fits exec latency = k_s * n + b_s by least squares;
it times pinned host -> HBM swap-ins of each expert size and fits
bytes / bandwidth + overhead.  Writes paper_2503_02354_b200/data/b200_exec.json,
which tools/make_configs.py turns into the shared device documents (read by
both the planner and the oracle).

    python tools/hwprofile.py
"""
import json, os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2503_02354_b200 import configs, runtime

shapes = set()
for name in configs.NAMES:
    cfg = json.load(open(os.path.join(configs.CONFIG_DIR, name, "config.json")))
    for s in cfg["shapes"].values():
        shapes.add((s["d"], s["h"], s["T"]))
table = {}
for d, h, T in sorted(shapes):
    nmax = 16
    shape = runtime.RuntimeShape(d, h, T)
    rt = runtime.B200Runtime(shape, num_experts=2, num_slots=2, max_requests=nmax, max_admissions=nmax,
                             max_wave_rows=nmax * T)
    rt.fill_inputs(nmax)
    xs, ys = [], []
    for n in range(1, nmax + 1):
        samples = []
        for _ in range(5):
            up, down = rt.bench_mlp(1, n, 5)
            samples.append(up + down)
        xs.append(n)
        ys.append(statistics.median(samples) / 1e3)
    k, b = np.polyfit(xs, ys, 1)
    # swap-in: pinned H2D of one expert (W1 | W2 halves, as the runtime issues them)
    nbytes = shape.expert_bytes
    host = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    dev = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
    times = []
    for _ in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        dev[: nbytes // 2].copy_(host[: nbytes // 2], non_blocking=True)
        dev[nbytes // 2:].copy_(host[nbytes // 2:], non_blocking=True)
        e1.record()
        e1.synchronize()
        times.append(e0.elapsed_time(e1) / 1e3)
    table[configs.shape_key(d, h, T)] = {
        "k_s": float(max(k, 1e-7)), "b_s": float(max(b, 0.0)), "source": "measured: K3 grouped MLP, 1..16 requests",
        "samples_s": ys, "swap_s": statistics.median(times[1:]), "expert_bytes": nbytes,
    }
    print(d, h, T, table[configs.shape_key(d, h, T)]["k_s"], table[configs.shape_key(d, h, T)]["b_s"],
          "swap", table[configs.shape_key(d, h, T)]["swap_s"], flush=True)
    rt.close()
    del host, dev
# host tier from the largest swap: bandwidth = bytes / time (overhead from a small copy)
big = max(table.values(), key=lambda e: e["expert_bytes"])
small = min(table.values(), key=lambda e: e["expert_bytes"])
bw = (big["expert_bytes"] - small["expert_bytes"]) / max(big["swap_s"] - small["swap_s"], 1e-9)
ovh = max(small["swap_s"] - small["expert_bytes"] / bw, 0.0)
out = {"shapes": table, "host_tier": {"read_bandwidth_bytes_per_s": bw, "fixed_load_overhead_s": ovh},
       "gpu": torch.cuda.get_device_name(0), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())}
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/b200_exec.json", "w"), indent=1)
print(json.dumps(out["host_tier"]))
