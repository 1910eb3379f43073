"""Probe the GPU box: host cores/RAM, GPU, pinned H2D/D2H bandwidth."""
import os, subprocess, time, json
import torch
out = {"cpu_count": os.cpu_count()}
try:
    out["meminfo"] = open("/proc/meminfo").read().split("\n")[:3]
except Exception as e:
    out["meminfo"] = str(e)
out["gpu"] = torch.cuda.get_device_name(0)
props = torch.cuda.get_device_properties(0)
out["sms"] = props.multi_processor_count
out["mem"] = props.total_memory
for gb in (1, 4):
    n = gb << 30
    t0 = time.time()
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    out[f"pin_alloc_{gb}GiB_s"] = time.time() - t0
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    for direction in ("h2d", "d2h"):
        best = 1e9
        for _ in range(5):
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                e0.record(s)
                if direction == "h2d":
                    d.copy_(h, non_blocking=True)
                else:
                    h.copy_(d, non_blocking=True)
                e1.record(s)
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1) / 1e3)
        out[f"{direction}_{gb}GiB_GBps"] = n / best / 1e9
    del h, d
out["nvidia_smi"] = subprocess.run(["nvidia-smi", "--query-gpu=name,pcie.link.gen.max,pcie.link.width.max,clocks.max.sm", "--format=csv"], capture_output=True, text=True).stdout
out["topo"] = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout[:2000]
print(json.dumps(out, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe_box.json", "w"), indent=1)
