"""Request-rate sweep on the B200 (BASELINE config 5's "request-rate sweep", run on a
single-GPU configuration).

    python tools/rate_sweep.py [config] [requests] [out.json]

The committed stream is re-timed to a fixed inter-arrival gap Δ (request i arrives at i·Δ;
same requests, components and branch draws), the native planner decides with the
reference's policy on the virtual clock, and the runtime executes the plan on the GPU
(device-resident inputs, CUDA-event timed after 2 warm-ups).  Rows: Δ, the offered load
1/Δ, the planner's virtual throughput, its batching (batches, mean requests per batch) and
swaps, and the measured B200 serving capacity for that schedule.
"""
import dataclasses
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2503_02354_b200 import configs, engine, runtime  # noqa: E402


def main() -> None:
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    nreq = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
    out = sys.argv[3] if len(sys.argv) > 3 else f"gpurun_out/rate_sweep_{name}_{nreq}.json"
    torch.cuda.set_device(0)
    base = configs.load(name, nreq)
    rows = []
    for gap in (1e-6, 1e-5, 1e-4, 3e-4, 1e-3):
        stream = [dataclasses.replace(r, arrival_time_s=i * gap) for i, r in enumerate(base.stream)]
        w = dataclasses.replace(base, stream=stream)
        cfg = configs.run_config(w, trace=False)
        if os.environ.get("ALLOC_COUNT"):  # expert budget as alloc_override={'gpu': N} (bench --alloc-count)
            cfg = configs.run_config(w, trace=False, alloc_override={"gpu": int(os.environ["ALLOC_COUNT"])},
                                     search_enabled=False)
        plan = engine.plan(cfg)
        metrics = engine.metrics_from_plan(plan)
        counts = [int(o["count"]) for o in plan.ops() if o["kind"] == 1]
        rt = runtime.B200Runtime.for_plan(plan, runtime.shape_of(w))
        n = len(plan.resolved.request_ids)
        rt.fill_inputs(n)
        stream_h = torch.cuda.ExternalStream(rt.stream_handle(0))
        for _ in range(2):
            rt.step(engine.plan(cfg))
        rt.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        keep = []
        steps = 3
        e0.record(stream_h)
        for _ in range(steps):
            p = engine.plan(cfg)
            st = rt.step(p)
            keep.append(p)
        e1.record(stream_h)
        rt.synchronize()
        ms = e0.elapsed_time(e1) / steps
        rt.close()
        row = {"interarrival_s": gap, "offered_rps": 1.0 / gap, "virtual_rps": metrics.throughput_rps,
               "measured_rps": n / (ms / 1e3), "ms_per_step": ms, "batches": len(counts),
               "mean_batch": sum(counts) / len(counts), "switches": metrics.expert_switches,
               "gb_swapped": st["load_bytes"] / 1e9, "waves": st["waves"]}
        rows.append(row)
        print(json.dumps(row), flush=True)
    json.dump({"config": name, "requests": nreq, "alloc_count": os.environ.get("ALLOC_COUNT"), "rows": rows,
               "note": "stream re-timed to arrival i*gap; measured = GPU capacity executing the planner's schedule "
                       "for that rate (device-resident inputs, CUDA events); virtual = the reference's simulated "
                       "throughput (bounded by the offered load)"}, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
