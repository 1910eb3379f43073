"""CoServe vs the Samba-CoE baselines, measured on the B200 (the reference's `coesim compare`
table, cli.py:306-380, with real expert execution instead of simulated seconds).

    python tools/compare_policies.py [config] [requests] [steps] [out.json]

For each policy of engine.POLICIES the native planner decides (bit-exact with the
reference), the runtime serves the plan on the GPU (device-resident inputs, CUDA-event
timed, `steps` steps after 2 warm-ups), and the row reports measured req/s, the planner's
virtual req/s, expert switches, GB swapped in, and -- as in the reference's table -- the
throughput ratio to samba_lru (xLRU) and the switch reduction against it (sw-red).
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2503_02354_b200 import configs, engine, runtime  # noqa: E402

ORDER = ("coserve", "coserve_em_ra", "coserve_em", "coserve_none", "samba_parallel", "samba_fifo", "samba_lru")


def measure(w, policy: str, steps: int) -> dict:
    cfg = configs.run_config(w, trace=False, policy=policy)
    plan = engine.plan(cfg)
    metrics = engine.metrics_from_plan(plan)
    rt = runtime.B200Runtime.for_plan(plan, runtime.shape_of(w))
    n = len(plan.resolved.request_ids)
    rt.fill_inputs(n)
    stream = torch.cuda.ExternalStream(rt.stream_handle(0))
    stats = None
    for _ in range(2):
        stats = rt.step(engine.plan(cfg))
    rt.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    keep = []
    e0.record(stream)
    for _ in range(steps):
        p = engine.plan(cfg)
        stats = rt.step(p)
        keep.append(p)
    e1.record(stream)
    rt.synchronize()
    ms = e0.elapsed_time(e1) / steps
    runs, violations = rt.check()
    rt.close()
    return {"policy": policy, "measured_rps": n / (ms / 1e3), "ms_per_step": ms, "virtual_rps": metrics.throughput_rps,
            "switches": metrics.expert_switches, "evictions": metrics.evictions,
            "gb_swapped": (stats["load_bytes"] + stats["restore_bytes"]) / 1e9, "batches": stats["batches"],
            "waves": stats["waves"], "grouping_violations": violations}


def main() -> None:
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    nreq = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    out = sys.argv[4] if len(sys.argv) > 4 else f"gpurun_out/compare_{name}_{nreq}.json"
    torch.cuda.set_device(0)
    w = configs.load(name, nreq)
    rows = []
    for policy in ORDER:
        t0 = time.time()
        rows.append(measure(w, policy, steps))
        rows[-1]["wall_s"] = time.time() - t0
        print(json.dumps(rows[-1]), flush=True)
    base = next(r for r in rows if r["policy"] == "samba_lru")
    for r in rows:
        r["xLRU_measured"] = r["measured_rps"] / base["measured_rps"]
        r["xLRU_virtual"] = r["virtual_rps"] / base["virtual_rps"]
        r["switch_reduction"] = 1.0 - r["switches"] / base["switches"] if base["switches"] else None
    lines = [f"{'policy':16s} {'req/s B200':>11s} {'xLRU':>6s} {'virtual':>9s} {'xLRU':>6s} {'switches':>8s} "
             f"{'sw-red':>7s} {'GB in':>7s}"]
    for r in rows:
        lines.append(f"{r['policy']:16s} {r['measured_rps']:11.1f} {r['xLRU_measured']:6.2f} {r['virtual_rps']:9.1f} "
                     f"{r['xLRU_virtual']:6.2f} {r['switches']:8d} {100 * (r['switch_reduction'] or 0):6.1f}% "
                     f"{r['gb_swapped']:7.1f}")
    table = "\n".join(lines)
    print(table)
    json.dump({"config": name, "requests": nreq, "steps": steps, "rows": rows, "table": table,
               "note": "device-resident inputs; CUDA-event timed per policy after 2 warm-up steps; planner decisions "
                       "bit-exact with the reference (virtual = the reference's simulated throughput with the "
                       "measured B200 cost constants)"}, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
