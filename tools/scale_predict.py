"""Planner-predicted multi-GPU balance (no GPU needed).

    python tools/scale_predict.py [config] [requests]

For N in 1/2/4/8 executors (one per GPU, 12 GB each: configs.load scales alloc_override)
the deterministic planner's op logs give each executor's admissions and swap-ins; the step
is bounded by the slowest executor's max(copy time at 55 GB/s, K3 time at the measured
in-step rate).  Hops between executors are counted (their NVLink time is negligible next to
either bound).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_02354_b200 import configs, engine, runtime  # noqa: E402

PCIE = 55e9
K3 = 1.3e15


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    nreq = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
    rows = []
    for n in (1, 2, 4, 8):
        w = configs.load(name, nreq, gpu_executors=n)
        plan = engine.plan(configs.run_config(w, trace=False))
        shapes = w.shapes
        reg = plan.resolved.config.registry
        ids = plan.resolved.expert_ids
        flops, copy_b = [0.0] * n, [0] * n
        adm = [0] * n
        for o in plan.ops():
            x, e = int(o["executor"]), ids[int(o["expert"])]
            d, h, T = shapes[reg.experts[e].arch]
            if o["kind"] == 1:
                adm[x] += int(o["count"])
                flops[x] += 4.0 * int(o["count"]) * T * d * h
            else:
                copy_b[x] += reg.experts[e].param_bytes
        step = [max(f / K3, b / PCIE) for f, b in zip(flops, copy_b)]
        rows.append({"gpus": n, "admissions": adm, "swap_in_gb": [round(b / 1e9, 2) for b in copy_b],
                     "step_ms": [round(s * 1e3, 1) for s in step], "predicted_rps": nreq / max(step),
                     "hops": len(runtime.hops_from_plan(plan)),
                     "expert_budget_gb": plan.resolved.alloc["gpu"]["expert_budget_bytes"] / 1e9})
        print(json.dumps(rows[-1]))
    base = rows[0]["predicted_rps"]
    for r in rows:
        print(f"{name} N={r['gpus']}: {r['predicted_rps']:9.0f} req/s  ({r['predicted_rps'] / base:4.1f}x)")


if __name__ == "__main__":
    main()
