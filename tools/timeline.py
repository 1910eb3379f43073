"""Run a few serving steps of a config and analyse the last step's timeline (debug tool).

    python tools/timeline.py [config] [requests] [out.json]

Prints one JSON summary: step / copy / K3 busy times, the K3 launch efficiency
split by wave size, the idle time of the GPU between K3 launches, and the
W2-wait gaps inside waves.  The raw per-wave phases go to out.json.
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_02354_b200 import configs, engine, runtime  # noqa: E402


def union(iv):
    iv = sorted(iv)
    tot, cur_s, cur_e = 0.0, None, None
    for s, e in iv:
        if cur_e is None or s > cur_e:
            if cur_e is not None:
                tot += cur_e - cur_s
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
    if cur_e is not None:
        tot += cur_e - cur_s
    return tot


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c3"
    nreq = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
    out = sys.argv[3] if len(sys.argv) > 3 else f"gpurun_out/timeline_{name}_{nreq}.json"
    e2e = len(sys.argv) > 4 and sys.argv[4] == "e2e"
    w = configs.load(name, nreq)
    shape = runtime.shape_of(w)
    cfg = configs.run_config(w, trace=False)
    if os.environ.get("ALLOC_COUNT"):  # expert budget as alloc_override={'gpu': N} (bench --alloc-count)
        cfg = configs.run_config(w, trace=False, alloc_override={"gpu": int(os.environ["ALLOC_COUNT"])},
                                 search_enabled=False)
    plan = engine.plan(cfg)
    rt = runtime.B200Runtime.for_plan(plan, shape, profile=True)
    rt.fill_inputs(len(plan.resolved.request_ids))
    keep = []
    kw = {}
    if e2e:
        import torch

        n = len(plan.resolved.request_ids)
        row = rt.shapes[0].T * rt.act_ld
        hin = torch.empty(n * row, dtype=torch.bfloat16).pin_memory()
        hout = torch.empty(n * row, dtype=torch.bfloat16).pin_memory()
        kw = dict(host_inputs=hin.data_ptr(), host_outputs=hout.data_ptr())
    for _ in range(4):
        p = engine.plan(cfg)
        st = rt.step(p, **kw)
        keep.append(p)
        rt.synchronize()
    timing = rt.timing()
    iv = rt.intervals()
    ph = rt.wave_phases()
    phases = np.array(ph["phases"])
    flops = np.array(ph["flops"])
    info = np.array(iv["wave_info"])
    up = phases[:, 1] - phases[:, 0]
    down = phases[:, 3] - phases[:, 2]
    w2wait = phases[:, 2] - phases[:, 1]
    k3_iv = [(a, b) for a, b in phases[:, 0:2]] + [(a, b) for a, b in phases[:, 2:4]]
    busy = union(k3_iv)
    rows = info[:, 1]
    buckets = {}
    for lo, hi in ((0, 2048), (2048, 8192), (8192, 16384), (16384, 1 << 30)):
        m = (rows >= lo) & (rows < hi)
        if m.any():
            t = float((up[m] + down[m]).sum())
            buckets[f"rows[{lo},{hi})"] = {"waves": int(m.sum()), "sum_launch_ms": t,
                                           "tflops_serial": float(flops[m].sum() / (t / 1e3) / 1e12) if t > 0 else None}
    cls = {}
    for c in sorted(set(info[:, 0].tolist())):
        m = info[:, 0] == c
        t = float((up[m] + down[m]).sum())
        cls[int(c)] = {"waves": int(m.sum()), "rows": int(rows[m].sum()), "sum_launch_ms": t,
                       "busy_union_ms": union([(a, b) for a, b in phases[m][:, 0:2]] +
                                              [(a, b) for a, b in phases[m][:, 2:4]]),
                       "tflops_serial": float(flops[m].sum() / (t / 1e3) / 1e12) if t > 0 else None}
    st = {k: v for k, v in st.items() if not isinstance(v, np.ndarray)}
    summary = {
        "config": name, "requests": nreq, "timing": timing, "stats": st,
        "k3": {"busy_ms": busy, "flops": float(flops.sum()), "tflops_busy": float(flops.sum() / (busy / 1e3) / 1e12),
               "sum_launch_ms": float((up + down).sum()), "w2_wait_ms_sum": float(w2wait.sum()),
               "waves": int(len(flops)), "mean_rows": float(rows.mean()), "median_rows": float(np.median(rows)),
               "idle_ms_in_step": timing["total_ms"] - busy, "by_rows": buckets, "by_stream_class": cls},
        "copies": {"n": len(iv["copies"]), "busy_ms": union([tuple(c) for c in iv["copies"]])},
    }
    if e2e:
        io = rt.io_intervals()
        h2d = [tuple(c) for c in iv["copies"]] + [tuple(c) for c in io["inputs"]]
        summary["e2e"] = {"h2d_busy_ms": union(h2d), "input_busy_ms": union([tuple(c) for c in io["inputs"]]),
                          "d2h_busy_ms": union([tuple(c) for c in io["outputs"]]),
                          "first_h2d_ms": min(a for a, _ in h2d) if h2d else None,
                          "last_h2d_end_ms": max(b for _, b in h2d) if h2d else None,
                          "last_d2h_end_ms": max((b for _, b in io["outputs"]), default=None),
                          "inputs": len(io["inputs"]), "outputs": len(io["outputs"])}
        summary["io"] = io
    print(json.dumps({k: v for k, v in summary.items() if k != "io"}))
    json.dump({"summary": summary, "phases": ph["phases"], "flops": ph["flops"], "wave_info": iv["wave_info"],
               "copies": iv["copies"]}, open(out, "w"))
    rt.close()


if __name__ == "__main__":
    main()
