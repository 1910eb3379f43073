"""Host-side cost of one serving step: planner (engine.plan) and runtime issue (rt.step returns
before the GPU finishes).  python tools/host_times.py [config] [requests] [e2e 0|1]"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2503_02354_b200 import configs, engine, runtime

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
nreq = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
e2e = len(sys.argv) > 3 and sys.argv[3] == "1"
w = configs.load(name, nreq)
cfg = configs.run_config(w, trace=False)
if os.environ.get("ALLOC_COUNT"):  # expert budget as alloc_override={'gpu': N} (bench --alloc-count)
    cfg = configs.run_config(w, trace=False, alloc_override={"gpu": int(os.environ["ALLOC_COUNT"])},
                             search_enabled=False)
plan = engine.plan(cfg)
rt = runtime.B200Runtime.for_plan(plan, runtime.shape_of(w))
n = len(plan.resolved.request_ids)
rt.fill_inputs(n)
kw = {}
if e2e:
    row = rt.shapes[0].T * rt.act_ld
    hin = torch.empty(n * row, dtype=torch.bfloat16).pin_memory()
    hout = torch.empty(n * row, dtype=torch.bfloat16).pin_memory()
    kw = dict(host_inputs=hin.data_ptr(), host_outputs=hout.data_ptr())
tp, ts, tg = [], [], []
for i in range(6):
    t0 = time.perf_counter()
    p = engine.plan(cfg)
    t1 = time.perf_counter()
    rt.step(p, **kw)
    t2 = time.perf_counter()
    rt.synchronize()
    t3 = time.perf_counter()
    if i >= 2:
        tp.append(t1 - t0); ts.append(t2 - t1); tg.append(t3 - t2)
print(json.dumps({"config": name, "requests": nreq, "e2e": e2e, "plan_ms": 1e3 * sum(tp) / len(tp),
                  "issue_ms": 1e3 * sum(ts) / len(ts), "gpu_tail_after_issue_ms": 1e3 * sum(tg) / len(tg)}))
