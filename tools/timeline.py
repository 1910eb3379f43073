"""Run a few serving steps of a config and dump the per-copy / per-wave timeline (debug tool)."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_02354_b200 import configs, engine, runtime

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
nreq = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
out = sys.argv[3] if len(sys.argv) > 3 else "gpurun_out/timeline.json"
w = configs.load(name, nreq)
shape = runtime.shape_of(w)
cfg = configs.run_config(w, trace=False)
plan = engine.plan(cfg)
rt = runtime.B200Runtime.for_plan(plan, shape, profile=True)
rt.fill_inputs(len(plan.resolved.request_ids))
res = []
for i in range(3):
    p = engine.plan(cfg)
    st = rt.step(p)
    rt.synchronize()
    res.append({"stats": st, "timing": rt.timing(), "iv": rt.intervals()})
    print(json.dumps(res[-1]["timing"]))
json.dump(res[-1], open(out, "w"))
