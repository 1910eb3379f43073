"""Sweep runtime scheduling knobs on one runtime (debug/tuning tool)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_02354_b200 import configs, engine, runtime

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
nreq = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
w = configs.load(name, nreq)
shape = runtime.shape_of(w)
cfg = configs.run_config(w, trace=False)
plan = engine.plan(cfg)
rt = runtime.B200Runtime.for_plan(plan, shape, profile=True)
rt.fill_inputs(len(plan.resolved.request_ids))
variants = [tuple(int(v) for v in x.split(",")) for x in sys.argv[3].split(";")] if len(sys.argv) > 3 else \
    [(0, 0, 16), (8192, 0, 16), (32768, 8192, 16)]
out = []
for wr, ur, rs in variants:
    rt.set_knobs(wr, ur, rs)
    times = []
    for i in range(3):
        p = engine.plan(cfg)
        rt.step(p)
        rt.synchronize()
        times.append(rt.timing()["total_ms"])
    rec = {"wave_rows": wr, "urgent_rows": ur, "reserve_sms": rs, "ms": times}
    print(json.dumps(rec), flush=True)
    out.append(rec)
json.dump(out, open("gpurun_out/knob_sweep.json", "w"))
