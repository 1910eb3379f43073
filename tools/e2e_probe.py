"""e2e step pipelining probe: ms/step for K back-to-back e2e steps with inputs+outputs, inputs only, outputs only."""
import os, sys, time, json
import torch
sys.path.insert(0, os.getcwd())
from paper_2503_02354_b200 import configs, engine, runtime

name = sys.argv[1] if len(sys.argv) > 1 else "c1"
w = configs.load(name, 10000)
shape = runtime.shape_of(w)
cfg = configs.run_config(w, trace=False)
plan0 = engine.plan(cfg)
rt = runtime.B200Runtime.for_plan(plan0, shape, executor=0)
n = len(plan0.resolved.request_ids)
rt.fill_inputs(n)
row = rt.shapes[0].T * rt.act_ld
hin = torch.empty(n * row, dtype=torch.bfloat16).pin_memory()
hout = torch.empty(n * row, dtype=torch.bfloat16).pin_memory()
rt.read_buffer(0, hin.data_ptr(), n * row * 2)
stream = torch.cuda.ExternalStream(rt.stream_handle(0))
res = {}
for mode in ("io", "in", "out", "none"):
    for K in (1, 2, 5):
        kw = {}
        if mode in ("io", "in"): kw["host_inputs"] = hin.data_ptr()
        if mode in ("io", "out"): kw["host_outputs"] = hout.data_ptr()
        plans = [engine.plan(cfg) for _ in range(K + 2)]
        for p in plans[:2]:
            rt.step(p, 0, **kw)
        rt.join(); rt.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(stream)
        for p in plans[2:]:
            rt.step(p, 0, **kw)
        rt.join()
        e1.record(stream)
        t_issue = time.perf_counter() - t0
        rt.synchronize()
        res[f"{mode}_K{K}"] = {"ms_per_step": e0.elapsed_time(e1) / K, "host_issue_ms_per_step": 1e3 * t_issue / K}
        print(mode, K, res[f"{mode}_K{K}"], flush=True)
json.dump(res, open(f"gpurun_out/e2e_probe_{name}.json", "w"), indent=1)
