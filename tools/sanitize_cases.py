"""Small serving cases for compute-sanitizer (racecheck / synccheck / memcheck), GPU box.

    compute-sanitizer --tool memcheck python tools/sanitize_cases.py [case ...]

Cases (each one runtime, two steps so cross-step slot / ring / staging reuse is covered):
  smoke   -- __graft_entry__.smoke(): C1 prefix, K1/K2/K3 + oracle check
  swaps   -- C3's 300-expert registry under the 12 GB budget with a mini expert shape:
             planned swap-ins and restores on the copy stream, release / swapped streams
  e2e     -- C2 prefix end to end twice back to back: inputs streamed into ring slots,
             finals through the output staging ring (small ring: wraps), D2H in completion order
  hops    -- C4 with 2 executors in one process, fused peer hops into landing rows
Exit code 0 and "case ok" lines mean the cases ran; the sanitizer's own summary decides.
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def trim(w, n):
    w.stream = w.stream[:n]
    w.docs = dict(w.docs, stream={"schema_version": 1, "requests": w.docs["stream"]["requests"][:n]})
    return w


def case_smoke():
    import __graft_entry__

    __graft_entry__.smoke()


def case_swaps():
    from paper_2503_02354_b200 import configs, engine, runtime

    w = trim(configs.load("c3", 1000), 120)
    plan = engine.plan(configs.run_config(w, trace=False))
    rt = runtime.B200Runtime.for_plan(plan, runtime.RuntimeShape(1024, 2048, 64))
    rt.fill_inputs(len(plan.resolved.request_ids))
    for _ in range(2):
        st = rt.step(plan)
    rt.synchronize()
    assert rt.check()[1] == 0 and st["loads"] > 0
    rt.close()


def case_e2e():
    import torch

    from paper_2503_02354_b200 import configs, engine, runtime

    w = trim(configs.load("c2", 1000), 60)
    plan = engine.plan(configs.run_config(w, trace=False))
    shape = runtime.RuntimeShape(1024, 2048, 64)
    rt = runtime.B200Runtime.for_plan(plan, shape, out_slots=24)
    n = len(plan.resolved.request_ids)
    rt.fill_inputs(n)
    row = shape.T * shape.d
    rt.step(plan)  # device-resident reference outputs (Y)
    rt.synchronize()
    ref = torch.empty(n * row, dtype=torch.bfloat16).pin_memory()
    rt.download_outputs(runtime.last_stages(plan), ref.data_ptr())
    rt.synchronize()
    ref = ref.view(n, -1)
    host_in = torch.empty(n * row, dtype=torch.bfloat16).pin_memory()
    rt.read_buffer(0, host_in.data_ptr(), n * row * 2)
    for _ in range(2):  # rows arrive in completion order, which may differ between steps
        h = torch.zeros(n * row, dtype=torch.bfloat16).pin_memory()
        rt.step(plan, host_inputs=host_in.data_ptr(), host_outputs=h.data_ptr())
        rt.synchronize()
        order = torch.from_numpy(rt.output_order()).long()
        assert torch.equal(h.view(n, -1), ref[order])
    rt.close()


def case_hops():
    from paper_2503_02354_b200 import configs, engine, runtime

    w = trim(configs.load("c4", 1000, gpu_executors=2), 80)
    plan = engine.plan(configs.run_config(w, trace=False))
    assert runtime.hops_from_plan(plan)
    rts = []
    for x in range(2):
        rt = runtime.B200Runtime.for_plan(plan, runtime.RuntimeShape(1024, 2048, 64), executor=x)
        rt.fill_inputs(len(plan.resolved.request_ids))
        rts.append(rt)
    hub = runtime.attach_peers_local(rts)
    for _ in range(2):
        runtime.step_executors(plan, rts, hub)
    for rt in rts:
        assert rt.check()[1] == 0
        rt.close()


CASES = {"smoke": case_smoke, "swaps": case_swaps, "e2e": case_e2e, "hops": case_hops}

if __name__ == "__main__":
    for name in sys.argv[1:] or list(CASES):
        CASES[name]()
        print("case ok:", name, flush=True)
