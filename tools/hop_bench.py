"""Follow-up hop transports on one GPU (several executors in one process).

    python tools/hop_bench.py [config] [requests] [executors] [out.json]

Serves the config's plan with N executors sharing the GPU (one runtime + host thread each)
and times a step for each transport: "peer" (hops fused into K3's down-pass epilogue: rows
stored straight into the consumer's buffer, readiness handed over as events) and "hub"
(send/receive pairs in the global hop order, each hop a separate device-to-device copy --
the protocol the NCCL transport follows).  Both produce identical outputs (checked).
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2503_02354_b200 import configs, engine, runtime  # noqa: E402


def serve(plan, shape, n_exec, transport, steps=3):
    rts = []
    hub = runtime.LocalHub(n_exec) if transport == "hub" else None
    for x in range(n_exec):
        rt = runtime.B200Runtime.for_plan(plan, shape, executor=x)
        if hub is not None:
            rt.attach_local(hub, x)
        rt.fill_inputs(len(plan.resolved.request_ids))
        rts.append(rt)
    if hub is None:
        hub = runtime.attach_peers_local(rts)
    runtime.step_executors(plan, rts, hub)  # warm-up
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        runtime.step_executors(plan, rts, hub)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) / steps * 1e3
    n = len(plan.resolved.request_ids)
    T, d = shape.T, shape.d
    outs = []
    for rt in rts:
        host = torch.empty(n * T * d, dtype=torch.bfloat16).pin_memory()
        rt.download_outputs(runtime.last_stages(plan), host.data_ptr())
        rt.synchronize()
        outs.append(host.view(n, T, d).float().numpy().copy())
        rt.close()
    return ms, outs


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c4"
    nreq = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
    n_exec = int(sys.argv[3]) if len(sys.argv) > 3 else 2
    out = sys.argv[4] if len(sys.argv) > 4 else f"gpurun_out/hop_bench_{name}_{nreq}_{n_exec}.json"
    w = configs.load(name, nreq, gpu_executors=n_exec)
    plan = engine.plan(configs.run_config(w, trace=False))
    hops = runtime.hops_from_plan(plan)
    shape = runtime.shape_of(w)
    res = {}
    outs = {}
    for transport in ("peer", "hub"):
        ms, o = serve(plan, shape, n_exec, transport)
        res[transport] = {"ms_per_step": ms}
        outs[transport] = o
    chains = plan.resolved.chains
    final_exec = {}
    for x in range(n_exec):
        for _e, members in runtime.batches_from_plan(plan, executor=x):
            for r, s in members:
                if s == len(chains[r]) - 1:
                    final_exec[r] = x
    same = all(np.array_equal(outs["peer"][final_exec[r]][r], outs["hub"][final_exec[r]][r]) for r in final_exec)
    row = {"config": name, "requests": nreq, "executors": n_exec, "hops": len(hops),
           "hop_bytes": len(hops) * shape.T * shape.d * 2, "identical_outputs": same, **res,
           "note": "wall time of one step of all executors sharing one GPU (host threads + synchronize)"}
    print(json.dumps(row))
    json.dump(row, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
