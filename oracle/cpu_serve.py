"""CPU restatement of the serving path, timed as the reference arm / cpu_baseline.

TEST / BENCH INFRASTRUCTURE ONLY.  The reference is a pure-Python simulator
with no expert math, so "the reference's CPU implementation of
the path" is restated here on the SAME workload the GPU arm serves (the whole
stream, e.g. config 3's 10k requests):

  * decisions: the oracle DES (``oracle.des``, single-threaded CPython, the
    reference's own algorithm: admission engine.py:588-626, step / load /
    batch engine.py:630-716, follow-ups engine.py:740-758, heap loop
    engine.py:762-781) over the FULL stream -- timed in full;
  * the decided work, executed on the host: a deterministic uniform sample of
    the plan's batches (numpy fp32 ``gelu(X W1^T) W2^T`` at the batch's real
    M = members * T rows and the expert's real (d, h); OpenBLAS on every host
    core) and of its swap-ins (a memcpy of the expert's ``param_bytes`` from a
    host store buffer into a pool buffer -- the host tier to "device" move of
    ``_start_load``, engine.py:643-677, whose bytes the GPU arm moves over
    PCIe).  The sampled times are scaled by the plan's total FLOPs / bytes over
    the sample's, which is exact for a uniform sample of work whose time is
    proportional to FLOPs (GEMMs) and bytes (memcpy).

Weight and activation *values* come from reusable buffers (timing-neutral);
numerical parity of the expert math is established separately in the tests.
"""

from __future__ import annotations

import math
import os
import time

import numpy as np

from . import des
from .mlp import gelu_tanh


def _threads() -> int:
    try:
        from threadpoolctl import threadpool_info

        n = [i.get("num_threads", 0) for i in threadpool_info() if i.get("user_api") == "blas"]
        if n:
            return int(max(n))
    except Exception:
        pass
    return os.cpu_count() or 1


def plan_full(docs: dict, run: dict) -> tuple:
    """The oracle DES over the whole stream: (plan, seconds)."""
    t0 = time.perf_counter()
    plan = des.simulate(docs["registry"], docs["device"], docs["stream"], routes=docs.get("routes"), trace=False,
                        **run)
    return plan, time.perf_counter() - t0


def _shape_of(docs: dict, shapes: dict) -> dict:
    return {e["expert_id"]: tuple(shapes[e["arch"]]) for e in docs["registry"]["experts"]}


def _param_bytes(docs: dict) -> dict:
    return {e["expert_id"]: int(e["param_bytes"]) for e in docs["registry"]["experts"]}


def serve_plan_sample(docs: dict, run: dict, shapes: dict, budget_s: float = 12.0, sample_index: int = 0,
                      plan=None, plan_seconds: float | None = None, seed: int = 0) -> dict:
    """Serve the whole workload on the host, executing a uniform sample of its work.

    ``budget_s`` bounds the sampled execution time (the sample is sized from a one-batch
    calibration); ``sample_index`` rotates which batches / loads are taken (deterministic:
    every ``stride``-th op starting at ``sample_index % stride``).  Returns the estimated
    seconds to serve the whole workload = DES time + scaled expert time + scaled swap time."""
    if plan is None:
        plan, plan_seconds = plan_full(docs, run)
    shape_of = _shape_of(docs, shapes)
    pbytes = _param_bytes(docs)
    batches = [op for op in plan["ops"] if op[0] == "batch"]
    loads = [op for op in plan["ops"] if op[0] == "load"]

    def flops(op):
        d, h, T = shape_of[op[2]]
        return 4.0 * len(op[3]) * T * d * h

    total_flops = sum(flops(op) for op in batches)
    total_bytes = sum(pbytes[op[2]] for op in loads)
    rng = np.random.default_rng(seed)
    bufs: dict = {}

    def weights(d, h):
        if (d, h) not in bufs:
            bufs[(d, h)] = (rng.standard_normal((h, d), dtype=np.float32) * np.float32(1.0 / math.sqrt(d)),
                            rng.standard_normal((d, h), dtype=np.float32) * np.float32(1.0 / math.sqrt(h)))
        return bufs[(d, h)]

    max_rows = max((len(op[3]) * shape_of[op[2]][2] for op in batches), default=1)
    max_d = max((s[0] for s in shape_of.values()), default=1)
    xbuf = rng.standard_normal((max_rows, max_d), dtype=np.float32)

    def run_batch(op) -> float:
        d, h, T = shape_of[op[2]]
        w1, w2 = weights(d, h)
        x = xbuf[:len(op[3]) * T, :d]
        t = time.perf_counter()
        y = gelu_tanh(x @ w1.T) @ w2.T
        dt = time.perf_counter() - t
        del y
        return dt

    # calibration: one average-sized batch (untimed for the estimate), then size the sample
    n_b = len(batches)
    mean_flops = total_flops / max(1, n_b)
    cal = min(batches, key=lambda op: abs(flops(op) - mean_flops)) if batches else None
    rate = None
    if cal is not None:
        run_batch(cal)  # warm (BLAS threads, page faults)
        rate = flops(cal) / max(run_batch(cal), 1e-9)
    exec_budget = 0.85 * budget_s
    want_b = n_b if rate is None else max(1, min(n_b, int(exec_budget * rate / max(mean_flops, 1.0))))
    stride_b = max(1, n_b // want_b) if n_b else 1
    pick_b = batches[sample_index % stride_b::stride_b] if n_b else []

    t_exec = 0.0
    f_exec = 0.0
    for op in pick_b:
        t_exec += run_batch(op)
        f_exec += flops(op)

    # swap-ins: memcpy of param_bytes host store -> pool buffer (sample ~15% of the budget)
    t_load = 0.0
    b_load = 0
    pick_l = []
    if loads:
        biggest = max(pbytes[op[2]] for op in loads)
        src = np.ones(biggest, np.uint8)
        dst = np.empty(biggest, np.uint8)
        np.copyto(dst, src)  # fault both buffers in
        t = time.perf_counter()
        np.copyto(dst, src)
        bw = biggest / max(time.perf_counter() - t, 1e-9)
        mean_b = total_bytes / len(loads)
        want_l = max(1, min(len(loads), int(0.15 * budget_s * bw / max(mean_b, 1.0))))
        stride_l = max(1, len(loads) // want_l)
        pick_l = loads[sample_index % stride_l::stride_l]
        for op in pick_l:
            nb = pbytes[op[2]]
            t = time.perf_counter()
            np.copyto(dst[:nb], src[:nb])
            t_load += time.perf_counter() - t
            b_load += nb

    exec_s = t_exec * (total_flops / f_exec) if f_exec > 0 else 0.0
    load_s = t_load * (total_bytes / b_load) if b_load > 0 else 0.0
    n_req = len(docs["stream"]["requests"])
    seconds = plan_seconds + exec_s + load_s
    return {
        "requests": n_req, "seconds": seconds, "plan_seconds": plan_seconds, "exec_seconds": exec_s,
        "load_seconds": load_s, "batches": n_b, "sampled_batches": len(pick_b), "loads": len(loads),
        "sampled_loads": len(pick_l), "total_flops": total_flops, "sampled_flops": f_exec,
        "total_load_bytes": total_bytes, "sampled_load_bytes": b_load,
        "cpu_tflops": (f_exec / t_exec / 1e12) if t_exec > 0 else None,
        "memcpy_gbs": (b_load / t_load / 1e9) if t_load > 0 else None,
        "sample_wall_seconds": t_exec + t_load, "threads": _threads(),
        "shapes": len(set(shape_of.values())),
    }


def describe(res: dict) -> str:
    return (f"the whole {res['requests']}-request plan: oracle DES over every request (1 thread, "
            f"{res['plan_seconds']:.2f}s, timed in full) + a uniform sample of {res['sampled_batches']}/"
            f"{res['batches']} planned batches as numpy fp32 expert MLPs at their real shapes "
            f"({res['threads']} threads, {res['cpu_tflops'] or 0:.2f} TFLOP/s) and {res['sampled_loads']}/"
            f"{res['loads']} swap-ins as host memcpys of param_bytes, scaled by total/sampled FLOPs and bytes")
