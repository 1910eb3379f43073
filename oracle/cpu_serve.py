"""CPU restatement of the serving path, timed as the reference arm / cpu_baseline.

TEST / BENCH INFRASTRUCTURE ONLY.  The reference is a pure-Python simulator
with no expert math, so "the reference's CPU implementation of
the path" is restated here as: the oracle DES (``oracle.des``, single-threaded
CPython, the reference's own algorithm) deciding every admission / eviction,
plus the decided work executed on the host -- numpy fp32 expert MLPs
(``oracle.mlp``; OpenBLAS on every host core) over the batches it groups,
and each planned swap-in as a host memcpy of the expert's weights into its
pool buffer.  Weight *values* come from one reusable buffer (timing-neutral;
numerical parity is established separately at small sizes in the tests).
"""

from __future__ import annotations

import os
import time

import numpy as np

from . import des
from .mlp import gelu_tanh


def serve_sample(docs: dict, run: dict, shapes: dict, num_requests: int, seed: int = 0) -> dict:
    """Serve the first ``num_requests`` requests of the workload on the CPU; returns timing."""
    stream = {"schema_version": 1, "requests": docs["stream"]["requests"][:num_requests]}
    archs = {e["expert_id"]: e["arch"] for e in docs["registry"]["experts"]}
    rng = np.random.default_rng(seed)
    (d, h, T), = set(tuple(v) for v in shapes.values())
    w1_src = (rng.standard_normal((h, d), dtype=np.float32) * np.float32(1.0 / np.sqrt(d)))
    w2_src = (rng.standard_normal((d, h), dtype=np.float32) * np.float32(1.0 / np.sqrt(h)))
    x0 = rng.standard_normal((num_requests, T, d), dtype=np.float32)

    t0 = time.perf_counter()
    plan = des.simulate(docs["registry"], docs["device"], stream, routes=docs.get("routes"), trace=False, **run)
    t_plan = time.perf_counter() - t0
    pool: dict = {}
    act = {}
    loads = 0
    moved = 0

    def swap_in(expert, reuse=None):
        nonlocal loads, moved
        w1 = reuse[0] if reuse is not None else np.empty((h, d), np.float32)
        w2 = reuse[1] if reuse is not None else np.empty((d, h), np.float32)
        np.copyto(w1, w1_src)
        np.copyto(w2, w2_src)
        pool[expert] = (w1, w2)
        loads += 1
        moved += w1.nbytes + w2.nbytes

    rid_index = {r["request_id"]: i for i, r in enumerate(stream["requests"])}
    for op in plan["ops"]:
        if op[0] == "load":
            _, _x, expert, victims = op
            reuse = None
            for v in victims:
                got = pool.pop(v, None)
                if got is not None and reuse is None:
                    reuse = got
            swap_in(expert, reuse)
            continue
        _, _x, expert, members = op
        if expert not in pool:  # initially resident: first touch materialises it
            swap_in(expert)
        w1, w2 = pool[expert]
        xs = np.concatenate([act.get(rid, x0[rid_index[rid]]) for rid, _stage in members])
        y = gelu_tanh(xs @ w1.T) @ w2.T
        for k, (rid, _stage) in enumerate(members):
            act[rid] = y[k * T:(k + 1) * T]
    elapsed = time.perf_counter() - t0
    return {"requests": num_requests, "seconds": elapsed, "plan_seconds": t_plan, "loads": loads,
            "bytes_moved": moved, "batches": len(plan["batches"]), "threads": os.cpu_count() or 1,
            "arch_count": len(set(archs.values()))}
