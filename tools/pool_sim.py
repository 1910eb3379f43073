"""Host-only simulation of the runtime's pooled expert allocator (csrc/runtime.cu issue_copy)
over C5's plans at several arrival gaps: does any LOAD / restore find no free run?

    python tools/pool_sim.py
Policies: "bestfit" (smallest fitting run, lowest address) and "split" (the runtime's: large
experts >= 256 MB take the top of their run, small ones the bottom); slack = k largest experts
on top of the planner's byte budget.  Three steps of the same plan (state carries over).
"""
import os, sys, dataclasses
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_02354_b200 import configs, engine, runtime, _native
UNIT = 2 << 20
def sim(plan, pool_bytes, policy="bestfit", steps=3):
    res = plan.resolved; ids = res.expert_ids; reg = res.config.registry
    nb = [ (reg.experts[i].param_bytes + UNIT - 1)//UNIT for i in ids]
    P = pool_bytes // UNIT if pool_bytes % UNIT == 0 else pool_bytes//UNIT + 1
    free = {0: P}; where = {}
    def alloc(e):
        n = nb[e]
        cands = [(l, s) for s, l in free.items() if l >= n]
        if not cands: return False
        if policy == "bestfit":
            l, s = min(cands, key=lambda t: (t[0], t[1]))
            u0 = s
        elif policy == "split":  # big experts from the top of their run, small from the bottom
            big = n * UNIT >= (256 << 20)
            l, s = min(cands, key=lambda t: (t[0], -t[1] if big else t[1]))
            u0 = s + l - n if big else s
        del free[s]
        if u0 > s: free[s] = u0 - s
        if u0 + n < s + l: free[u0 + n] = s + l - u0 - n
        where[e] = (u0, n); return True
    def release(e):
        u0, n = where.pop(e)
        free[u0] = n
        # coalesce
        keys = sorted(free)
        merged = {}
        cs, cl = None, 0
        for k in keys:
            if cs is not None and cs + cl == k: cl += free[k]
            else:
                if cs is not None: merged[cs] = cl
                cs, cl = k, free[k]
        if cs is not None: merged[cs] = cl
        free.clear(); free.update(merged)
    ops = plan.ops(); args = plan.op_args(); init = set(plan.initial_residency()[0])
    for st in range(steps):
        for e in list(where):
            if e not in init: release(e)
        pending = {e for e in init if e not in where}
        for o in ops:
            e = int(o["expert"])
            if o["kind"] == _native.OP_LOAD:
                for v in args[int(o["offset"]):int(o["offset"])+int(o["count"])]:
                    v = int(v); pending.discard(v)
                    if v in where: release(v)
                pending.discard(e)
                if e in where: release(e)
                if not alloc(e): return f"fail step {st} load {e} ({nb[e]} units) free={sorted(free.values())[-5:]}"
            else:
                if e not in where:
                    pending.discard(e)
                    if not alloc(e): return f"fail step {st} restore {e}"
    return "ok"
if __name__ == "__main__":
    for gap in ():  # (single-slack table: see the sweep below)
        base = configs.load("c5", 10000)
        stream = [dataclasses.replace(r, arrival_time_s=i * gap) for i, r in enumerate(base.stream)]
        w = dataclasses.replace(base, stream=stream)
        cfg = configs.run_config(w, trace=False, alloc_override={"gpu": 201}, search_enabled=False)
        p = engine.plan(cfg)
        budget = p.resolved.executors[0][1]
        # the runtime's pool: min(budget, held) + largest + peak * unit  (approximate with budget + largest + 300 units)
        largest = max(e.param_bytes for e in p.resolved.config.registry.experts.values())
        pool = int(budget) + largest + 300 * UNIT
        print(gap, "bestfit", sim(p, pool), "| split", sim(p, pool, "split"))
    print("--- slack sweep")
    for gap in (1e-4, 3e-4, 1e-3):
        base = configs.load("c5", 10000)
        stream = [dataclasses.replace(r, arrival_time_s=i * gap) for i, r in enumerate(base.stream)]
        w = dataclasses.replace(base, stream=stream)
        cfg = configs.run_config(w, trace=False, alloc_override={"gpu": 201}, search_enabled=False)
        p = engine.plan(cfg)
        budget = p.resolved.executors[0][1]
        largest = max(e.param_bytes for e in p.resolved.config.registry.experts.values())
        for k in (2, 3, 4, 6):
            pool = int(budget) + k * largest + 300 * UNIT
            print(gap, k, sim(p, pool), sim(p, pool, "split"))
