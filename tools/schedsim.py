"""Offline model of the runtime's physical schedule (prototype for list scheduling).

Usage: python tools/schedsim.py [config] [requests]
Simulates the copy engine + main stream + release stream for a plan under
different wave-ordering policies, using measured rates (PCIe 55.3 GB/s,
K3 ~1.25 PFLOP/s), to compare makespans before porting a policy to C++.
"""
import heapq, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2503_02354_b200 import configs, engine, runtime, _native

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
nreq = int(sys.argv[2]) if len(sys.argv) > 2 else 10000
w = configs.load(name, nreq)
shape = runtime.shape_of(w)
plan = engine.plan(configs.run_config(w, trace=False))
ops, args = plan.ops(), plan.op_args()
T, d, h = shape.T, shape.d, shape.h
PCIE = 55.3e9
EB = shape.expert_bytes
F = 1.25e15
RES_FRAC = 16 / 148
LAUNCH = 8e-6
MAXROWS = 32768

# ---- build batch list and copy list as the runtime does (no restores in steady state) ----
batches = []   # dict: expert, members, copy (index or -1), release
copies = []    # dict: expert, slot victim readers
rel = [False] * len(ops)
nxt = {}
for k in range(len(ops) - 1, -1, -1):
    o = ops[k]
    if o["kind"] == 0:
        for j in range(o["count"]):
            nxt[int(args[o["offset"] + j])] = "E"
        nxt[int(o["expert"])] = None
    else:
        rel[k] = nxt.get(int(o["expert"])) == "E"
        nxt[int(o["expert"])] = "U"
last_reader = {}   # expert -> batch index (last reader so far)
cur_copy = {}      # expert -> copy index that loaded it this step
for k, o in enumerate(ops):
    e = int(o["expert"])
    if o["kind"] == 0:
        victims = [int(args[o["offset"] + j]) for j in range(o["count"])]
        dep = [last_reader[v] for v in victims if v in last_reader]
        copies.append({"expert": e, "after": dep})
        cur_copy[e] = len(copies) - 1
        for v in victims:
            last_reader.pop(v, None)
            cur_copy.pop(v, None)
    else:
        n = int(o["count"])
        mem = [(int(args[o["offset"] + 2 * j]), int(args[o["offset"] + 2 * j + 1])) for j in range(n)]
        batches.append({"expert": e, "members": mem, "copy": cur_copy.get(e, -1), "release": rel[k], "rows": n * T})
        last_reader[e] = len(batches) - 1
producer = {}
for bi, b in enumerate(batches):
    b["deps"] = [producer[(r, s - 1)] for r, s in b["members"] if s > 0]
    for r, s in b["members"]:
        producer[(r, s)] = bi
copy_t = EB / PCIE


def simulate(policy):
    nb = len(batches)
    done = [None] * nb          # batch completion time
    copy_end = [None] * len(copies)
    copy_ptr = 0
    t_copy = 0.0
    t_main = 0.0
    t_rel = 0.0
    pending = list(range(nb))
    main_order = [i for i in range(nb) if not batches[i]["release"]]
    rel_order = [i for i in range(nb) if batches[i]["release"]]
    mi = ri = 0
    # event-driven: repeatedly advance the earliest resource that can make progress
    scheduled = [False] * nb
    while True:
        progressed = False
        # copy engine: next copy can start when its victim readers are done
        if copy_ptr < len(copies):
            c = copies[copy_ptr]
            if all(done[b] is not None for b in c["after"]):
                start = max([t_copy] + [done[b] for b in c["after"]])
                t_copy = start + copy_t
                copy_end[copy_ptr] = t_copy
                copy_ptr += 1
                progressed = True
        # release stream: in order
        if ri < len(rel_order):
            b = batches[rel_order[ri]]
            deps_ok = all(done[x] is not None for x in b["deps"]) and (b["copy"] < 0 or copy_end[b["copy"]] is not None)
            if deps_ok:
                start = max([t_rel] + [done[x] for x in b["deps"]] + ([copy_end[b["copy"]]] if b["copy"] >= 0 else []))
                t_rel = start + b["rows"] * 4 * d * h / (F * RES_FRAC) + 2 * LAUNCH
                done[rel_order[ri]] = t_rel
                ri += 1
                progressed = True
        # main stream
        if mi < len(main_order):
            if policy == "inorder":
                wave = []
                rows = 0
                reqs = set()
                j = mi
                while j < len(main_order):
                    b = batches[main_order[j]]
                    if wave and (rows + b["rows"] > MAXROWS or any(r in reqs for r, _ in b["members"]) or
                                 (b["copy"] >= 0 and b["copy"] not in waited)):
                        break
                    if not (all(done[x] is not None or x in wave for x in b["deps"]) and
                            (b["copy"] < 0 or copy_end[b["copy"]] is not None)):
                        break
                    if any(x in wave for x in b["deps"]):
                        break
                    wave.append(main_order[j]); rows += b["rows"]; reqs |= {r for r, _ in b["members"]}
                    if b["copy"] >= 0:
                        waited.add(b["copy"])
                    j += 1
                if wave:
                    start = max([t_main] + [done[x] for i2 in wave for x in batches[i2]["deps"] if done[x] is not None] +
                                [copy_end[batches[i2]["copy"]] for i2 in wave if batches[i2]["copy"] >= 0])
                    t_main = start + rows * 4 * d * h / (F * (1 - RES_FRAC)) + 2 * LAUNCH
                    for i2 in wave:
                        done[i2] = t_main
                    mi = j
                    progressed = True
        if not progressed:
            break
    return max([t_copy, t_main, t_rel]), t_copy, t_main, t_rel, mi, ri, copy_ptr


waited = set()
print("batches", len(batches), "copies", len(copies), "copy floor ms", len(copies) * copy_t * 1e3)
res = simulate("inorder")
print("inorder: makespan %.1f ms copy_end %.1f main_end %.1f rel_end %.1f (progress %d/%d main, %d rel, %d copies)" %
      (res[0] * 1e3, res[1] * 1e3, res[2] * 1e3, res[3] * 1e3, res[4], sum(not b['release'] for b in batches), res[5], res[6]))
