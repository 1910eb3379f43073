"""Pure-Python restatement of the reference discrete-event engine (oracle).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).  Works on plain JSON
documents (registry / device / stream, optional N-stage ``routes``) and does
not import the product package.  Every step cites the reference line it
restates (``/root/reference/pkg/src/coesim/...``); data structures are the
reference's own (a Python list per queue with a backward scan for arranging),
so this is deliberately the slow, literal form the product planner is checked
against.

Returns ``{"metrics": <metrics doc>, "trace": [records], "batches": [...],
"loads": [...], "initial": [...]}`` where each batch is ``(executor, expert,
[(request_id, stage), ...])`` in start order and each load is ``(executor,
expert, victims, tier)``.
"""

from __future__ import annotations

import hashlib
import heapq
import math
import random

# engine.py:68-76 -- (assign, arrange, evict, single_gpu, host_mode)
POLICY_TABLE = {
    "coserve": ("makespan", True, "two_stage", False, "prob"),
    "coserve_em_ra": ("round_robin", True, "two_stage", False, "prob"),
    "coserve_em": ("round_robin", False, "two_stage", False, "prob"),
    "coserve_none": ("round_robin", False, "fifo", False, "fifo"),
    "samba_lru": ("round_robin", False, "lru", True, "lru"),
    "samba_fifo": ("round_robin", False, "fifo", True, "fifo"),
    "samba_parallel": ("round_robin", False, "lru", False, "lru"),
}


class OracleStarvation(RuntimeError):
    pass


def _subseed(seed, *labels):  # seeding.py:15-19
    text = str(int(seed)) + "".join(f"/{x}" for x in labels)
    return int.from_bytes(hashlib.sha256(text.encode()).digest()[:8], "big")


class Device:
    """Closed forms of costmodel.py:55-92 over a device document."""

    def __init__(self, doc):
        self.arch = doc["architecture"]
        self.tiers = {t["tier"]: (t["capacity_bytes"], float(t["read_bandwidth_bytes_per_s"]),
                                  float(t.get("fixed_load_overhead_s", 0.0))) for t in doc["tiers"]}
        self.const = {}
        for c in doc["exec_constants"]:
            self.const[(c["arch"], c["proc"])] = (float(c["k_s"]), float(c["b_s"]), int(c.get("n_sat", 1_000_000)),
                                                   float(c.get("gamma", 1.0)), int(c.get("intermediate_base_bytes", 0)),
                                                   int(c.get("intermediate_per_item_bytes", 0)))

    def exec_latency(self, arch, proc, n, k_scale=1.0):  # costmodel.py:55-64
        k_s, b_s, n_sat, gamma, _, _ = self.const[(arch, proc)]
        k = k_s * k_scale
        if n <= n_sat:
            return k * n + b_s
        return k * n_sat + b_s + gamma * k * (n - n_sat)

    def load_latency(self, tier, nbytes):  # costmodel.py:69-73
        _, bw, ovh = self.tiers[tier]
        return nbytes / bw + ovh

    def inference_memory(self, arch, proc, n):  # costmodel.py:75-82
        if n == 0:
            return 0
        _, _, _, _, base, item = self.const[(arch, proc)]
        return base + n * item

    def feasible_batch(self, arch, proc, free, hard_cap=4096):  # costmodel.py:84-92
        _, _, _, _, base, item = self.const[(arch, proc)]
        if free < base + item:
            return 0
        if item == 0:
            return hard_cap
        return min(int((free - base) // item), hard_cap)


def _fit(xs, ys):  # profiler.py:166-174 (CPython sum moments)
    n = len(xs)
    mx = sum(xs) / n
    my = sum(ys) / n
    var = sum((x - mx) ** 2 for x in xs)
    cov = sum((x - mx) * (y - my) for x, y in zip(xs, ys))
    k = cov / var
    return k, my - k * mx


def perf_profile(experts, device, mem_by_proc, plateau=0.02):
    """profiler.py:119-216 -> {(arch, proc): (max_batch, k, b)}"""
    biggest = {}
    for e in experts.values():
        biggest[e["arch"]] = max(biggest.get(e["arch"], 0), e["param_bytes"])
    out = {}
    for arch in sorted(biggest):
        for proc in sorted(mem_by_proc):
            if mem_by_proc[proc] <= 0:
                continue
            feasible = device.feasible_batch(arch, proc, mem_by_proc[proc])
            if feasible < 1:
                raise ValueError("memory budget cannot hold a single-item batch")
            mb = feasible
            for n in range(1, feasible):
                a = device.exec_latency(arch, proc, n) / n
                b = device.exec_latency(arch, proc, n + 1) / (n + 1)
                if (a - b) / a < plateau:
                    mb = n
                    break
            if mb >= 2:
                xs = list(range(1, mb + 1))
                ys = [device.exec_latency(arch, proc, n) for n in xs]
                s0 = ys[1] - ys[0]
                cut = len(xs)
                for i in range(2, len(xs)):
                    if abs((ys[i] - ys[i - 1]) - s0) > 1e-9 * max(abs(s0), 1e-300):
                        cut = i
                        break
                k, b = _fit(xs[:cut], ys[:cut])
            else:
                k, b = device.const[(arch, proc)][0], device.const[(arch, proc)][1]
            out[(arch, proc)] = (mb, k, b)
    return out


def partition(device, gpu, cpu, cpu_frac):  # engine.py:192-224
    per = {}
    if device.arch == "numa":
        if gpu:
            per["gpu"] = device.tiers["device"][0] / gpu
        host = device.tiers["host"][0]
        cpu_total = host * cpu_frac if cpu else 0.0
        if cpu:
            per["cpu"] = cpu_total / cpu
        return per, host - cpu_total
    share = device.tiers["device"][0] / (gpu + cpu)
    if gpu:
        per["gpu"] = share
    if cpu:
        per["cpu"] = share
    return per, 0.0


class _Run:
    """One simulation (engine.py:356-824) on documents."""

    def __init__(self, registry, device_doc, requests, opts, perf=None):
        self.opts = opts
        self.experts = {e["expert_id"]: e for e in registry["experts"]}
        self.usage = {eid: float(e["usage_prob"]) for eid, e in self.experts.items()}
        self.device = Device(device_doc)
        self.assign_mode, self.arrange, self.evict, single, self.host_mode = POLICY_TABLE[opts["policy"]]
        gpu, cpu = opts["gpu_executors"], opts["cpu_executors"]
        if single and opts.get("samba_gpu_only", True):
            gpu, cpu = 1, 0
        self.gpu, self.cpu = gpu, cpu
        self.per_exec, self.host_budget = partition(self.device, gpu, cpu, opts["cpu_mem_fraction"])
        self.perf = perf or perf_profile(self.experts, self.device, self.per_exec, opts["plateau_threshold"])
        self.registry = registry
        self.alloc = self._allocation()
        self.ex = []
        for proc, n in (("gpu", gpu), ("cpu", cpu)):
            for _ in range(n):
                self.ex.append({
                    "id": len(self.ex), "proc": proc, "budget": self.alloc[proc]["expert_budget_bytes"],
                    "inf": self.alloc[proc]["inference_budget_bytes"],
                    "k_scale": opts["contention_factor"] ** (n - 1),
                    "resident": {}, "used": 0, "pinned": set(), "stamp": {}, "clock": 0,
                    "queue": [], "counts": {}, "total": 0.0, "busy": False, "busy_s": 0.0, "switches": 0,
                })
        self.routes = opts.get("routes") or {}
        self.rules = {r["component_type"]: r for r in registry["rules"]}
        self.requests = {}
        for r in requests:
            self.requests[r["request_id"]] = dict(r)
        self.rr = 0
        peer = opts.get("peer_tier")
        self.peer = None if peer is None else (float(peer["read_bandwidth_bytes_per_s"]),
                                               float(peer["fixed_load_overhead_s"]))

    # -- allocation (engine.py:412-495) --------------------------------------
    def _desc(self):
        return sorted(self.experts.values(), key=lambda e: (-float(e["usage_prob"]), e["expert_id"]))

    def _allocation(self):
        desc = self._desc()
        cum = [0]
        for e in desc:
            cum.append(cum[-1] + e["param_bytes"])
        biggest = max(e["param_bytes"] for e in desc)
        arches = sorted({e["arch"] for e in desc})
        lanes = {"gpu": self.gpu, "cpu": self.cpu}
        overrides = dict(self.opts.get("alloc_override") or {})
        alloc = {}
        self.window = {}
        for proc in sorted(self.per_exec):
            mem = self.per_exec[proc]
            min_inf = max(self.device.inference_memory(a, proc, 1) for a in arches)
            if mem < biggest + min_inf:
                raise OracleStarvation("executor memory cannot hold the largest expert plus one item")
            chosen = None
            if proc in overrides:
                chosen = max(1, min(int(overrides[proc]), len(desc)))
                budget = cum[chosen] / lanes[proc]
            else:
                search = False
                for a in arches:
                    mb = self.perf[(a, proc)][0]
                    if not self.device.inference_memory(a, proc, mb) <= self.opts["alloc_threshold"] * mem:
                        search = True
                if search and self.opts.get("search_enabled", False):
                    lo, hi, chosen = self._window_search(proc)
                    self.window[proc] = (lo, hi, chosen)
                    chosen = max(1, min(chosen, len(desc)))
                    budget = cum[chosen] / lanes[proc]
                else:
                    budget = mem - max(self.device.inference_memory(a, proc, self.perf[(a, proc)][0]) for a in arches)
            budget = min(max(budget, biggest), mem - min_inf)
            alloc[proc] = {"expert_budget_bytes": budget, "inference_budget_bytes": mem - budget,
                           "experts_chosen": chosen}
        return alloc

    def _window_search(self, proc):  # profiler.py:281-354 with engine.py:462-495 probes
        opts = self.opts
        sample = self._stream_list[: min(opts.get("search_sample_requests", 400), len(self._stream_list))]
        overrides = dict(opts.get("alloc_override") or {})

        def probe(count):
            sub = dict(opts, seed=_subseed(opts["seed"], "alloc-sample"), alloc_override={**overrides, proc: count},
                       search_enabled=False, trace=False)
            r = _Run(self.registry, self._device_doc, sample, sub, perf=self.perf)
            return r.run()["metrics"]["throughput_rps"]

        desc = self._desc()
        arches = sorted({e["arch"] for e in desc})
        per, _ = partition(self.device, self.gpu, self.cpu, opts["cpu_mem_fraction"])
        cap = (per[proc] - max(self.device.inference_memory(a, proc, 1) for a in arches)) * \
            (self.gpu if proc == "gpu" else self.cpu)
        max_count = len(desc)
        acc = 0
        for n, e in enumerate(desc, start=1):
            acc += e["param_bytes"]
            if acc >= cap:
                max_count = n
                break
        w0 = opts.get("initial_window", 15)
        margin = opts.get("error_margin", 0.05)
        fit_points = opts.get("fit_points", 3)
        decay = 1.0 - w0 / 100.0
        size = float(w0)
        lo, hi = 0, min(w0, max_count)
        samples = []
        fit = None
        while True:
            thr = probe(hi)
            samples.append((hi, thr))
            m = len(samples)
            if m == fit_points:
                fit = _fit(list(range(1, m + 1)), [t for _, t in samples])
            if fit is not None and m > fit_points:
                pred = fit[0] * m + fit[1]
                if pred > 0:
                    if (pred - thr) / pred > margin:
                        break
                else:
                    break
            if hi >= max_count or decay <= 0.0:
                break
            size *= decay
            lo, hi = hi, min(hi + max(1, math.ceil(size)), max_count)
        if opts.get("window_choose", "random") == "midpoint":
            chosen = max(1, (lo + hi + 1) // 2)
        else:
            chosen = random.Random(_subseed(_subseed(opts["seed"], "alloc", proc), "window-choice")).randint(
                max(1, lo), max(1, hi))
        return lo, hi, chosen

    # -- residency (expert_pool.py:62-87, engine.py:528-548) -------------------
    def _initial(self):
        desc = self._desc()
        turn = 0
        placed = [[] for _ in self.ex]
        for e in desc:
            target = None
            for s in range(len(self.ex)):
                i = (turn + s) % len(self.ex)
                x = self.ex[i]
                if e["param_bytes"] <= x["budget"] - x["used"]:
                    target = i
                    break
            if target is None:
                break
            x = self.ex[target]
            x["resident"][e["expert_id"]] = e["param_bytes"]
            x["used"] += e["param_bytes"]
            placed[target].append(e["expert_id"])
            turn = (target + 1) % len(self.ex)
        for x, ids in zip(self.ex, placed):
            if self.evict in ("lru", "fifo"):
                for eid in ids:
                    x["stamp"][eid] = x["clock"]
                    x["clock"] += 1
        self.initial = placed
        self.hc = None
        if self.device.arch == "numa" and self.host_budget > 0:
            self.hc = {"res": {}, "used": 0, "stamp": {}, "clock": 0}
            anywhere = {eid for x in self.ex for eid in x["resident"]}
            for e in desc:
                if e["expert_id"] in anywhere:
                    continue
                if self.hc["used"] + e["param_bytes"] <= self.host_budget:
                    self._hc_insert(e["expert_id"], e["param_bytes"])

    def _hc_insert(self, eid, nbytes):  # engine.py:308-330
        hc = self.hc
        if eid in hc["res"]:
            if self.host_mode == "lru":
                hc["stamp"][eid] = hc["clock"]
                hc["clock"] += 1
            return
        if nbytes > self.host_budget:
            return
        while hc["used"] + nbytes > self.host_budget:
            if self.host_mode == "prob":
                v = min(hc["res"], key=lambda k: (self.usage.get(k, 0.0), -hc["res"][k], k))
            else:
                v = min(hc["res"], key=lambda k: (hc["stamp"].get(k, -1), k))
            hc["used"] -= hc["res"].pop(v)
            hc["stamp"].pop(v, None)
        hc["res"][eid] = nbytes
        hc["used"] += nbytes
        hc["stamp"][eid] = hc["clock"]
        hc["clock"] += 1

    def _tier(self, eid):  # engine.py:579-582
        return "host" if self.hc is not None and eid in self.hc["res"] else "ssd"

    def _peer_src(self, eid):
        """(f3) lowest-id GPU executor holding eid and not loading it right now, else None."""
        if self.peer is None:
            return None
        for x in self.ex:
            if x["proc"] == "gpu" and eid in x["resident"] and x.get("loading") != eid:
                return x["id"]
        return None

    def _load_s(self, eid):  # engine.py:583-586 (predictions keep the host/ssd tier)
        return self.device.load_latency(self._tier(eid), self.experts[eid]["param_bytes"])

    # -- event loop ----------------------------------------------------------
    def _push(self, t, kind, data):
        heapq.heappush(self.heap, (t, self.seq, kind, data))
        self.seq += 1

    def _rec(self, t, ex, ev, eid, rid):
        if self.opts.get("trace", True):
            self.trace.append({"time_s": t, "executor": ex, "event": ev, "expert_id": eid, "request_id": rid})

    def _admit(self, t, req, follow_up):  # engine.py:588-626
        eid = req["chain"][0]
        arch = self.experts[eid]["arch"]

        def parts(x, load_s):  # scheduler.py:51-61
            mb, k, b = self.perf[(arch, x["proc"])]
            queued = x["counts"].get(eid, 0) > 0
            ex_part = k if queued else k + b
            sw = 0.0 if (queued or eid in x["resident"]) else load_s
            return ex_part, sw

        if self.assign_mode == "makespan":  # scheduler.py:72-97
            load_s = self._load_s(eid)
            totals = [x["total"] for x in self.ex]
            best = None
            for i, x in enumerate(self.ex):
                e_p, s_p = parts(x, load_s)
                added = e_p + s_p
                span = max(totals[i] + added, max((v for j, v in enumerate(totals) if j != i), default=0.0))
                key = (span, added, x["id"])
                if best is None or key < best:
                    best = key
            target = self.ex[best[2]]
        else:
            target = self.ex[self.rr]
            self.rr = (self.rr + 1) % len(self.ex)
        e_p, s_p = parts(target, self._load_s(eid))
        entry = [req["request_id"], eid, e_p, s_p, False, False, follow_up, req["stage"]]
        q = target["queue"]
        pos = len(q)
        if self.arrange:  # scheduler.py:100-108
            for i in range(len(q) - 1, -1, -1):
                if q[i][1] == eid:
                    pos = i + 1
                    break
        q.insert(pos, entry)
        target["counts"][eid] = target["counts"].get(eid, 0) + 1
        target["total"] += e_p + s_p
        self._rec(t, target["id"], "assign", eid, req["request_id"])
        if not target["busy"]:
            self._push(t, "wake", target["id"])

    def _select(self, x, need):
        deficit = need - (x["budget"] - x["used"])
        if deficit <= 0:
            return []
        victims, got = [], 0.0
        if self.evict == "two_stage":  # expert_pool.py:96-148
            pending = {e[1] for e in x["queue"] if not e[4]}
            one = []
            for eid, nb in x["resident"].items():
                ups = self.experts[eid]["upstream"]
                if eid in x["pinned"] or eid in pending or not ups:
                    continue
                if any(u in x["resident"] for u in ups):
                    continue
                one.append((eid, nb))
            one.sort(key=lambda p: (-p[1], p[0]))
            for eid, nb in one:
                if got >= deficit:
                    break
                victims.append(eid)
                got += nb
            if got >= deficit:
                return victims
            rest = [(eid, nb) for eid, nb in x["resident"].items() if eid not in x["pinned"] and eid not in victims]
            rest.sort(key=lambda p: (self.usage[p[0]], -p[1], p[0]))
        else:  # baselines.py:54-73
            rest = sorted(((eid, nb) for eid, nb in x["resident"].items() if eid not in x["pinned"]),
                          key=lambda p: (x["stamp"].get(p[0], -1), p[0]))
        for eid, nb in rest:
            if got >= deficit:
                break
            victims.append(eid)
            got += nb
        if got < deficit:
            raise OracleStarvation("evicting every unpinned expert is not enough")
        return victims

    def _step(self, t, x):  # engine.py:630-716
        if x["busy"]:
            return
        q = x["queue"]
        start = 0
        while start < len(q) and q[start][4]:
            start += 1
        if start == len(q):
            return
        eid = q[start][1]
        run = []
        for e in q[start:]:
            if e[4] or e[1] != eid:
                break
            run.append(e)
        spec = self.experts[eid]
        if eid not in x["resident"]:
            if spec["param_bytes"] > x["budget"]:
                raise OracleStarvation("expert exceeds the expert budget")
            victims = self._select(x, spec["param_bytes"])
            for v in victims:
                nb = x["resident"].pop(v)
                x["used"] -= nb
                self.evictions += 1
                self._rec(t, x["id"], "evict", v, None)
                if self.hc is not None and x["proc"] == "gpu":
                    self._hc_insert(v, nb)
                if x["counts"].get(v, 0):  # engine.py:679-691
                    for e in q:
                        if e[1] == v and not e[4]:
                            if e[3] == 0.0 and not e[5]:
                                lat = self._load_s(v)
                                e[3] = lat
                                e[5] = True
                                x["total"] += lat
                            break
            src = self._peer_src(eid)
            if src is not None:  # (f3) NVLink copy from another GPU's pool
                tier = "peer"
                lat = spec["param_bytes"] / self.peer[0] + self.peer[1]
            else:
                tier = self._tier(eid)
                lat = self.device.load_latency(tier, spec["param_bytes"])
            x["loading"] = eid
            x["resident"][eid] = spec["param_bytes"]
            x["used"] += spec["param_bytes"]
            if self.evict in ("lru", "fifo"):
                x["stamp"][eid] = x["clock"]
                x["clock"] += 1
            if tier == "host" and self.host_mode == "lru":
                self.hc["stamp"][eid] = self.hc["clock"]
                self.hc["clock"] += 1
            x["switches"] += 1
            head = run[0]
            if head[5] or head[3] == 0.0:
                self.stale += 1
                head[5] = False
            x["busy"] = True
            x["busy_s"] += lat
            self.loads.append((x["id"], eid, victims, tier))
            self.load_src.append(src)
            self.ops.append(("load", x["id"], eid, list(victims)))
            self._rec(t, x["id"], "load", eid, None)
            self._push(t + lat, "load_done", x["id"])
            return
        mb, _, _ = self.perf[(spec["arch"], x["proc"])]
        cap = 0
        while cap < mb and self.device.inference_memory(spec["arch"], x["proc"], cap + 1) <= x["inf"]:
            cap += 1
        if cap < 1:
            raise OracleStarvation("no single-item batch fits")
        batch = run[:cap]
        for e in batch:
            e[4] = True
        x["pinned"].add(eid)
        if self.evict == "lru":
            x["stamp"][eid] = x["clock"]
            x["clock"] += 1
        dur = self.device.exec_latency(spec["arch"], x["proc"], len(batch), k_scale=x["k_scale"])
        x["busy"] = True
        x["busy_s"] += dur
        self.batches.append((x["id"], eid, [(e[0], e[7]) for e in batch]))
        self.ops.append(("batch", x["id"], eid, [(e[0], e[7]) for e in batch]))
        self._rec(t, x["id"], "batch_start", eid, None)
        self._push(t + dur, "batch_done", (x["id"], len(batch), eid))

    def _batch_done(self, t, x, n, eid):  # engine.py:740-758
        x["busy"] = False
        x["pinned"].discard(eid)
        done = x["queue"][:n]
        del x["queue"][:n]
        for e in done:
            c = x["counts"][e[1]] - 1
            if c:
                x["counts"][e[1]] = c
            else:
                del x["counts"][e[1]]
            x["total"] -= e[2] + e[3]
        if not x["queue"]:
            x["total"] = 0.0
        self._rec(t, x["id"], "batch_done", eid, None)
        for e in done:
            req = self.requests[e[0]]
            req["chain"].pop(0)
            req["stage"] += 1
            if e[6]:
                self.fu_done += 1
            if req["chain"]:
                self.fu_made += 1
                self._push(t, "follow_up", e[0])
            else:
                self.completed += 1
                self.last = t
                self._rec(t, x["id"], "complete", eid, e[0])
        self._push(t, "wake", x["id"])

    def _chain(self, req):  # engine.py:720-727 (+ N-stage routes)
        route = self.routes.get(req["component_type"])
        if route is None:
            rule = self.rules[req["component_type"]]
            experts = [rule["classification_expert_id"]]
            prob = 0.0
            if rule.get("detection_expert_id") is not None:
                experts.append(rule["detection_expert_id"])
                prob = float(rule.get("detection_prob", 0.0))
        else:
            experts, prob = list(route["experts"]), float(route["branch_prob"])
        if len(experts) > 1 and req["detect_u"] < prob:
            return experts
        return experts[:1]

    def run(self):
        self._initial()
        self.heap, self.seq, self.trace = [], 0, []
        self.batches, self.loads, self.ops, self.load_src = [], [], [], []
        self.completed = self.fu_made = self.fu_done = self.evictions = self.stale = 0
        self.last = 0.0
        for rid in self.requests:
            self._push(self.requests[rid]["arrival_time_s"], "arrival", rid)
        while self.heap:
            t, _, kind, data = heapq.heappop(self.heap)
            if kind == "arrival":
                req = self.requests[data]
                req["chain"] = self._chain(req)
                req["stage"] = 0
                self._rec(t, None, "arrival", None, data)
                self._admit(t, req, False)
            elif kind == "follow_up":
                req = self.requests[data]
                self._rec(t, None, "follow_up", req["chain"][0], data)
                self._admit(t, req, True)
            elif kind == "wake":
                self._step(t, self.ex[data])
            elif kind == "load_done":
                self.ex[data]["busy"] = False
                self.ex[data]["loading"] = None
                self._rec(t, data, "load_done", None, None)
                self._step(t, self.ex[data])
            else:
                self._batch_done(t, self.ex[data[0]], data[1], data[2])
        if self.completed != len(self.requests) or self.fu_made != self.fu_done:
            raise RuntimeError("conservation violated")
        span = self.last
        per = [{"executor": x["id"], "proc": x["proc"], "busy_s": x["busy_s"],
                "busy_fraction": x["busy_s"] / span if span > 0 else 0.0, "switches": x["switches"]}
               for x in self.ex]
        metrics = {
            "schema_version": 1, "policy": self.opts["policy"], "seed": self.opts["seed"],
            "completed_requests": self.completed, "follow_ups": self.fu_done, "makespan_s": span,
            "throughput_rps": self.completed / span if span > 0 else 0.0,
            "expert_switches": sum(x["switches"] for x in self.ex), "evictions": self.evictions,
            "stale_predictions": self.stale, "busy_s_total": sum(x["busy_s"] for x in self.ex),
            "per_executor": per, "alloc": {p: self.alloc[p] for p in sorted(self.alloc)},
        }
        return {"metrics": metrics, "trace": self.trace, "batches": self.batches, "loads": self.loads,
                "ops": self.ops, "initial": self.initial, "load_src": self.load_src}


DEFAULTS = {
    "policy": "coserve", "seed": 0, "gpu_executors": 3, "cpu_executors": 1, "contention_factor": 1.15,
    "cpu_mem_fraction": 0.4, "alloc_override": None, "alloc_threshold": 0.15, "plateau_threshold": 0.02,
    "initial_window": 15, "error_margin": 0.05, "fit_points": 3, "search_enabled": True,
    "search_sample_requests": 400, "window_choose": "random", "samba_gpu_only": True, "trace": True,
    "routes": None, "peer_tier": None,
}


def simulate(registry_doc, device_doc, stream_doc, **opts):
    """Run one configuration; ``opts`` mirror RunConfig fields (engine.py:79-103)."""
    full = dict(DEFAULTS)
    full.update(opts)
    requests = [dict(r) for r in stream_doc["requests"]]
    run = _Run.__new__(_Run)
    run._stream_list = requests
    run._device_doc = device_doc
    _Run.__init__(run, registry_doc, device_doc, requests, full)
    return run.run()


def metrics_json(doc) -> str:
    import json
    return json.dumps(doc, sort_keys=True, indent=2) + "\n"


def trace_jsonl(trace) -> str:
    import json
    return "".join(json.dumps(r, sort_keys=True, separators=(",", ":")) + "\n" for r in trace)
