// planner.cpp -- bit-exact virtual-clock planner of the CoE serving path.
//
// Re-states the reference engine's decision cycle
// (/root/reference/pkg/src/coesim/engine.py:588-795) as a native event loop
// over struct-of-arrays state.  What is *different* from the reference, and
// why it is still bit-exact:
//
//  * Queues are kept as a deque of runs, each run a FIFO of entries.  Under
//    the `arrange` policy an admission joins its expert's live run or opens a
//    new run at the tail (run_rank = creation counter); under FCFS it joins
//    the tail run iff that run has the same expert.  The queue order is then
//    exactly the stable sort by (run_rank, admission seq) that the
//    reference's arrange_position + list.insert produces (scheduler.py:100-108,
//    engine.py:251-254), in O(1) per admission instead of an
//    O(queue) backward scan.
//  * Per (executor, expert) FIFOs give the live count (QueueView.expert_counts,
//    engine.py:569-577) and the first pending same-expert entry that
//    _invalidate_prediction charges (engine.py:679-691).
//  * All float64 arithmetic keeps the reference's operation order; the file is
//    compiled with -ffp-contract=off so no FMA can change a rounding.
//
// The loop additionally emits the physical op log (LOAD / BATCH per executor)
// and one admission record per (request, stage) for the GPU grouping kernel.

#include "coe_planner.h"
#include "hops.h"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <deque>
#include <queue>
#include <string>
#include <vector>

namespace {

thread_local std::string g_error;

struct PlanError {
  int code;
  std::string msg;
};

[[noreturn]] void fail(int code, const std::string &msg) { throw PlanError{code, msg}; }

std::string fmt_num(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", v);
  return buf;
}

enum EvKind : uint8_t { K_ARRIVAL, K_FOLLOW_UP, K_WAKE, K_LOAD_DONE, K_BATCH_DONE };

struct Event {
  double t;
  uint64_t seq;
  uint8_t kind;
  int32_t a, b, c;
};

struct EventLater {
  bool operator()(const Event &x, const Event &y) const {
    if (x.t != y.t) return x.t > y.t;
    return x.seq > y.seq;
  }
};

struct Entry {
  int32_t req;
  int32_t stage;
  int32_t expert;
  double pred_exec;
  double pred_switch;
  bool in_flight;
  bool stale;
  bool follow_up;
};

struct Run {
  int32_t expert;
  int32_t rank;
  std::vector<int32_t> ents;  // entry ids in seq order
  size_t head = 0;            // ents[head:] still queued
  size_t size() const { return ents.size() - head; }
};

struct Executor {
  int32_t id;
  int32_t proc;
  double expert_budget;
  double inference_budget;
  double k_scale;
  // ModelPool (expert_pool.py:27-59)
  std::vector<uint8_t> resident;
  std::vector<int32_t> res_list;   // resident experts (order irrelevant: selections sort on unique keys)
  std::vector<int32_t> res_pos;
  std::vector<uint8_t> pinned;
  int64_t used_bytes = 0;
  // LRU / FIFO stamps (baselines.py:20-51)
  int64_t clock = 0;
  std::vector<int64_t> stamp;
  // queue
  std::deque<int32_t> runs;        // run ids, queue order
  std::vector<int32_t> live_run;   // expert -> run id holding its entries (arrange)
  std::vector<std::deque<int32_t>> by_expert;  // expert -> entry ids in queue order
  int64_t queue_len = 0;
  double total_pending = 0.0;
  int32_t next_rank = 0;
  bool busy = false;
  double busy_s = 0.0;
  int64_t switches = 0;
  int32_t batches = 0;
  int32_t loading = -1;            // expert of the load in flight (f3 peer tier), else -1

  double free_bytes() const { return expert_budget - (double)used_bytes; }
};

struct HostCache {
  bool enabled = false;
  int mode = 0;  // 0 prob, 1 lru, 2 fifo
  double budget = 0.0;
  int64_t used = 0;
  int64_t clock = 0;
  std::vector<uint8_t> resident;
  std::vector<int64_t> size;
  std::vector<int64_t> stamp;
  std::vector<int32_t> res_list;
  std::vector<int32_t> res_pos;
};

}  // namespace

struct coe_plan {
  // ---- configuration (copied) ----
  int32_t E = 0, A = 0, X = 0, R = 0;
  std::vector<int64_t> bytes;
  std::vector<double> usage;
  std::vector<int32_t> arch;
  std::vector<int32_t> up_off, up_idx;
  std::vector<int32_t> desc;
  std::vector<uint8_t> perf_valid, cost_valid;
  std::vector<int32_t> perf_max_batch;
  std::vector<double> perf_k, perf_b, cost_k, cost_b, cost_gamma;
  std::vector<int64_t> cost_nsat, cost_base, cost_item;
  int32_t numa = 1;
  double host_bw = 1, host_ovh = 0, ssd_bw = 1, ssd_ovh = 0;
  int32_t peer_enabled = 0;
  double peer_bw = 1, peer_ovh = 0;
  int32_t host_mode = -1;
  double host_budget = 0;
  int32_t assign_makespan = 1, arrange = 1, evict = 0;
  std::vector<int64_t> req_id;
  std::vector<double> arrival;
  std::vector<int32_t> chain_off, chain_exp;
  bool record_trace = false, record_ops = false;

  // ---- state ----
  std::vector<Executor> ex;
  HostCache hc;
  std::vector<Entry> entries;
  std::vector<Run> runs;
  std::vector<int32_t> req_stage;
  std::priority_queue<Event, std::vector<Event>, EventLater> heap;
  uint64_t seq = 0;
  int32_t rr_next = 0;
  std::vector<int32_t> init_off, init_exp;

  // ---- outputs ----
  int64_t completed = 0, fu_generated = 0, fu_completed = 0, evictions = 0, stale = 0;
  double last_completion = 0.0;
  double sched_wall = 0.0;
  int64_t sched_calls = 0;
  std::vector<double> tr_t;
  std::vector<int32_t> tr_ex, tr_ev, tr_exp;
  std::vector<int64_t> tr_req;
  std::vector<coe_op> ops;
  std::vector<int32_t> op_args;
  std::vector<coe_admission> adms;
  bool ran = false;

  // ------------------------------------------------------------------
  int pa(int32_t a, int32_t proc) const { return a * 2 + proc; }

  void push(double t, uint8_t kind, int32_t a = 0, int32_t b = 0, int32_t c = 0) {
    heap.push(Event{t, seq++, kind, a, b, c});
  }

  void record(double t, int32_t exid, int32_t ev, int32_t expert, int32_t req) {
    if (!record_trace) return;
    tr_t.push_back(t);
    tr_ex.push_back(exid);
    tr_ev.push_back(ev);
    tr_exp.push_back(expert);
    tr_req.push_back(req < 0 ? -1 : req_id[req]);
  }

  // costmodel.py:69-73
  double load_latency_from(int tier, int64_t nbytes) const {
    if (tier == COE_TIER_HOST) return (double)nbytes / host_bw + host_ovh;
    if (tier == COE_TIER_PEER) return (double)nbytes / peer_bw + peer_ovh;
    return (double)nbytes / ssd_bw + ssd_ovh;
  }
  int source_tier(int32_t e) const {  // engine.py:579-582
    return (hc.enabled && hc.resident[e]) ? COE_TIER_HOST : COE_TIER_SSD;
  }
  // switch-cost predictions (engine.py:583-586): the reference's tier, also with a peer tier
  double load_latency(int32_t e) const { return load_latency_from(source_tier(e), bytes[e]); }
  // (f3) lowest-id GPU executor holding e that is not loading it right now, else -1
  int32_t peer_source(int32_t e) const {
    if (!peer_enabled) return -1;
    for (const Executor &y : ex)
      if (y.proc == 0 && y.resident[e] && y.loading != e) return y.id;
    return -1;
  }

  // costmodel.py:55-64
  double exec_latency(int32_t a, int32_t proc, int64_t n, double k_scale) const {
    int i = pa(a, proc);
    if (!cost_valid[i]) fail(COE_ERR_CONFIG, "device has no execution constants for arch on processor");
    double k = cost_k[i] * k_scale;
    int64_t nsat = cost_nsat[i];
    if (n <= nsat) return k * (double)n + cost_b[i];
    return k * (double)nsat + cost_b[i] + cost_gamma[i] * k * (double)(n - nsat);
  }
  // costmodel.py:75-82
  int64_t inference_memory(int32_t a, int32_t proc, int64_t n) const {
    if (n == 0) return 0;
    int i = pa(a, proc);
    if (!cost_valid[i]) fail(COE_ERR_CONFIG, "device has no execution constants for arch on processor");
    return cost_base[i] + n * cost_item[i];
  }
  void need_perf(int32_t a, int32_t proc) const {
    if (!perf_valid[pa(a, proc)]) fail(COE_ERR_CONFIG, "profile has no entry for arch on processor");
  }

  // ---- pool (expert_pool.py:27-59) -------------------------------------
  void pool_add(Executor &x, int32_t e) {
    if (x.resident[e]) fail(COE_ERR_VALUE, "expert already resident in pool " + std::to_string(x.id));
    if ((double)bytes[e] > x.free_bytes())
      fail(COE_ERR_STARVATION, "pool " + std::to_string(x.id) + ": " + std::to_string(bytes[e]) +
                                   " bytes do not fit in " + fmt_num(x.free_bytes()) + " free");
    x.resident[e] = 1;
    x.res_pos[e] = (int32_t)x.res_list.size();
    x.res_list.push_back(e);
    x.used_bytes += bytes[e];
  }
  int64_t pool_remove(Executor &x, int32_t e) {
    if (x.pinned[e]) fail(COE_ERR_VALUE, "expert is pinned and cannot be removed");
    if (!x.resident[e]) fail(COE_ERR_VALUE, "expert not resident");
    int32_t pos = x.res_pos[e];
    int32_t last = x.res_list.back();
    x.res_list[pos] = last;
    x.res_pos[last] = pos;
    x.res_list.pop_back();
    x.resident[e] = 0;
    x.used_bytes -= bytes[e];
    return bytes[e];
  }

  // ---- host cache (engine.py:289-330) -----------------------------------
  void hc_note_read(int32_t e) {
    if (hc.mode == 1 && hc.resident[e]) hc.stamp[e] = hc.clock++;
  }
  int32_t hc_victim() const {
    int32_t best = -1;
    for (int32_t e : hc.res_list) {
      if (best < 0) { best = e; continue; }
      bool less;
      if (hc.mode == 0) {  // (usage_prob, -bytes, id)
        if (usage[e] != usage[best]) less = usage[e] < usage[best];
        else if (hc.size[e] != hc.size[best]) less = hc.size[e] > hc.size[best];
        else less = e < best;
      } else {  // (stamp, id)
        if (hc.stamp[e] != hc.stamp[best]) less = hc.stamp[e] < hc.stamp[best];
        else less = e < best;
      }
      if (less) best = e;
    }
    return best;
  }
  void hc_insert(int32_t e, int64_t nbytes) {
    if (hc.resident[e]) { hc_note_read(e); return; }
    if ((double)nbytes > hc.budget) return;
    while ((double)(hc.used + nbytes) > hc.budget) {
      int32_t v = hc_victim();
      hc.used -= hc.size[v];
      hc.resident[v] = 0;
      hc.stamp[v] = -1;
      int32_t pos = hc.res_pos[v];
      int32_t last = hc.res_list.back();
      hc.res_list[pos] = last;
      hc.res_pos[last] = pos;
      hc.res_list.pop_back();
    }
    hc.resident[e] = 1;
    hc.size[e] = nbytes;
    hc.res_pos[e] = (int32_t)hc.res_list.size();
    hc.res_list.push_back(e);
    hc.used += nbytes;
    hc.stamp[e] = hc.clock++;
  }

  // ---- evictors ----------------------------------------------------------
  bool has_live_upstream(const Executor &x, int32_t e) const {
    for (int32_t i = up_off[e]; i < up_off[e + 1]; ++i)
      if (x.resident[up_idx[i]]) return true;
    return false;
  }

  // expert_pool.py:96-148
  std::vector<int32_t> select_two_stage(const Executor &x, int64_t needed) const {
    std::vector<int32_t> victims;
    double deficit = (double)needed - x.free_bytes();
    if (deficit <= 0) return victims;
    std::vector<int32_t> one;
    for (int32_t e : x.res_list) {
      if (x.pinned[e] || !x.by_expert[e].empty()) continue;  // pending targets
      if (up_off[e] == up_off[e + 1]) continue;
      if (has_live_upstream(x, e)) continue;
      one.push_back(e);
    }
    std::sort(one.begin(), one.end(), [&](int32_t p, int32_t q) {
      if (bytes[p] != bytes[q]) return bytes[p] > bytes[q];
      return p < q;
    });
    double reclaimed = 0.0;
    for (int32_t e : one) {
      if (reclaimed >= deficit) break;
      victims.push_back(e);
      reclaimed += (double)bytes[e];
    }
    if (reclaimed >= deficit) return victims;
    std::vector<uint8_t> taken(E, 0);
    for (int32_t e : victims) taken[e] = 1;
    std::vector<int32_t> two;
    for (int32_t e : x.res_list)
      if (!x.pinned[e] && !taken[e]) two.push_back(e);
    std::sort(two.begin(), two.end(), [&](int32_t p, int32_t q) {
      if (usage[p] != usage[q]) return usage[p] < usage[q];
      if (bytes[p] != bytes[q]) return bytes[p] > bytes[q];
      return p < q;
    });
    for (int32_t e : two) {
      if (reclaimed >= deficit) break;
      victims.push_back(e);
      reclaimed += (double)bytes[e];
    }
    if (reclaimed < deficit)
      fail(COE_ERR_STARVATION, "pool " + std::to_string(x.id) + ": evicting every unpinned expert frees " +
                                   fmt_num(reclaimed) + " bytes, still short of " + fmt_num(deficit));
    return victims;
  }

  // baselines.py:54-73
  std::vector<int32_t> select_stamped(const Executor &x, int64_t needed) const {
    std::vector<int32_t> victims;
    double deficit = (double)needed - x.free_bytes();
    if (deficit <= 0) return victims;
    std::vector<int32_t> cand;
    for (int32_t e : x.res_list)
      if (!x.pinned[e]) cand.push_back(e);
    std::sort(cand.begin(), cand.end(), [&](int32_t p, int32_t q) {
      if (x.stamp[p] != x.stamp[q]) return x.stamp[p] < x.stamp[q];
      return p < q;
    });
    double reclaimed = 0.0;
    for (int32_t e : cand) {
      if (reclaimed >= deficit) break;
      victims.push_back(e);
      reclaimed += (double)bytes[e];
    }
    if (reclaimed < deficit)
      fail(COE_ERR_STARVATION, "pool " + std::to_string(x.id) + ": evicting every unpinned expert frees " +
                                   fmt_num(reclaimed) + " bytes, still short of " + fmt_num(deficit));
    return victims;
  }

  // ---- queue -------------------------------------------------------------
  int32_t queue_insert(Executor &x, int32_t entry_id) {
    Entry &en = entries[entry_id];
    int32_t e = en.expert;
    int32_t run_id = -1;
    if (arrange) {
      if (!x.by_expert[e].empty()) run_id = x.live_run[e];
    } else if (!x.runs.empty()) {
      int32_t tail = x.runs.back();
      if (runs[tail].expert == e && runs[tail].size() > 0) run_id = tail;
    }
    if (run_id < 0) {
      run_id = (int32_t)runs.size();
      runs.push_back(Run{e, x.next_rank++, {}, 0});
      x.runs.push_back(run_id);
      if (arrange) x.live_run[e] = run_id;
    }
    runs[run_id].ents.push_back(entry_id);
    x.by_expert[e].push_back(entry_id);
    x.queue_len += 1;
    x.total_pending += en.pred_exec + en.pred_switch;  // engine.py:254
    return runs[run_id].rank;
  }

  // head_run (engine.py:270-283): queue order is run order; the executor is
  // idle whenever this is asked, so no entry is in flight.
  int32_t head_run(const Executor &x) const {
    for (int32_t rid : x.runs)
      if (runs[rid].size() > 0) return rid;
    return -1;
  }

  // ---- event handlers ----------------------------------------------------
  void admit(double t, int32_t r, bool follow_up) {
    int32_t stage = req_stage[r];
    int32_t e = chain_exp[chain_off[r] + stage];
    int32_t a = arch[e];
    auto started = std::chrono::steady_clock::now();
    int32_t target;
    if (assign_makespan) {
      // scheduler.assign (scheduler.py:72-97) over engine._view snapshots
      double load_s = load_latency(e);
      double top1 = -INFINITY, top2 = -INFINITY;
      int32_t top1_i = -1;
      for (int32_t i = 0; i < X; ++i) {
        double v = ex[i].total_pending;
        if (top1_i < 0 || v > top1) { top2 = top1; top1 = v; top1_i = i; }
        else if (v > top2) top2 = v;
      }
      bool have = false;
      double best_span = 0, best_added = 0;
      int32_t best_id = 0;
      for (int32_t i = 0; i < X; ++i) {
        Executor &x = ex[i];
        need_perf(a, x.proc);
        int pi = pa(a, x.proc);
        bool queued = !x.by_expert[e].empty();
        double exec_part = queued ? perf_k[pi] : perf_k[pi] + perf_b[pi];
        double switch_part = (queued || x.resident[e]) ? 0.0 : load_s;
        double added = exec_part + switch_part;
        double others = (X == 1) ? 0.0 : (i == top1_i ? top2 : top1);
        double own = x.total_pending + added;
        double span = (others > own) ? others : own;  // python max(own, others)
        if (!have || span < best_span || (span == best_span && (added < best_added ||
                                                                  (added == best_added && i < best_id)))) {
          have = true;
          best_span = span;
          best_added = added;
          best_id = i;
        }
      }
      target = best_id;
    } else {
      target = rr_next;
      rr_next = (rr_next + 1) % X;
    }
    Executor &x = ex[target];
    need_perf(a, x.proc);
    int pi = pa(a, x.proc);
    bool queued = !x.by_expert[e].empty();
    double exec_part = queued ? perf_k[pi] : perf_k[pi] + perf_b[pi];
    double switch_part = (queued || x.resident[e]) ? 0.0 : load_latency(e);
    int32_t entry_id = (int32_t)entries.size();
    entries.push_back(Entry{r, stage, e, exec_part, switch_part, false, false, follow_up});
    int32_t rank = queue_insert(x, entry_id);
    sched_wall += std::chrono::duration<double>(std::chrono::steady_clock::now() - started).count();
    sched_calls += 1;
    if (record_ops) adms.push_back(coe_admission{target, rank, r, stage});
    record(t, target, COE_EV_ASSIGN, e, r);
    if (!x.busy) push(t, K_WAKE, target);
  }

  void invalidate_prediction(Executor &x, int32_t victim) {  // engine.py:679-691
    if (x.by_expert[victim].empty()) return;
    Entry &en = entries[x.by_expert[victim].front()];
    if (en.pred_switch == 0.0 && !en.stale) {
      double lat = load_latency(victim);
      en.pred_switch = lat;
      en.stale = true;
      x.total_pending += lat;
    }
  }

  void start_load(double t, Executor &x, int32_t run_id) {  // engine.py:643-677
    Run &run = runs[run_id];
    int32_t e = run.expert;
    if ((double)bytes[e] > x.expert_budget)
      fail(COE_ERR_STARVATION, "expert " + std::to_string(e) + " (" + std::to_string(bytes[e]) +
                                   " bytes) exceeds the expert budget of executor " + std::to_string(x.id));
    std::vector<int32_t> victims =
        evict == 0 ? select_two_stage(x, bytes[e]) : select_stamped(x, bytes[e]);
    for (int32_t v : victims) {
      int64_t nb = pool_remove(x, v);
      evictions += 1;
      record(t, x.id, COE_EV_EVICT, v, -1);
      if (hc.enabled && x.proc == 0) hc_insert(v, nb);
      invalidate_prediction(x, v);
    }
    const int32_t peer_src = peer_source(e);
    int tier = peer_src >= 0 ? COE_TIER_PEER : source_tier(e);
    double latency = load_latency_from(tier, bytes[e]);
    pool_add(x, e);
    x.loading = e;
    if (evict == 1 || evict == 2) x.stamp[e] = x.clock++;  // LRU touch / FIFO on_resident
    if (tier == COE_TIER_HOST) hc_note_read(e);
    x.switches += 1;
    Entry &head = entries[run.ents[run.head]];
    if (head.stale || head.pred_switch == 0.0) {
      stale += 1;
      head.stale = false;
    }
    x.busy = true;
    x.busy_s += latency;
    if (record_ops) {
      coe_op op{};
      op.executor = x.id;
      op.kind = COE_OP_LOAD;
      op.expert = e;
      op.count = (int32_t)victims.size();
      op.offset = (int64_t)op_args.size();
      op.time_s = t;
      op.tier = tier;
      op.seq = peer_src;
      for (int32_t v : victims) op_args.push_back(v);
      ops.push_back(op);
    }
    record(t, x.id, COE_EV_LOAD, e, -1);
    push(t + latency, K_LOAD_DONE, x.id);
  }

  void start_batch(double t, Executor &x, int32_t run_id) {  // engine.py:693-716
    Run &run = runs[run_id];
    int32_t e = run.expert;
    int32_t a = arch[e];
    need_perf(a, x.proc);
    int64_t max_batch = perf_max_batch[pa(a, x.proc)];
    int64_t cap = 0;  // scheduler.batch_cap, scheduler.py:111-118
    while (cap < max_batch && (double)inference_memory(a, x.proc, cap + 1) <= x.inference_budget) cap += 1;
    if (cap < 1)
      fail(COE_ERR_STARVATION, "executor " + std::to_string(x.id) +
                                   " cannot fit a single-item batch in its inference memory");
    int64_t n = std::min<int64_t>(cap, (int64_t)run.size());
    if (record_ops) {
      coe_op op{};
      op.executor = x.id;
      op.kind = COE_OP_BATCH;
      op.expert = e;
      op.count = (int32_t)n;
      op.offset = (int64_t)op_args.size();
      op.time_s = t;
      op.tier = -1;
      op.seq = x.batches;
      ops.push_back(op);
    }
    x.batches += 1;
    for (int64_t i = 0; i < n; ++i) {
      Entry &en = entries[run.ents[run.head + i]];
      en.in_flight = true;
      if (record_ops) {
        op_args.push_back(en.req);
        op_args.push_back(en.stage);
      }
    }
    x.pinned[e] = 1;
    if (evict == 1) x.stamp[e] = x.clock++;  // LRU touch at batch start
    double duration = exec_latency(a, x.proc, n, x.k_scale);
    x.busy = true;
    x.busy_s += duration;
    record(t, x.id, COE_EV_BATCH_START, e, -1);
    push(t + duration, K_BATCH_DONE, x.id, (int32_t)n, e);
  }

  void step(double t, Executor &x) {  // engine.py:630-641
    if (x.busy) return;
    int32_t rid = head_run(x);
    if (rid < 0) return;
    if (!x.resident[runs[rid].expert]) start_load(t, x, rid);
    else start_batch(t, x, rid);
  }

  void on_batch_done(double t, Executor &x, int32_t n, int32_t e) {  // engine.py:740-758
    x.busy = false;
    x.pinned[e] = 0;
    // remove_prefix (engine.py:256-268): the batch is the head of the queue
    std::vector<int32_t> batch;
    batch.reserve(n);
    while ((int32_t)batch.size() < n) {
      int32_t rid = x.runs.front();
      Run &run = runs[rid];
      if (run.size() == 0) { x.runs.pop_front(); continue; }
      int32_t id = run.ents[run.head++];
      batch.push_back(id);
      Entry &en = entries[id];
      x.by_expert[en.expert].pop_front();
      x.queue_len -= 1;
      x.total_pending -= en.pred_exec + en.pred_switch;
      if (run.size() == 0) x.runs.pop_front();
    }
    if (x.queue_len == 0) x.total_pending = 0.0;
    record(t, x.id, COE_EV_BATCH_DONE, e, -1);
    for (int32_t id : batch) {
      Entry &en = entries[id];
      int32_t r = en.req;
      req_stage[r] += 1;
      if (en.follow_up) fu_completed += 1;
      if (chain_off[r] + req_stage[r] < chain_off[r + 1]) {
        fu_generated += 1;
        push(t, K_FOLLOW_UP, r);
      } else {
        completed += 1;
        last_completion = t;
        record(t, x.id, COE_EV_COMPLETE, e, r);
      }
    }
    push(t, K_WAKE, x.id);
  }

  // ---- setup (engine.py:497-548) -----------------------------------------
  void initialize() {
    // initialize_pools (expert_pool.py:62-87)
    for (int32_t i = 0; i < X; ++i) {
      Executor &x = ex[i];
      x.id = i;
      x.resident.assign(E, 0);
      x.res_pos.assign(E, -1);
      x.pinned.assign(E, 0);
      x.stamp.assign(E, -1);
      x.live_run.assign(E, -1);
      x.by_expert.assign(E, std::deque<int32_t>());
    }
    std::vector<std::vector<int32_t>> placed(X);
    int32_t turn = 0;
    for (int32_t k = 0; k < E && X > 0; ++k) {
      int32_t e = desc[k];
      int32_t target = -1;
      for (int32_t s = 0; s < X; ++s) {
        int32_t i = (turn + s) % X;
        if ((double)bytes[e] <= ex[i].free_bytes()) { target = i; break; }
      }
      if (target < 0) break;
      pool_add(ex[target], e);
      placed[target].push_back(e);
      turn = (target + 1) % X;
    }
    init_off.assign(1, 0);
    init_exp.clear();
    for (int32_t i = 0; i < X; ++i) {
      for (int32_t e : placed[i]) {
        if (evict == 1 || evict == 2) ex[i].stamp[e] = ex[i].clock++;
        init_exp.push_back(e);
      }
      init_off.push_back((int32_t)init_exp.size());
    }
    hc = HostCache();
    if (numa && host_mode >= 0 && host_budget > 0) {
      hc.enabled = true;
      hc.mode = host_mode;
      hc.budget = host_budget;
      hc.resident.assign(E, 0);
      hc.size.assign(E, 0);
      hc.stamp.assign(E, -1);
      hc.res_pos.assign(E, -1);
      std::vector<uint8_t> anywhere(E, 0);
      for (auto &x : ex)
        for (int32_t e : x.res_list) anywhere[e] = 1;
      for (int32_t k = 0; k < E; ++k) {
        int32_t e = desc[k];
        if (anywhere[e]) continue;
        if ((double)(hc.used + bytes[e]) <= hc.budget) hc_insert(e, bytes[e]);
      }
    }
  }

  void run_loop() {
    req_stage.assign(R, 0);
    for (int32_t r = 0; r < R; ++r) push(arrival[r], K_ARRIVAL, r);
    while (!heap.empty()) {
      Event ev = heap.top();
      heap.pop();
      switch (ev.kind) {
        case K_ARRIVAL:
          record(ev.t, -1, COE_EV_ARRIVAL, -1, ev.a);
          admit(ev.t, ev.a, false);
          break;
        case K_FOLLOW_UP: {
          int32_t r = ev.a;
          record(ev.t, -1, COE_EV_FOLLOW_UP, chain_exp[chain_off[r] + req_stage[r]], r);
          admit(ev.t, r, true);
          break;
        }
        case K_WAKE:
          step(ev.t, ex[ev.a]);
          break;
        case K_LOAD_DONE:
          ex[ev.a].busy = false;
          ex[ev.a].loading = -1;
          record(ev.t, ev.a, COE_EV_LOAD_DONE, -1, -1);
          step(ev.t, ex[ev.a]);
          break;
        case K_BATCH_DONE:
          on_batch_done(ev.t, ex[ev.a], ev.b, ev.c);
          break;
      }
    }
    // engine.py:783-795
    if (completed != R)
      fail(COE_ERR_RUNTIME, "conservation violated: " + std::to_string(completed) + " of " + std::to_string(R) +
                                " requests completed");
    if (fu_generated != fu_completed)
      fail(COE_ERR_RUNTIME, "conservation violated: " + std::to_string(fu_generated) +
                                " follow-ups generated, " + std::to_string(fu_completed) + " completed");
    for (auto &x : ex)
      if (x.queue_len)
        fail(COE_ERR_RUNTIME, "executor " + std::to_string(x.id) + " finished with " +
                                  std::to_string(x.queue_len) + " stranded entries");
  }
};

template <class T>
static std::vector<T> copy_vec(const T *p, int64_t n) {
  return p ? std::vector<T>(p, p + n) : std::vector<T>((size_t)n, T());
}

extern "C" {

const char *coe_plan_last_error(void) { return g_error.c_str(); }

int coe_plan_create(const coe_plan_config *c, coe_plan **out) {
  try {
    if (!c || !out) fail(COE_ERR_CONFIG, "null argument");
    if (c->num_executors < 1) fail(COE_ERR_CONFIG, "need at least one executor");
    if (c->num_requests < 1) fail(COE_ERR_CONFIG, "request stream is empty");
    auto *p = new coe_plan();
    p->E = c->num_experts;
    p->A = c->num_arches;
    p->X = c->num_executors;
    p->R = c->num_requests;
    p->bytes = copy_vec(c->expert_bytes, p->E);
    p->usage = copy_vec(c->usage_prob, p->E);
    p->arch = copy_vec(c->expert_arch, p->E);
    p->up_off = copy_vec(c->upstream_offsets, p->E + 1);
    p->up_idx = copy_vec(c->upstream_index, p->up_off.empty() ? 0 : p->up_off.back());
    p->desc = copy_vec(c->desc_order, p->E);
    int64_t ap = (int64_t)p->A * 2;
    p->perf_valid = copy_vec(c->perf_valid, ap);
    p->perf_max_batch = copy_vec(c->perf_max_batch, ap);
    p->perf_k = copy_vec(c->perf_k, ap);
    p->perf_b = copy_vec(c->perf_b, ap);
    p->cost_valid = copy_vec(c->cost_valid, ap);
    p->cost_k = copy_vec(c->cost_k, ap);
    p->cost_b = copy_vec(c->cost_b, ap);
    p->cost_nsat = copy_vec(c->cost_n_sat, ap);
    p->cost_gamma = copy_vec(c->cost_gamma, ap);
    p->cost_base = copy_vec(c->cost_base_bytes, ap);
    p->cost_item = copy_vec(c->cost_per_item_bytes, ap);
    p->numa = c->numa;
    p->host_bw = c->host_bw;
    p->host_ovh = c->host_overhead;
    p->ssd_bw = c->ssd_bw;
    p->ssd_ovh = c->ssd_overhead;
    p->peer_enabled = c->peer_enabled;
    p->peer_bw = c->peer_bw;
    p->peer_ovh = c->peer_overhead;
    if (p->peer_enabled && !(p->peer_bw > 0)) fail(COE_ERR_CONFIG, "peer tier bandwidth must be positive");
    p->host_mode = c->host_mode;
    p->host_budget = c->host_cache_budget;
    p->assign_makespan = c->assign_makespan;
    p->arrange = c->arrange;
    p->evict = c->evict;
    p->req_id = copy_vec(c->request_id, p->R);
    p->arrival = copy_vec(c->arrival_s, p->R);
    p->chain_off = copy_vec(c->chain_offsets, p->R + 1);
    p->chain_exp = copy_vec(c->chain_experts, p->chain_off.back());
    p->record_trace = c->record_trace != 0;
    p->record_ops = c->record_ops != 0;
    for (int32_t r = 0; r < p->R; ++r)
      if (p->chain_off[r + 1] <= p->chain_off[r]) {
        delete p;
        fail(COE_ERR_CONFIG, "request with an empty expert chain");
      }
    p->ex.resize(p->X);
    for (int32_t i = 0; i < p->X; ++i) {
      p->ex[i].proc = c->exec_proc[i];
      p->ex[i].expert_budget = c->exec_expert_budget[i];
      p->ex[i].inference_budget = c->exec_inference_budget[i];
      p->ex[i].k_scale = c->exec_k_scale[i];
    }
    *out = p;
    return COE_OK;
  } catch (const PlanError &e) {
    g_error = e.msg;
    return e.code;
  } catch (const std::exception &e) {
    g_error = e.what();
    return COE_ERR_RUNTIME;
  }
}

int coe_plan_run(coe_plan *p) {
  try {
    if (p->ran) fail(COE_ERR_RUNTIME, "plan already ran");
    p->ran = true;
    p->initialize();
    p->run_loop();
    return COE_OK;
  } catch (const PlanError &e) {
    g_error = e.msg;
    return e.code;
  } catch (const std::exception &e) {
    g_error = e.what();
    return COE_ERR_RUNTIME;
  }
}

void coe_plan_destroy(coe_plan *p) { delete p; }

int coe_plan_metrics_get(const coe_plan *p, coe_plan_metrics *m) {
  m->completed = p->completed;
  m->follow_ups = p->fu_completed;
  m->makespan_s = p->last_completion;
  m->evictions = p->evictions;
  m->stale_predictions = p->stale;
  m->sched_wall_s = p->sched_wall;
  m->sched_calls = p->sched_calls;
  return COE_OK;
}

int coe_plan_executor_stats(const coe_plan *p, double *busy_s, int64_t *switches) {
  for (int32_t i = 0; i < p->X; ++i) {
    busy_s[i] = p->ex[i].busy_s;
    switches[i] = p->ex[i].switches;
  }
  return COE_OK;
}

int64_t coe_plan_trace_len(const coe_plan *p) { return (int64_t)p->tr_t.size(); }

int coe_plan_trace(const coe_plan *p, double *t, int32_t *exid, int32_t *ev, int32_t *expert, int64_t *req) {
  size_t n = p->tr_t.size();
  if (n == 0) return COE_OK;
  std::memcpy(t, p->tr_t.data(), n * sizeof(double));
  std::memcpy(exid, p->tr_ex.data(), n * sizeof(int32_t));
  std::memcpy(ev, p->tr_ev.data(), n * sizeof(int32_t));
  std::memcpy(expert, p->tr_exp.data(), n * sizeof(int32_t));
  std::memcpy(req, p->tr_req.data(), n * sizeof(int64_t));
  return COE_OK;
}

int coe_plan_initial_residency(const coe_plan *p, int32_t *offsets, int32_t *experts) {
  if (!p->ran) return COE_ERR_RUNTIME;
  std::memcpy(offsets, p->init_off.data(), p->init_off.size() * sizeof(int32_t));
  if (!p->init_exp.empty()) std::memcpy(experts, p->init_exp.data(), p->init_exp.size() * sizeof(int32_t));
  return COE_OK;
}

int64_t coe_plan_num_ops(const coe_plan *p) { return (int64_t)p->ops.size(); }
const coe_op *coe_plan_ops(const coe_plan *p) { return p->ops.data(); }
int64_t coe_plan_num_op_args(const coe_plan *p) { return (int64_t)p->op_args.size(); }
const int32_t *coe_plan_op_args(const coe_plan *p) { return p->op_args.data(); }
int64_t coe_plan_num_admissions(const coe_plan *p) { return (int64_t)p->adms.size(); }

int64_t coe_plan_hops(const coe_plan *p, int64_t capacity, int64_t *index, int32_t *src, int32_t *dst,
                      int32_t *request, int32_t *stage) {
  std::vector<coe::Hop> hops = coe::hop_schedule(p->adms.data(), (int64_t)p->adms.size(), p->R);
  int64_t n = (int64_t)hops.size();
  for (int64_t i = 0; i < n && i < capacity; ++i) {
    index[i] = hops[i].index;
    src[i] = hops[i].src;
    dst[i] = hops[i].dst;
    request[i] = hops[i].request;
    stage[i] = hops[i].stage;
  }
  return n;
}
const coe_admission *coe_plan_admissions(const coe_plan *p) { return p->adms.data(); }

}  // extern "C"
