// act_rows.h -- activation rows of one executor's step: the request-slot ring.
//
// The reference keeps no activations; physically each request carries a
// T x d activation between its stages.  Instead of one row block per request (memory
// growing with the stream), an executor holds activations in A = [landing | ring]:
//
//   * ring slots: a request's activation lives in one slot from its first batch on this
//     executor until its output leaves (final stage -> Y / the output staging ring, or a
//     fused hop into another executor's landing rows).  Every stage runs IN PLACE: the up
//     pass reads the slot into H, the down pass (a separate launch, after every up tile)
//     writes the stage output back into the same slot.  A freed slot returns to the tail
//     of a FIFO free list, so reuse is as far apart in op order as the ring allows; the
//     batch that freed it becomes a producer of the batch that next writes it (in-step
//     write-after-read order, enforced by the runtime's wave dependencies);
//   * landing rows: where other executors' fused hops store a request's activation
//     (indexed by the hop's position among this executor's hop-ins in the global hop
//     order, hops.h, so producer and consumer agree without exchanging anything); not
//     recycled inside a step -- the step fence orders them across steps.
//
// Which rows a member reads and writes is decided here in op order and carried to the GPU
// as two codes per admission (coe_grouped_mlp_routed): in = (row << 1) | from_X and
// out = (row << 4) | kind.  The same pass, run without a ring limit, sizes the ring
// (coe_runtime_plan_rows), so capacity and use can never disagree.
#pragma once

#include <stdint.h>

#include <algorithm>
#include <deque>
#include <string>
#include <unordered_map>
#include <vector>

#include "coe_planner.h"
#include "hops.h"

namespace coe {

enum : int32_t { OUT_RING = 0, OUT_Y = 1, OUT_STAGE = 2, OUT_PEER0 = 3 };
constexpr int ROW_STAGES = 8;  // (request, stage) keys: stage < 8 (same bound as the hop tables)

struct RowPlan {
  // per admission of this executor (admission order): routes for K3
  std::vector<int32_t> in_code, out_code;
  std::vector<uint8_t> is_final;             // out kind to be filled with a staging position
  // per batch (op order among this executor's batches): in-step slot predecessors
  std::vector<std::vector<int32_t>> preds;
  // e2e inputs: per request whose stage 0 runs here, its slot, in-step predecessor batch
  // (-1: none) and the previous occupant's slot index (for cross-step waits)
  std::vector<int32_t> in_slot, in_pred;     // indexed by request (-1: none)
  // NCCL transport: rows of each local hop (my_hops order): send source / receive target
  std::vector<int32_t> hop_row;
  // ring slots (absolute A rows) freed this step and the batch that freed them
  std::vector<int32_t> freed_slot, freed_by;
  std::vector<int32_t> free_after;           // free-list order at the end of the step
  int32_t peak_ring = 0, landing = 0;
  bool nccl_hold = false;                    // NCCL hop-outs keep their rows until the step ends
};

// ops / op_args / adm: the plan; batch_ops: op indices of this executor's BATCH ops in op
// order; adm_index: (request * ROW_STAGES + stage) -> admission index on this executor;
// all_hops: global hop order; my_hops: indices into all_hops touching this executor;
// final_stage: per request.  ring_order: the free list at step start (absolute A rows,
// landing .. landing + ring); an empty list with ring_cap < 0 sizes instead (unlimited).
inline bool plan_rows(const coe_op *ops, const int32_t *op_args, const std::vector<int64_t> &batch_ops,
                      const std::unordered_map<int64_t, int32_t> &adm_index, const std::vector<Hop> &all_hops,
                      const std::vector<int32_t> &my_hops, const std::vector<int32_t> &final_stage, int32_t executor,
                      bool e2e_in, bool e2e_out, bool peer_mode, int32_t landing_cap, int32_t ring_cap,
                      const std::vector<int32_t> &ring_order, int32_t num_requests, int64_t num_admissions,
                      RowPlan &out, std::string &err) {
  const bool sizing = ring_cap < 0;
  auto key = [](int32_t r, int32_t s) { return (int64_t)r * ROW_STAGES + s; };
  // landing row of every hop (position among its destination's hop-ins, global order)
  std::vector<int32_t> landing_of(all_hops.size(), -1);
  {
    std::unordered_map<int32_t, int32_t> per_dst;
    for (size_t i = 0; i < all_hops.size(); ++i) landing_of[i] = per_dst[all_hops[i].dst]++;
  }
  std::unordered_map<int64_t, int32_t> hop_in, hop_out;  // (request, stage) -> my_hops position
  for (size_t i = 0; i < my_hops.size(); ++i) {
    const Hop &h = all_hops[my_hops[i]];
    if (h.dst == executor) {
      hop_in[key(h.request, h.stage + 1)] = (int32_t)i;
      out.landing = std::max(out.landing, landing_of[my_hops[i]] + 1);
    }
    if (h.src == executor) hop_out[key(h.request, h.stage)] = (int32_t)i;
  }
  if (!sizing && out.landing > landing_cap) {
    err = "activation landing rows too few for this step's hop-ins (" + std::to_string(out.landing) + " > " +
          std::to_string(landing_cap) + ")";
    return false;
  }
  out.in_code.assign(num_admissions, 0);
  out.out_code.assign(num_admissions, 0);
  out.is_final.assign(num_admissions, 0);
  out.preds.assign(batch_ops.size(), {});
  out.in_slot.assign(num_requests, -1);
  out.in_pred.assign(num_requests, -1);
  out.hop_row.assign(my_hops.size(), -1);
  out.freed_slot.clear();
  out.freed_by.clear();
  std::deque<int32_t> free_list(ring_order.begin(), ring_order.end());
  std::unordered_map<int32_t, int32_t> freed_by_batch;  // ring slot -> batch that freed it this step
  int32_t next_new = landing_cap;                        // sizing: fresh slots past the landing rows
  int32_t live = 0;
  std::vector<int32_t> held;                            // NCCL hop-out slots, released at step end
  std::vector<int32_t> cur(num_requests, -1);           // A row holding the request's activation
  std::vector<uint8_t> in_ring(num_requests, 0);        // cur is a ring slot (not a landing row)
  auto alloc = [&](int32_t b, int32_t &slot, int32_t &pred) -> bool {
    if (free_list.empty()) {
      if (!sizing) {
        err = "activation ring too small for this step (" + std::to_string(ring_cap) + " slots)";
        return false;
      }
      free_list.push_back(next_new++);
    }
    slot = free_list.front();
    free_list.pop_front();
    auto it = freed_by_batch.find(slot);
    pred = it == freed_by_batch.end() ? -1 : it->second;
    if (pred >= 0 && pred != b && std::find(out.preds[b].begin(), out.preds[b].end(), pred) == out.preds[b].end())
      out.preds[b].push_back(pred);
    out.peak_ring = std::max(out.peak_ring, ++live);
    return true;
  };
  for (size_t b = 0; b < batch_ops.size(); ++b) {
    const coe_op &op = ops[batch_ops[b]];
    std::vector<int32_t> frees;
    for (int32_t j = 0; j < op.count; ++j) {
      const int32_t r = op_args[op.offset + 2 * j], s = op_args[op.offset + 2 * j + 1];
      if (s >= ROW_STAGES) {
        err = "activation rows: chains longer than 8 stages";
        return false;
      }
      auto ai_it = adm_index.find(key(r, s));
      if (ai_it == adm_index.end()) {
        err = "activation rows: batch member without an admission";
        return false;
      }
      const int32_t ai = ai_it->second;
      // ---- input rows ----
      auto hi = hop_in.find(key(r, s));
      if (hi != hop_in.end()) {
        cur[r] = landing_of[my_hops[hi->second]];
        in_ring[r] = 0;
        out.hop_row[hi->second] = cur[r];
        out.in_code[ai] = cur[r] << 1;
      } else if (s == 0) {
        if (e2e_in) {
          int32_t q, pred;
          if (!alloc((int32_t)b, q, pred)) return false;
          cur[r] = q;
          in_ring[r] = 1;
          out.in_slot[r] = q;
          out.in_pred[r] = pred;
          out.in_code[ai] = q << 1;
        } else {
          cur[r] = -1;
          out.in_code[ai] = (r << 1) | 1;  // the device-resident inputs X
        }
      } else {
        if (cur[r] < 0) {
          err = "activation rows: a later stage without its predecessor's rows on this executor";
          return false;
        }
        out.in_code[ai] = cur[r] << 1;
      }
      // ---- output rows ----
      auto ho = hop_out.find(key(r, s));
      if (s == final_stage[r]) {
        out.is_final[ai] = 1;
        out.out_code[ai] = e2e_out ? OUT_STAGE : ((r << 4) | OUT_Y);  // staging row set at issue
        if (in_ring[r]) frees.push_back(cur[r]);
        cur[r] = -1;
        in_ring[r] = 0;
      } else if (ho != hop_out.end()) {
        const int32_t hidx = my_hops[ho->second];
        if (peer_mode) {
          out.out_code[ai] = (landing_of[hidx] << 4) | (OUT_PEER0 + all_hops[hidx].dst);
          if (in_ring[r]) frees.push_back(cur[r]);
        } else {  // NCCL: the row stays here until the hop stream has sent it (step end)
          if (cur[r] < 0) {
            int32_t q, pred;
            if (!alloc((int32_t)b, q, pred)) return false;
            cur[r] = q;
            in_ring[r] = 1;
          }
          if (in_ring[r]) held.push_back(cur[r]);
          out.out_code[ai] = (cur[r] << 4) | OUT_RING;
          out.hop_row[ho->second] = cur[r];
          out.nccl_hold = true;
        }
        cur[r] = -1;
        in_ring[r] = 0;
      } else {  // the next stage runs here: in place, or into a fresh slot after X
        if (cur[r] < 0) {
          int32_t q, pred;
          if (!alloc((int32_t)b, q, pred)) return false;
          cur[r] = q;
          in_ring[r] = 1;
        }
        out.out_code[ai] = (cur[r] << 4) | OUT_RING;
      }
    }
    for (int32_t q : frees) {  // after the batch's allocations: its up pass is the last reader
      free_list.push_back(q);
      freed_by_batch[q] = (int32_t)b;
      out.freed_slot.push_back(q);
      out.freed_by.push_back((int32_t)b);
      --live;
    }
  }
  out.free_after.assign(free_list.begin(), free_list.end());
  out.free_after.insert(out.free_after.end(), held.begin(), held.end());  // free once the step has ended
  return true;
}

}  // namespace coe
