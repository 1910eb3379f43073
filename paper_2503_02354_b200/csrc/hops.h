// hops.h -- cross-executor follow-up hops, shared by the planner (host API, tests)
// and the GPU runtime (NCCL exchange).
//
// A follow-up admitted to executor x whose previous stage ran on executor y != x
// needs that stage's T x d activation moved y -> x (engine.py:751-753 admits the
// follow-up; the reference moves no data).  The global hop order is the planner's
// admission order: a hop is admitted when its producer batch finishes, and any batch
// consuming hop h starts after h is admitted, so every hop a batch *produces* comes
// after every hop it *consumes*.  Ranks issue their own sends / receives in this
// order, which keeps NCCL point-to-point matching consistent and deadlock-free.
#pragma once

#include <stdint.h>

#include <vector>

#include "coe_planner.h"

namespace coe {

struct Hop {
  int64_t index;    // position in the global hop order
  int32_t src;      // executor holding the data (ran stage `stage`)
  int32_t dst;      // executor running stage `stage` + 1
  int32_t request;  // request index
  int32_t stage;    // stage whose output moves
};

inline std::vector<Hop> hop_schedule(const coe_admission *adm, int64_t n, int32_t num_requests) {
  std::vector<int32_t> last_exec(num_requests > 0 ? num_requests : 0, -1);
  std::vector<Hop> hops;
  for (int64_t i = 0; i < n; ++i) {
    const coe_admission &a = adm[i];
    if (a.request < 0 || a.request >= num_requests) continue;
    int32_t prev = last_exec[a.request];
    if (a.stage > 0 && prev >= 0 && prev != a.executor)
      hops.push_back(Hop{(int64_t)hops.size(), prev, a.executor, a.request, a.stage - 1});
    last_exec[a.request] = a.executor;
  }
  return hops;
}

}  // namespace coe
