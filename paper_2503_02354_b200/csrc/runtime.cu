// runtime.cu -- GPU serving runtime: executes one executor's op log on a B200.
//
// The reference advances a virtual clock through load / batch events
// (Simulation._start_load / _start_batch / _on_batch_done,
// /root/reference/pkg/src/coesim/engine.py:643-758); here the same op log is
// *executed*:
//
//   compute stream: upload the step's admissions -> K1 group sort -> K2 run
//                   compaction -> waves of K3 grouped expert MLPs
//   copy stream:    K4 swap-ins, pinned host expert store -> HBM slot,
//                   each issued as soon as its slot's last wave completed
//
// Physical layout (HBM): a slab of `num_slots` fixed expert slots
// ([W1 h*d | W2 d*h] bf16 each; budget/bytes of the planner's ModelPool), the
// request inputs X, two ping-pong activation buffers P0/P1, the H scratch of
// the current wave, and small grouping arrays.  Host: one pinned store of
// every expert (the "host tier", types.py:17).
//
// Host pass 1 turns the op log into actions (COPY / WAVE): slot assignment
// (victim slots are reused; initial-residency experts missing after the
// previous step are restored lazily, at first use, so a step always starts
// from initialize_pools' placement), wave cuts (a wave closes before a batch
// that must wait for a copy, that touches a request already in the wave, or
// that overflows the H scratch; and before a copy into a slot the open wave
// still reads).  Pass 2 issues them.  Timing never feeds back into decisions.

#include <cuda_bf16.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <unordered_set>
#include <vector>

#include "coe_cuda.h"
#include "coe_planner.h"
#include "common.cuh"

namespace {

thread_local std::string g_last_error;

constexpr int BM = 128;
constexpr int BN = 256;

uint64_t splitmix64_host(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void gather_outputs(const __nv_bfloat16 *p0, const __nv_bfloat16 *p1, const int32_t *last_stage,
                               int32_t num_requests, int64_t row_elems, __nv_bfloat16 *out) {
  // one block per request; 16-byte vectors
  int32_t r = blockIdx.x;
  if (r >= num_requests) return;
  const __nv_bfloat16 *src = (last_stage[r] & 1) ? p1 : p0;
  const uint4 *s = reinterpret_cast<const uint4 *>(src + r * row_elems);
  uint4 *d = reinterpret_cast<uint4 *>(out + r * row_elems);
  for (int64_t i = threadIdx.x; i < row_elems / 8; i += blockDim.x) d[i] = s[i];
}

struct CopyAct {
  int32_t expert;
  int32_t slot;
  int32_t wait_wave;  // wave whose completion frees the slot (-1: none this step)
  bool restore;
};

struct WaveAct {
  int32_t first_group;
  int32_t num_groups;
  int32_t tiles_up;
  int32_t tiles_down;
  int64_t rows;
  std::vector<int32_t> wait_copies;
};

struct Action {
  bool is_copy;
  int32_t index;
};

bool ok(cudaError_t e, const char *what) { return coe_cuda_ok(e, what); }

}  // namespace

void coe_set_error(const std::string &msg) { g_last_error = msg; }

struct coe_runtime {
  coe_runtime_config cfg{};
  int64_t expert_bytes = 0;
  int64_t row_elems = 0;  // T * d
  cudaStream_t compute = nullptr, copy = nullptr;
  // device memory
  char *slab = nullptr;
  __nv_bfloat16 *x = nullptr, *p0 = nullptr, *p1 = nullptr, *hbuf = nullptr, *outbuf = nullptr;
  int32_t *d_adm = nullptr;       // [4][max_adm]: exec, rank, req, stage
  int32_t *d_perm = nullptr, *d_keys = nullptr, *d_mreq = nullptr, *d_mstage = nullptr;
  int32_t *d_batch = nullptr;     // [2][max_batches]: exec, size
  int32_t *d_boff = nullptr;
  int32_t *d_flags = nullptr;     // runs, violations
  int32_t *d_last = nullptr;
  coe_mlp_group *d_groups = nullptr;  // [2][max_batches]
  void *d_sort_scratch = nullptr, *d_compact_scratch = nullptr;
  // host
  char *host_store = nullptr;
  char *staging[2] = {nullptr, nullptr};
  int64_t staging_bytes = 0;
  cudaEvent_t staging_done[2] = {nullptr, nullptr};
  int staging_idx = 0;
  int32_t *h_last = nullptr;
  coe_mlp *mlp = nullptr;
  // slot state (persists across steps)
  std::vector<int32_t> slot_expert, expert_slot;
  // events
  std::vector<cudaEvent_t> wave_ev, copy_ev;
  std::vector<cudaEvent_t> t_copy_start, t_copy_end, t_wave_start, t_wave_end;
  cudaEvent_t t_step_start = nullptr, t_group_end = nullptr, t_step_end = nullptr, copy_drained = nullptr;
  cudaEvent_t prev_step_end = nullptr;
  bool have_prev = false;
  int32_t last_waves = 0, last_copies = 0;
  int64_t last_adm = 0, last_batches = 0;

  ~coe_runtime() {
    if (compute) cudaStreamSynchronize(compute);
    if (copy) cudaStreamSynchronize(copy);
    if (mlp) coe_mlp_destroy(mlp);
    for (void *p : {(void *)slab, (void *)x, (void *)p0, (void *)p1, (void *)hbuf, (void *)outbuf, (void *)d_adm,
                    (void *)d_perm, (void *)d_keys, (void *)d_mreq, (void *)d_mstage, (void *)d_batch, (void *)d_boff,
                    (void *)d_flags, (void *)d_last, (void *)d_groups, d_sort_scratch, d_compact_scratch})
      if (p) cudaFree(p);
    for (void *p : {(void *)host_store, (void *)staging[0], (void *)staging[1], (void *)h_last})
      if (p) cudaFreeHost(p);
    auto kill = [](std::vector<cudaEvent_t> &v) {
      for (auto e : v) cudaEventDestroy(e);
      v.clear();
    };
    kill(wave_ev);
    kill(copy_ev);
    kill(t_copy_start);
    kill(t_copy_end);
    kill(t_wave_start);
    kill(t_wave_end);
    for (cudaEvent_t e : {t_step_start, t_group_end, t_step_end, copy_drained, prev_step_end, staging_done[0],
                          staging_done[1]})
      if (e) cudaEventDestroy(e);
    if (compute) cudaStreamDestroy(compute);
    if (copy) cudaStreamDestroy(copy);
  }

  bool ensure_events(std::vector<cudaEvent_t> &v, size_t n, bool timing) {
    while (v.size() < n) {
      cudaEvent_t e;
      if (!ok(cudaEventCreateWithFlags(&e, timing ? cudaEventDefault : cudaEventDisableTiming), "event create"))
        return false;
      v.push_back(e);
    }
    return true;
  }
};

namespace {

template <class T>
bool dmalloc(T **p, size_t bytes, const char *what) {
  return ok(cudaMalloc(reinterpret_cast<void **>(p), bytes < 16 ? 16 : bytes), what);
}

int fail_cuda() { return COE_CUDA_ERR_CUDA; }

float elapsed(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

// union length of [s, e) intervals
float union_len(std::vector<std::pair<float, float>> v) {
  std::sort(v.begin(), v.end());
  float total = 0.f, cs = -1.f, ce = -1.f;
  for (auto &iv : v) {
    if (iv.first > ce) {
      if (ce > cs) total += ce - cs;
      cs = iv.first;
      ce = iv.second;
    } else {
      ce = std::max(ce, iv.second);
    }
  }
  if (ce > cs) total += ce - cs;
  return total;
}

float intersect_len(std::vector<std::pair<float, float>> a, std::vector<std::pair<float, float>> b) {
  auto norm = [](std::vector<std::pair<float, float>> v) {
    std::sort(v.begin(), v.end());
    std::vector<std::pair<float, float>> out;
    for (auto &iv : v) {
      if (!out.empty() && iv.first <= out.back().second) out.back().second = std::max(out.back().second, iv.second);
      else out.push_back(iv);
    }
    return out;
  };
  a = norm(a);
  b = norm(b);
  size_t i = 0, j = 0;
  float total = 0.f;
  while (i < a.size() && j < b.size()) {
    float lo = std::max(a[i].first, b[j].first), hi = std::min(a[i].second, b[j].second);
    if (hi > lo) total += hi - lo;
    if (a[i].second < b[j].second) ++i;
    else ++j;
  }
  return total;
}

}  // namespace

extern "C" {

const char *coe_cuda_last_error(void) { return g_last_error.c_str(); }

uint64_t coe_expert_seed(uint64_t weight_seed, int32_t expert, int32_t matrix) {
  return splitmix64_host(weight_seed ^ (uint64_t)(2 * (int64_t)expert + matrix + 1) * 0xD1B54A32D192ED03ull);
}

int coe_runtime_create(const coe_runtime_config *cfg, coe_runtime **out) {
  auto *rt = new coe_runtime();
  rt->cfg = *cfg;
  const auto &c = rt->cfg;
  rt->expert_bytes = 2LL * c.d * c.h * 2;
  rt->row_elems = (int64_t)c.T * c.d;
  const int64_t act_bytes = (int64_t)c.max_requests * rt->row_elems * 2;
  bool good = ok(cudaStreamCreateWithFlags(&rt->compute, cudaStreamNonBlocking), "stream") &&
              ok(cudaStreamCreateWithFlags(&rt->copy, cudaStreamNonBlocking), "stream") &&
              dmalloc(&rt->slab, (size_t)rt->expert_bytes * c.num_slots, "slab alloc") &&
              dmalloc(&rt->x, act_bytes, "X alloc") && dmalloc(&rt->p0, act_bytes, "P0 alloc") &&
              dmalloc(&rt->p1, act_bytes, "P1 alloc") && dmalloc(&rt->outbuf, act_bytes, "out alloc") &&
              dmalloc(&rt->hbuf, (size_t)c.max_wave_rows * c.h * 2, "H alloc") &&
              dmalloc(&rt->d_adm, 16 * (size_t)c.max_admissions, "adm alloc") &&
              dmalloc(&rt->d_perm, 4 * (size_t)c.max_admissions, "perm alloc") &&
              dmalloc(&rt->d_keys, 4 * (size_t)c.max_admissions, "keys alloc") &&
              dmalloc(&rt->d_mreq, 4 * (size_t)c.max_admissions, "member alloc") &&
              dmalloc(&rt->d_mstage, 4 * (size_t)c.max_admissions, "member alloc") &&
              dmalloc(&rt->d_batch, 8 * (size_t)c.max_batches, "batch alloc") &&
              dmalloc(&rt->d_boff, 4 * (size_t)c.max_batches, "boff alloc") &&
              dmalloc(&rt->d_flags, 64, "flags alloc") && dmalloc(&rt->d_last, 4 * (size_t)c.max_requests, "last") &&
              dmalloc(&rt->d_groups, 2 * sizeof(coe_mlp_group) * (size_t)c.max_batches, "group alloc") &&
              dmalloc(&rt->d_sort_scratch, (size_t)coe_group_sort_scratch_bytes(c.max_admissions), "sort scratch") &&
              dmalloc(&rt->d_compact_scratch, (size_t)coe_run_compact_scratch_bytes(c.max_admissions, (int)c.max_batches, 1),
                      "compact scratch");
  if (good) {
    rt->staging_bytes = 16 * c.max_admissions + 8 * c.max_batches + 2 * sizeof(coe_mlp_group) * c.max_batches + 256;
    good = ok(cudaHostAlloc(reinterpret_cast<void **>(&rt->staging[0]), rt->staging_bytes, cudaHostAllocDefault), "staging") &&
           ok(cudaHostAlloc(reinterpret_cast<void **>(&rt->staging[1]), rt->staging_bytes, cudaHostAllocDefault), "staging") &&
           ok(cudaHostAlloc(reinterpret_cast<void **>(&rt->h_last), 4 * (size_t)c.max_requests, cudaHostAllocDefault), "last") &&
           ok(cudaHostAlloc(reinterpret_cast<void **>(&rt->host_store), (size_t)rt->expert_bytes * c.num_experts,
                            cudaHostAllocDefault),
              "pinned expert store") &&
           ok(cudaEventCreateWithFlags(&rt->staging_done[0], cudaEventDisableTiming), "event") &&
           ok(cudaEventCreateWithFlags(&rt->staging_done[1], cudaEventDisableTiming), "event") &&
           ok(cudaEventCreateWithFlags(&rt->prev_step_end, cudaEventDisableTiming), "event") &&
           ok(cudaEventCreateWithFlags(&rt->copy_drained, cudaEventDisableTiming), "event") &&
           ok(cudaEventCreate(&rt->t_step_start), "event") && ok(cudaEventCreate(&rt->t_group_end), "event") &&
           ok(cudaEventCreate(&rt->t_step_end), "event");
  }
  if (good) {
    coe_mlp_config mc{};
    mc.d = c.d;
    mc.h = c.h;
    mc.T = c.T;
    mc.x = rt->x;
    mc.act0 = rt->p0;
    mc.act1 = rt->p1;
    mc.act_rows = (int64_t)c.max_requests * c.T;
    mc.h_scratch = rt->hbuf;
    mc.h_rows = c.max_wave_rows;
    mc.slab = rt->slab;
    mc.num_slots = c.num_slots;
    mc.slot_stride_bytes = rt->expert_bytes;
    if (coe_mlp_create(&mc, &rt->mlp) != COE_CUDA_OK) good = false;
  }
  if (!good) {
    std::string msg = g_last_error;
    delete rt;
    g_last_error = msg;
    return COE_CUDA_ERR_CUDA;
  }
  rt->slot_expert.assign(c.num_slots, -1);
  rt->expert_slot.assign(c.num_experts, -1);
  *out = rt;
  return COE_CUDA_OK;
}

void coe_runtime_destroy(coe_runtime *rt) { delete rt; }

void *coe_runtime_buffer(coe_runtime *rt, int which) {
  switch (which) {
    case 0: return rt->x;
    case 1: return rt->p0;
    case 2: return rt->p1;
    case 3: return rt->hbuf;
    case 4: return rt->slab;
    case 5: return rt->host_store;
    case 6: return rt->outbuf;
    default: return nullptr;
  }
}

cudaStream_t coe_runtime_stream(coe_runtime *rt, int which) { return which == 0 ? rt->compute : rt->copy; }

int coe_runtime_read_buffer(coe_runtime *rt, int which, void *host, int64_t bytes) {
  void *src = coe_runtime_buffer(rt, which);
  if (!src || which == 5) {
    coe_set_error("read_buffer: not a device buffer");
    return COE_CUDA_ERR_CONFIG;
  }
  if (!ok(cudaStreamSynchronize(rt->compute), "read_buffer sync")) return fail_cuda();
  return ok(cudaMemcpy(host, src, (size_t)bytes, cudaMemcpyDeviceToHost), "read_buffer") ? COE_CUDA_OK : fail_cuda();
}

int coe_runtime_slot_of(coe_runtime *rt, int32_t expert) {
  if (expert < 0 || expert >= (int32_t)rt->expert_slot.size()) return -1;
  return rt->expert_slot[expert];
}

int coe_runtime_init_experts(coe_runtime *rt) {
  const auto &c = rt->cfg;
  const int64_t half = (int64_t)c.d * c.h;  // elements per matrix
  // generate into slot 0 of the slab, stage to the pinned store
  for (int32_t e = 0; e < c.num_experts; ++e) {
    __nv_bfloat16 *w = reinterpret_cast<__nv_bfloat16 *>(rt->slab);
    if (coe_fill_uniform_bf16(w, half, coe_expert_seed(c.weight_seed, e, 0), sqrtf(3.0f / c.d), rt->compute) ||
        coe_fill_uniform_bf16(w + half, half, coe_expert_seed(c.weight_seed, e, 1), sqrtf(3.0f / c.h), rt->compute))
      return COE_CUDA_ERR_CUDA;
    if (!ok(cudaMemcpyAsync(rt->host_store + e * rt->expert_bytes, rt->slab, rt->expert_bytes,
                            cudaMemcpyDeviceToHost, rt->compute),
            "expert store D2H"))
      return fail_cuda();
  }
  if (!ok(cudaStreamSynchronize(rt->compute), "init experts")) return fail_cuda();
  std::fill(rt->slot_expert.begin(), rt->slot_expert.end(), -1);
  std::fill(rt->expert_slot.begin(), rt->expert_slot.end(), -1);
  rt->have_prev = false;
  return COE_CUDA_OK;
}

int coe_runtime_fill_inputs(coe_runtime *rt, uint64_t seed, int32_t num_requests) {
  if (num_requests > rt->cfg.max_requests) {
    coe_set_error("fill_inputs: more requests than the runtime was sized for");
    return COE_CUDA_ERR_CONFIG;
  }
  int rc = coe_fill_uniform_bf16(rt->x, (int64_t)num_requests * rt->row_elems, seed, sqrtf(3.0f), rt->compute);
  if (rc) return rc;
  return ok(cudaStreamSynchronize(rt->compute), "fill inputs") ? COE_CUDA_OK : fail_cuda();
}

int coe_runtime_upload_inputs(coe_runtime *rt, const void *host, int32_t num_requests) {
  if (num_requests > rt->cfg.max_requests) {
    coe_set_error("upload_inputs: more requests than the runtime was sized for");
    return COE_CUDA_ERR_CONFIG;
  }
  return ok(cudaMemcpyAsync(rt->x, host, (size_t)num_requests * rt->row_elems * 2, cudaMemcpyHostToDevice,
                            rt->compute),
            "input H2D")
             ? COE_CUDA_OK
             : fail_cuda();
}

int coe_runtime_download_outputs(coe_runtime *rt, const int32_t *last_stage_host, int32_t num_requests, void *host) {
  if (num_requests <= 0) return COE_CUDA_OK;
  std::memcpy(rt->h_last, last_stage_host, 4 * (size_t)num_requests);
  if (!ok(cudaMemcpyAsync(rt->d_last, rt->h_last, 4 * (size_t)num_requests, cudaMemcpyHostToDevice, rt->compute),
          "last stage H2D"))
    return fail_cuda();
  gather_outputs<<<num_requests, 256, 0, rt->compute>>>(rt->p0, rt->p1, rt->d_last, num_requests, rt->row_elems,
                                                        rt->outbuf);
  if (!ok(cudaGetLastError(), "gather outputs")) return fail_cuda();
  return ok(cudaMemcpyAsync(host, rt->outbuf, (size_t)num_requests * rt->row_elems * 2, cudaMemcpyDeviceToHost,
                            rt->compute),
            "output D2H")
             ? COE_CUDA_OK
             : fail_cuda();
}

int coe_runtime_synchronize(coe_runtime *rt) {
  bool a = ok(cudaStreamSynchronize(rt->copy), "sync copy");
  bool b = ok(cudaStreamSynchronize(rt->compute), "sync compute");
  return (a && b) ? COE_CUDA_OK : fail_cuda();
}

int coe_runtime_check(coe_runtime *rt, int32_t *runs, int32_t *violations) {
  int32_t flags[2];
  if (!ok(cudaMemcpy(flags, rt->d_flags, 8, cudaMemcpyDeviceToHost), "flags D2H")) return fail_cuda();
  *runs = flags[0];
  *violations = flags[1];
  return COE_CUDA_OK;
}

int coe_runtime_members(coe_runtime *rt, int32_t *member_req, int32_t *member_stage, int32_t *batch_off) {
  bool good = ok(cudaMemcpy(member_req, rt->d_mreq, 4 * rt->last_adm, cudaMemcpyDeviceToHost), "members D2H") &&
              ok(cudaMemcpy(member_stage, rt->d_mstage, 4 * rt->last_adm, cudaMemcpyDeviceToHost), "members D2H") &&
              ok(cudaMemcpy(batch_off, rt->d_boff, 4 * rt->last_batches, cudaMemcpyDeviceToHost), "boff D2H");
  return good ? COE_CUDA_OK : fail_cuda();
}

int coe_runtime_timing(coe_runtime *rt, coe_step_timing *out) {
  if (!rt->cfg.profile) {
    coe_set_error("runtime created without profile events");
    return COE_CUDA_ERR_CONFIG;
  }
  std::memset(out, 0, sizeof(*out));
  out->total_ms = elapsed(rt->t_step_start, rt->t_step_end);
  out->group_ms = elapsed(rt->t_step_start, rt->t_group_end);
  std::vector<std::pair<float, float>> cp, wv;
  for (int i = 0; i < rt->last_copies; ++i)
    cp.emplace_back(elapsed(rt->t_step_start, rt->t_copy_start[i]), elapsed(rt->t_step_start, rt->t_copy_end[i]));
  wv.emplace_back(0.f, out->group_ms);
  for (int i = 0; i < rt->last_waves; ++i) {
    float s = elapsed(rt->t_step_start, rt->t_wave_start[i]), e = elapsed(rt->t_step_start, rt->t_wave_end[i]);
    wv.emplace_back(s, e);
    out->mlp_ms += e - s;
  }
  out->copy_busy_ms = union_len(cp);
  out->compute_busy_ms = union_len(wv);
  out->overlap_ms = intersect_len(cp, wv);
  return COE_CUDA_OK;
}

int coe_runtime_step(coe_runtime *rt, const coe_step_input *in, coe_step_stats *stats) {
  const auto &c = rt->cfg;
  const coe_op *ops = static_cast<const coe_op *>(in->ops);
  const coe_admission *adm = static_cast<const coe_admission *>(in->admissions);
  const int32_t x = in->executor;
  coe_step_stats st{};

  // ---- admissions of this executor (admission order) ----
  std::vector<int32_t> a_rank, a_req, a_stage;
  int32_t max_rank = 0;
  for (int64_t i = 0; i < in->num_admissions; ++i) {
    if (adm[i].executor != x) continue;
    a_rank.push_back(adm[i].run_rank);
    a_req.push_back(adm[i].request);
    a_stage.push_back(adm[i].stage);
    max_rank = std::max(max_rank, adm[i].run_rank);
    if (adm[i].request >= c.max_requests) {
      coe_set_error("request index beyond the runtime's activation capacity");
      return COE_CUDA_ERR_CONFIG;
    }
  }
  const int64_t n_adm = (int64_t)a_rank.size();
  if (n_adm > c.max_admissions) {
    coe_set_error("more admissions than the runtime was sized for");
    return COE_CUDA_ERR_CONFIG;
  }
  int rank_bits = 1;
  while ((1LL << rank_bits) <= max_rank) ++rank_bits;
  const int passes = (rank_bits + 7) / 8;  // executor field is 0 (one executor per runtime)
  st.rank_bits = rank_bits;

  // ---- pass 1: slots, copies, waves ----
  std::vector<uint8_t> plan_res(c.num_experts, 0), pending_restore(c.num_experts, 0);
  std::vector<int32_t> slot_use_wave(c.num_slots, -1), slot_copy(c.num_slots, -1);
  std::vector<uint8_t> slot_copy_waited(c.num_slots, 1);
  // slots holding experts outside the initial placement become stale
  for (int32_t i = 0; i < in->num_initial; ++i) plan_res[in->initial[i]] = 1;
  for (int32_t s = 0; s < c.num_slots; ++s) {
    int32_t e = rt->slot_expert[s];
    if (e >= 0 && !plan_res[e]) {
      rt->expert_slot[e] = -1;
      rt->slot_expert[s] = -1;
    }
  }
  for (int32_t i = 0; i < in->num_initial; ++i) {
    int32_t e = in->initial[i];
    if (rt->expert_slot[e] < 0) pending_restore[e] = 1;
  }

  std::vector<CopyAct> copies;
  std::vector<WaveAct> waves;
  std::vector<Action> actions;
  std::vector<coe_mlp_group> g_up, g_down;
  std::vector<int32_t> b_size;
  std::unordered_set<int32_t> wave_reqs;
  WaveAct open{};
  open.first_group = 0;
  bool open_used = false;

  auto flush = [&]() {
    if (!open_used) return;
    int32_t id = (int32_t)waves.size();
    waves.push_back(open);
    actions.push_back(Action{false, id});
    st.max_wave_groups = std::max(st.max_wave_groups, open.num_groups);
    st.max_wave_rows = std::max(st.max_wave_rows, open.rows);
    open = WaveAct{};
    open.first_group = (int32_t)g_up.size();
    open_used = false;
    wave_reqs.clear();
  };
  auto open_id = [&]() { return (int32_t)waves.size(); };
  auto alloc_slot = [&](int32_t &slot) -> bool {
    int32_t best = -1;
    for (int32_t s = 0; s < c.num_slots; ++s) {
      if (rt->slot_expert[s] >= 0) continue;
      if (best < 0 || slot_use_wave[s] < slot_use_wave[best]) best = s;
    }
    if (best < 0) return false;
    if (open_used && slot_use_wave[best] == open_id()) flush();
    slot = best;
    return true;
  };
  auto issue_copy = [&](int32_t e, bool restore) -> bool {
    int32_t s;
    if (!alloc_slot(s)) {
      coe_set_error("no free HBM expert slot (planner residency exceeds the slot count)");
      return false;
    }
    int32_t cid = (int32_t)copies.size();
    copies.push_back(CopyAct{e, s, slot_use_wave[s], restore});
    actions.push_back(Action{true, cid});
    rt->slot_expert[s] = e;
    rt->expert_slot[e] = s;
    slot_copy[s] = cid;
    slot_copy_waited[s] = 0;
    if (restore) {
      st.restores += 1;
      st.restore_bytes += rt->expert_bytes;
    } else {
      st.loads += 1;
      st.load_bytes += rt->expert_bytes;
    }
    return true;
  };

  for (int64_t i = 0; i < in->num_ops; ++i) {
    const coe_op &op = ops[i];
    if (op.executor != x) continue;
    if (op.kind == COE_OP_LOAD) {
      for (int32_t k = 0; k < op.count; ++k) {
        int32_t v = in->op_args[op.offset + k];
        plan_res[v] = 0;
        pending_restore[v] = 0;
        int32_t s = rt->expert_slot[v];
        if (s >= 0) {
          rt->expert_slot[v] = -1;
          rt->slot_expert[s] = -1;
        }
      }
      plan_res[op.expert] = 1;
      if (rt->expert_slot[op.expert] >= 0) {  // never reuse bytes: every planned load moves them
        int32_t s = rt->expert_slot[op.expert];
        rt->slot_expert[s] = -1;
        rt->expert_slot[op.expert] = -1;
      }
      if (!issue_copy(op.expert, false)) return COE_CUDA_ERR_CHECK;
    } else {
      const int32_t e = op.expert;
      if (rt->expert_slot[e] < 0) {
        if (!pending_restore[e]) {
          coe_set_error("batch on an expert that is neither resident nor loaded");
          return COE_CUDA_ERR_CHECK;
        }
        pending_restore[e] = 0;
        if (!issue_copy(e, true)) return COE_CUDA_ERR_CHECK;
      }
      const int32_t s = rt->expert_slot[e];
      const int64_t rows = (int64_t)op.count * c.T;
      bool clash = false;
      for (int32_t k = 0; k < op.count && !clash; ++k) clash = wave_reqs.count(in->op_args[op.offset + 2 * k]) > 0;
      const bool need_wait = !slot_copy_waited[s];
      if (open_used && (need_wait || clash || open.rows + rows > c.max_wave_rows ||
                        open.num_groups >= coe_mlp_max_groups()))
        flush();
      if (rows > c.max_wave_rows) {
        coe_set_error("a single batch exceeds the H scratch rows");
        return COE_CUDA_ERR_CONFIG;
      }
      if (need_wait) {
        open.wait_copies.push_back(slot_copy[s]);
        slot_copy_waited[s] = 1;
      }
      const int32_t m_tiles = (int32_t)((rows + BM - 1) / BM);
      coe_mlp_group gu{};
      gu.rows = (int32_t)rows;
      gu.slot = s;
      gu.batch = (int32_t)b_size.size();
      gu.h_row = (int32_t)open.rows;
      gu.tile_start = open.tiles_up;
      coe_mlp_group gd = gu;
      gd.tile_start = open.tiles_down;
      g_up.push_back(gu);
      g_down.push_back(gd);
      b_size.push_back(op.count);
      open.num_groups += 1;
      open.rows += rows;
      open.tiles_up += m_tiles * (c.h / BN);
      open.tiles_down += m_tiles * (c.d / BN);
      open_used = true;
      slot_use_wave[s] = open_id();
      for (int32_t k = 0; k < op.count; ++k) wave_reqs.insert(in->op_args[op.offset + 2 * k]);
    }
  }
  flush();
  const int64_t n_batches = (int64_t)b_size.size();
  if (n_batches > c.max_batches) {
    coe_set_error("more batches than the runtime was sized for");
    return COE_CUDA_ERR_CONFIG;
  }
  st.admissions = n_adm;
  st.batches = n_batches;
  st.waves = (int64_t)waves.size();

  // ---- pass 2: issue ----
  if (!rt->ensure_events(rt->wave_ev, waves.size(), false) || !rt->ensure_events(rt->copy_ev, copies.size(), false))
    return fail_cuda();
  if (c.profile && (!rt->ensure_events(rt->t_wave_start, waves.size(), true) ||
                    !rt->ensure_events(rt->t_wave_end, waves.size(), true) ||
                    !rt->ensure_events(rt->t_copy_start, copies.size(), true) ||
                    !rt->ensure_events(rt->t_copy_end, copies.size(), true)))
    return fail_cuda();

  // staging (double-buffered pinned upload of admissions, batches, groups)
  const int sidx = rt->staging_idx;
  rt->staging_idx ^= 1;
  if (!ok(cudaEventSynchronize(rt->staging_done[sidx]), "staging reuse")) return fail_cuda();
  char *stg = rt->staging[sidx];
  int32_t *s_adm = reinterpret_cast<int32_t *>(stg);
  for (int64_t i = 0; i < n_adm; ++i) {
    s_adm[i] = 0;
    s_adm[n_adm + i] = a_rank[i];
    s_adm[2 * n_adm + i] = a_req[i];
    s_adm[3 * n_adm + i] = a_stage[i];
  }
  int32_t *s_batch = s_adm + 4 * n_adm;
  for (int64_t b = 0; b < n_batches; ++b) {
    s_batch[b] = 0;
    s_batch[n_batches + b] = b_size[b];
  }
  coe_mlp_group *s_groups = reinterpret_cast<coe_mlp_group *>(
      (reinterpret_cast<uintptr_t>(s_batch + 2 * n_batches) + 31) & ~uintptr_t(31));
  if (n_batches) {
    std::memcpy(s_groups, g_up.data(), sizeof(coe_mlp_group) * n_batches);
    std::memcpy(s_groups + n_batches, g_down.data(), sizeof(coe_mlp_group) * n_batches);
  }
  const size_t adm_bytes = 16 * (size_t)n_adm, batch_bytes = 8 * (size_t)n_batches,
               group_bytes = 2 * sizeof(coe_mlp_group) * (size_t)n_batches;

  cudaStream_t cs = rt->compute, ks = rt->copy;
  if (c.profile && !ok(cudaEventRecord(rt->t_step_start, cs), "record")) return fail_cuda();
  if (rt->have_prev && !ok(cudaStreamWaitEvent(ks, rt->prev_step_end, 0), "copy waits previous step"))
    return fail_cuda();
  int32_t *d_exec = rt->d_adm, *d_rank = rt->d_adm + n_adm, *d_req = rt->d_adm + 2 * n_adm,
          *d_stage = rt->d_adm + 3 * n_adm;
  if (n_adm && !ok(cudaMemcpyAsync(rt->d_adm, s_adm, adm_bytes, cudaMemcpyHostToDevice, cs), "adm H2D"))
    return fail_cuda();
  if (n_batches) {
    if (!ok(cudaMemcpyAsync(rt->d_batch, s_batch, batch_bytes, cudaMemcpyHostToDevice, cs), "batch H2D") ||
        !ok(cudaMemcpyAsync(rt->d_groups, s_groups, group_bytes, cudaMemcpyHostToDevice, cs), "group H2D"))
      return fail_cuda();
  }
  if (!ok(cudaEventRecord(rt->staging_done[sidx], cs), "record")) return fail_cuda();
  // K1 + K2
  if (n_adm) {
    int rc = coe_group_sort(d_exec, d_rank, n_adm, rank_bits, passes, rt->d_perm, rt->d_keys, rt->d_sort_scratch, cs);
    if (rc) return rc;
  }
  {
    int rc = coe_run_compact(rt->d_perm, rt->d_keys, d_req, d_stage, n_adm, rank_bits, rt->d_batch,
                             rt->d_batch + n_batches, (int)n_batches, 1, rt->d_boff, rt->d_mreq, rt->d_mstage,
                             rt->d_flags, rt->d_flags + 1, rt->d_compact_scratch, cs);
    if (rc) return rc;
  }
  if (c.profile && !ok(cudaEventRecord(rt->t_group_end, cs), "record")) return fail_cuda();

  const coe_mlp_group *dg_up = rt->d_groups, *dg_down = rt->d_groups + n_batches;
  for (const Action &a : actions) {
    if (a.is_copy) {
      const CopyAct &cp = copies[a.index];
      if (cp.wait_wave >= 0 && !ok(cudaStreamWaitEvent(ks, rt->wave_ev[cp.wait_wave], 0), "copy waits slot"))
        return fail_cuda();
      if (c.profile && !ok(cudaEventRecord(rt->t_copy_start[a.index], ks), "record")) return fail_cuda();
      if (!ok(cudaMemcpyAsync(rt->slab + (int64_t)cp.slot * rt->expert_bytes,
                              rt->host_store + (int64_t)cp.expert * rt->expert_bytes, rt->expert_bytes,
                              cudaMemcpyHostToDevice, ks),
              "swap-in H2D"))
        return fail_cuda();
      if (c.profile && !ok(cudaEventRecord(rt->t_copy_end[a.index], ks), "record")) return fail_cuda();
      if (!ok(cudaEventRecord(rt->copy_ev[a.index], ks), "record")) return fail_cuda();
    } else {
      const WaveAct &w = waves[a.index];
      for (int32_t cid : w.wait_copies)
        if (!ok(cudaStreamWaitEvent(cs, rt->copy_ev[cid], 0), "wave waits copy")) return fail_cuda();
      if (c.profile && !ok(cudaEventRecord(rt->t_wave_start[a.index], cs), "record")) return fail_cuda();
      int rc = coe_grouped_mlp(rt->mlp, dg_up + w.first_group, dg_down + w.first_group, w.num_groups, w.tiles_up,
                               w.tiles_down, rt->d_boff, rt->d_mreq, rt->d_mstage, 3, cs);
      if (rc) return rc;
      st.launches += 2;
      if (c.profile && !ok(cudaEventRecord(rt->t_wave_end[a.index], cs), "record")) return fail_cuda();
      if (!ok(cudaEventRecord(rt->wave_ev[a.index], cs), "record")) return fail_cuda();
    }
  }
  // join: compute waits for the copy stream, step end on compute
  if (!ok(cudaEventRecord(rt->copy_drained, ks), "record") || !ok(cudaStreamWaitEvent(cs, rt->copy_drained, 0), "join"))
    return fail_cuda();
  if (c.profile && !ok(cudaEventRecord(rt->t_step_end, cs), "record")) return fail_cuda();
  if (!ok(cudaEventRecord(rt->prev_step_end, cs), "record")) return fail_cuda();
  rt->have_prev = true;
  rt->last_waves = (int32_t)waves.size();
  rt->last_copies = (int32_t)copies.size();
  rt->last_adm = n_adm;
  rt->last_batches = n_batches;
  if (stats) *stats = st;
  return COE_CUDA_OK;
}

}  // extern "C"
