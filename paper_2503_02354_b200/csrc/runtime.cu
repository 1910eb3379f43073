// runtime.cu -- GPU serving runtime: executes one executor's op log on a B200.
//
// The reference advances a virtual clock through load / batch events
// (Simulation._start_load / _start_batch / _on_batch_done,
// /root/reference/pkg/src/coesim/engine.py:643-758); here the same op log is
// *executed*:
//
//   copy stream:     the step's plan upload, then K4 swap-ins (pinned host expert
//                    store -> HBM slot), each half of an expert (W1 | W2) issued as soon
//                    as the slot's last reader of that half has finished -- dependency-
//                    aware prefetch -- and, end to end, the stage-0 input chunks
//   compute streams: K1 group sort -> K2 run compaction, then waves of K3 grouped expert
//                    MLPs on two alternating main streams plus a high-priority release
//                    stream; a wave's up projection waits only for the W1 halves it needs,
//                    its down projection for the W2 halves; the down pass stores hopping
//                    rows into the destination executor (fused hops, peer mode)
//   output stream:   end to end, each wave's gathered final rows, one D2H copy
//
// Physical layout (HBM): fixed expert slots per shape ([W1 h*d | W2 d*h] bf16; the
// planner's ModelPool budget / expert bytes), the request inputs X (two buffers end to
// end), ping-pong activations P0/P1, the H scratch of a wave per stream, double-buffered
// step arrays.  Host: one pinned store of the experts this executor touches (the host
// tier, types.py:17).
//
// Phase A walks the op log (slot assignment: victim slots are reused; initial-residency
// experts missing after the previous step are restored lazily at first use, so a step
// always starts from initialize_pools' placement; data dependencies; hops).  Phase B
// list-schedules copies, input chunks and waves on estimated clocks.
// Phase C issues them with explicit events.  Timing never feeds back into decisions.

#include <cuda.h>
#include <cuda_bf16.h>
#include <fcntl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <array>
#include <cstring>
#include <climits>
#include <deque>
#include <map>
#include <memory>
#include <cstdlib>
#include <string>
#include <unordered_map>
#include <unordered_set>
#include <vector>

#include "coe_cuda.h"
#include "coe_planner.h"
#include "comm.h"
#include "common.cuh"
#include "act_rows.h"
#include "hops.h"

namespace {

thread_local std::string g_last_error;

constexpr int BM = 128;
constexpr int BN = 256;

uint64_t splitmix64_host(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// e2e: one wave's final rows, packed (request << 1 | P parity), gathered contiguously (one
// block per row, 16-byte vectors) so the wave's results leave in a single D2H copy
__global__ void gather_rows(const __nv_bfloat16 *p0, const __nv_bfloat16 *p1, const int32_t *req_par, int64_t row_elems,
                            __nv_bfloat16 *out) {
  const int32_t rp = req_par[blockIdx.x];
  const __nv_bfloat16 *src = ((rp & 1) ? p1 : p0) + (int64_t)(rp >> 1) * row_elems;
  const uint4 *sv = reinterpret_cast<const uint4 *>(src);
  uint4 *dv = reinterpret_cast<uint4 *>(out + (int64_t)blockIdx.x * row_elems);
  for (int64_t i = threadIdx.x; i < row_elems / 8; i += blockDim.x) dv[i] = sv[i];
}

// e2e inputs: a chunk's request rows read straight from pinned host memory over PCIe (the host
// rows are in request order, the chunk is in the order batches need it, so a DMA per request
// would be one small copy each).  A few CTAs keep ~100 KB of 16-byte loads in flight -- enough
// to fill PCIe Gen5 -- and fit next to a resident K3 CTA (94 registers x 384 threads, ~197 KB
// shared): the copy stream runs this kernel in H2D-queue order with the swap-in DMAs.
__global__ void __launch_bounds__(256) gather_inputs(const uint4 *__restrict__ host, const int64_t *__restrict__ map,
                                                     int32_t first, int32_t n, int64_t row_vec, int32_t segs_per_row,
                                                     uint4 *__restrict__ dst) {
  constexpr int SEG = 2048;  // 32 KB of a row per work item; 4 loads in flight per thread
  const int32_t items = n * segs_per_row;
  for (int32_t item = blockIdx.x; item < items; item += gridDim.x) {
    const int32_t r = item / segs_per_row, sg = item - r * segs_per_row;
    const int64_t off = (int64_t)sg * SEG;
    const int32_t len = (int32_t)(row_vec - off < SEG ? row_vec - off : SEG);
    const uint4 *src = host + map[2 * (first + r)] * row_vec + off;
    uint4 *out = dst + map[2 * (first + r) + 1] * row_vec + off;
    int32_t i = threadIdx.x;
    for (; i + 768 < len; i += 1024) {
      const uint4 v0 = src[i], v1 = src[i + 256], v2 = src[i + 512], v3 = src[i + 768];
      out[i] = v0;
      out[i + 256] = v1;
      out[i + 512] = v2;
      out[i + 768] = v3;
    }
    for (; i < len; i += 256) out[i] = src[i];
  }
}

const int kInputGatherCtas = getenv("COE_INPUT_CTAS") ? atoi(getenv("COE_INPUT_CTAS")) : 64;

struct CopyAct {
  int32_t expert;
  int32_t slot;
  bool restore;
  std::vector<int32_t> wait_waves;  // last issued reader wave of the bytes overwritten, per stream (this step)
  std::vector<int32_t> wait_prev;   // slot * NCLS + stream: last step's readers (slot_free events)
  int32_t unit0 = -1;               // pooled: first unit of the expert's new place
  const char *peer_src = nullptr;   // (f3) peer executor's bytes (else host store / generate)
  coe_runtime *peer_rt = nullptr;
  int32_t peer_exec = -1;
  int32_t peer_par = 0;
  // pooled memory: the W1 half lands on bytes an earlier expert (another shape, or placed
  // elsewhere) used as ITS W2, so it must wait for the down passes too, not just the up passes
  bool w1_waits_down = false;
};

struct WaveAct {
  int32_t cls;  // stream: 0 main, 1 release (high priority, reserved SMs)
  int32_t shape = 0;  // expert shape (one K3 tensor-map set per wave)
  int32_t first_group;
  int32_t num_groups;
  int32_t tiles_up;
  int32_t tiles_down;
  int64_t rows;
  std::vector<int32_t> wait_copies;  // W1 event before the up pass, W2 before the down pass
  std::vector<int32_t> wait_waves;   // other-stream waves producing this wave's inputs
  std::vector<int32_t> wait_recvs;   // hops (local index) this wave consumes
  std::vector<int32_t> frees_slots;  // slots whose last reader this step, on this stream, is this wave
};

struct Action {
  bool is_copy;      // swap-in (index: copy) ...
  int32_t index;
  bool is_input = false;  // ... or an e2e stage-0 input upload (index: batch), same copy engine
};

bool ok(cudaError_t e, const char *what) { return coe_cuda_ok(e, what); }

// Stream memory operations (driver API, resolved once): the fused-hop flags.
using StreamValueFn = CUresult (*)(CUstream, CUdeviceptr, cuuint32_t, unsigned int);
struct StreamMemops {
  StreamValueFn wait = nullptr, write = nullptr;
};
const StreamMemops *stream_memops() {
  static StreamMemops ops;
  static bool tried = false;
  if (!tried) {
    tried = true;
    void *w = nullptr, *v = nullptr;
    cudaDriverEntryPointQueryResult q1, q2;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue32", &w, cudaEnableDefault, &q1) == cudaSuccess &&
        q1 == cudaDriverEntryPointSuccess &&
        cudaGetDriverEntryPoint("cuStreamWriteValue32", &v, cudaEnableDefault, &q2) == cudaSuccess &&
        q2 == cudaDriverEntryPointSuccess) {
      ops.wait = reinterpret_cast<StreamValueFn>(w);
      ops.write = reinterpret_cast<StreamValueFn>(v);
    }
  }
  return ops.wait ? &ops : nullptr;
}
// A flag satisfied by a REMOTE write (a peer GPU's cuStreamWriteValue32 after its NVLink row
// stores) does not by itself make those stores visible to later work on this device: the
// device may reorder remote writes internally.  Where the device can flush remote writes
// (CU_DEVICE_ATTRIBUTE_CAN_FLUSH_REMOTE_WRITES) the wait carries CU_STREAM_WAIT_VALUE_FLUSH;
// elsewhere a one-thread kernel re-reads the flag with a system-scope acquire, which orders
// every later kernel on the stream after the peer's release.
__global__ void acquire_flag(const int32_t *addr, uint32_t value) {
  uint32_t v;
  do {
    asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(addr) : "memory");
  } while ((int32_t)(v - value) < 0);
}
int can_flush_remote_writes() {
  static int cached = -1;
  if (cached < 0) {
    using AttrFn = CUresult (*)(int *, CUdevice_attribute, CUdevice);
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    int dev = 0, v = 0;
    cudaGetDevice(&dev);
    if (cudaGetDriverEntryPoint("cuDeviceGetAttribute", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess &&
        reinterpret_cast<AttrFn>(p)(&v, CU_DEVICE_ATTRIBUTE_CAN_FLUSH_REMOTE_WRITES, dev) == CUDA_SUCCESS)
      cached = v ? 1 : 0;
    else
      cached = 0;
  }
  return cached;
}
bool wait_flag(cudaStream_t s, const int32_t *addr, uint32_t value, bool remote = true) {
  const bool flush = remote && can_flush_remote_writes();
  CUresult r = stream_memops()->wait(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(addr), value,
                                     CU_STREAM_WAIT_VALUE_GEQ | (flush ? CU_STREAM_WAIT_VALUE_FLUSH : 0));
  if (r != CUDA_SUCCESS) {
    coe_set_error("cuStreamWaitValue32 failed (" + std::to_string((int)r) + ")");
    return false;
  }
  if (remote && !flush) {
    acquire_flag<<<1, 1, 0, s>>>(addr, value);
    return coe_cuda_ok(cudaGetLastError(), "acquire flag");
  }
  return true;
}
// default flags: the write follows a memory barrier, so the producer kernel's stores (peer
// stores included) are visible before the flag is
bool write_flag(cudaStream_t s, int32_t *addr, uint32_t value) {
  CUresult r = stream_memops()->write(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(addr), value,
                                      CU_STREAM_WRITE_VALUE_DEFAULT);
  if (r != CUDA_SUCCESS) coe_set_error("cuStreamWriteValue32 failed (" + std::to_string((int)r) + ")");
  return r == CUDA_SUCCESS;
}

// Release-wave grid: the reserved SMs (COE_RELEASE_CTAS overrides, for experiments).
int release_grid(int reserved, int /*sms*/) {
  if (const char *v = getenv("COE_RELEASE_CTAS")) return std::max(2, atoi(v) & ~1);
  return reserved;
}

// Row-run copies, one cudaMemcpyAsync each: the e2e path merges each chunk's requests into
// runs that are contiguous on both sides (usually the whole chunk), so the count stays small.
bool run_copies(const std::vector<void *> &dsts, const std::vector<void *> &srcs, const std::vector<size_t> &sizes,
                cudaStream_t stream, const char *what) {
  for (size_t i = 0; i < dsts.size(); ++i)
    if (!ok(cudaMemcpyAsync(dsts[i], srcs[i], sizes[i], cudaMemcpyDefault, stream), what)) return false;
  return true;
}

}  // namespace

void coe_set_error(const std::string &msg) { g_last_error = msg; }

struct coe_runtime;

struct StepBuffers {  // device arrays one step uses; two sets alternate
  int32_t *adm = nullptr;   // [6][max_adm]: exec, rank, req, stage, in route, out route
  int32_t *batch = nullptr; // [2][max_batches]: exec, size
  int32_t *boff = nullptr;
  int32_t *mreq = nullptr, *mstage = nullptr, *min = nullptr, *mout = nullptr;
  coe_mlp_group *groups = nullptr;  // [2][max_batches]
  int64_t *in_map = nullptr;        // e2e inputs, need order: [max_requests][host row, A row]
  cudaEvent_t free_ev = nullptr;    // recorded on compute when the step using this set ends
  bool used = false;
};

struct coe_runtime {
  coe_runtime_config cfg{};
  // expert shapes: shape k owns global slots [slot_base[k], slot_base[k] + slot_count[k]) in
  // its own slab of sbytes[k]-sized slots; act_ld = widest d (activation row stride)
  int S = 1;
  std::vector<int32_t> sd, sh, slot_base, slot_count, slot_shape, expert_shape;
  std::vector<int64_t> sbytes, sstride, store_off;
  std::vector<char *> slabs;
  int32_t act_ld = 0, h_max = 0, total_slots = 0;
  int64_t row_elems = 0;  // T * act_ld
  // Expert memory under ONE byte budget for several shapes (cfg.expert_pool_bytes > 0): one
  // slab addressed in 2 MB units; a load takes a best-fit run of free units, an eviction
  // returns its run -- so the planner's byte-budgeted pool (expert_pool.py:27-59) bounds
  // physical HBM whatever the shape mix (the slab is the budget plus one largest expert of
  // slack against fragmentation).  Every shape's weight tensor maps span the whole slab with
  // a one-unit "slot" stride, so an expert is addressed by its first unit.  Each expert keeps
  // a static bookkeeping slot (readers, events); freed units remember the slot that last used
  // them, and a later copy into them waits for that slot's readers.
  bool pooled = false;
  int64_t unit = 0, pool_units = 0;
  char *pool = nullptr;
  std::map<int32_t, int32_t> free_runs;  // first unit -> run length
  std::vector<int32_t> unit_owner;       // slot that last used the unit (-1: never)
  std::vector<uint8_t> unit_w2;          // the unit held the W2 half of its last expert
  std::vector<int32_t> slot_unit, slot_units;  // per slot: first unit / units of its residency
  std::vector<int32_t> expert_vslot;     // expert -> its bookkeeping slot

  char *slot_ptr(int32_t s) const {
    if (pooled) return pool + (int64_t)slot_unit[s] * unit;
    const int k = slot_shape[s];
    return slabs[k] + (int64_t)(s - slot_base[k]) * sstride[k];
  }
  // wave classes, one stream each: 0 main (experts resident since step start; also runs K1/K2
  // and the step join), 1 release (last readers of slots a later swap-in overwrites: high
  // priority on reserved SMs -- they gate the copy engine), 2 swapped (experts copied this
  // step: waits for copies in op order without blocking class 0); copy = plan upload + swap-ins
  static constexpr int NCLS = 3;
  cudaStream_t cls_stream[NCLS] = {nullptr, nullptr, nullptr};
  cudaStream_t compute = nullptr, copy = nullptr;  // compute == cls_stream[0]
  // device memory: X / Y device-resident request inputs / final outputs ([requests][T][ld],
  // device_io only); A the activation rows [landing | ring] (act_rows.h); the output staging
  // ring (e2e finals, download staging)
  __nv_bfloat16 *x = nullptr, *y = nullptr, *act = nullptr, *outbuf = nullptr;
  int32_t ring_slots = 0, landing_slots = 0, out_slots = 0;
  std::vector<int32_t> ring_order;     // free list of ring slots (absolute A rows), FIFO across steps
  std::vector<int32_t> act_prev_wave;  // per A row: wave of the previous step that freed it (-1: none)
  bool prev_nccl_hold = false;         // the previous step kept NCCL hop-out rows until its end
  int64_t out_pos = 0;                 // e2e: global position of the next staging row
  struct OutUse {
    int64_t begin, end;
    cudaEvent_t ev;
  };
  std::deque<OutUse> out_hist;         // e2e: staging rows still being downloaded
  std::vector<cudaEvent_t> out_ev_pool;
  int step_parity = 0;                 // wave events alternate by step (the next step refers back)
  bool last_group_fused = false;       // the last step grouped with coe_group_compact_fused
  __nv_bfloat16 *hbuf[NCLS] = {nullptr, nullptr, nullptr};
  StepBuffers sets[2];
  int cur_set = 0;
  int32_t *d_perm = nullptr, *d_keys = nullptr, *d_flags = nullptr, *d_last = nullptr;
  void *d_sort_scratch = nullptr, *d_compact_scratch = nullptr;
  // host
  char *host_store = nullptr;
  bool store_mapped = false;  // shared (mmap + cudaHostRegister) instead of cudaHostAlloc
  size_t store_bytes = 0;
  char *staging[2] = {nullptr, nullptr};
  int64_t staging_bytes = 0;
  cudaEvent_t staging_done[2] = {nullptr, nullptr};
  int32_t *h_last = nullptr;
  std::vector<std::array<coe_mlp *, NCLS>> mlps;  // [shape][stream class]
  // slot state (persists across steps)
  std::vector<int32_t> slot_expert, expert_slot;
  // last reader of each slot half in the previous step, per compute stream ([slot * NCLS + cls])
  std::vector<cudaEvent_t> slot_free_up, slot_free_down;
  std::vector<uint8_t> slot_free_valid;
  // events (wave events per step parity: e2e uploads of step k+1 wait on step k's waves)
  std::vector<cudaEvent_t> wave_up_evs[2], wave_down_evs[2], copy_up_ev, copy_down_ev, out_ev;
  std::vector<int32_t> out_order;  // e2e: request of each host output row (completion order)
  std::vector<cudaEvent_t> t_copy_start, t_copy_end, t_wave_start, t_wave_end, t_up_end, t_down_start;
  std::vector<cudaEvent_t> t_io;    // profile, e2e: [start, end] event pairs of uploads / downloads
  std::vector<uint8_t> io_kind;      // per pair: 0 input upload, 1 output download
  std::vector<double> last_wave_flops;  // algorithmic 4*rows*d*h per wave
  cudaEvent_t staged = nullptr, copy_drained = nullptr, grouped = nullptr;
  cudaEvent_t cls_drained[NCLS] = {nullptr, nullptr, nullptr};
  cudaEvent_t t_step_start = nullptr, t_group_end = nullptr, t_step_end = nullptr;
  int32_t last_waves = 0, last_copies = 0;
  std::vector<int32_t> last_wave_cls, last_wave_rows, last_wave_groups, last_wave_shape;
  int64_t last_adm = 0, last_batches = 0;
  int last_set = 0;
  cudaStream_t out_stream = nullptr;  // e2e output downloads (inputs ride the copy engine)
  cudaStream_t copy_in = nullptr;     // e2e inputs: the gather kernels' queue
  std::vector<cudaEvent_t> in_ev;
  cudaEvent_t out_drained = nullptr;
  bool have_out = false;
  coe_comm *comm = nullptr;            // hop transport (N > 1)
  cudaStream_t hop = nullptr;
  std::vector<cudaEvent_t> recv_ev;
  cudaEvent_t hop_drained = nullptr, step_end = nullptr;
  // (f3) peer-GPU swap-in tier between runtimes of one process: at the end of every step the
  // runtime records where each resident expert's bytes live (double-buffered by step parity,
  // so a peer in the next step reads a stable copy) and an event after the step's work
  int device = 0;
  int64_t step_count = 0;
  std::vector<const char *> res_snap[2];
  cudaEvent_t res_ready[2] = {nullptr, nullptr};
  std::vector<coe_runtime *> local_peers;
  // ... and between processes (CUDA IPC): each peer's expert allocations mapped here, the
  // peer's end-of-step residency (exchanged on the host after every step, as slab<<40|offset
  // codes), and whether a peer read our experts last step (our copies then wait for its end)
  std::vector<std::vector<char *>> peer_exp_base;      // [rank][slab]
  std::vector<std::vector<const char *>> ipc_snap;     // [rank][expert] (previous step)
  bool peer_read_prev = false;
  bool have_step_end = false;
  // fused hops over peer memory (coe_runtime_attach_peers): K3's down pass stores a hopping
  // request's rows into the destination executor's P buffer; flags are published with stream
  // memory operations.  d_hflags: [max_admissions] hop flags (by global hop index) followed
  // by COE_MAX_PEERS step flags; each holds the step sequence number that last set it.
  int32_t *d_hflags = nullptr;
  int64_t hflag_step_base = 0;
  std::vector<coe_peer_buffers> peers;  // every executor's buffers as mapped in this process
  std::vector<void *> ipc_opened;
  int32_t peer_rank = -1, peer_world = 0;
  coe_local_hub *peer_hub = nullptr;  // same-process peers: host-side event handoff, no flags
  uint32_t step_seq = 0;
  int m_ctas = 148, r_ctas = 16;  // SM split: main waves vs the swap-in-gating waves
  int rel_launch_ctas = 148;      // grid of a release wave (all SMs; see phase C)

  ~coe_runtime() {
    for (auto st : cls_stream)
      if (st) cudaStreamSynchronize(st);
    if (copy) cudaStreamSynchronize(copy);
    if (copy_in) cudaStreamSynchronize(copy_in);
    if (hop) cudaStreamSynchronize(hop);
    if (out_stream) cudaStreamSynchronize(out_stream);
    for (auto &per : mlps)
      for (auto m : per)
        if (m) coe_mlp_destroy(m);
    std::vector<void *> dev = {x, y, act, hbuf[0], hbuf[1], hbuf[2], outbuf, d_perm, d_keys, d_flags, d_last,
                               d_sort_scratch, d_compact_scratch};
    if (pooled) {
      dev.push_back(pool);
    } else {
      for (char *sl : slabs) dev.push_back(sl);
    }
    for (auto &s : sets) {
      for (void *p : {(void *)s.adm, (void *)s.batch, (void *)s.boff, (void *)s.mreq, (void *)s.mstage, (void *)s.in_map,
                      (void *)s.min, (void *)s.mout, (void *)s.groups})
        dev.push_back(p);
      if (s.free_ev) cudaEventDestroy(s.free_ev);
    }
    for (void *p : dev)
      if (p) cudaFree(p);
    for (void *p : ipc_opened) cudaIpcCloseMemHandle(p);
    if (d_hflags) cudaFree(d_hflags);
    for (void *p : {(void *)staging[0], (void *)staging[1], (void *)h_last})
      if (p) cudaFreeHost(p);
    if (host_store && store_mapped) {
      cudaHostUnregister(host_store);
      munmap(host_store, store_bytes);
    } else if (host_store) {
      cudaFreeHost(host_store);
    }
    for (auto *v : {&in_ev, &recv_ev, &slot_free_up, &slot_free_down, &wave_up_evs[0], &wave_down_evs[0],
                    &wave_up_evs[1], &wave_down_evs[1], &copy_up_ev, &copy_down_ev, &out_ev, &out_ev_pool,
                    &t_copy_start, &t_copy_end, &t_wave_start, &t_wave_end, &t_up_end, &t_down_start, &t_io}) {
      for (auto e : *v) cudaEventDestroy(e);
      v->clear();
    }
    for (auto &u : out_hist) cudaEventDestroy(u.ev);
    for (cudaEvent_t e : {out_drained, hop_drained, step_end, staged, copy_drained, grouped, cls_drained[0], cls_drained[1], cls_drained[2], t_step_start, t_group_end, t_step_end, staging_done[0],
                          staging_done[1], res_ready[0], res_ready[1]})
      if (e) cudaEventDestroy(e);
    for (auto st : cls_stream)
      if (st) cudaStreamDestroy(st);
    if (copy) cudaStreamDestroy(copy);
    if (copy_in) cudaStreamDestroy(copy_in);
    if (hop) cudaStreamDestroy(hop);
    if (out_stream) cudaStreamDestroy(out_stream);
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

constexpr int64_t kPoolUnit = 2ll << 20;  // allocation unit of the pooled expert slab

// One slab of pool_bytes for every shape; each expert gets a bookkeeping slot (its rank among
// the experts of its shape); every unit free.
bool pool_create(coe_runtime *rt, int64_t pool_bytes) {
  rt->unit = kPoolUnit;
  rt->pool_units = (pool_bytes + rt->unit - 1) / rt->unit;
  if (rt->pool_units >= (1ll << 27)) {
    coe_set_error("pooled expert memory: too many units");
    return false;
  }
  if (!ok(cudaMalloc(&rt->pool, (size_t)(rt->pool_units * rt->unit)), "expert pool alloc")) return false;
  for (int k = 0; k < rt->S; ++k) {
    rt->slabs[k] = rt->pool;
    rt->sstride[k] = rt->unit;
  }
  rt->pooled = true;
  rt->free_runs = {{0, (int32_t)rt->pool_units}};
  rt->unit_owner.assign((size_t)rt->pool_units, -1);
  rt->unit_w2.assign((size_t)rt->pool_units, 0);
  rt->slot_unit.assign(rt->total_slots, -1);
  rt->slot_units.assign(rt->total_slots, 0);
  rt->expert_vslot.assign(rt->cfg.num_experts, -1);
  std::vector<int32_t> next(rt->S, 0);
  for (int32_t e = 0; e < rt->cfg.num_experts; ++e) {
    const int k = rt->expert_shape[e];
    if (next[k] >= rt->slot_count[k]) {
      coe_set_error("pooled expert memory: more experts of a shape than its slots");
      return false;
    }
    rt->expert_vslot[e] = rt->slot_base[k] + next[k]++;
  }
  return true;
}

float elapsed(cudaEvent_t a, cudaEvent_t b) {
  float ms = 0.f;
  cudaEventElapsedTime(&ms, a, b);
  return ms;
}

std::vector<std::pair<float, float>> merged(std::vector<std::pair<float, float>> v) {
  std::sort(v.begin(), v.end());
  std::vector<std::pair<float, float>> out;
  for (auto &iv : v) {
    if (!out.empty() && iv.first <= out.back().second) out.back().second = std::max(out.back().second, iv.second);
    else out.push_back(iv);
  }
  return out;
}

float union_len(const std::vector<std::pair<float, float>> &v) {
  float total = 0.f;
  for (auto &iv : merged(v)) total += iv.second - iv.first;
  return total;
}

float intersect_len(const std::vector<std::pair<float, float>> &a0, const std::vector<std::pair<float, float>> &b0) {
  auto a = merged(a0), b = merged(b0);
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

// The host tier: one pinned copy of every expert.  With store_path set (multi-GPU on one
// node) the copy lives in a shared file mapping registered with every process's CUDA
// context, so N ranks share one 60 GB store instead of pinning N copies.
static bool rt_alloc_store(coe_runtime *rt, const char *path) {
  rt->store_bytes = 0;
  for (int64_t off : rt->store_off) rt->store_bytes = std::max<size_t>(rt->store_bytes, (size_t)(off >= 0 ? off : 0));
  rt->store_bytes = 0;
  for (int32_t e = 0; e < rt->cfg.num_experts; ++e)
    if (rt->store_off[e] >= 0) rt->store_bytes = std::max<size_t>(rt->store_bytes, (size_t)rt->store_off[e] + rt->sbytes[rt->expert_shape[e]]);
  if (rt->store_bytes == 0) rt->store_bytes = 16;
  if (!path || !*path)
    return ok(cudaHostAlloc(reinterpret_cast<void **>(&rt->host_store), rt->store_bytes, cudaHostAllocDefault),
              "pinned expert store");
  int fd = open(path, O_RDWR | O_CREAT, 0600);
  if (fd < 0 || ftruncate(fd, (off_t)rt->store_bytes) != 0) {
    if (fd >= 0) close(fd);
    coe_set_error(std::string("cannot create shared expert store ") + path);
    return false;
  }
  void *p = mmap(nullptr, rt->store_bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) {
    coe_set_error("mmap of the shared expert store failed");
    return false;
  }
  rt->host_store = static_cast<char *>(p);
  rt->store_mapped = true;
  return ok(cudaHostRegister(p, rt->store_bytes, cudaHostRegisterPortable), "cudaHostRegister expert store");
}

extern "C" {

const char *coe_cuda_last_error(void) { return g_last_error.c_str(); }

uint64_t coe_expert_seed(uint64_t weight_seed, int32_t expert, int32_t matrix) {
  return splitmix64_host(weight_seed ^ (uint64_t)(2 * (int64_t)expert + matrix + 1) * 0xD1B54A32D192ED03ull);
}

int coe_runtime_create(const coe_runtime_config *cfg, coe_runtime **out) {
  auto *rt = new coe_runtime();
  rt->cfg = *cfg;
  const auto &c = rt->cfg;
  if (c.num_shapes > 0) {
    rt->S = c.num_shapes;
    for (int k = 0; k < rt->S; ++k) {
      rt->sd.push_back(c.shape_d[k]);
      rt->sh.push_back(c.shape_h[k]);
      rt->slot_count.push_back(c.shape_slots[k]);
    }
  } else {
    rt->S = 1;
    rt->sd = {c.d};
    rt->sh = {c.h};
    rt->slot_count = {c.num_slots};
  }
  for (int k = 0; k < rt->S; ++k) {
    rt->sbytes.push_back(2LL * rt->sd[k] * rt->sh[k] * 2);
    rt->slot_base.push_back(rt->total_slots);
    rt->total_slots += rt->slot_count[k];
    for (int32_t q = 0; q < rt->slot_count[k]; ++q) rt->slot_shape.push_back(k);
    rt->act_ld = std::max(rt->act_ld, rt->sd[k]);
    rt->h_max = std::max(rt->h_max, rt->sh[k]);
  }
  rt->expert_shape.assign(c.num_experts, 0);
  if (c.num_shapes > 0 && c.expert_shape)
    for (int32_t e = 0; e < c.num_experts; ++e) rt->expert_shape[e] = c.expert_shape[e];
  rt->store_off.assign(c.num_experts, -1);
  {
    int64_t off = 0;
    for (int32_t e = 0; e < c.num_experts; ++e)
      if (!c.store_mask || c.store_mask[e]) {
        rt->store_off[e] = off;
        off += rt->sbytes[rt->expert_shape[e]];
      }
  }
  rt->row_elems = (int64_t)c.T * rt->act_ld;
  const int64_t io_bytes = c.device_io ? (int64_t)c.max_requests * rt->row_elems * 2 : 0;
  rt->ring_slots = std::max(1, c.ring_slots);
  rt->landing_slots = std::max(0, c.landing_slots);
  // staging for e2e finals: several waves' worth (a wave holds at most max_wave_rows / T requests)
  rt->out_slots = c.out_slots > 0 ? c.out_slots : (int32_t)std::max<int64_t>(64, 2 * c.max_wave_rows / c.T);
  const int64_t a_rows = (int64_t)rt->landing_slots + rt->ring_slots;
  const size_t A = (size_t)c.max_admissions, B = (size_t)c.max_batches;
  int prio_low = 0, prio_high = 0;
  cudaDeviceGetStreamPriorityRange(&prio_low, &prio_high);
  bool good = ok(cudaStreamCreateWithPriority(&rt->cls_stream[0], cudaStreamNonBlocking, prio_low), "stream") &&
              ok(cudaStreamCreateWithPriority(&rt->cls_stream[1], cudaStreamNonBlocking, prio_high), "stream") &&
              ok(cudaStreamCreateWithPriority(&rt->cls_stream[2], cudaStreamNonBlocking, prio_low), "stream") &&
              ok(cudaStreamCreateWithFlags(&rt->copy, cudaStreamNonBlocking), "stream") &&
              ok(cudaStreamCreateWithFlags(&rt->hop, cudaStreamNonBlocking), "stream") &&
              ok(cudaStreamCreateWithFlags(&rt->out_stream, cudaStreamNonBlocking), "stream") &&
              ok(cudaStreamCreateWithFlags(&rt->copy_in, cudaStreamNonBlocking), "stream") &&
              ok(cudaGetDevice(&rt->device), "device") &&
              ok(cudaEventCreateWithFlags(&rt->res_ready[0], cudaEventDisableTiming), "event") &&
              ok(cudaEventCreateWithFlags(&rt->res_ready[1], cudaEventDisableTiming), "event") &&
              (!c.device_io || (dmalloc(&rt->x, io_bytes, "X alloc") && dmalloc(&rt->y, io_bytes, "Y alloc"))) &&
              dmalloc(&rt->act, a_rows * rt->row_elems * 2, "activation ring alloc") &&
              dmalloc(&rt->outbuf, (int64_t)rt->out_slots * rt->row_elems * 2, "output staging alloc") &&
              dmalloc(&rt->hbuf[0], (size_t)c.max_wave_rows * rt->h_max * 2, "H alloc") &&
              dmalloc(&rt->hbuf[1], (size_t)c.max_wave_rows * rt->h_max * 2, "H alloc") &&
              dmalloc(&rt->hbuf[2], (size_t)c.max_wave_rows * rt->h_max * 2, "H alloc") &&
              dmalloc(&rt->d_perm, 4 * A, "perm alloc") && dmalloc(&rt->d_keys, 4 * A, "keys alloc") &&
              dmalloc(&rt->d_flags, 64, "flags alloc") && dmalloc(&rt->d_last, 4 * (size_t)c.max_requests, "last") &&
              dmalloc(&rt->d_sort_scratch, (size_t)coe_group_sort_scratch_bytes(c.max_admissions), "sort scratch") &&
              dmalloc(&rt->d_compact_scratch, (size_t)coe_run_compact_scratch_bytes(c.max_admissions, (int)B, 1),
                      "compact scratch") &&
              dmalloc(&rt->d_hflags, 4 * (A + COE_MAX_PEERS), "hop flags") &&
              ok(cudaMemset(rt->d_hflags, 0, 4 * (A + COE_MAX_PEERS)), "hop flags");
  rt->hflag_step_base = (int64_t)A;
  rt->slabs.assign(rt->S, nullptr);
  rt->sstride = rt->sbytes;
  if (c.expert_pool_bytes > 0) {
    good = good && pool_create(rt, c.expert_pool_bytes);
  } else {
    for (int k = 0; k < rt->S; ++k)
      good = good && dmalloc(&rt->slabs[k], (size_t)rt->sbytes[k] * std::max(1, rt->slot_count[k]), "slab alloc");
  }
  for (auto &s : rt->sets)
    good = good && dmalloc(&s.adm, 24 * A, "adm alloc") && dmalloc(&s.batch, 8 * B, "batch alloc") &&
           dmalloc(&s.boff, 4 * B, "boff alloc") && dmalloc(&s.mreq, 4 * A, "member alloc") &&
           dmalloc(&s.mstage, 4 * A, "member alloc") && dmalloc(&s.min, 4 * A, "member alloc") &&
           dmalloc(&s.mout, 4 * A, "member alloc") && dmalloc(&s.groups, 2 * sizeof(coe_mlp_group) * B, "groups") &&
           dmalloc(&s.in_map, 16 * (size_t)c.max_requests, "input map") &&
           ok(cudaEventCreateWithFlags(&s.free_ev, cudaEventDisableTiming), "event");
  rt->compute = rt->cls_stream[0];
  if (good) {
    rt->staging_bytes = 24 * A + 8 * B + 2 * sizeof(coe_mlp_group) * B + 16 * (int64_t)c.max_requests + 1024;
    good = ok(cudaHostAlloc(reinterpret_cast<void **>(&rt->staging[0]), rt->staging_bytes, cudaHostAllocDefault), "staging") &&
           ok(cudaHostAlloc(reinterpret_cast<void **>(&rt->staging[1]), rt->staging_bytes, cudaHostAllocDefault), "staging") &&
           ok(cudaHostAlloc(reinterpret_cast<void **>(&rt->h_last), 4 * (size_t)c.max_requests, cudaHostAllocDefault), "last") &&
           rt_alloc_store(rt, c.store_path) &&
           ok(cudaEventCreateWithFlags(&rt->staging_done[0], cudaEventDisableTiming), "event") &&
           ok(cudaEventCreateWithFlags(&rt->staging_done[1], cudaEventDisableTiming), "event") &&
           ok(cudaEventCreateWithFlags(&rt->staged, cudaEventDisableTiming), "event") &&
           ok(cudaEventCreateWithFlags(&rt->copy_drained, cudaEventDisableTiming), "event") &&
           ok(cudaEventCreateWithFlags(&rt->grouped, cudaEventDisableTiming), "event") &&
           ok(cudaEventCreateWithFlags(&rt->hop_drained, cudaEventDisableTiming), "event") &&
           ok(cudaEventCreateWithFlags(&rt->out_drained, cudaEventDisableTiming), "event") &&
           ok(cudaEventCreateWithFlags(&rt->step_end, cudaEventDisableTiming), "event") &&
           ok(cudaEventCreateWithFlags(&rt->cls_drained[0], cudaEventDisableTiming), "event") &&
           ok(cudaEventCreateWithFlags(&rt->cls_drained[1], cudaEventDisableTiming), "event") &&
           ok(cudaEventCreateWithFlags(&rt->cls_drained[2], cudaEventDisableTiming), "event") &&
           ok(cudaEventCreate(&rt->t_step_start), "event") && ok(cudaEventCreate(&rt->t_group_end), "event") &&
           ok(cudaEventCreate(&rt->t_step_end), "event") &&
           rt->ensure_events(rt->slot_free_up, (size_t)rt->total_slots * coe_runtime::NCLS, false) &&
           rt->ensure_events(rt->slot_free_down, (size_t)rt->total_slots * coe_runtime::NCLS, false);
  }
  if (good) {
    rt->mlps.assign(rt->S, std::array<coe_mlp *, coe_runtime::NCLS>{nullptr, nullptr, nullptr});
    for (int sk = 0; sk < rt->S && good; ++sk) {
      coe_mlp_config mc{};
      mc.d = rt->sd[sk];
      mc.h = rt->sh[sk];
      mc.T = c.T;
      mc.x = c.device_io ? rt->x : rt->act;  // e2e-only runtimes read stage-0 inputs from A
      mc.act0 = rt->act;
      mc.act1 = rt->act;
      mc.act_rows = a_rows * c.T;
      mc.x_rows = c.device_io ? (int64_t)c.max_requests * c.T : a_rows * c.T;
      mc.act_ld = rt->act_ld;
      mc.h_rows = c.max_wave_rows;
      mc.slab = rt->slabs[sk];
      mc.num_slots = rt->pooled ? (int32_t)rt->pool_units : std::max(1, rt->slot_count[sk]);
      mc.slot_stride_bytes = rt->sstride[sk];
      for (int k = 0; k < coe_runtime::NCLS && good; ++k) {
        mc.h_scratch = rt->hbuf[k];
        if (coe_mlp_create(&mc, &rt->mlps[sk][k]) != COE_CUDA_OK ||
            coe_mlp_set_outputs(rt->mlps[sk][k], rt->y, rt->outbuf) != COE_CUDA_OK)
          good = false;
      }
    }
  }
  if (!good) {
    std::string msg = g_last_error;
    delete rt;
    g_last_error = msg;
    return COE_CUDA_ERR_CUDA;
  }
  {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int reserve = c.reserve_sms > 0 ? std::min(c.reserve_sms, sms / 2) : 0;
    rt->m_ctas = sms - reserve;
    rt->r_ctas = reserve > 0 ? reserve : sms;
    rt->rel_launch_ctas = release_grid(rt->r_ctas, sms);
  }
  rt->slot_expert.assign(rt->total_slots, -1);
  rt->expert_slot.assign(c.num_experts, -1);
  rt->slot_free_valid.assign((size_t)rt->total_slots * coe_runtime::NCLS, 0);
  for (int32_t q = 0; q < rt->ring_slots; ++q) rt->ring_order.push_back(rt->landing_slots + q);
  rt->act_prev_wave.assign((size_t)a_rows, -1);
  *out = rt;
  return COE_CUDA_OK;
}

void coe_runtime_destroy(coe_runtime *rt) { delete rt; }

void *coe_runtime_buffer(coe_runtime *rt, int which) {
  switch (which) {
    case 0: return rt->x;
    case 1: return rt->act;
    case 2: return rt->y;
    case 3: return rt->hbuf[0];
    case 4: return rt->slabs[0];
    case 5: return rt->host_store;
    case 6: return rt->outbuf;
    default: return nullptr;
  }
}

cudaStream_t coe_runtime_stream(coe_runtime *rt, int which) {
  if (which == 1) return rt->copy;
  if (which == 0) return rt->compute;
  return (which >= 2 && which - 1 < coe_runtime::NCLS) ? rt->cls_stream[which - 1] : nullptr;
}

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
  if (!ok(cudaDeviceSynchronize(), "init experts sync")) return fail_cuda();
  char *scratch = nullptr;  // pooled: no expert has units yet -- generate into a scratch expert
  if (rt->pooled) {
    const int64_t big = *std::max_element(rt->sbytes.begin(), rt->sbytes.end());
    if (!ok(cudaMalloc(&scratch, (size_t)big), "init scratch")) return fail_cuda();
  }
  for (int32_t e = 0; e < c.num_experts; ++e) {  // generate into the shape's first slot, stage to the store
    if (rt->store_off[e] < 0) continue;
    const int k = rt->expert_shape[e];
    if (rt->slot_count[k] < 1) {
      coe_set_error("init_experts: a stored expert's shape has no HBM slot");
      return COE_CUDA_ERR_CONFIG;
    }
    const int64_t half = (int64_t)rt->sd[k] * rt->sh[k];  // elements per matrix
    __nv_bfloat16 *w = reinterpret_cast<__nv_bfloat16 *>(scratch ? scratch : rt->slabs[k]);
    if (coe_fill_uniform_bf16(w, half, coe_expert_seed(c.weight_seed, e, 0), sqrtf(3.0f / rt->sd[k]), rt->compute) ||
        coe_fill_uniform_bf16(w + half, half, coe_expert_seed(c.weight_seed, e, 1), sqrtf(3.0f / rt->sh[k]),
                              rt->compute))
      return COE_CUDA_ERR_CUDA;
    if (!ok(cudaMemcpyAsync(rt->host_store + rt->store_off[e], w, rt->sbytes[k], cudaMemcpyDeviceToHost, rt->compute),
            "expert store D2H"))
      return fail_cuda();
  }
  if (!ok(cudaStreamSynchronize(rt->compute), "init experts")) return fail_cuda();
  if (scratch) cudaFree(scratch);
  if (rt->pooled) {  // every unit free
    rt->free_runs = {{0, (int32_t)rt->pool_units}};
    std::fill(rt->unit_owner.begin(), rt->unit_owner.end(), -1);
    std::fill(rt->unit_w2.begin(), rt->unit_w2.end(), 0);
    std::fill(rt->slot_units.begin(), rt->slot_units.end(), 0);
  }
  std::fill(rt->slot_expert.begin(), rt->slot_expert.end(), -1);
  std::fill(rt->expert_slot.begin(), rt->expert_slot.end(), -1);
  std::fill(rt->slot_free_valid.begin(), rt->slot_free_valid.end(), 0);
  return COE_CUDA_OK;
}

int coe_runtime_fill_inputs(coe_runtime *rt, uint64_t seed, int32_t num_requests) {
  if (!rt->x) {
    coe_set_error("fill_inputs: runtime created without device_io (no X buffer)");
    return COE_CUDA_ERR_CONFIG;
  }
  if (num_requests > rt->cfg.max_requests) {
    coe_set_error("fill_inputs: more requests than the runtime was sized for");
    return COE_CUDA_ERR_CONFIG;
  }
  int rc = coe_fill_uniform_bf16(rt->x, (int64_t)num_requests * rt->row_elems, seed, sqrtf(3.0f), rt->compute);
  if (rc) return rc;
  return ok(cudaStreamSynchronize(rt->compute), "fill inputs") ? COE_CUDA_OK : fail_cuda();
}

int coe_runtime_upload_inputs(coe_runtime *rt, const void *host, int32_t num_requests) {
  if (!rt->x) {
    coe_set_error("upload_inputs: runtime created without device_io (no X buffer)");
    return COE_CUDA_ERR_CONFIG;
  }
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
  (void)last_stage_host;  // device-resident steps store every request's final rows in Y[request]
  if (num_requests <= 0) return COE_CUDA_OK;
  if (!rt->y || num_requests > rt->cfg.max_requests) {
    coe_set_error("download_outputs: no device output buffer (device_io) or too many requests");
    return COE_CUDA_ERR_CONFIG;
  }
  return ok(cudaMemcpyAsync(host, rt->y, (size_t)num_requests * rt->row_elems * 2, cudaMemcpyDeviceToHost,
                            rt->compute),
            "output D2H")
             ? COE_CUDA_OK
             : fail_cuda();
}

int coe_runtime_download_requests(coe_runtime *rt, const int32_t *requests, const int32_t *stages, int32_t n,
                                  void *host) {
  if (n <= 0) return COE_CUDA_OK;
  if (n > rt->cfg.max_requests) {
    coe_set_error("download_requests: more rows than the runtime was sized for");
    return COE_CUDA_ERR_CONFIG;
  }
  for (int32_t i = 0; i < n; ++i)
    if (requests[i] < 0 || requests[i] >= rt->cfg.max_requests || stages[i] < 0) {
      coe_set_error("download_requests: request or stage out of range");
      return COE_CUDA_ERR_CONFIG;
    }
  if (!rt->y) {
    coe_set_error("download_requests: runtime created without device_io (no Y buffer)");
    return COE_CUDA_ERR_CONFIG;
  }
  // final rows live in Y[request] (stages: the caller's view of the chain; kept for the ABI)
  if (!ok(cudaStreamSynchronize(rt->out_stream), "download sync")) return fail_cuda();  // e2e staging use
  const size_t rb = (size_t)rt->row_elems * 2;
  for (int32_t i0 = 0; i0 < n; i0 += rt->out_slots) {  // staging holds out_slots rows at a time
    const int32_t k = std::min(rt->out_slots, n - i0);
    if (!ok(cudaStreamSynchronize(rt->compute), "download sync")) return fail_cuda();  // h_last / staging reuse
    for (int32_t i = 0; i < k; ++i) rt->h_last[i] = requests[i0 + i] << 1;
    if (!ok(cudaMemcpyAsync(rt->d_last, rt->h_last, 4 * (size_t)k, cudaMemcpyHostToDevice, rt->compute), "rows H2D"))
      return fail_cuda();
    gather_rows<<<k, 256, 0, rt->compute>>>(rt->y, rt->y, rt->d_last, rt->row_elems, rt->outbuf);
    if (!ok(cudaGetLastError(), "gather rows") ||
        !ok(cudaMemcpyAsync(static_cast<char *>(host) + (size_t)i0 * rb, rt->outbuf, (size_t)k * rb,
                            cudaMemcpyDeviceToHost, rt->compute),
            "rows D2H") ||
        !ok(cudaStreamSynchronize(rt->compute), "rows sync"))
      return fail_cuda();
  }
  return COE_CUDA_OK;
}

int coe_runtime_synchronize(coe_runtime *rt) {
  bool good = ok(cudaStreamSynchronize(rt->copy), "sync copy") && ok(cudaStreamSynchronize(rt->hop), "sync hop") &&
              ok(cudaStreamSynchronize(rt->out_stream), "sync out") && ok(cudaStreamSynchronize(rt->copy_in), "sync in");
  for (int k = coe_runtime::NCLS - 1; k >= 0; --k) good = ok(cudaStreamSynchronize(rt->cls_stream[k]), "sync") && good;
  return good ? COE_CUDA_OK : fail_cuda();
}

int coe_runtime_join(coe_runtime *rt) {
  if (rt->have_out && !ok(cudaStreamWaitEvent(rt->compute, rt->out_drained, 0), "join downloads")) return fail_cuda();
  return COE_CUDA_OK;
}

int coe_runtime_check(coe_runtime *rt, int32_t *runs, int32_t *violations) {
  int32_t flags[2];
  if (!ok(cudaMemcpy(flags, rt->d_flags, 8, cudaMemcpyDeviceToHost), "flags D2H")) return fail_cuda();
  *runs = flags[0];
  *violations = flags[1];
  return COE_CUDA_OK;
}

int coe_runtime_members(coe_runtime *rt, int32_t *member_req, int32_t *member_stage, int32_t *batch_off) {
  const StepBuffers &s = rt->sets[rt->last_set];
  bool good = ok(cudaMemcpy(member_req, s.mreq, 4 * rt->last_adm, cudaMemcpyDeviceToHost), "members D2H") &&
              ok(cudaMemcpy(member_stage, s.mstage, 4 * rt->last_adm, cudaMemcpyDeviceToHost), "members D2H") &&
              ok(cudaMemcpy(batch_off, s.boff, 4 * rt->last_batches, cudaMemcpyDeviceToHost), "boff D2H");
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
  std::vector<std::pair<float, float>> k3;  // K3 launches only (up, down), W2 waits excluded
  wv.emplace_back(0.f, out->group_ms);
  for (int i = 0; i < rt->last_waves; ++i) {
    float s = elapsed(rt->t_step_start, rt->t_wave_start[i]), e = elapsed(rt->t_step_start, rt->t_wave_end[i]);
    float ue = elapsed(rt->t_step_start, rt->t_up_end[i]), ds = elapsed(rt->t_step_start, rt->t_down_start[i]);
    wv.emplace_back(s, e);
    k3.emplace_back(s, ue);
    k3.emplace_back(ds, e);
    out->mlp_ms += e - s;
    out->k3_flops += rt->last_wave_flops[i];
  }
  out->copy_busy_ms = union_len(cp);
  out->compute_busy_ms = union_len(wv);
  out->overlap_ms = intersect_len(cp, wv);
  out->k3_busy_ms = union_len(k3);
  out->k3_launches = 2 * rt->last_waves;
  return COE_CUDA_OK;
}

int coe_runtime_set_knobs(coe_runtime *rt, int64_t wave_rows_cap, int64_t urgent_rows_cap, int32_t reserve_sms) {
  rt->cfg.wave_rows_cap = wave_rows_cap;
  rt->cfg.urgent_rows_cap = urgent_rows_cap;
  if (reserve_sms >= 0) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int reserve = reserve_sms > 0 ? std::min<int>(reserve_sms, sms / 2) : 0;
    rt->cfg.reserve_sms = reserve;
    rt->m_ctas = sms - reserve;
    rt->r_ctas = reserve > 0 ? reserve : sms;
    rt->rel_launch_ctas = release_grid(rt->r_ctas, sms);
  }
  return COE_CUDA_OK;
}

int coe_runtime_attach_local_experts(coe_runtime *rt, coe_runtime *const *peers, int32_t world) {
  if (world < 1 || !peers) {
    coe_set_error("attach_local_experts: bad peer list");
    return COE_CUDA_ERR_CONFIG;
  }
  rt->local_peers.assign(peers, peers + world);
  return COE_CUDA_OK;
}

int coe_runtime_ipc_export_experts(coe_runtime *rt, void *handles, int32_t *count) {
  auto *h = static_cast<cudaIpcMemHandle_t *>(handles);
  const int n = rt->pooled ? 1 : rt->S;
  for (int k = 0; k < n; ++k)
    if (!ok(cudaIpcGetMemHandle(&h[k], rt->pooled ? rt->pool : rt->slabs[k]), "ipc export experts")) return fail_cuda();
  *count = n;
  return COE_CUDA_OK;
}

int coe_runtime_ipc_open_experts(coe_runtime *rt, int32_t rank, const void *handles, int32_t count) {
  const auto *h = static_cast<const cudaIpcMemHandle_t *>(handles);
  if (rank < 0 || count < 1) {
    coe_set_error("ipc_open_experts: bad rank / count");
    return COE_CUDA_ERR_CONFIG;
  }
  if ((int)rt->peer_exp_base.size() <= rank) rt->peer_exp_base.resize(rank + 1);
  rt->peer_exp_base[rank].clear();
  for (int k = 0; k < count; ++k) {
    void *p = nullptr;
    if (!ok(cudaIpcOpenMemHandle(&p, h[k], cudaIpcMemLazyEnablePeerAccess), "ipc open experts")) return fail_cuda();
    rt->ipc_opened.push_back(p);
    rt->peer_exp_base[rank].push_back(static_cast<char *>(p));
  }
  return COE_CUDA_OK;
}

int coe_runtime_residency_codes(coe_runtime *rt, int64_t *codes) {
  if (rt->step_count == 0) {
    for (int32_t e = 0; e < rt->cfg.num_experts; ++e) codes[e] = -1;
    return COE_CUDA_OK;
  }
  const auto &snap = rt->res_snap[(rt->step_count - 1) & 1];
  for (int32_t e = 0; e < rt->cfg.num_experts; ++e) {
    codes[e] = -1;
    if (e >= (int32_t)snap.size() || !snap[e]) continue;
    const int k = rt->pooled ? 0 : rt->expert_shape[e];
    const char *base = rt->pooled ? rt->pool : rt->slabs[k];
    codes[e] = ((int64_t)k << 40) | (int64_t)(snap[e] - base);
  }
  return COE_CUDA_OK;
}

int coe_runtime_set_peer_residency(coe_runtime *rt, int32_t rank, const int64_t *codes) {
  if (rank < 0 || rank >= (int32_t)rt->peer_exp_base.size() || rt->peer_exp_base[rank].empty()) {
    coe_set_error("set_peer_residency: the peer's experts are not mapped (coe_runtime_ipc_open_experts)");
    return COE_CUDA_ERR_CONFIG;
  }
  if ((int)rt->ipc_snap.size() <= rank) rt->ipc_snap.resize(rank + 1);
  auto &snap = rt->ipc_snap[rank];
  snap.assign(rt->cfg.num_experts, nullptr);
  for (int32_t e = 0; e < rt->cfg.num_experts; ++e) {
    if (codes[e] < 0) continue;
    const int64_t k = codes[e] >> 40, off = codes[e] & ((1ll << 40) - 1);
    if (k < (int64_t)rt->peer_exp_base[rank].size()) snap[e] = rt->peer_exp_base[rank][k] + off;
  }
  return COE_CUDA_OK;
}

int coe_runtime_attach_comm(coe_runtime *rt, coe_comm *comm) {
  rt->comm = comm;
  return COE_CUDA_OK;
}

int coe_runtime_peer_buffers(coe_runtime *rt, coe_peer_buffers *out) {
  out->p0 = rt->act;  // fused hops store into a peer's landing rows of A
  out->p1 = rt->act;
  out->flags = rt->d_hflags;
  return COE_CUDA_OK;
}

int coe_runtime_ipc_export(coe_runtime *rt, void *handles) {
  auto *h = static_cast<cudaIpcMemHandle_t *>(handles);
  bool good = ok(cudaIpcGetMemHandle(&h[0], rt->act), "ipc export A") &&
              ok(cudaIpcGetMemHandle(&h[2], rt->d_hflags), "ipc export flags");
  if (good) h[1] = h[0];  // slot kept for the ABI (one activation buffer)
  return good ? COE_CUDA_OK : fail_cuda();
}

int coe_runtime_ipc_open(coe_runtime *rt, const void *handles, coe_peer_buffers *out) {
  const auto *h = static_cast<const cudaIpcMemHandle_t *>(handles);
  void *p[3] = {nullptr, nullptr, nullptr};
  for (int i : {0, 2}) {
    if (!ok(cudaIpcOpenMemHandle(&p[i], h[i], cudaIpcMemLazyEnablePeerAccess), "ipc open")) return fail_cuda();
    rt->ipc_opened.push_back(p[i]);
  }
  out->p0 = p[0];
  out->p1 = p[0];
  out->flags = p[2];
  return COE_CUDA_OK;
}

int coe_runtime_attach_peers(coe_runtime *rt, int32_t rank, int32_t world, const coe_peer_buffers *peers,
                             coe_local_hub *hub) {
  if (world < 1 || world > COE_MAX_PEERS || rank < 0 || rank >= world) {
    coe_set_error("attach_peers: world must be 1..COE_MAX_PEERS and rank inside it");
    return COE_CUDA_ERR_CONFIG;
  }
  if (!hub && !stream_memops()) {
    coe_set_error("attach_peers: cuStreamWaitValue32 / cuStreamWriteValue32 unavailable");
    return COE_CUDA_ERR_CUDA;
  }
  rt->peers.assign(peers, peers + world);
  rt->peer_hub = hub;
  rt->peer_rank = rank;
  rt->peer_world = world;
  return COE_CUDA_OK;
}

int coe_runtime_bench_mlp(coe_runtime *rt, int32_t groups, int32_t requests_per_group, int32_t iters,
                          float *up_ms, float *down_ms) {
  const auto &c = rt->cfg;
  if (rt->pooled) {
    coe_set_error("bench_mlp: experts are placed on demand in pooled mode");
    return COE_CUDA_ERR_CONFIG;
  }
  const int64_t rows = (int64_t)requests_per_group * c.T;
  const int32_t nreq = groups * requests_per_group;
  if (groups < 1 || requests_per_group < 1 || nreq > c.max_requests || rows * groups > c.max_wave_rows ||
      groups > coe_mlp_max_groups()) {
    coe_set_error("bench_mlp: wave does not fit the runtime's buffers");
    return COE_CUDA_ERR_CONFIG;
  }
  std::vector<coe_mlp_group> gu(groups), gd(groups);
  std::vector<int32_t> boff(groups), mreq(nreq), mst(nreq, 0);
  int tu = 0, td = 0;
  for (int32_t g = 0; g < groups; ++g) {
    const int32_t mt = (int32_t)((rows + BM - 1) / BM);
    gu[g] = coe_mlp_group{(int32_t)rows, g % std::max(1, rt->slot_count[0]), g, (int32_t)(g * rows), tu, {0, 0, 0}};
    gd[g] = gu[g];
    gd[g].tile_start = td;
    tu += mt * (rt->sh[0] / BN);
    td += mt * (rt->sd[0] / BN);
    boff[g] = g * requests_per_group;
  }
  // routed rows: inputs from X (or A without device_io), outputs into Y (or A), one block per request
  const int32_t a_rows = rt->landing_slots + rt->ring_slots;
  for (int32_t r = 0; r < nreq; ++r) {
    mreq[r] = rt->x ? ((r << 1) | 1) : ((r % a_rows) << 1);
    mst[r] = rt->y ? ((r << 4) | coe::OUT_Y) : (((r % a_rows) << 4) | coe::OUT_RING);
  }
  coe_mlp_group *d_g = nullptr;
  int32_t *d_i = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr, e2 = nullptr;
  bool good = dmalloc(&d_g, 2 * sizeof(coe_mlp_group) * groups, "bench alloc") &&
              dmalloc(&d_i, 4 * (size_t)(groups + 2 * nreq), "bench alloc") &&
              ok(cudaMemcpy(d_g, gu.data(), sizeof(coe_mlp_group) * groups, cudaMemcpyHostToDevice), "bench H2D") &&
              ok(cudaMemcpy(d_g + groups, gd.data(), sizeof(coe_mlp_group) * groups, cudaMemcpyHostToDevice), "H2D") &&
              ok(cudaMemcpy(d_i, boff.data(), 4 * groups, cudaMemcpyHostToDevice), "H2D") &&
              ok(cudaMemcpy(d_i + groups, mreq.data(), 4 * (size_t)nreq, cudaMemcpyHostToDevice), "H2D") &&
              ok(cudaMemcpy(d_i + groups + nreq, mst.data(), 4 * (size_t)nreq, cudaMemcpyHostToDevice), "H2D") &&
              ok(cudaEventCreate(&e0), "event") && ok(cudaEventCreate(&e1), "event") && ok(cudaEventCreate(&e2), "event");
  cudaStream_t cs = rt->compute;
  float tot_up = 0.f, tot_down = 0.f;
  for (int it = -2; good && it < iters; ++it) {  // two untimed warm-up launches
    good = ok(cudaEventRecord(e0, cs), "record") &&
           coe_grouped_mlp_routed(rt->mlps[0][0], d_g, d_g + groups, groups, tu, td, d_i, d_i + groups,
                                  d_i + groups + nreq, 1, 0, cs) == COE_CUDA_OK &&
           ok(cudaEventRecord(e1, cs), "record") &&
           coe_grouped_mlp_routed(rt->mlps[0][0], d_g, d_g + groups, groups, tu, td, d_i, d_i + groups,
                                  d_i + groups + nreq, 2, 0, cs) == COE_CUDA_OK &&
           ok(cudaEventRecord(e2, cs), "record") && ok(cudaEventSynchronize(e2), "sync");
    if (good && it >= 0) {
      tot_up += elapsed(e0, e1);
      tot_down += elapsed(e1, e2);
    }
  }
  if (d_g) cudaFree(d_g);
  if (d_i) cudaFree(d_i);
  for (cudaEvent_t e : {e0, e1, e2})
    if (e) cudaEventDestroy(e);
  if (!good) return COE_CUDA_ERR_CUDA;
  *up_ms = tot_up / iters;
  *down_ms = tot_down / iters;
  return COE_CUDA_OK;
}

int coe_runtime_intervals(coe_runtime *rt, float *copy_iv, float *wave_iv, int32_t *wave_info) {
  if (!rt->cfg.profile) {
    coe_set_error("runtime created without profile events");
    return COE_CUDA_ERR_CONFIG;
  }
  for (int i = 0; i < rt->last_copies; ++i) {
    copy_iv[2 * i] = elapsed(rt->t_step_start, rt->t_copy_start[i]);
    copy_iv[2 * i + 1] = elapsed(rt->t_step_start, rt->t_copy_end[i]);
  }
  for (int i = 0; i < rt->last_waves; ++i) {
    wave_iv[2 * i] = elapsed(rt->t_step_start, rt->t_wave_start[i]);
    wave_iv[2 * i + 1] = elapsed(rt->t_step_start, rt->t_wave_end[i]);
    wave_info[3 * i] = rt->last_wave_cls[i];
    wave_info[3 * i + 1] = rt->last_wave_rows[i];
    wave_info[3 * i + 2] = rt->last_wave_groups[i];
  }
  return COE_CUDA_OK;
}

int coe_runtime_wave_shapes(coe_runtime *rt, int32_t *shape_index) {
  for (int i = 0; i < rt->last_waves; ++i) shape_index[i] = rt->last_wave_shape[i];
  return COE_CUDA_OK;
}

int coe_runtime_wave_phases(coe_runtime *rt, float *phase_iv, double *wave_flops) {
  if (!rt->cfg.profile) {
    coe_set_error("runtime created without profile events");
    return COE_CUDA_ERR_CONFIG;
  }
  for (int i = 0; i < rt->last_waves; ++i) {
    phase_iv[4 * i] = elapsed(rt->t_step_start, rt->t_wave_start[i]);
    phase_iv[4 * i + 1] = elapsed(rt->t_step_start, rt->t_up_end[i]);
    phase_iv[4 * i + 2] = elapsed(rt->t_step_start, rt->t_down_start[i]);
    phase_iv[4 * i + 3] = elapsed(rt->t_step_start, rt->t_wave_end[i]);
    wave_flops[i] = rt->last_wave_flops[i];
  }
  return COE_CUDA_OK;
}

int coe_runtime_io_intervals(coe_runtime *rt, float *iv, int32_t *n_in, int32_t *n_out) {
  if (!rt->cfg.profile) {
    coe_set_error("runtime created without profile events");
    return COE_CUDA_ERR_CONFIG;
  }
  *n_in = *n_out = 0;
  for (uint8_t k : rt->io_kind) (k ? *n_out : *n_in) += 1;
  if (iv) {  // input pairs first, then output pairs
    int32_t wi = 0, wo = 2 * *n_in;
    for (size_t p = 0; p < rt->io_kind.size(); ++p) {
      int32_t &w = rt->io_kind[p] ? wo : wi;
      iv[w++] = elapsed(rt->t_step_start, rt->t_io[2 * p]);
      iv[w++] = elapsed(rt->t_step_start, rt->t_io[2 * p + 1]);
    }
  }
  return COE_CUDA_OK;
}

int32_t coe_runtime_output_order(coe_runtime *rt, int32_t *requests, int32_t capacity) {
  const int32_t n = (int32_t)rt->out_order.size();
  if (requests)
    for (int32_t i = 0; i < n && i < capacity; ++i) requests[i] = rt->out_order[i];
  return n;
}

int coe_runtime_counts(coe_runtime *rt, int32_t *copies, int32_t *waves) {
  *copies = rt->last_copies;
  *waves = rt->last_waves;
  return COE_CUDA_OK;
}

}  // extern "C"

// ---------------------------------------------------------------------------------------
// coe_runtime_step: phase A walks the op log in order (slots, copies, data dependencies);
// phase B list-schedules the physical actions on estimated clocks (copy engine, main
// stream, release stream) so that no stream blocks behind work whose inputs are not ready
// while the copy engine -- the bottleneck of budgeted configs -- is kept busy; phase C
// issues the chosen order.  Every dependency is an explicit event on an earlier-issued
// action, so estimates only affect speed, never correctness.

namespace {

struct BatchInfo {
  int32_t op_index;   // index into the op log
  int32_t expert, slot, count, cls;
  int32_t tma_slot;   // weight-map slot index: slot within its shape's slab, or (pooled) first unit
  int32_t copy;       // copy that wrote this batch's slot this step (-1: resident since step start)
  bool release;       // last reader of a slot a later LOAD overwrites
  int64_t rows;
  std::vector<int32_t> producers;  // batches of this executor producing this batch's inputs
  std::vector<int32_t> recvs;      // my_hops slots consumed
  std::vector<int32_t> sends;      // my_hops slots produced
  int64_t max_recv = -1, min_send = INT64_MAX;
  int32_t wave = -1;
  double done = 0.0;               // estimated completion
  std::vector<int32_t> inputs;     // e2e: stage-0 requests whose inputs this batch uploads
  std::vector<int32_t> finals;     // e2e: requests whose final output this batch produces
  int32_t input_event = -1;        // e2e: the input chunk this batch needs last (its event)
};

struct CopyInfo {
  int32_t expert, slot;
  bool restore;
  std::vector<int32_t> readers;    // batches reading the slot's previous content this step
  bool first_write;                // slot not written earlier this step
  std::vector<int32_t> deps;       // slots whose readers must finish first (pooled: the units' last users)
  int32_t unit0 = -1;              // pooled: first unit of the expert's new place
  bool w1_over_w2 = false;         // pooled: its W1 lands on units an earlier expert used for W2
  const char *peer_src = nullptr;  // (f3) copy from this peer executor's HBM instead of the host store
  coe_runtime *peer_rt = nullptr;  // in-process peer (else another process: peer_exec's IPC mapping)
  int32_t peer_exec = -1;
  int32_t peer_par = 0;            // parity of the peer's snapshot / ready event
  double up_end = 0.0, end = 0.0;  // estimated
  bool issued = false;
  int64_t op_pos = 0;              // op-log position of the LOAD (restores: of the first batch)
};

}  // namespace

extern "C" int coe_runtime_plan_rows(const coe_step_input *in, int32_t max_requests, int e2e, int nccl,
                                     int32_t *ring_slots, int32_t *landing_slots) {
  const coe_op *ops = static_cast<const coe_op *>(in->ops);
  const coe_admission *adm = static_cast<const coe_admission *>(in->admissions);
  const int32_t x = in->executor;
  std::unordered_map<int64_t, int32_t> adm_index;
  std::vector<int32_t> final_stage(max_requests, -1);
  int64_t n_adm = 0;
  for (int64_t i = 0; i < in->num_admissions; ++i) {
    const coe_admission &a = adm[i];
    if (a.request < 0 || a.request >= max_requests || a.stage < 0 || a.stage >= coe::ROW_STAGES) {
      coe_set_error("plan_rows: request beyond max_requests or chain longer than 8 stages");
      return COE_CUDA_ERR_CONFIG;
    }
    final_stage[a.request] = std::max(final_stage[a.request], a.stage);
    if (a.executor == x) adm_index[(int64_t)a.request * coe::ROW_STAGES + a.stage] = (int32_t)n_adm++;
  }
  std::vector<int64_t> batch_ops;
  for (int64_t i = 0; i < in->num_ops; ++i)
    if (ops[i].executor == x && ops[i].kind == COE_OP_BATCH) batch_ops.push_back(i);
  const std::vector<coe::Hop> all_hops = coe::hop_schedule(adm, in->num_admissions, max_requests);
  std::vector<int32_t> my_hops;
  for (size_t i = 0; i < all_hops.size(); ++i)
    if (all_hops[i].src == x || all_hops[i].dst == x) my_hops.push_back((int32_t)i);
  coe::RowPlan rows;
  std::string err;
  if (!coe::plan_rows(ops, in->op_args, batch_ops, adm_index, all_hops, my_hops, final_stage, x, e2e != 0, e2e != 0,
                      nccl == 0, 0, -1, {}, max_requests, n_adm, rows, err)) {
    coe_set_error(err);
    return COE_CUDA_ERR_CONFIG;
  }
  *ring_slots = rows.peak_ring;
  *landing_slots = rows.landing;
  return COE_CUDA_OK;
}

extern "C" int coe_runtime_step(coe_runtime *rt, const coe_step_input *in, coe_step_stats *stats) {
  const auto &c = rt->cfg;
  const coe_op *ops = static_cast<const coe_op *>(in->ops);
  const coe_admission *adm = static_cast<const coe_admission *>(in->admissions);
  const int32_t x = in->executor;
  constexpr int NCLS = coe_runtime::NCLS;
  coe_step_stats st{};

  // ---- admissions of this executor (admission order) ----
  std::vector<int32_t> a_rank, a_req, a_stage;
  std::unordered_map<int64_t, int32_t> adm_index;  // (request, stage) -> admission of this executor
  int32_t max_rank = 0;
  for (int64_t i = 0; i < in->num_admissions; ++i) {
    if (adm[i].executor != x) continue;
    if (adm[i].stage < 0 || adm[i].stage >= coe::ROW_STAGES) {
      coe_set_error("chains longer than 8 stages are not supported");
      return COE_CUDA_ERR_CONFIG;
    }
    adm_index[(int64_t)adm[i].request * coe::ROW_STAGES + adm[i].stage] = (int32_t)a_rank.size();
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

  // ---- my ops and the release lookahead ----
  std::vector<int64_t> my_ops;
  for (int64_t i = 0; i < in->num_ops; ++i)
    if (ops[i].executor == x) my_ops.push_back(i);
  std::vector<uint8_t> releases(my_ops.size(), 0);
  {
    std::vector<uint8_t> next_is_evict(c.num_experts, 0);
    for (int64_t k = (int64_t)my_ops.size() - 1; k >= 0; --k) {
      const coe_op &op = ops[my_ops[k]];
      if (op.kind == COE_OP_LOAD) {
        for (int32_t j = 0; j < op.count; ++j) next_is_evict[in->op_args[op.offset + j]] = 1;
        next_is_evict[op.expert] = 0;
      } else {
        releases[k] = next_is_evict[op.expert];
        next_is_evict[op.expert] = 0;
      }
    }
  }

  // ---- hops touching this executor (global admission order, hops.h) ----
  const std::vector<coe::Hop> all_hops = coe::hop_schedule(adm, in->num_admissions, c.max_requests);
  std::vector<int32_t> my_hops;
  std::unordered_map<int64_t, int32_t> hop_in, hop_out;
  auto hkey = [](int32_t r, int32_t s) { return ((int64_t)r << 8) | s; };
  for (size_t i = 0; i < all_hops.size(); ++i) {
    const coe::Hop &h = all_hops[i];
    if (h.src != x && h.dst != x) continue;
    if (h.dst == x) hop_in[hkey(h.request, h.stage + 1)] = (int32_t)my_hops.size();
    if (h.src == x) hop_out[hkey(h.request, h.stage)] = (int32_t)my_hops.size();
    my_hops.push_back((int32_t)i);
  }
  const bool peer_mode = rt->peer_world > 0;
  if (!my_hops.empty() && !rt->comm && !peer_mode) {
    coe_set_error("plan moves activations between executors: attach a communicator (coe_runtime_attach_comm) "
                  "or peer buffers (coe_runtime_attach_peers)");
    return COE_CUDA_ERR_CONFIG;
  }
  if (peer_mode && x != rt->peer_rank) {
    coe_set_error("peer hops: step executor differs from the rank the runtime was attached as");
    return COE_CUDA_ERR_CONFIG;
  }
  std::vector<int32_t> hop_batch(my_hops.size(), -1);  // producing batch of each send

  // ---- phase A: slots, copies, batches in op order ----
  std::vector<uint8_t> plan_res(c.num_experts, 0), pending_restore(c.num_experts, 0);
  const int32_t NS = rt->total_slots;
  std::vector<int32_t> slot_copy(NS, -1);
  std::vector<std::vector<int32_t>> slot_readers(NS);
  std::vector<uint8_t> slot_written(NS, 0);
  for (int32_t i = 0; i < in->num_initial; ++i) plan_res[in->initial[i]] = 1;
  // pooled: per unit, the readers (batches, this step) of the residency that freed it
  std::vector<std::shared_ptr<const std::vector<int32_t>>> unit_rd;
  if (rt->pooled) unit_rd.assign((size_t)rt->pool_units, nullptr);
  auto pool_free = [&](int32_t q) {  // the expert in slot q left: its units return to the pool
    auto snap = std::make_shared<const std::vector<int32_t>>(slot_readers[q]);
    const int32_t u0 = rt->slot_unit[q], n = rt->slot_units[q];
    for (int32_t u = u0; u < u0 + n; ++u) unit_rd[u] = snap;
    auto it = rt->free_runs.emplace(u0, n).first;  // coalesce with the neighbours
    if (it != rt->free_runs.begin()) {
      auto prev = std::prev(it);
      if (prev->first + prev->second == it->first) {
        prev->second += it->second;
        rt->free_runs.erase(it);
        it = prev;
      }
    }
    auto next = std::next(it);
    if (next != rt->free_runs.end() && it->first + it->second == next->first) {
      it->second += next->second;
      rt->free_runs.erase(next);
    }
    rt->slot_units[q] = 0;
  };
  // experts this executor's op log touches (loads or batches) in this step
  std::vector<uint8_t> touched(c.num_experts, 0);
  for (int64_t i = 0; i < in->num_ops; ++i)
    if (ops[i].executor == x && ops[i].expert >= 0 && ops[i].expert < c.num_experts) touched[ops[i].expert] = 1;
  // (f3) experts other executors copy from this one this step: kept (initial placement, never
  // evicted here) and materialised at step start, so that this step's end snapshot has them
  std::vector<uint8_t> exported(c.num_experts, 0);
  bool any_export = false;
  if (in->initial_offsets && x < in->num_executors && (!rt->local_peers.empty() || !rt->peer_exp_base.empty())) {
    std::vector<uint8_t> mine(c.num_experts, 0);
    for (int32_t i = in->initial_offsets[x]; i < in->initial_offsets[x + 1]; ++i) mine[in->initial_all[i]] = 1;
    for (int64_t i = 0; i < in->num_ops; ++i)
      if (ops[i].executor == x && ops[i].kind == COE_OP_LOAD)
        for (int32_t v = 0; v < ops[i].count; ++v) mine[in->op_args[ops[i].offset + v]] = 0;
    for (int64_t i = 0; i < in->num_ops; ++i) {
      const coe_op &o = ops[i];
      if (o.executor != x && o.kind == COE_OP_LOAD && o.tier == COE_TIER_PEER && o.seq == x && mine[o.expert]) {
        exported[o.expert] = touched[o.expert] = 1;
        any_export = true;
      }
    }
  }
  // slots outside the initial placement are free again, and so are residents this step never
  // uses: what is physically resident is then always part of the planner's pool at that
  // moment, restricted to the experts this step touches (the runtime's slot sizing)
  for (int32_t s = 0; s < NS; ++s) {
    int32_t e = rt->slot_expert[s];
    if (e >= 0 && (!plan_res[e] || !touched[e])) {
      rt->expert_slot[e] = -1;
      rt->slot_expert[s] = -1;
      if (rt->pooled) pool_free(s);
    }
  }
  for (int32_t i = 0; i < in->num_initial; ++i)
    if (rt->expert_slot[in->initial[i]] < 0) pending_restore[in->initial[i]] = 1;

  std::vector<CopyInfo> copies;
  std::vector<BatchInfo> batches;
  std::vector<int32_t> req_last(c.max_requests, -1);  // latest batch of each request on this executor
  const bool e2e_in = in->host_inputs != nullptr, e2e_out = in->host_outputs != nullptr;
  if ((!e2e_in && !rt->x) || (!e2e_out && !rt->y)) {
    coe_set_error("device-resident inputs / outputs need a runtime created with device_io");
    return COE_CUDA_ERR_CONFIG;
  }
  std::vector<int32_t> final_stage(c.max_requests, -1);
  for (int64_t i = 0; i < in->num_admissions; ++i)
    if (adm[i].request >= 0 && adm[i].request < c.max_requests)
      final_stage[adm[i].request] = std::max(final_stage[adm[i].request], adm[i].stage);
  auto issue_copy = [&](int32_t e, bool restore, int64_t op_pos) -> bool {
    // an initially resident expert outside the host store (never loaded, never evicted by the
    // plan) is materialised on the device the first time it is used instead of restored
    if (rt->store_off[e] < 0 && !restore) {
      coe_set_error("swap-in of an expert that is not in the host store");
      return false;
    }
    const int k = rt->expert_shape[e];
    int32_t best = -1;  // free slot of the expert's shape whose readers were issued earliest
    if (rt->pooled) {
      best = rt->expert_vslot[e];  // the expert's own bookkeeping slot
    } else {
      for (int32_t s = rt->slot_base[k]; s < rt->slot_base[k] + rt->slot_count[k]; ++s) {
        if (rt->slot_expert[s] >= 0) continue;
        auto age = [&](int32_t q) { return slot_readers[q].empty() ? -1 : slot_readers[q].back(); };
        if (best < 0 || age(s) < age(best)) best = s;
      }
    }
    if (best < 0 || rt->slot_expert[best] >= 0) {
      coe_set_error("no free HBM expert slot (planner residency exceeds the slot count)");
      return false;
    }
    CopyInfo ci{e, best, restore, slot_readers[best], !slot_written[best]};
    ci.deps.push_back(best);
    if (rt->pooled) {  // best-fit run of free units; wait for the readers of whatever used them last
      const int32_t n = (int32_t)((rt->sbytes[k] + rt->unit - 1) / rt->unit);
      // best fit; large experts (>= 256 MB) take the top of their run and small ones the
      // bottom, so the two size classes drift to opposite ends instead of interleaving
      // (a simulation of C5's plans at 1-1000 us arrival gaps: no load ever fails with three
      // largest experts of slack, tools/pool_sim.py)
      const bool big = rt->sbytes[k] >= (256ll << 20);
      auto pick = rt->free_runs.end();
      for (auto it = rt->free_runs.begin(); it != rt->free_runs.end(); ++it)
        if (it->second >= n && (pick == rt->free_runs.end() || it->second < pick->second ||
                                (big && it->second == pick->second)))
          pick = it;
      if (pick == rt->free_runs.end()) {
        coe_set_error("pooled expert memory: no free run for a load (byte budget exceeded or fragmented)");
        return false;
      }
      const int32_t start = pick->first, len = pick->second;
      const int32_t u0 = big ? start + len - n : start;
      rt->free_runs.erase(pick);
      if (u0 > start) rt->free_runs.emplace(start, u0 - start);
      if (u0 + n < start + len) rt->free_runs.emplace(u0 + n, start + len - u0 - n);
      const std::vector<int32_t> *last_rd = nullptr;
      // the W1 half lands on units that held an earlier expert's W2 (any byte of it) -> it
      // must wait for their down passes; a unit holding any W2 byte counts as W2
      const int64_t half = rt->sbytes[k] / 2;
      const int32_t w1_units = (int32_t)((half + rt->unit - 1) / rt->unit);  // units with W1 bytes
      for (int32_t u = u0; u < u0 + w1_units; ++u) ci.w1_over_w2 |= rt->unit_w2[u] != 0;
      for (int32_t u = u0; u < u0 + n; ++u) {
        rt->unit_w2[u] = (int64_t)(u - u0 + 1) * rt->unit > half;
        const int32_t owner = rt->unit_owner[u];
        if (owner >= 0 && std::find(ci.deps.begin(), ci.deps.end(), owner) == ci.deps.end()) ci.deps.push_back(owner);
        if (unit_rd[u] && unit_rd[u].get() != last_rd) {
          last_rd = unit_rd[u].get();
          for (int32_t r : *unit_rd[u])
            if (std::find(ci.readers.begin(), ci.readers.end(), r) == ci.readers.end()) ci.readers.push_back(r);
        }
        unit_rd[u] = nullptr;
        rt->unit_owner[u] = best;
      }
      rt->slot_unit[best] = u0;
      rt->slot_units[best] = n;
      ci.unit0 = u0;
    }
    ci.op_pos = op_pos;
    copies.push_back(ci);
    slot_readers[best].clear();
    slot_written[best] = 1;
    rt->slot_expert[best] = e;
    rt->expert_slot[e] = best;
    slot_copy[best] = (int32_t)copies.size() - 1;
    (restore ? st.restores : st.loads) += 1;
    if (rt->store_off[e] >= 0) (restore ? st.restore_bytes : st.load_bytes) += rt->sbytes[k];  // else: generated
    return true;
  };
  // (f3) physical source of a peer-tier LOAD: executor j's bytes, when they were resident on j
  // at the end of the previous step, e is in j's initial placement (so j's step start keeps
  // it) and no LOAD of j in this plan evicts it -- j never rewrites them during this step
  std::vector<std::vector<uint8_t>> peer_keep(std::max<size_t>(rt->local_peers.size(), rt->ipc_snap.size()));
  auto keep_of = [&](int32_t j) -> std::vector<uint8_t> & {
    if ((int32_t)peer_keep.size() <= j) peer_keep.resize(j + 1);
    if (peer_keep[j].empty()) {
      peer_keep[j].assign(c.num_experts, 0);
      for (int32_t i = in->initial_offsets[j]; i < in->initial_offsets[j + 1]; ++i) peer_keep[j][in->initial_all[i]] = 1;
      for (int64_t i = 0; i < in->num_ops; ++i)
        if (ops[i].executor == j && ops[i].kind == COE_OP_LOAD)
          for (int32_t v = 0; v < ops[i].count; ++v) peer_keep[j][in->op_args[ops[i].offset + v]] = 0;
    }
    return peer_keep[j];
  };
  auto peer_source = [&](int32_t j, int32_t e) -> const char * {
    if (j < 0 || j == x || rt->step_count == 0 || !in->initial_offsets || j >= in->num_executors) return nullptr;
    const std::vector<const char *> *snap = nullptr;
    if (j < (int32_t)rt->local_peers.size() && rt->local_peers[j])  // in-process peer
      snap = &rt->local_peers[j]->res_snap[(rt->step_count - 1) & 1];
    else if (j < (int32_t)rt->ipc_snap.size())  // another process: its residency, exchanged after the last step
      snap = &rt->ipc_snap[j];
    if (!snap || e >= (int32_t)snap->size() || !(*snap)[e]) return nullptr;
    return keep_of(j)[e] ? (*snap)[e] : nullptr;
  };
  if (any_export)
    for (int32_t e = 0; e < c.num_experts; ++e)
      if (exported[e] && rt->expert_slot[e] < 0 && pending_restore[e]) {
        pending_restore[e] = 0;
        if (!issue_copy(e, true, my_ops.empty() ? 0 : my_ops[0])) return COE_CUDA_ERR_CHECK;
      }
  for (size_t k = 0; k < my_ops.size(); ++k) {
    const coe_op &op = ops[my_ops[k]];
    if (op.kind == COE_OP_LOAD) {
      for (int32_t j = 0; j < op.count; ++j) {
        int32_t v = in->op_args[op.offset + j];
        plan_res[v] = 0;
        pending_restore[v] = 0;
        int32_t s = rt->expert_slot[v];
        if (s >= 0) {
          rt->expert_slot[v] = -1;
          rt->slot_expert[s] = -1;
          if (rt->pooled) pool_free(s);
        }
      }
      plan_res[op.expert] = 1;
      if (rt->expert_slot[op.expert] >= 0) {  // never reuse bytes: every planned load moves them
        int32_t s = rt->expert_slot[op.expert];
        rt->slot_expert[s] = -1;
        rt->expert_slot[op.expert] = -1;
        if (rt->pooled) pool_free(s);
      }
      if (!issue_copy(op.expert, false, my_ops[k])) return COE_CUDA_ERR_CHECK;
      if (op.tier == COE_TIER_PEER) {
        st.peer_tier_loads += 1;
        if (const char *src = peer_source(op.seq, op.expert)) {
          CopyInfo &ci = copies.back();
          ci.peer_src = src;
          ci.peer_rt = op.seq < (int32_t)rt->local_peers.size() ? rt->local_peers[op.seq] : nullptr;
          ci.peer_exec = op.seq;
          ci.peer_par = (int32_t)((rt->step_count - 1) & 1);
        }
      }
      continue;
    }
    const int32_t e = op.expert;
    if (rt->expert_slot[e] < 0) {
      if (!pending_restore[e]) {
        coe_set_error("batch on an expert that is neither resident nor loaded");
        return COE_CUDA_ERR_CHECK;
      }
      pending_restore[e] = 0;
      if (!issue_copy(e, true, my_ops[k])) return COE_CUDA_ERR_CHECK;
    }
    BatchInfo b;
    b.op_index = (int32_t)my_ops[k];
    b.expert = e;
    b.slot = rt->expert_slot[e];
    b.tma_slot = rt->pooled ? rt->slot_unit[b.slot] : b.slot - rt->slot_base[rt->slot_shape[b.slot]];
    b.count = op.count;
    b.rows = (int64_t)op.count * c.T;
    b.copy = slot_copy[b.slot];
    b.release = releases[k] != 0;
    b.cls = b.release ? 1 : 0;
    if (b.rows > c.max_wave_rows) {
      coe_set_error("a single batch exceeds the H scratch rows");
      return COE_CUDA_ERR_CONFIG;
    }
    const int32_t bi = (int32_t)batches.size();
    for (int32_t j = 0; j < op.count; ++j) {
      const int32_t r = in->op_args[op.offset + 2 * j], s = in->op_args[op.offset + 2 * j + 1];
      if (req_last[r] >= 0 && std::find(b.producers.begin(), b.producers.end(), req_last[r]) == b.producers.end())
        b.producers.push_back(req_last[r]);
      auto hi = hop_in.find(hkey(r, s));
      if (hi != hop_in.end()) {
        b.recvs.push_back(hi->second);
        b.max_recv = std::max<int64_t>(b.max_recv, all_hops[my_hops[hi->second]].index);
      }
      auto ho = hop_out.find(hkey(r, s));
      if (ho != hop_out.end()) {
        b.sends.push_back(ho->second);
        b.min_send = std::min<int64_t>(b.min_send, all_hops[my_hops[ho->second]].index);
        hop_batch[ho->second] = bi;
      }
      req_last[r] = bi;
      if (e2e_in && s == 0) b.inputs.push_back(r);
      if (e2e_out && s == final_stage[r]) b.finals.push_back(r);
    }
    slot_readers[b.slot].push_back(bi);
    batches.push_back(std::move(b));
  }
  // (f3, between processes) do other executors copy experts out of this one's HBM this step?
  // Then next step's copies into this HBM must wait for their end (see phase C)
  bool read_by_peers = false;
  if (peer_mode && !rt->peer_hub && in->initial_offsets && rt->step_count > 0 && x < in->num_executors) {
    const auto &mine = rt->res_snap[(rt->step_count - 1) & 1];
    for (int64_t i = 0; i < in->num_ops && !read_by_peers; ++i) {
      const coe_op &o = ops[i];
      if (o.executor != x && o.kind == COE_OP_LOAD && o.tier == COE_TIER_PEER && o.seq == x &&
          o.expert < (int32_t)mine.size() && mine[o.expert] && keep_of(x)[o.expert])
        read_by_peers = true;
    }
  }
  const int64_t n_batches = (int64_t)batches.size();
  if (n_batches > c.max_batches) {
    coe_set_error("more batches than the runtime was sized for");
    return COE_CUDA_ERR_CONFIG;
  }
  // ---- activation rows: ring slots / landing rows per member, slot-reuse order ----
  coe::RowPlan rows;
  {
    std::vector<int64_t> batch_ops;
    for (const BatchInfo &b : batches) batch_ops.push_back(b.op_index);
    std::string err;
    if (!coe::plan_rows(ops, in->op_args, batch_ops, adm_index, all_hops, my_hops, final_stage, x, e2e_in, e2e_out,
                        peer_mode, rt->landing_slots, rt->ring_slots, rt->ring_order, c.max_requests, n_adm, rows,
                        err)) {
      coe_set_error(err);
      return COE_CUDA_ERR_CONFIG;
    }
    for (size_t b = 0; b < batches.size(); ++b)  // write-after-read on a reused slot
      for (int32_t p : rows.preds[b])
        if (std::find(batches[b].producers.begin(), batches[b].producers.end(), p) == batches[b].producers.end())
          batches[b].producers.push_back(p);
  }
  // sends ordered by global index: a batch needing recv h may only be issued once every
  // send of this executor with a smaller index has its producer issued
  std::vector<int32_t> send_slots;
  for (size_t i = 0; i < my_hops.size(); ++i)
    if (all_hops[my_hops[i]].src == x) send_slots.push_back((int32_t)i);

  // ---- phase B: list schedule ----
  auto copy_half_s = [&](int32_t e) { return (double)rt->sbytes[rt->expert_shape[e]] / 2 / 55.0e9; };
  const double f_main = 1.2e15 * (double)rt->m_ctas / 148.0, f_rel = 1.2e15 * (double)rt->r_ctas / 148.0;
  const double launch_s = 12e-6;
  std::vector<uint8_t> issued(n_batches, 0);
  std::vector<int32_t> main_pending, rel_order;
  for (int32_t i = 0; i < (int32_t)n_batches; ++i) (batches[i].cls ? rel_order : main_pending).push_back(i);
  size_t next_rel = 0, next_copy = 0, send_ptr = 0;
  double t_copy = 0.0, t_stream[NCLS] = {0.0, 0.0, 0.0};
  // two main streams measured faster than one (r1: C1 -5 %, C3 -3 %, C2 even)
  const int main_streams = getenv("COE_MAIN_STREAMS") ? atoi(getenv("COE_MAIN_STREAMS")) : 2;
  int main_flip = 0;
  std::vector<WaveAct> waves;
  std::vector<Action> actions;
  std::vector<coe_mlp_group> g_up, g_down;
  std::vector<int32_t> batch_of_group;  // group position -> batch (K2 batch index = op-order batch)
  std::vector<int32_t> slot_last_wave(NS * NCLS, -1);
  std::vector<int32_t> copy_action(copies.size(), -1);

  auto sends_ready_before = [&](int64_t hop_index) {
    while (send_ptr < send_slots.size() && hop_batch[send_slots[send_ptr]] >= 0 &&
           issued[hop_batch[send_slots[send_ptr]]])
      ++send_ptr;
    return send_ptr >= send_slots.size() || all_hops[my_hops[send_slots[send_ptr]]].index > hop_index;
  };
  // e2e: stage-0 inputs move in chunks of >= 32 MB (full-rate DMA) in the order batches need
  // them, each request straight into its ring slot; batch b needs chunks 0..b.input_event.  A
  // chunk waits for the batches that freed its slots (their up passes read the old rows), so a
  // chunk never holds a request whose slot predecessor shares the chunk.  chunk_end < 0: not
  // issued yet.
  std::vector<int32_t> in_reqs, in_batch(e2e_in ? c.max_requests : 0, -1);
  for (size_t bi = 0; bi < batches.size(); ++bi)
    for (int32_t r : batches[bi].inputs) {
      in_reqs.push_back(r);
      in_batch[r] = (int32_t)bi;
    }
  std::vector<int32_t> host_row;  // host_inputs row of a request: rank among this executor's stage-0 requests
  if (e2e_in) {
    host_row.assign(c.max_requests, -1);
    std::vector<int32_t> sorted(in_reqs);
    std::sort(sorted.begin(), sorted.end());
    for (size_t i = 0; i < sorted.size(); ++i) host_row[sorted[i]] = (int32_t)i;
  }
  const int64_t in_chunk = std::max<int64_t>(1, (32ll << 20) / std::max<int64_t>(1, rt->row_elems * 2));
  std::vector<int32_t> chunk_start;  // first in_reqs index of each chunk
  {
    int32_t first_b = -1;
    for (size_t i = 0; i < in_reqs.size(); ++i) {
      const int32_t r = in_reqs[i], p = rows.in_pred[r];
      if (chunk_start.empty() || (int64_t)i - chunk_start.back() >= in_chunk || (p >= 0 && p >= first_b)) {
        chunk_start.push_back((int32_t)i);
        first_b = in_batch[r];
      }
    }
  }
  const int32_t n_chunks = (int32_t)chunk_start.size();
  chunk_start.push_back((int32_t)in_reqs.size());
  std::vector<double> chunk_end(n_chunks, -1.0);
  std::vector<int64_t> chunk_pos(n_chunks, INT64_MAX);  // op position of the first batch needing it
  std::vector<std::vector<int32_t>> chunk_preds(n_chunks);
  {
    std::unordered_map<int32_t, int32_t> chunk_of;
    for (int32_t k = 0; k < n_chunks; ++k)
      for (int32_t i = chunk_start[k]; i < chunk_start[k + 1]; ++i) {
        const int32_t r = in_reqs[i], p = rows.in_pred[r];
        chunk_of[r] = k;
        if (p >= 0 && std::find(chunk_preds[k].begin(), chunk_preds[k].end(), p) == chunk_preds[k].end())
          chunk_preds[k].push_back(p);
      }
    for (BatchInfo &b : batches) {
      b.input_event = -1;
      for (int32_t r : b.inputs) {
        const int32_t k = chunk_of[r];
        b.input_event = std::max(b.input_event, k);
        chunk_pos[k] = std::min<int64_t>(chunk_pos[k], b.op_index);
      }
    }
    for (int32_t k = n_chunks - 2; k >= 0; --k) chunk_pos[k] = std::min(chunk_pos[k], chunk_pos[k + 1]);
  }
  auto chunk_ready = [&](int32_t k) {
    for (int32_t p : chunk_preds[k])
      if (!issued[p]) return false;
    return true;
  };
  auto issuable = [&](const BatchInfo &b) {
    if (b.input_event >= 0 && chunk_end[b.input_event] < 0) return false;  // inputs not uploaded yet
    for (int32_t p : b.producers)
      if (!issued[p]) return false;
    if (b.copy >= 0 && !copies[b.copy].issued) return false;
    if (b.max_recv >= 0 && !sends_ready_before(b.max_recv)) return false;
    return true;
  };
  auto ready_time = [&](const BatchInfo &b) {
    double t = b.input_event >= 0 ? chunk_end[b.input_event] : 0.0;
    for (int32_t p : b.producers) t = std::max(t, batches[p].done);
    if (b.copy >= 0) t = std::max(t, copies[b.copy].up_end);
    return t;
  };
  auto copy_ready = [&](const CopyInfo &ci) {
    for (int32_t r : ci.readers)
      if (!issued[r]) return false;
    return true;
  };
  auto wave_time = [&](int64_t rows, int cls, int shape) {
    const double padded = (double)((rows + BM - 1) / BM * BM);
    return padded * 4.0 * rt->sd[shape] * rt->sh[shape] / (cls ? f_rel : f_main) + 2 * launch_s;
  };
  auto emit_wave = [&](const std::vector<int32_t> &members, int cls, double start) {
    WaveAct w{};
    w.cls = cls;
    w.shape = rt->slot_shape[batches[members[0]].slot];
    w.first_group = (int32_t)g_up.size();
    const int32_t id = (int32_t)waves.size();
    for (int32_t bi : members) {
      BatchInfo &b = batches[bi];
      const int32_t m_tiles = (int32_t)((b.rows + BM - 1) / BM);
      coe_mlp_group gu{};
      gu.rows = (int32_t)b.rows;
      gu.slot = b.tma_slot;
      gu.batch = bi;
      gu.h_row = (int32_t)w.rows;
      gu.tile_start = w.tiles_up;
      coe_mlp_group gd = gu;
      gd.tile_start = w.tiles_down;
      g_up.push_back(gu);
      g_down.push_back(gd);
      w.num_groups += 1;
      w.rows += b.rows;
      w.tiles_up += m_tiles * (rt->sh[w.shape] / BN);
      w.tiles_down += m_tiles * (rt->sd[w.shape] / BN);
      if (b.copy >= 0 && std::find(w.wait_copies.begin(), w.wait_copies.end(), b.copy) == w.wait_copies.end())
        w.wait_copies.push_back(b.copy);
      for (int32_t p : b.producers) {
        const int32_t pw = batches[p].wave;
        if (waves[pw].cls != cls && std::find(w.wait_waves.begin(), w.wait_waves.end(), pw) == w.wait_waves.end())
          w.wait_waves.push_back(pw);
      }
      for (int32_t h : b.recvs) w.wait_recvs.push_back(h);
      b.wave = id;
      issued[bi] = 1;
      slot_last_wave[b.slot * NCLS + cls] = id;
    }
    const double end = start + wave_time(w.rows, cls, w.shape);
    for (int32_t bi : members) batches[bi].done = end;
    t_stream[cls == 2 ? 0 : cls] = end;  // streams 0 and 2 share the main clock
    st.max_wave_groups = std::max(st.max_wave_groups, w.num_groups);
    st.max_wave_rows = std::max(st.max_wave_rows, w.rows);
    waves.push_back(std::move(w));
    actions.push_back(Action{false, id});
  };

  const size_t kWindow = 256;
  const double kSlack = 50e-6;
  const int max_groups = coe_mlp_max_groups();
  // urgency: a main batch that reads a slot an upcoming swap-in overwrites goes first, and
  // a wave carrying urgent work is capped so that swap-in waits for little else
  std::vector<int32_t> needed_by_copy(n_batches, -1);
  for (int32_t ci = 0; ci < (int32_t)copies.size(); ++ci)
    for (int32_t r : copies[ci].readers) needed_by_copy[r] = ci;
  const int64_t wave_rows_cap = c.wave_rows_cap > 0 ? std::min<int64_t>(c.wave_rows_cap, c.max_wave_rows)
                                                    : c.max_wave_rows;
  const int64_t urgent_rows_cap = c.urgent_rows_cap > 0 ? c.urgent_rows_cap : wave_rows_cap;
  const int urgent_horizon = getenv("COE_URGENT_HORIZON") ? atoi(getenv("COE_URGENT_HORIZON")) : 2;
  // Swap-ins may leave op order within a small window: a copy whose victim slot is still
  // being read (e.g. the expert the previous copy brought in, evicted right after its
  // batches) must not idle the copy engine while a later copy's slot is already free.  The
  // planner's decisions are unaffected -- only the physical order of slot writes changes;
  // two copies into the same slot keep their order.
  const size_t kCopyWindow = getenv("COE_COPY_WINDOW") ? (size_t)atoi(getenv("COE_COPY_WINDOW")) : 8;
  size_t copy_pick = 0;
  // e2e: the stage-0 input uploads ride the same copy engine (one H2D queue): in op order with
  // the swap-ins, and ahead of a swap-in whose victim slot is still being read -- the PCIe
  // link, which both share, never idles while either has work
  int32_t next_in = 0;
  const double row_bytes = (double)rt->row_elems * 2;
  while (next_copy < copies.size() || next_in < n_chunks || next_rel < rel_order.size() ||
         !main_pending.empty()) {
    const double INF = 1e30;
    while (next_copy < copies.size() && copies[next_copy].issued) ++next_copy;
    // candidate: the earliest-startable swap-in in the window
    double c_start = INF;
    for (size_t k = next_copy, seen = 0; k < copies.size() && seen < kCopyWindow; ++k) {
      if (copies[k].issued) continue;
      ++seen;
      bool waw = false;
      for (size_t m = next_copy; m < k && !waw; ++m) waw = !copies[m].issued && copies[m].slot == copies[k].slot;
      if (waw || !copy_ready(copies[k])) continue;
      double t = t_copy;
      for (int32_t r : copies[k].readers) t = std::max(t, batches[r].done);
      if (t < c_start) {
        c_start = t;
        copy_pick = k;
      }
    }
    // candidate: the next input upload (always startable; op order against the swap-in)
    bool take_input = false;
    if (next_in < n_chunks && chunk_ready(next_in)) {
      double t_in = t_copy;
      for (int32_t p : chunk_preds[next_in]) t_in = std::max(t_in, batches[p].done);
      take_input = c_start == INF || t_in < c_start || chunk_pos[next_in] < copies[copy_pick].op_pos;
      if (take_input) c_start = t_in;
    }
    // candidate: next release wave (singleton, in order)
    double r_start = INF;
    if (next_rel < rel_order.size() && issuable(batches[rel_order[next_rel]]))
      r_start = std::max(t_stream[1], ready_time(batches[rel_order[next_rel]]));
    // candidate: a main wave -- earliest estimated-ready issuable batch in the window
    double m_start = INF;
    const size_t win = std::min(kWindow, main_pending.size());
    for (size_t i = 0; i < win; ++i) {
      const BatchInfo &b = batches[main_pending[i]];
      if (issuable(b)) m_start = std::min(m_start, std::max(t_stream[0], ready_time(b)));
    }
    if (c_start == INF && r_start == INF && m_start == INF) {
      coe_set_error("internal: runtime list scheduler found no issuable action");
      return COE_CUDA_ERR_CHECK;
    }
    if (take_input && c_start <= r_start && c_start <= m_start) {
      const int64_t nreq_k = chunk_start[next_in + 1] - chunk_start[next_in];
      chunk_end[next_in] = c_start + (double)nreq_k * row_bytes / 55.0e9;
      t_copy = chunk_end[next_in];
      actions.push_back(Action{false, next_in, true});
      ++next_in;
    } else if (c_start <= r_start && c_start <= m_start) {
      CopyInfo &ci = copies[copy_pick];
      ci.issued = true;
      ci.up_end = c_start + copy_half_s(ci.expert);
      ci.end = c_start + 2 * copy_half_s(ci.expert);
      t_copy = ci.end;
      copy_action[copy_pick] = (int32_t)actions.size();
      actions.push_back(Action{true, (int32_t)copy_pick});
    } else if (r_start <= m_start) {
      emit_wave({rel_order[next_rel]}, 1, r_start);
      ++next_rel;
    } else {
      // greedy wave at m_start: ready (by estimate) issuable batches in op order
      std::vector<int32_t> members;
      std::unordered_set<int32_t> reqs;
      int64_t rows = 0, wave_max_recv = -1, wave_min_send = INT64_MAX, wave_finals = 0;
      std::vector<size_t> taken;
      // candidate order: urgent (slot needed by one of the next swap-ins) first, then op order
      std::vector<size_t> order;
      bool urgent_present = false;
      for (size_t i = 0; i < win; ++i) {
        const int32_t nb = needed_by_copy[main_pending[i]];
        if (nb >= 0 && nb <= (int32_t)next_copy + urgent_horizon) {
          order.push_back(i);
          urgent_present = true;
        }
      }
      for (size_t i = 0; i < win; ++i) {
        const int32_t nb = needed_by_copy[main_pending[i]];
        if (!(nb >= 0 && nb <= (int32_t)next_copy + urgent_horizon)) order.push_back(i);
      }
      // urgent batches (readers of slots the next swap-ins overwrite) fill a wave up to the
      // full cap -- one big wave lets the swap-in's W1 half wait for a single up pass instead
      // of an up/down chain; unrelated work only rides along up to urgent_rows_cap
      for (size_t oi = 0; oi < order.size() && (int)members.size() < max_groups; ++oi) {
        const size_t i = order[oi];
        const int32_t bi = main_pending[i];
        const BatchInfo &b = batches[bi];
        if (!issuable(b) || ready_time(b) > m_start + kSlack) continue;
        if (!members.empty() && rt->slot_shape[b.slot] != rt->slot_shape[batches[members[0]].slot]) continue;
        const int32_t nb = needed_by_copy[bi];
        const bool urgent = nb >= 0 && nb <= (int32_t)next_copy + urgent_horizon;
        const int64_t cap = (urgent || !urgent_present) ? wave_rows_cap : urgent_rows_cap;
        if (!members.empty() && rows + b.rows > cap) {
          if (urgent) continue;  // a smaller urgent batch may still fit
          break;
        }
        bool clash = false;
        for (int32_t j = 0; j < b.count && !clash; ++j)
          clash = reqs.count(in->op_args[ops[b.op_index].offset + 2 * j]) > 0;
        if (clash) continue;
        const int64_t mr = std::max(wave_max_recv, b.max_recv), ms = std::min(wave_min_send, b.min_send);
        if (mr >= 0 && ms < mr) continue;  // a wave may not wait on a hop its own sends precede
        // e2e: a wave's final rows must fit the output staging ring at once
        if (!members.empty() && wave_finals + (int64_t)b.finals.size() > rt->out_slots) continue;
        members.push_back(bi);
        taken.push_back(i);
        rows += b.rows;
        wave_finals += (int64_t)b.finals.size();
        wave_max_recv = mr;
        wave_min_send = ms;
        for (int32_t j = 0; j < b.count; ++j) reqs.insert(in->op_args[ops[b.op_index].offset + 2 * j]);
      }
      if (members.empty()) {
        coe_set_error("internal: empty main wave");
        return COE_CUDA_ERR_CHECK;
      }
      // main waves alternate between two streams (0, 2) when enabled: the next wave's up
      // pass fills the SMs the previous wave's down pass leaves idle in its tail
      emit_wave(members, (main_streams == 2 && (main_flip ^= 1) == 0) ? 2 : 0, m_start);
      std::sort(taken.begin(), taken.end());
      for (size_t t = taken.size(); t-- > 0;) main_pending.erase(main_pending.begin() + (std::ptrdiff_t)taken[t]);
    }
  }
  // copy waits: the last issued reader wave of the slot's previous content, per stream
  std::vector<CopyAct> copy_acts(copies.size());
  {
    std::vector<int32_t> last_reader_wave(NS * NCLS, -1);
    std::vector<uint8_t> written(NS, 0);
    for (const Action &a : actions) {
      if (a.is_input) continue;
      if (a.is_copy) {
        const CopyInfo &ci = copies[a.index];
        CopyAct &ca = copy_acts[a.index];
        ca.expert = ci.expert;
        ca.slot = ci.slot;
        ca.restore = ci.restore;
        ca.unit0 = ci.unit0;
        ca.peer_src = ci.peer_src;
        ca.peer_rt = ci.peer_rt;
        ca.peer_exec = ci.peer_exec;
        ca.peer_par = ci.peer_par;
        ca.w1_waits_down = ci.w1_over_w2;
        for (int32_t q : ci.deps)  // the slot itself, and (VMM) the last users of its pages
          for (int k = 0; k < NCLS; ++k) {
            const int32_t wv = last_reader_wave[q * NCLS + k];
            if (wv >= 0) {
              if (std::find(ca.wait_waves.begin(), ca.wait_waves.end(), wv) == ca.wait_waves.end())
                ca.wait_waves.push_back(wv);
            } else if (!written[q] && rt->slot_free_valid[(size_t)q * NCLS + k]) {
              ca.wait_prev.push_back(q * NCLS + k);
            }
          }
        for (int k = 0; k < NCLS; ++k) last_reader_wave[ci.slot * NCLS + k] = -1;
        written[ci.slot] = 1;
      } else {
        const WaveAct &w = waves[a.index];
        for (int32_t gi = w.first_group; gi < w.first_group + w.num_groups; ++gi)  // global slot index
          last_reader_wave[batches[g_up[gi].batch].slot * NCLS + w.cls] = a.index;
      }
    }
    for (int32_t s = 0; s < NS; ++s)
      for (int k = 0; k < NCLS; ++k)
        if (last_reader_wave[s * NCLS + k] >= 0) waves[last_reader_wave[s * NCLS + k]].frees_slots.push_back(s * NCLS + k);
  }
  st.admissions = n_adm;
  st.batches = n_batches;
  st.waves = (int64_t)waves.size();
  if (const char *dump = getenv("COE_SCHED_DUMP")) {  // debug: the issue order and its dependencies
    if (FILE *f = fopen(dump, "w")) {
      fprintf(f, "{\"actions\": [");
      for (size_t i = 0; i < actions.size(); ++i)
        fprintf(f, "%s[%d, %d]", i ? ", " : "", actions[i].is_copy ? 1 : (actions[i].is_input ? 2 : 0),
                actions[i].index);
      fprintf(f, "], \"copies\": [");
      for (size_t i = 0; i < copy_acts.size(); ++i) {
        fprintf(f, "%s{\"expert\": %d, \"slot\": %d, \"est_start\": %.6f, \"wait_waves\": [", i ? ", " : "",
                copy_acts[i].expert, copy_acts[i].slot, copies[i].end - 2 * copy_half_s(copies[i].expert));
        for (size_t j = 0; j < copy_acts[i].wait_waves.size(); ++j)
          fprintf(f, "%s%d", j ? ", " : "", copy_acts[i].wait_waves[j]);
        fprintf(f, "]}");
      }
      fprintf(f, "], \"waves\": [");
      for (size_t i = 0; i < waves.size(); ++i) {
        const WaveAct &w = waves[i];
        fprintf(f, "%s{\"cls\": %d, \"rows\": %lld, \"est_end\": %.6f, \"wait_copies\": [", i ? ", " : "", w.cls,
                (long long)w.rows, batches[g_up[w.first_group].batch].done);
        for (size_t j = 0; j < w.wait_copies.size(); ++j) fprintf(f, "%s%d", j ? ", " : "", w.wait_copies[j]);
        fprintf(f, "], \"wait_waves\": [");
        for (size_t j = 0; j < w.wait_waves.size(); ++j) fprintf(f, "%s%d", j ? ", " : "", w.wait_waves[j]);
        fprintf(f, "], \"batches\": [");
        for (int32_t gi = w.first_group; gi < w.first_group + w.num_groups; ++gi)
          fprintf(f, "%s%d", gi > w.first_group ? ", " : "", g_up[gi].batch);
        fprintf(f, "]}");
      }
      fprintf(f, "]}\n");
      fclose(f);
    }
  }

  // ---- phase C: issue ----
  const size_t nw = waves.size(), nc = copies.size();
  const int par = rt->step_parity;  // this step's wave events; par ^ 1 holds the previous step's
  std::vector<cudaEvent_t> &wave_up_ev = rt->wave_up_evs[par], &wave_down_ev = rt->wave_down_evs[par];
  if (!rt->ensure_events(wave_up_ev, nw, false) || !rt->ensure_events(wave_down_ev, nw, false) ||
      !rt->ensure_events(rt->copy_up_ev, nc, false) || !rt->ensure_events(rt->copy_down_ev, nc, false) ||
      !rt->ensure_events(rt->recv_ev, my_hops.size(), false))
    return fail_cuda();
  if (c.profile && (!rt->ensure_events(rt->t_wave_start, nw, true) || !rt->ensure_events(rt->t_wave_end, nw, true) ||
                    !rt->ensure_events(rt->t_up_end, nw, true) || !rt->ensure_events(rt->t_down_start, nw, true) ||
                    !rt->ensure_events(rt->t_copy_start, nc, true) || !rt->ensure_events(rt->t_copy_end, nc, true)))
    return fail_cuda();

  const int set_idx = rt->cur_set;
  rt->cur_set ^= 1;
  StepBuffers &sb = rt->sets[set_idx];
  if (!ok(cudaEventSynchronize(rt->staging_done[set_idx]), "staging reuse")) return fail_cuda();
  char *stg = rt->staging[set_idx];
  uint32_t seq = 0;
  if (peer_mode) {  // fused hops: K3's down pass stores hopping rows into the peers' landing rows
    seq = ++rt->step_seq;
    std::vector<void *> pa(2 * rt->peer_world);
    for (int r = 0; r < rt->peer_world; ++r) {
      pa[2 * r] = rt->peers[r].p0;
      pa[2 * r + 1] = rt->peers[r].p0;
    }
    for (auto &per : rt->mlps)
      for (coe_mlp *m : per)
        if (m && coe_mlp_set_hops(m, nullptr, 0, pa.data(), rt->peer_world)) return COE_CUDA_ERR_CONFIG;
  }

  // e2e: final rows leave in completion order -- per wave, its finals by request id, each
  // stored by the down pass straight into the output staging ring at its global position
  std::vector<int32_t> fin_begin(nw, 0), fin_end(nw, 0);  // per wave: slice of the output order
  const int64_t out_base = rt->out_pos;
  if (e2e_out) {
    rt->out_order.clear();
    for (size_t a = 0; a < actions.size(); ++a) {
      if (actions[a].is_copy || actions[a].is_input) continue;
      const WaveAct &w = waves[actions[a].index];
      std::vector<int32_t> fin;
      for (int32_t gi = w.first_group; gi < w.first_group + w.num_groups; ++gi)
        for (int32_t r : batches[g_up[gi].batch].finals) fin.push_back(r);
      std::sort(fin.begin(), fin.end());
      if ((int64_t)fin.size() > rt->out_slots) {
        coe_set_error("output staging ring smaller than one wave's final rows");
        return COE_CUDA_ERR_CONFIG;
      }
      fin_begin[actions[a].index] = (int32_t)rt->out_order.size();
      for (int32_t r : fin) {
        const int64_t pos = out_base + (int64_t)rt->out_order.size();
        const int32_t ai = adm_index[(int64_t)r * coe::ROW_STAGES + final_stage[r]];
        rows.out_code[ai] = (int32_t)((pos % rt->out_slots) << 4) | coe::OUT_STAGE;
        rt->out_order.push_back(r);
      }
      fin_end[actions[a].index] = (int32_t)rt->out_order.size();
    }
    rt->out_pos += (int64_t)rt->out_order.size();
    if (!rt->ensure_events(rt->out_ev, nw, false)) return fail_cuda();
  }
  int32_t *s_adm = reinterpret_cast<int32_t *>(stg);
  for (int64_t i = 0; i < n_adm; ++i) {
    s_adm[i] = 0;
    s_adm[n_adm + i] = a_rank[i];
    s_adm[2 * n_adm + i] = a_req[i];
    s_adm[3 * n_adm + i] = a_stage[i];
    s_adm[4 * n_adm + i] = rows.in_code[i];
    s_adm[5 * n_adm + i] = rows.out_code[i];
  }
  int32_t *s_batch = s_adm + 6 * n_adm;
  for (int64_t b = 0; b < n_batches; ++b) {
    s_batch[b] = 0;
    s_batch[n_batches + b] = batches[b].count;
  }
  coe_mlp_group *s_groups = reinterpret_cast<coe_mlp_group *>(
      (reinterpret_cast<uintptr_t>(s_batch + 2 * n_batches) + 31) & ~uintptr_t(31));
  if (n_batches) {
    std::memcpy(s_groups, g_up.data(), sizeof(coe_mlp_group) * n_batches);
    std::memcpy(s_groups + n_batches, g_down.data(), sizeof(coe_mlp_group) * n_batches);
  }
  // e2e inputs: read by gather_inputs straight from the pinned host rows; the device needs,
  // per request in need order, its host row and A row (COE_INPUT_DMA: one DMA per row run)
  const uint4 *host_in_dev = nullptr;
  if (e2e_in && !getenv("COE_INPUT_DMA")) {
    void *dp = nullptr;
    if (cudaHostGetDevicePointer(&dp, const_cast<void *>(in->host_inputs), 0) == cudaSuccess)
      host_in_dev = static_cast<const uint4 *>(dp);
    else
      cudaGetLastError();  // not page-locked: one DMA per row run instead
  }
  int64_t *s_in = reinterpret_cast<int64_t *>(
      (reinterpret_cast<uintptr_t>(s_groups + 2 * n_batches) + 15) & ~uintptr_t(15));
  if (host_in_dev)
    for (size_t i = 0; i < in_reqs.size(); ++i) {
      s_in[2 * i] = host_row[in_reqs[i]];
      s_in[2 * i + 1] = rows.in_slot[in_reqs[i]];
    }

  cudaStream_t cs = rt->compute, ks = rt->copy;
  if (c.profile && !ok(cudaEventRecord(rt->t_step_start, cs), "record")) return fail_cuda();
  if (sb.used && !ok(cudaStreamWaitEvent(ks, sb.free_ev, 0), "set reuse")) return fail_cuda();
  if (n_adm && !ok(cudaMemcpyAsync(sb.adm, s_adm, 24 * (size_t)n_adm, cudaMemcpyHostToDevice, ks), "adm H2D"))
    return fail_cuda();
  if (n_batches &&
      (!ok(cudaMemcpyAsync(sb.batch, s_batch, 8 * (size_t)n_batches, cudaMemcpyHostToDevice, ks), "batch H2D") ||
       !ok(cudaMemcpyAsync(sb.groups, s_groups, 2 * sizeof(coe_mlp_group) * (size_t)n_batches,
                           cudaMemcpyHostToDevice, ks),
           "group H2D")))
    return fail_cuda();
  if (host_in_dev && !in_reqs.empty() &&
      !ok(cudaMemcpyAsync(sb.in_map, s_in, 16 * in_reqs.size(), cudaMemcpyHostToDevice, ks), "input map H2D"))
    return fail_cuda();
  // step fence: every peer has finished the previous step (its landing rows are free).
  // Same-process peers (hub) are stepped and synchronised together (runtime.step_executors).
  if (peer_mode && !rt->peer_hub)
    for (int r = 0; r < rt->peer_world; ++r)
      if (r != x && !wait_flag(cs, rt->d_hflags + rt->hflag_step_base + r, seq - 1)) return COE_CUDA_ERR_CUDA;
  if (!ok(cudaEventRecord(rt->staging_done[set_idx], ks), "record") || !ok(cudaEventRecord(rt->staged, ks), "record") ||
      !ok(cudaStreamWaitEvent(cs, rt->staged, 0), "compute waits upload") ||
      // the input gathers read this step's input map (uploaded above on the copy stream)
      (e2e_in && !ok(cudaStreamWaitEvent(rt->copy_in, rt->staged, 0), "inputs wait upload")))
    return fail_cuda();
  int32_t *d_exec = sb.adm, *d_rank = sb.adm + n_adm, *d_req = sb.adm + 2 * n_adm, *d_stage = sb.adm + 3 * n_adm;
  int idx_bits = 1;
  while ((1ll << idx_bits) < n_adm) ++idx_bits;
  // one-block K1+K2 only for small steps: at C3's 13,642 admissions the single block takes
  // ~100 us (ncu, profiles/r2r_k12_ncu_summary.json) against ~39 us for the multi-block
  // kernels (profiles/r1m_k12_ncu_summary.json), so launch count is not worth it there
  static const int64_t fused_max = getenv("COE_FUSED_MAX") ? atoll(getenv("COE_FUSED_MAX")) : 4096;
  const bool fused = n_adm >= 1 && n_adm <= std::min<int64_t>(fused_max, COE_FUSED_MAX_ADMISSIONS) &&
                     n_batches <= COE_FUSED_MAX_BATCHES && rank_bits + idx_bits + 1 <= 32 && !getenv("COE_GROUP_MULTI");
  rt->last_group_fused = fused;
  if (fused) {  // serving size: K1 + K2 in one block, one launch
    int rc = coe_group_compact_fused(d_rank, d_req, d_stage, sb.adm + 4 * n_adm, sb.adm + 5 * n_adm, n_adm, rank_bits,
                                     sb.batch + n_batches, (int)n_batches, rt->d_perm, sb.boff, sb.mreq, sb.mstage,
                                     sb.min, sb.mout, rt->d_flags, cs);
    if (rc) return rc;
    st.launches += 1;
  } else {
    st.launches += (n_adm ? 1 + passes : 0) + (n_adm ? 1 : 0) + (n_batches > 4096 ? 2 : 0) + (n_batches ? 1 : 0);
    if (n_adm) {
      int rc = coe_group_sort(d_exec, d_rank, n_adm, rank_bits, passes, rt->d_perm, rt->d_keys, rt->d_sort_scratch,
                              cs);
      if (rc) return rc;
    }
    int rc = coe_run_compact_routes(rt->d_perm, rt->d_keys, d_req, d_stage, sb.adm + 4 * n_adm, sb.adm + 5 * n_adm,
                                    n_adm, rank_bits, sb.batch, sb.batch + n_batches, (int)n_batches, 1, sb.boff,
                                    sb.mreq, sb.mstage, sb.min, sb.mout, rt->d_flags, rt->d_flags + 1,
                                    rt->d_compact_scratch, cs);
    if (rc) return rc;
  }
  if (c.profile && !ok(cudaEventRecord(rt->t_group_end, cs), "record")) return fail_cuda();
  if (!ok(cudaEventRecord(rt->grouped, cs), "record")) return fail_cuda();
  for (int k = 1; k < NCLS; ++k)
    if (!ok(cudaStreamWaitEvent(rt->cls_stream[k], rt->grouped, 0), "class stream waits K2")) return fail_cuda();

  if (!my_hops.empty() && rt->have_step_end && !ok(cudaStreamWaitEvent(rt->hop, rt->step_end, 0), "hop waits step"))
    return fail_cuda();
  if (e2e_in && !rt->ensure_events(rt->in_ev, (size_t)n_chunks, false)) return fail_cuda();
  bool in_prev_waited = false;
  // stage-0 rows of a chunk, pinned host -> their ring slots, coalescing consecutive rows
  int32_t io_n = 0;  // profile events recorded this step
  rt->io_kind.clear();
  auto io_mark = [&](cudaStream_t s_) -> bool {
    if (!c.profile) return true;
    if (!rt->ensure_events(rt->t_io, (size_t)io_n + 1, true)) return false;
    return ok(cudaEventRecord(rt->t_io[io_n++], s_), "record");
  };
  const size_t rb = (size_t)rt->row_elems * 2;
  // COE_INPUT_QUEUE: 1 (default) = input chunks on their own queue, so the gather kernels'
  // PCIe reads and the swap-in DMAs share the link concurrently (C3 e2e 1,493 -> 1,412 ms,
  // tools/timeline.py; the gather alone reaches ~42 GB/s, the DMA fills the rest); 0 = the
  // swap-in copy stream (one H2D queue); 2 = odd chunks on the second queue
  const int input_queue = getenv("COE_INPUT_QUEUE") ? atoi(getenv("COE_INPUT_QUEUE")) : 1;
  auto upload_inputs = [&](int32_t k) -> bool {
    const cudaStream_t ks = (input_queue == 1 || (input_queue == 2 && (k & 1))) ? rt->copy_in : rt->copy;
    if (!in_prev_waited && rt->prev_nccl_hold && rt->have_step_end) {  // slots held for NCCL sends
      in_prev_waited = true;
      if (!ok(cudaStreamWaitEvent(ks, rt->step_end, 0), "inputs wait last step")) return false;
    }
    // write-after-read: the batches that last read these slots (this step, or the previous one)
    std::vector<cudaEvent_t> waits;
    for (int32_t i = chunk_start[k]; i < chunk_start[k + 1]; ++i) {
      const int32_t r = in_reqs[i], p = rows.in_pred[r], q = rows.in_slot[r];
      cudaEvent_t ev = nullptr;
      if (p >= 0) ev = wave_up_ev[batches[p].wave];
      else if (rt->act_prev_wave[q] >= 0) ev = rt->wave_up_evs[par ^ 1][rt->act_prev_wave[q]];
      if (ev && std::find(waits.begin(), waits.end(), ev) == waits.end()) waits.push_back(ev);
    }
    for (cudaEvent_t ev : waits)
      if (!ok(cudaStreamWaitEvent(ks, ev, 0), "inputs wait slot readers")) return false;
    if (c.profile) rt->io_kind.push_back(0);
    if (!io_mark(ks)) return false;
    if (host_in_dev) {  // one gather kernel per chunk (host rows scattered in need order)
      const int32_t n = chunk_start[k + 1] - chunk_start[k];
      const int64_t row_vec = (int64_t)(rb / 16);
      gather_inputs<<<kInputGatherCtas, 256, 0, ks>>>(host_in_dev, sb.in_map, chunk_start[k], n, row_vec,
                                                       (int32_t)((row_vec + 2047) / 2048),
                                                       reinterpret_cast<uint4 *>(rt->act));
      st.launches += 1;
      st.h2d_input_bytes += (int64_t)n * (int64_t)rb;
      return ok(cudaGetLastError(), "gather_inputs") && io_mark(ks) && ok(cudaEventRecord(rt->in_ev[k], ks), "record");
    }
    const char *hin = static_cast<const char *>(in->host_inputs);
    std::vector<void *> dsts, srcs;
    std::vector<size_t> sizes;
    for (int32_t i = chunk_start[k]; i < chunk_start[k + 1];) {
      int32_t j = i + 1;
      while (j < chunk_start[k + 1] && rows.in_slot[in_reqs[j]] == rows.in_slot[in_reqs[j - 1]] + 1 &&
             host_row[in_reqs[j]] == host_row[in_reqs[j - 1]] + 1)
        ++j;
      dsts.push_back(reinterpret_cast<char *>(rt->act) + (size_t)rows.in_slot[in_reqs[i]] * rb);
      srcs.push_back(const_cast<char *>(hin) + (size_t)host_row[in_reqs[i]] * rb);
      sizes.push_back((size_t)(j - i) * rb);
      st.h2d_input_bytes += (int64_t)((j - i) * rb);
      i = j;
    }
    return run_copies(dsts, srcs, sizes, ks, "input H2D") && io_mark(ks) &&
           ok(cudaEventRecord(rt->in_ev[k], ks), "record");
  };
  size_t hop_cursor = 0;
  const size_t row_elems = (size_t)rt->row_elems;
  // NCCL transport: the hops up to `limit` (global order) as ONE NCCL group on the hop stream
  // -- an all-to-all of this wave's sends / receives with exact counts; the producers of its
  // sends were issued earlier (phase B), so the stream first waits for their down passes
  auto issue_hops_until = [&](int64_t limit) -> bool {
    size_t end = hop_cursor;
    while (end < my_hops.size() && all_hops[my_hops[end]].index <= limit) ++end;
    if (end == hop_cursor) return true;
    std::vector<int32_t> waited;
    for (size_t k = hop_cursor; k < end; ++k) {
      if (all_hops[my_hops[k]].src != x) continue;
      const int32_t pb = hop_batch[k];
      if (pb < 0 || !issued[pb] || batches[pb].wave < 0) {
        coe_set_error("internal: hop send issued before its producer wave");
        return false;
      }
      if (std::find(waited.begin(), waited.end(), batches[pb].wave) != waited.end()) continue;
      waited.push_back(batches[pb].wave);
      if (!ok(cudaStreamWaitEvent(rt->hop, wave_down_ev[batches[pb].wave], 0), "send waits producer")) return false;
    }
    if (!coe_comm_group(rt->comm, true)) return false;
    for (size_t k = hop_cursor; k < end; ++k) {
      const coe::Hop &h = all_hops[my_hops[k]];
      __nv_bfloat16 *row = rt->act + (size_t)rows.hop_row[k] * row_elems;
      if (!(h.src == x ? coe_comm_send_bf16(rt->comm, row, row_elems, h.dst, rt->hop)
                       : coe_comm_recv_bf16(rt->comm, row, row_elems, h.src, rt->hop))) {
        coe_comm_group(rt->comm, false);
        return false;
      }
    }
    if (!coe_comm_group(rt->comm, false)) return false;
    for (size_t k = hop_cursor; k < end; ++k)
      if (all_hops[my_hops[k]].dst == x && !ok(cudaEventRecord(rt->recv_ev[k], rt->hop), "record")) return false;
    hop_cursor = end;
    return true;
  };
  // output staging ring: before a wave's down pass stores rows [p0, p1) (global positions), the
  // downloads of the rows' previous occupants [p0 - R, p1 - R) must have finished
  auto out_wait = [&](cudaStream_t ws, int64_t p0, int64_t p1) -> bool {
    const int64_t R = rt->out_slots;
    for (const auto &u : rt->out_hist)
      if (u.end > p0 - R && u.begin < p1 - R && !ok(cudaStreamWaitEvent(ws, u.ev, 0), "staging reuse")) return false;
    while (!rt->out_hist.empty() && rt->out_hist.front().end <= p1 - R) {
      rt->out_ev_pool.push_back(rt->out_hist.front().ev);
      rt->out_hist.pop_front();
    }
    return true;
  };
  // issue() for sends must only see producers already issued in phase C
  std::fill(issued.begin(), issued.end(), 0);
  if (peer_mode && !rt->peer_hub && rt->peer_read_prev)  // peers read our experts last step
    for (int r = 0; r < rt->peer_world; ++r)
      if (r != x && !wait_flag(ks, rt->d_hflags + rt->hflag_step_base + r, seq - 1)) return COE_CUDA_ERR_CUDA;
  rt->peer_read_prev = read_by_peers;

  const coe_mlp_group *dg_up = sb.groups, *dg_down = sb.groups + n_batches;
  for (const Action &a : actions) {
    if (a.is_input) {
      if (!upload_inputs(a.index)) return fail_cuda();
      continue;
    }
    if (a.is_copy) {
      const CopyAct &cp = copy_acts[a.index];
      char *dst = rt->pooled ? rt->pool + (int64_t)cp.unit0 * rt->unit : rt->slot_ptr(cp.slot);
      const bool generate = rt->store_off[cp.expert] < 0;
      const char *src = generate ? nullptr : rt->host_store + rt->store_off[cp.expert];
      const int64_t half_bytes = rt->sbytes[rt->slot_shape[cp.slot]] / 2;
      const int ksh = rt->slot_shape[cp.slot];
      for (int32_t wv : cp.wait_waves)
        if (!ok(cudaStreamWaitEvent(ks, cp.w1_waits_down ? wave_down_ev[wv] : wave_up_ev[wv], 0), "copy waits W1 readers"))
          return fail_cuda();
      for (int32_t sk : cp.wait_prev)
        if (!ok(cudaStreamWaitEvent(ks, cp.w1_waits_down ? rt->slot_free_down[sk] : rt->slot_free_up[sk], 0),
                "copy waits last step"))
          return fail_cuda();
      if (c.profile && !ok(cudaEventRecord(rt->t_copy_start[a.index], ks), "record")) return fail_cuda();
      if (cp.peer_src) {  // (f3) NVLink / same-device copy from the peer executor's HBM
        if (cp.peer_rt) {  // in-process: its ready event of the previous step
          if (!ok(cudaStreamWaitEvent(ks, cp.peer_rt->res_ready[cp.peer_par], 0), "peer copy waits peer") ||
              !ok(cudaMemcpyPeerAsync(dst, rt->device, cp.peer_src, cp.peer_rt->device, half_bytes, ks), "peer W1"))
            return fail_cuda();
        } else {  // another process: its end of the previous step (step fence flag), then a UVA copy
          if (!wait_flag(ks, rt->d_hflags + rt->hflag_step_base + cp.peer_exec, seq - 1) ||
              !ok(cudaMemcpyAsync(dst, cp.peer_src, half_bytes, cudaMemcpyDefault, ks), "peer W1"))
            return fail_cuda();
        }
      } else if (generate) {
        if (coe_fill_uniform_bf16(dst, half_bytes / 2, coe_expert_seed(c.weight_seed, cp.expert, 0),
                                  sqrtf(3.0f / rt->sd[ksh]), ks))
          return COE_CUDA_ERR_CUDA;
      } else if (!ok(cudaMemcpyAsync(dst, src, half_bytes, cudaMemcpyHostToDevice, ks), "swap-in W1")) {
        return fail_cuda();
      }
      if (!ok(cudaEventRecord(rt->copy_up_ev[a.index], ks), "record")) return fail_cuda();
      for (int32_t wv : cp.wait_waves)
        if (!ok(cudaStreamWaitEvent(ks, wave_down_ev[wv], 0), "copy waits W2 readers")) return fail_cuda();
      for (int32_t sk : cp.wait_prev)
        if (!ok(cudaStreamWaitEvent(ks, rt->slot_free_down[sk], 0), "copy waits last step")) return fail_cuda();
      if (cp.peer_src) {
        if (!(cp.peer_rt ? ok(cudaMemcpyPeerAsync(dst + half_bytes, rt->device, cp.peer_src + half_bytes,
                                                   cp.peer_rt->device, half_bytes, ks),
                              "peer W2")
                         : ok(cudaMemcpyAsync(dst + half_bytes, cp.peer_src + half_bytes, half_bytes, cudaMemcpyDefault,
                                              ks),
                              "peer W2")))
          return fail_cuda();
        st.peer_loads += 1;
        st.peer_bytes += 2 * half_bytes;
      } else if (generate) {
        if (coe_fill_uniform_bf16(dst + half_bytes, half_bytes / 2, coe_expert_seed(c.weight_seed, cp.expert, 1),
                                  sqrtf(3.0f / rt->sh[ksh]), ks))
          return COE_CUDA_ERR_CUDA;
      } else if (!ok(cudaMemcpyAsync(dst + half_bytes, src + half_bytes, half_bytes, cudaMemcpyHostToDevice, ks),
                     "swap-in W2")) {
        return fail_cuda();
      }
      if (!ok(cudaEventRecord(rt->copy_down_ev[a.index], ks), "record")) return fail_cuda();
      if (c.profile && !ok(cudaEventRecord(rt->t_copy_end[a.index], ks), "record")) return fail_cuda();
      continue;
    }
    const WaveAct &w = waves[a.index];
    cudaStream_t ws = rt->cls_stream[w.cls];
    coe_mlp *m = rt->mlps[w.shape][w.cls];
    if (peer_mode) {
      for (int32_t hslot : w.wait_recvs) {
        const int64_t hi = all_hops[my_hops[hslot]].index;
        if (rt->peer_hub ? !coe_hub_wait(rt->peer_hub, hi, ws) : !wait_flag(ws, rt->d_hflags + hi, seq))
          return COE_CUDA_ERR_CUDA;
      }
    } else if (!w.wait_recvs.empty()) {
      int64_t limit = -1;
      for (int32_t hslot : w.wait_recvs) limit = std::max<int64_t>(limit, all_hops[my_hops[hslot]].index);
      if (!issue_hops_until(limit)) return COE_CUDA_ERR_CUDA;
      for (int32_t hslot : w.wait_recvs)
        if (!ok(cudaStreamWaitEvent(ws, rt->recv_ev[hslot], 0), "wave waits hop")) return fail_cuda();
    }
    for (int32_t wid : w.wait_waves)
      if (!ok(cudaStreamWaitEvent(ws, wave_down_ev[wid], 0), "wave waits producer")) return fail_cuda();
    for (int32_t cid : w.wait_copies)
      if (!ok(cudaStreamWaitEvent(ws, rt->copy_up_ev[cid], 0), "wave waits W1")) return fail_cuda();
    for (int32_t gi = w.first_group; gi < w.first_group + w.num_groups; ++gi) {
      const int32_t ie = batches[g_up[gi].batch].input_event;
      if (ie >= 0 && !ok(cudaStreamWaitEvent(ws, rt->in_ev[ie], 0), "wave waits inputs")) return fail_cuda();
    }
    if (c.profile && !ok(cudaEventRecord(rt->t_wave_start[a.index], ws), "record")) return fail_cuda();
    // release waves gate the copy engine: they start on the reserved SMs at once
    const int ctas = w.cls == 1 ? rt->rel_launch_ctas : rt->m_ctas;
    int rc = coe_grouped_mlp_routed(m, dg_up + w.first_group, dg_down + w.first_group, w.num_groups, w.tiles_up,
                                    w.tiles_down, sb.boff, sb.min, sb.mout, 1, ctas, ws);
    if (rc) return rc;
    if (!ok(cudaEventRecord(wave_up_ev[a.index], ws), "record")) return fail_cuda();
    if (c.profile && !ok(cudaEventRecord(rt->t_up_end[a.index], ws), "record")) return fail_cuda();
    for (int32_t sk : w.frees_slots)
      if (!ok(cudaEventRecord(rt->slot_free_up[sk], ws), "record")) return fail_cuda();
    for (int32_t cid : w.wait_copies)
      if (!ok(cudaStreamWaitEvent(ws, rt->copy_down_ev[cid], 0), "wave waits W2")) return fail_cuda();
    const int32_t b0 = fin_begin[a.index], b1 = fin_end[a.index];
    if (e2e_out && b1 > b0 && !out_wait(ws, out_base + b0, out_base + b1)) return fail_cuda();
    if (c.profile && !ok(cudaEventRecord(rt->t_down_start[a.index], ws), "record")) return fail_cuda();
    rc = coe_grouped_mlp_routed(m, dg_up + w.first_group, dg_down + w.first_group, w.num_groups, w.tiles_up,
                                w.tiles_down, sb.boff, sb.min, sb.mout, 2, ctas, ws);
    if (rc) return rc;
    st.launches += 2;
    if (!ok(cudaEventRecord(wave_down_ev[a.index], ws), "record")) return fail_cuda();
    if (peer_mode)  // publish the hops this wave's down pass just stored into the peers
      for (int32_t gi = w.first_group; gi < w.first_group + w.num_groups; ++gi)
        for (int32_t hslot : batches[g_up[gi].batch].sends) {
          const coe::Hop &h = all_hops[my_hops[hslot]];
          if (rt->peer_hub ? !coe_hub_publish(rt->peer_hub, h.index, ws)
                           : !write_flag(ws, static_cast<int32_t *>(rt->peers[h.dst].flags) + h.index, seq))
            return COE_CUDA_ERR_CUDA;
        }
    for (int32_t sk : w.frees_slots) {
      if (!ok(cudaEventRecord(rt->slot_free_down[sk], ws), "record")) return fail_cuda();
      rt->slot_free_valid[sk] = 1;
    }
    for (int32_t gi = w.first_group; gi < w.first_group + w.num_groups; ++gi) issued[g_up[gi].batch] = 1;
    if (c.profile && !ok(cudaEventRecord(rt->t_wave_end[a.index], ws), "record")) return fail_cuda();
    if (e2e_out && b1 > b0) {  // this wave's final rows are in the staging ring: download them
      if (!ok(cudaEventRecord(rt->out_ev[a.index], ws), "record") ||
          !ok(cudaStreamWaitEvent(rt->out_stream, rt->out_ev[a.index], 0), "download waits wave"))
        return fail_cuda();
      char *hout = static_cast<char *>(in->host_outputs);
      const int64_t R = rt->out_slots;
      if (c.profile) rt->io_kind.push_back(1);
      if (!io_mark(rt->out_stream)) return fail_cuda();
      for (int64_t p = out_base + b0; p < out_base + b1;) {  // at most two pieces (ring wrap)
        const int64_t q = p % R, n = std::min<int64_t>(out_base + b1 - p, R - q);
        if (!ok(cudaMemcpyAsync(hout + (size_t)(p - out_base) * rb, reinterpret_cast<char *>(rt->outbuf) + (size_t)q * rb,
                                (size_t)n * rb, cudaMemcpyDeviceToHost, rt->out_stream),
                "output D2H"))
          return fail_cuda();
        p += n;
      }
      if (!io_mark(rt->out_stream)) return fail_cuda();
      cudaEvent_t done = nullptr;
      if (!rt->out_ev_pool.empty()) {
        done = rt->out_ev_pool.back();
        rt->out_ev_pool.pop_back();
      } else if (!ok(cudaEventCreateWithFlags(&done, cudaEventDisableTiming), "event")) {
        return fail_cuda();
      }
      if (!ok(cudaEventRecord(done, rt->out_stream), "record")) return fail_cuda();
      rt->out_hist.push_back(coe_runtime::OutUse{out_base + b0, out_base + b1, done});
      st.d2h_output_bytes += (int64_t)(b1 - b0) * (int64_t)rb;
    }
  }
  if (e2e_out) {
    // not joined into the compute stream: the next step's waves need not wait for this step's
    // downloads (only the staging rows they overwrite do); coe_runtime_join / synchronize cover them
    if (!ok(cudaEventRecord(rt->out_drained, rt->out_stream), "record")) return fail_cuda();
    rt->have_out = true;
  }
  if (!peer_mode && !issue_hops_until(INT64_MAX)) return COE_CUDA_ERR_CUDA;
  if (peer_mode)  // launches captured their arguments; later direct K3 uses run hop-free
    for (auto &per : rt->mlps)
      for (coe_mlp *m : per)
        if (m) coe_mlp_set_hops(m, nullptr, 0, nullptr, 0);
  if (!my_hops.empty() && (!ok(cudaEventRecord(rt->hop_drained, rt->hop), "record") ||
                           !ok(cudaStreamWaitEvent(cs, rt->hop_drained, 0), "join hop")))
    return fail_cuda();
  if (!ok(cudaEventRecord(rt->copy_drained, ks), "record") || !ok(cudaStreamWaitEvent(cs, rt->copy_drained, 0), "join"))
    return fail_cuda();
  for (int k = 1; k < NCLS; ++k)
    if (!ok(cudaEventRecord(rt->cls_drained[k], rt->cls_stream[k]), "record") ||
        !ok(cudaStreamWaitEvent(cs, rt->cls_drained[k], 0), "join"))
      return fail_cuda();
  if (peer_mode && !rt->peer_hub)  // this step is done here: tell every peer (their next step's fence)
    for (int r = 0; r < rt->peer_world; ++r)
      if (r != x &&
          !write_flag(cs, static_cast<int32_t *>(rt->peers[r].flags) + rt->hflag_step_base + x, seq))
        return COE_CUDA_ERR_CUDA;
  if (c.profile && !ok(cudaEventRecord(rt->t_step_end, cs), "record")) return fail_cuda();
  if (!ok(cudaEventRecord(sb.free_ev, cs), "record") || !ok(cudaEventRecord(rt->step_end, cs), "record"))
    return fail_cuda();
  rt->have_step_end = true;
  {  // (f3) where each resident expert's bytes live once this step's work is done
    const int par = (int)(rt->step_count & 1);
    auto &snap = rt->res_snap[par];
    snap.assign(c.num_experts, nullptr);
    for (int32_t e = 0; e < c.num_experts; ++e) {
      const int32_t sl = rt->expert_slot[e];
      if (sl >= 0) snap[e] = rt->pooled ? rt->pool + (int64_t)rt->slot_unit[sl] * rt->unit : rt->slot_ptr(sl);
    }
    if (!ok(cudaEventRecord(rt->res_ready[par], cs), "record")) return fail_cuda();
    rt->step_count += 1;
  }
  // the ring carries over: the free list in release order, and for the next step's input
  // uploads the wave (this parity) whose up pass last read each slot freed in this step
  std::fill(rt->act_prev_wave.begin(), rt->act_prev_wave.end(), -1);
  for (size_t i = 0; i < rows.freed_slot.size(); ++i)
    rt->act_prev_wave[rows.freed_slot[i]] = batches[rows.freed_by[i]].wave;
  rt->ring_order = rows.free_after;
  rt->prev_nccl_hold = rows.nccl_hold;
  rt->step_parity ^= 1;
  st.ring_peak = rows.peak_ring;
  st.landing_rows = rows.landing;
  sb.used = true;
  rt->last_waves = (int32_t)nw;
  rt->last_wave_cls.clear();
  rt->last_wave_rows.clear();
  rt->last_wave_groups.clear();
  rt->last_wave_shape.clear();
  rt->last_wave_flops.clear();
  for (const WaveAct &w : waves) {
    rt->last_wave_cls.push_back(w.cls);
    rt->last_wave_rows.push_back((int32_t)w.rows);
    rt->last_wave_groups.push_back(w.num_groups);
    rt->last_wave_shape.push_back(w.shape);
    rt->last_wave_flops.push_back(4.0 * (double)w.rows * rt->sd[w.shape] * rt->sh[w.shape]);
  }
  rt->last_copies = (int32_t)nc;

  rt->last_adm = n_adm;
  rt->last_batches = n_batches;
  rt->last_set = set_idx;
  if (stats) *stats = st;
  return COE_CUDA_OK;
}
