// comm.cu -- NCCL point-to-point for follow-up hops (loaded with dlopen).
//
// The runtime moves a hopped request's T x d activation from the GPU that ran
// its previous stage to the GPU its next stage was assigned to
// (engine.py:751-753 admits the follow-up there).  NCCL 2.28 (the library
// torch ships, site-packages/nvidia/nccl) is dlopen'ed so the kernel library
// has no link-time NCCL dependency; one communicator per runtime, all hop
// traffic on the runtime's hop stream, one ncclSend / ncclRecv per hop in the
// global hop order (hops.h).
#include <cuda_bf16.h>
#include <dlfcn.h>

#include <condition_variable>
#include <cstring>
#include <deque>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "coe_cuda.h"
#include "comm.h"
#include "common.cuh"

namespace {

struct NcclApi {
  void *handle = nullptr;
  ncclResult_t (*get_unique_id)(ncclUniqueId *) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char *(*error_string)(ncclResult_t) = nullptr;
};

NcclApi g_nccl;

bool load_nccl(const char *path) {
  if (g_nccl.handle) return true;
  void *h = dlopen(path && *path ? path : "libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    coe_set_error(std::string("dlopen NCCL failed: ") + dlerror());
    return false;
  }
  g_nccl.handle = h;
  g_nccl.get_unique_id = reinterpret_cast<decltype(g_nccl.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
  g_nccl.comm_init_rank = reinterpret_cast<decltype(g_nccl.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
  g_nccl.comm_destroy = reinterpret_cast<decltype(g_nccl.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
  g_nccl.send = reinterpret_cast<decltype(g_nccl.send)>(dlsym(h, "ncclSend"));
  g_nccl.recv = reinterpret_cast<decltype(g_nccl.recv)>(dlsym(h, "ncclRecv"));
  g_nccl.error_string = reinterpret_cast<decltype(g_nccl.error_string)>(dlsym(h, "ncclGetErrorString"));
  g_nccl.group_start = reinterpret_cast<decltype(g_nccl.group_start)>(dlsym(h, "ncclGroupStart"));
  g_nccl.group_end = reinterpret_cast<decltype(g_nccl.group_end)>(dlsym(h, "ncclGroupEnd"));
  if (!g_nccl.get_unique_id || !g_nccl.comm_init_rank || !g_nccl.send || !g_nccl.recv || !g_nccl.group_start ||
      !g_nccl.group_end) {
    coe_set_error("NCCL library lacks point-to-point symbols");
    return false;
  }
  return true;
}

bool nccl_ok(ncclResult_t r, const char *what) {
  if (r == ncclSuccess) return true;
  coe_set_error(std::string(what) + ": " + (g_nccl.error_string ? g_nccl.error_string(r) : "nccl error"));
  return false;
}

}  // namespace

// In-process transport: several runtimes on ONE device (one host thread each), e.g. the
// reference's multiple logical executors per GPU, and the single-GPU test of the hop
// protocol.  Point-to-point messages match in order per (src, dst) pair like NCCL's; a
// send publishes (rows, event-after-producer) and returns, a receive blocks on the host
// until its match is published, then makes its stream wait and copies device to device.
// Callers synchronise every runtime between steps (the sender does not wait for the copy).
struct LocalMsg {
  const void *buf;
  size_t bytes;
  cudaEvent_t ready;
};

struct coe_local_hub {
  int world = 1;
  std::mutex mu;
  std::condition_variable cv;
  std::map<std::pair<int, int>, std::deque<LocalMsg>> queues;
  std::map<int64_t, cudaEvent_t> published;  // fused peer hops in one process: hop index -> event
  std::vector<cudaEvent_t> events;  // owned, reused round-robin
  size_t next_event = 0;
  ~coe_local_hub() {
    for (auto e : events) cudaEventDestroy(e);
  }
};

struct coe_comm {
  ncclComm_t comm = nullptr;
  coe_local_hub *hub = nullptr;
  int rank = 0, world = 1;
};

bool coe_comm_send_bf16(coe_comm *c, const void *buf, size_t count, int peer, cudaStream_t stream) {
  if (c->hub) {
    std::lock_guard<std::mutex> lk(c->hub->mu);
    auto &hub = *c->hub;
    if (hub.next_event >= hub.events.size()) {
      cudaEvent_t e;
      if (!coe_cuda_ok(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "local hub event")) return false;
      hub.events.push_back(e);
    }
    cudaEvent_t ev = hub.events[hub.next_event++];
    if (!coe_cuda_ok(cudaEventRecord(ev, stream), "local send record")) return false;
    hub.queues[{c->rank, peer}].push_back(LocalMsg{buf, count * 2, ev});
    hub.cv.notify_all();
    return true;
  }
  return nccl_ok(g_nccl.send(buf, count, ncclBfloat16, peer, c->comm, stream), "ncclSend");
}

bool coe_comm_recv_bf16(coe_comm *c, void *buf, size_t count, int peer, cudaStream_t stream) {
  if (c->hub) {
    LocalMsg m;
    {
      std::unique_lock<std::mutex> lk(c->hub->mu);
      auto &q = c->hub->queues[{peer, c->rank}];
      c->hub->cv.wait(lk, [&] { return !q.empty(); });
      m = q.front();
      q.pop_front();
    }
    if (m.bytes != count * 2) {
      coe_set_error("local hop: message size mismatch");
      return false;
    }
    return coe_cuda_ok(cudaStreamWaitEvent(stream, m.ready, 0), "local recv wait") &&
           coe_cuda_ok(cudaMemcpyAsync(buf, m.buf, m.bytes, cudaMemcpyDeviceToDevice, stream), "local recv copy");
  }
  return nccl_ok(g_nccl.recv(buf, count, ncclBfloat16, peer, c->comm, stream), "ncclRecv");
}

int coe_comm_rank(const coe_comm *c) { return c->rank; }

// One NCCL group around a run of sends / receives: NCCL fuses them into one launch that
// progresses every transfer concurrently (the all-to-all of a wave's hops).  The in-process
// hub has nothing to fuse.
bool coe_comm_group(coe_comm *c, bool start) {
  if (c->hub) return true;
  return nccl_ok(start ? g_nccl.group_start() : g_nccl.group_end(), start ? "ncclGroupStart" : "ncclGroupEnd");
}

// Fused peer hops between runtimes of one process: the producer publishes an event recorded
// after the down pass that stored the rows; the consumer blocks on the host until it is
// published and makes its stream wait on it.  (Stream memory-op flags are not used in one
// process: a waiting stream can share a hardware queue with the stream that would write the
// flag.)
bool coe_hub_publish(coe_local_hub *hub, int64_t key, cudaStream_t stream) {
  std::lock_guard<std::mutex> lk(hub->mu);
  if (hub->next_event >= hub->events.size()) {
    cudaEvent_t e;
    if (!coe_cuda_ok(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "hub event")) return false;
    hub->events.push_back(e);
  }
  cudaEvent_t ev = hub->events[hub->next_event++];
  if (!coe_cuda_ok(cudaEventRecord(ev, stream), "hub publish")) return false;
  hub->published[key] = ev;
  hub->cv.notify_all();
  return true;
}

bool coe_hub_wait(coe_local_hub *hub, int64_t key, cudaStream_t stream) {
  cudaEvent_t ev;
  {
    std::unique_lock<std::mutex> lk(hub->mu);
    hub->cv.wait(lk, [&] { return hub->published.count(key) > 0; });
    ev = hub->published[key];
  }
  return coe_cuda_ok(cudaStreamWaitEvent(stream, ev, 0), "hub wait");
}

extern "C" {

int coe_comm_unique_id(const char *nccl_path, void *out128) {
  if (!load_nccl(nccl_path)) return COE_CUDA_ERR_CONFIG;
  ncclUniqueId id;
  if (!nccl_ok(g_nccl.get_unique_id(&id), "ncclGetUniqueId")) return COE_CUDA_ERR_CUDA;
  std::memcpy(out128, &id, sizeof(id));
  return COE_CUDA_OK;
}

int coe_comm_create(const char *nccl_path, int rank, int world, const void *id128, coe_comm **out) {
  if (!load_nccl(nccl_path)) return COE_CUDA_ERR_CONFIG;
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  auto *c = new coe_comm();
  c->rank = rank;
  c->world = world;
  if (!nccl_ok(g_nccl.comm_init_rank(&c->comm, world, id, rank), "ncclCommInitRank")) {
    delete c;
    return COE_CUDA_ERR_CUDA;
  }
  *out = c;
  return COE_CUDA_OK;
}

void coe_comm_destroy(coe_comm *c) {
  if (!c) return;
  if (c->comm && g_nccl.comm_destroy) g_nccl.comm_destroy(c->comm);
  delete c;
}

coe_local_hub *coe_local_hub_create(int world) {
  auto *h = new coe_local_hub();
  h->world = world;
  return h;
}

void coe_local_hub_destroy(coe_local_hub *h) { delete h; }

void coe_local_hub_reset(coe_local_hub *h) {
  std::lock_guard<std::mutex> lk(h->mu);
  h->queues.clear();
  h->published.clear();
  h->next_event = 0;
}

int coe_swap_in(void *dst_slot, const void *src_pinned, int64_t bytes, cudaStream_t copy_stream,
                cudaEvent_t done_event) {
  if (bytes < 0 || (bytes && (!dst_slot || !src_pinned))) {
    coe_set_error("coe_swap_in: bad buffer or size");
    return COE_CUDA_ERR_CONFIG;
  }
  if (bytes && !coe_cuda_ok(cudaMemcpyAsync(dst_slot, src_pinned, (size_t)bytes, cudaMemcpyHostToDevice, copy_stream),
                            "coe_swap_in"))
    return COE_CUDA_ERR_CUDA;
  if (done_event && !coe_cuda_ok(cudaEventRecord(done_event, copy_stream), "coe_swap_in record"))
    return COE_CUDA_ERR_CUDA;
  return COE_CUDA_OK;
}

int coe_hop(coe_comm *comm, const void *sendbuf, const int64_t *send_counts, void *recvbuf,
            const int64_t *recv_counts, cudaStream_t stream) {
  if (!comm || !send_counts || !recv_counts) {
    coe_set_error("coe_hop: communicator and counts required");
    return COE_CUDA_ERR_CONFIG;
  }
  const int W = comm->world, me = comm->rank;
  std::vector<int64_t> soff(W + 1, 0), roff(W + 1, 0);
  for (int r = 0; r < W; ++r) {
    if (send_counts[r] < 0 || recv_counts[r] < 0) {
      coe_set_error("coe_hop: negative count");
      return COE_CUDA_ERR_CONFIG;
    }
    soff[r + 1] = soff[r] + send_counts[r];
    roff[r + 1] = roff[r] + recv_counts[r];
  }
  if (send_counts[me] != recv_counts[me]) {
    coe_set_error("coe_hop: the self segment must send what it receives");
    return COE_CUDA_ERR_CONFIG;
  }
  const auto *sb = static_cast<const __nv_bfloat16 *>(sendbuf);
  auto *rb = static_cast<__nv_bfloat16 *>(recvbuf);
  if (send_counts[me] &&
      !coe_cuda_ok(cudaMemcpyAsync(rb + roff[me], sb + soff[me], 2 * (size_t)send_counts[me], cudaMemcpyDeviceToDevice,
                                   stream),
                   "coe_hop self copy"))
    return COE_CUDA_ERR_CUDA;
  if (!coe_comm_group(comm, true)) return COE_CUDA_ERR_CUDA;
  bool good = true;
  for (int k = 1; k < W && good; ++k) {  // ring order: every rank sends to me+k while receiving from me-k
    const int to = (me + k) % W, from = (me - k + W) % W;
    if (send_counts[to]) good = coe_comm_send_bf16(comm, sb + soff[to], (size_t)send_counts[to], to, stream);
    if (good && recv_counts[from])
      good = coe_comm_recv_bf16(comm, rb + roff[from], (size_t)recv_counts[from], from, stream);
  }
  if (!coe_comm_group(comm, false) || !good) return COE_CUDA_ERR_CUDA;
  return COE_CUDA_OK;
}

int coe_comm_create_local(coe_local_hub *hub, int rank, coe_comm **out) {
  auto *c = new coe_comm();
  c->hub = hub;
  c->rank = rank;
  c->world = hub->world;
  *out = c;
  return COE_CUDA_OK;
}

}  // extern "C"
