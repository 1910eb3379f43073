/*
 * coe_cuda.h -- C-ABI of the sm_100a kernels and the GPU serving runtime.
 *
 * Plain pointers and sizes only (device pointers unless stated otherwise);
 * every call is stream-ordered on the caller's cudaStream_t, returns 0 or a
 * COE_CUDA_ERR_* code, and leaves the message in coe_cuda_last_error().
 *
 * Reference interfaces each entry point replaces (the reference models these
 * steps with closed-form costs; SURVEY.md §2 "Kernels and collectives"):
 *   coe_group_sort   <- scheduler.arrange_position + engine._Queue.insert
 *                       (scheduler.py:100-108, engine.py:251-254)
 *   coe_run_compact  <- engine._Queue.head_run + scheduler.batch_cap/split_batch
 *                       (engine.py:270-283, scheduler.py:111-137)
 *   coe_grouped_mlp  <- CostModel.exec_latency as used by Simulation._start_batch
 *                       (costmodel.py:55-64, engine.py:693-716)
 *   coe_swap_in      <- CostModel.load_latency_from as used by Simulation._start_load
 *                       (costmodel.py:69-73, engine.py:643-677)
 *   coe_runtime_*    <- Simulation.run's physical side (engine.py:762-781)
 */
#ifndef COE_CUDA_H
#define COE_CUDA_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st *cudaStream_t;
typedef struct CUevent_st *cudaEvent_t;

enum { COE_CUDA_OK = 0, COE_CUDA_ERR_CONFIG = 2, COE_CUDA_ERR_CHECK = 4, COE_CUDA_ERR_CUDA = 6 };

const char *coe_cuda_last_error(void);

/* ---------------- K1 / K2: GPU grouping ---------------------------------- */

/* Stable LSD radix sort of n admissions by key = executor << rank_bits | run_rank.
 * executor/run_rank: [n] int32 (admission order); out_perm: [n] sorted indices.
 * scratch: coe_group_sort_scratch_bytes(n) bytes.  This is the segmented
 * (per-executor) stable sort by run-rank that reproduces the reference's
 * arranged queue order. */
int64_t coe_group_sort_scratch_bytes(int64_t n);
int coe_group_sort(const int32_t *executor, const int32_t *run_rank, int64_t n, int rank_bits, int num_passes,
                   int32_t *out_perm, int32_t *out_keys, void *scratch, cudaStream_t stream);

/* Compaction: gathers the sorted admissions into per-member arrays, finds
 * each planned batch's offset inside its executor's segment, and checks that
 * every batch is a single run (one key) -- the head-run/split contract.
 *   batch_exec/batch_size: [num_batches] in per-executor op order
 *   out_batch_off: [num_batches]; out_member_req/stage: [n]
 *   out_run_count: [1] number of distinct runs; out_violations: [1] batches
 *   spanning more than one run (must be 0). */
int coe_run_compact(const int32_t *perm, const int32_t *sorted_keys, const int32_t *adm_request,
                    const int32_t *adm_stage, int64_t n, int rank_bits, const int32_t *batch_exec,
                    const int32_t *batch_size, int num_batches, int num_executors, int32_t *out_batch_off,
                    int32_t *out_member_req,
                    int32_t *out_member_stage, int32_t *out_run_count, int32_t *out_violations, void *scratch,
                    cudaStream_t stream);
int64_t coe_run_compact_scratch_bytes(int64_t n, int num_batches, int num_executors);
/* coe_run_compact that also gathers each admission's activation-row routes (adm_in /
 * adm_out -> out_member_in / out_member_out, same permutation; see coe_grouped_mlp_routed) */
int coe_run_compact_routes(const int32_t *perm, const int32_t *sorted_keys, const int32_t *adm_request,
                           const int32_t *adm_stage, const int32_t *adm_in, const int32_t *adm_out, int64_t n,
                           int rank_bits, const int32_t *batch_exec, const int32_t *batch_size, int num_batches,
                           int num_executors, int32_t *out_batch_off, int32_t *out_member_req,
                           int32_t *out_member_stage, int32_t *out_member_in, int32_t *out_member_out,
                           int32_t *out_run_count, int32_t *out_violations, void *scratch, cudaStream_t stream);

/* K1 + K2 of ONE executor in one launch (serving size): one 1,024-thread block sorts the
 * keys (run_rank << idx_bits | admission) in shared memory -- the stable sort by run-rank --
 * then gathers members (and their row routes, adm_in / adm_out may be NULL), scans the batch
 * sizes into offsets and checks that no batch straddles two runs: out_flags[0] = runs,
 * out_flags[1] = violations, like coe_run_compact.  COE_CUDA_ERR_CONFIG (no launch) when
 * n > COE_FUSED_MAX_ADMISSIONS, num_batches > COE_FUSED_MAX_BATCHES or the key needs more
 * than 32 bits; callers then use coe_group_sort + coe_run_compact. */
#define COE_FUSED_MAX_ADMISSIONS 32768
#define COE_FUSED_MAX_BATCHES 4096
int coe_group_compact_fused(const int32_t *run_rank, const int32_t *adm_request, const int32_t *adm_stage,
                            const int32_t *adm_in, const int32_t *adm_out, int64_t n, int rank_bits,
                            const int32_t *batch_size, int num_batches, int32_t *out_perm, int32_t *out_batch_off,
                            int32_t *out_member_req, int32_t *out_member_stage, int32_t *out_member_in,
                            int32_t *out_member_out, int32_t *out_flags, cudaStream_t stream);

/* ---------------- K3: grouped expert MLP (tcgen05) ------------------------ */

typedef struct coe_mlp_config {
  int32_t d, h, T;              /* model dim, hidden dim, rows per request       */
  void *x;                      /* request inputs (stage 0) [act_rows, d] bf16   */
  void *act0, *act1;            /* stage s>0 reads act[(s-1)&1], writes act[s&1] */
  int64_t act_rows;             /* requests * T                                  */
  void *h_scratch;              /* [h_rows, h] bf16                              */
  int64_t h_rows;
  void *slab;                   /* expert slots: [num_slots][W1 h*d | W2 d*h]    */
  int32_t num_slots;
  int64_t slot_stride_bytes;
  int32_t act_ld;               /* row stride of X / P0 / P1 in elements (0: d);
                                   > d when experts of several widths share them */
  int64_t x_rows;               /* rows of x (0: act_rows)                       */
} coe_mlp_config;

/* One planned batch inside a wave.  tile_start is the wave-relative prefix of
 * tiles (ceil(rows/128) * N/256) for the pass the array is used with. */
typedef struct coe_mlp_group {
  int32_t rows;        /* members * T                                        */
  int32_t slot;        /* expert slot holding W1/W2                          */
  int32_t batch;       /* index into batch_off                               */
  int32_t h_row;       /* first row of this group in h_scratch               */
  int32_t tile_start;
  int32_t pad[3];
} coe_mlp_group;

typedef struct coe_mlp coe_mlp;
int coe_mlp_create(const coe_mlp_config *cfg, coe_mlp **out);
void coe_mlp_destroy(coe_mlp *m);
int coe_mlp_max_groups(void);
/* which: bit0 = up projection (gelu(X W1^T) -> H), bit1 = down (H W2^T -> Y).
 * max_ctas: persistent grid cap (0 = one CTA per SM).  tiles_up / tiles_down and each
 * group's tile_start count 128-row x 256-column tiles (m fastest inside (group, n-block));
 * the default CTA-pair kernel (COE_K3_CG=2) walks 256-row pair tiles and derives them from
 * the groups' row counts itself, so callers always pass the 128-row figures. */
int coe_grouped_mlp(coe_mlp *m, const coe_mlp_group *groups_up, const coe_mlp_group *groups_down, int num_groups,
                    int tiles_up, int tiles_down, const int32_t *batch_off, const int32_t *member_req,
                    const int32_t *member_stage, int which, int max_ctas, cudaStream_t stream);
/* Fused follow-up hops for the down projection of later launches: a member whose
 * hop_dst[req * hop_stride + stage] = r >= 0 has its output rows stored into
 * peer_act[2 * r + (stage & 1)] (executor r's P0 / P1, same row layout) instead of the
 * local buffer.  hop_dst == NULL turns it off.  world <= COE_MAX_PEERS. */
#define COE_MAX_PEERS 8
int coe_mlp_set_hops(coe_mlp *m, const int8_t *hop_dst, int hop_stride, void *const *peer_act, int world);
/* Routed mode: each member (sorted admission) names its own activation rows instead of
 * (request, stage) ping-pong addressing.  member_in[i] = (row << 1) | from_x: the A operand
 * is request-row block `row` of cfg.x (from_x = 1) or of cfg.act0 (the activation ring A);
 * member_out[i] = (row << 4) | kind: the down pass stores the member's rows into block `row`
 * of kind 0 = cfg.act0 (in place: the up pass has consumed the input), 1 = the device output
 * buffer y, 2 = the output staging ring, 3 + r = executor r's act0 (peer_act of
 * coe_mlp_set_hops; a fused hop).  Up passes only read member_in, down passes member_out. */
int coe_mlp_set_outputs(coe_mlp *m, void *y, void *out_stage);
int coe_grouped_mlp_routed(coe_mlp *m, const coe_mlp_group *groups_up, const coe_mlp_group *groups_down,
                           int num_groups, int tiles_up, int tiles_down, const int32_t *batch_off,
                           const int32_t *member_in, const int32_t *member_out, int which, int max_ctas,
                           cudaStream_t stream);
/* Stage-0 inputs of later launches from `x` (same shape / stride as cfg.x; NULL or cfg.x:
 * back to cfg.x) -- lets e2e steps double-buffer their input uploads. */
int coe_mlp_set_input(coe_mlp *m, void *x);

/* ---------------- GPU serving runtime (one executor per GPU) --------------- */

/* The physical half of the serving path: executes the planner's op log for
 * one executor -- GPU grouping (K1/K2) of the step's admissions, waves of
 * grouped expert MLPs (K3) on the compute stream, swap-ins (K4) from the
 * pinned host expert store into fixed HBM slots on a copy-engine stream,
 * issued as soon as the victim slot's last wave has finished (dependency-
 * aware prefetch).  Decisions are never changed by physical timing. */
typedef struct coe_runtime_config {
  int32_t d, h, T;
  int32_t num_experts;
  int32_t num_slots;        /* HBM expert slots = expert budget / expert bytes       */
  int32_t max_requests;     /* capacity of the X / P0 / P1 activation buffers        */
  int64_t max_wave_rows;    /* rows of the H scratch (caps a wave)                   */
  int64_t max_admissions;
  int64_t max_batches;
  uint64_t weight_seed;     /* synthetic expert weights, see coe_expert_seed         */
  int32_t profile;          /* record per-copy / per-wave events for overlap stats   */
  int32_t reserve_sms;      /* SMs kept for the swap-in-gating waves (0: no split)   */
  int32_t swapped_stream;   /* reserved (ignored)                                    */
  const char *store_path;   /* NULL: private pinned store; else a shared file mapping
                               (one copy per node for N ranks; host-registered)     */
  int64_t wave_rows_cap;    /* main-stream wave size cap (0: max_wave_rows)          */
  int64_t urgent_rows_cap;  /* cap when a wave carries reads an imminent swap-in
                               waits for (0: wave_rows_cap)                          */
  /* heterogeneous experts: per-shape (d, h) slabs; activations are [requests][T][max d]
   * and an expert of width d uses the first d columns (d is constant along a chain) */
  int32_t num_shapes;       /* 0: a single shape (d, h, num_slots above)            */
  const int32_t *shape_d, *shape_h, *shape_slots;   /* [num_shapes]                  */
  const int32_t *expert_shape;                       /* [num_experts] shape index     */
  const uint8_t *store_mask; /* [num_experts] experts held in the host store (NULL: all) */
  /* activation memory (act_rows.h): A = [landing_slots | ring_slots] request-row blocks of
   * T x max-d bf16 -- a request's activation occupies one ring slot from its first batch
   * here until its output leaves (stages run in place), hop-ins land in landing rows;
   * size both with coe_runtime_plan_rows.  out_slots: e2e output staging rows (0: auto). */
  int32_t ring_slots, landing_slots, out_slots;
  int32_t device_io;        /* 1: X / Y of max_requests rows for device-resident steps
                               (fill_inputs, value-mode steps, download_*); 0: e2e only */
  /* > 0: experts of every shape share ONE slab of this many bytes (the planner's byte budget
   * + unit rounding + fragmentation slack), addressed in 2 MB units: a load takes a best-fit
   * run of free units, an eviction returns it; shape_slots[k] = experts of shape k (one
   * bookkeeping slot each).  0: fixed per-shape slabs of shape_slots[k] slots. */
  int64_t expert_pool_bytes;
} coe_runtime_config;


typedef struct coe_step_input {
  int32_t executor;                         /* ops / admissions of other executors ignored */
  int64_t num_admissions;
  const void *admissions;                   /* coe_admission[] (coe_planner.h)            */
  int64_t num_ops;
  const void *ops;                          /* coe_op[] (coe_planner.h)                   */
  int64_t num_op_args;
  const int32_t *op_args;
  int32_t num_initial;                      /* initial residency of this executor          */
  const int32_t *initial;
  /* end-to-end serving (optional, pinned host memory, [rows][T][ld] bf16): input row i holds
   * the i-th smallest request whose stage 0 runs on this executor (with one executor: row r =
   * request r), uploaded just in time on the copy engine; outputs are streamed
   * back in COMPLETION order -- each wave's final rows are gathered on the GPU and leave in
   * one D2H copy -- and coe_runtime_output_order names the request of every output row */
  const void *host_inputs;
  void *host_outputs;
  /* (f3) initial residency of EVERY executor, CSR over executors (optional: null disables
   * physical peer copies -- peer-tier LOADs are then served from the host tier) */
  int32_t num_executors;
  const int32_t *initial_offsets;           /* [num_executors + 1]                          */
  const int32_t *initial_all;
} coe_step_input;

/* Activation rows one step of `in` needs on executor in->executor (host only, no GPU):
 * the ring's peak occupancy and the landing rows for hop-ins.  e2e: stage-0 inputs also
 * occupy slots; nccl: hop-outs keep their slots until the step ends (the NCCL transport). */
int coe_runtime_plan_rows(const coe_step_input *in, int32_t max_requests, int e2e, int nccl,
                          int32_t *ring_slots, int32_t *landing_slots);

typedef struct coe_step_stats {
  int64_t admissions, batches, waves, launches;
  int64_t h2d_input_bytes, d2h_output_bytes;
  int64_t loads, load_bytes, restores, restore_bytes;
  int64_t max_wave_rows;
  int32_t max_wave_groups;
  int32_t rank_bits;
  int32_t ring_peak;        /* activation ring slots occupied at most during the step  */
  int32_t landing_rows;     /* landing rows the step's hop-ins used                     */
  int64_t peer_loads;       /* (f3) peer-tier LOADs copied from another executor's HBM  */
  int64_t peer_bytes;
  int64_t peer_tier_loads;  /* peer-tier LOADs in the plan (the rest came from the host) */
} coe_step_stats;

typedef struct coe_step_timing {
  float total_ms;           /* step start -> both streams drained                    */
  float copy_busy_ms;       /* union of swap-in copy intervals                        */
  float compute_busy_ms;    /* union of wave intervals (grouping included)           */
  float overlap_ms;         /* intersection of the two                               */
  float mlp_ms;             /* sum of K3 wave durations                              */
  float group_ms;           /* K1 + K2                                                */
  float k3_busy_ms;         /* union of K3 launch intervals (up and down passes; waits
                               for a swap-in's W2 half between them excluded)          */
  int32_t k3_launches;      /* K3 launches in the step (2 per wave)                   */
  double k3_flops;          /* algorithmic 4*rows*d*h over the step's waves          */
} coe_step_timing;

typedef struct coe_runtime coe_runtime;
int coe_runtime_create(const coe_runtime_config *cfg, coe_runtime **out);
void coe_runtime_destroy(coe_runtime *rt);
/* generate every expert's W1/W2 on the GPU and stage them in the pinned host store */
int coe_runtime_init_experts(coe_runtime *rt);
/* seeded request inputs straight into the device X buffer (device-resident runs) */
int coe_runtime_fill_inputs(coe_runtime *rt, uint64_t seed, int32_t num_requests);
/* host (pinned) -> X for the first num_requests requests, on the compute stream */
int coe_runtime_upload_inputs(coe_runtime *rt, const void *host, int32_t num_requests);
int coe_runtime_step(coe_runtime *rt, const coe_step_input *in, coe_step_stats *stats);
/* gather each request's final activation (stage last_stage[r]) and copy to host */
int coe_runtime_download_outputs(coe_runtime *rt, const int32_t *last_stage_host, int32_t num_requests, void *host);
/* the activation rows of (requests[i], stage stages[i]) -- normally each request's final
 * stage -- gathered on the GPU into host[i] ([n][T][ld] bf16, pageable or pinned); synchronous */
int coe_runtime_download_requests(coe_runtime *rt, const int32_t *requests, const int32_t *stages, int32_t n,
                                  void *host);
int coe_runtime_synchronize(coe_runtime *rt);
/* after synchronize: K2 run count / violations, and the grouped members */
/* make the compute stream (coe_runtime_stream(rt, 0)) wait for the last step's output
 * downloads -- e2e steps do not join them, so an event recorded after this covers them */
int coe_runtime_join(coe_runtime *rt);
int coe_runtime_check(coe_runtime *rt, int32_t *runs, int32_t *violations);
int coe_runtime_members(coe_runtime *rt, int32_t *member_req, int32_t *member_stage, int32_t *batch_off);
int coe_runtime_timing(coe_runtime *rt, coe_step_timing *out);
/* profile mode: per-copy [start,end) and per-wave [start,end) ms since step start,
 * wave_info = (stream class, rows, groups) per wave; sizes from coe_runtime_counts */
int coe_runtime_counts(coe_runtime *rt, int32_t *copies, int32_t *waves);
/* e2e: request id of each row of host_outputs after the last step (completion order);
 * returns the row count, copies at most `capacity` ids (requests may be NULL) */
int32_t coe_runtime_output_order(coe_runtime *rt, int32_t *requests, int32_t capacity);
/* K3 in isolation on the runtime's buffers: one wave of `groups` batches x
 * `requests_per_group` requests; average up / down projection launch times */
int coe_runtime_bench_mlp(coe_runtime *rt, int32_t groups, int32_t requests_per_group, int32_t iters,
                          float *up_ms, float *down_ms);
int coe_runtime_intervals(coe_runtime *rt, float *copy_iv, float *wave_iv, int32_t *wave_info);

/* ---- fused follow-up hops over peer memory (N executors, N <= COE_MAX_PEERS) ----
 * Instead of a send / receive pair, the producer's K3 down pass stores a hopping request's
 * output rows directly into the destination executor's P buffer (NVLink peer stores when
 * the executors are different GPUs), then its stream publishes the hop's flag in the
 * destination's flag array (cuStreamWriteValue32, after a memory barrier); the consumer's
 * wave waits on its own flag (cuStreamWaitValue32) -- no copy, no extra kernel.  Every
 * executor sees the same global hop order (hops.h), so flags are indexed by hop index and
 * hold the step sequence number.  A per-step device-side fence keeps a producer from
 * writing into a destination still running the previous step.
 * Buffers come from coe_runtime_peer_buffers (same process) or, across processes, from
 * coe_runtime_ipc_export (3 x 64-byte cudaIpcMemHandle_t) + coe_runtime_ipc_open. */
typedef struct coe_local_hub coe_local_hub;  /* in-process transport, declared below */
typedef struct coe_peer_buffers {
  void *p0, *p1, *flags;
} coe_peer_buffers;
int coe_runtime_peer_buffers(coe_runtime *rt, coe_peer_buffers *out);
int coe_runtime_ipc_export(coe_runtime *rt, void *handles);
int coe_runtime_ipc_open(coe_runtime *rt, const void *handles, coe_peer_buffers *out);
/* peers[world]: every executor's buffers (peers[rank] = this runtime's own).  hub != NULL:
 * the peers are runtimes of THIS process (several executors on one GPU, stepped together):
 * hops are handed over as events through the hub instead of stream-memop flags, since a
 * flag-waiting stream may share a hardware queue with the stream that would write it. */
int coe_runtime_attach_peers(coe_runtime *rt, int32_t rank, int32_t world, const coe_peer_buffers *peers,
                             coe_local_hub *hub);
/* profile mode: per wave [up start, up end, down start, down end] ms since step start and
 * the wave's algorithmic FLOPs (4 * rows * d * h) */
int coe_runtime_wave_phases(coe_runtime *rt, float *phase_iv, double *wave_flops);
/* after a step: the expert-shape index (coe_runtime_config.shape_d / shape_h order) of each wave */
int coe_runtime_wave_shapes(coe_runtime *rt, int32_t *shape_index);
/* profile mode, e2e steps: [start, end] ms of each stage-0 input upload (copy engine) then of
 * each output download (output stream); iv == NULL queries the counts only */
int coe_runtime_io_intervals(coe_runtime *rt, float *iv, int32_t *n_in, int32_t *n_out);
/* device pointers (tests / benches): 0 X, 1 P0, 2 P1, 3 H scratch, 4 slot slab */
void *coe_runtime_buffer(coe_runtime *rt, int which);
/* synchronous device -> host copy of the first `bytes` of buffer `which` */
int coe_runtime_read_buffer(coe_runtime *rt, int which, void *host, int64_t bytes);
int coe_runtime_slot_of(coe_runtime *rt, int32_t expert);
cudaStream_t coe_runtime_stream(coe_runtime *rt, int which);
uint64_t coe_expert_seed(uint64_t weight_seed, int32_t expert, int32_t matrix);

/* ---------------- follow-up hops (NCCL over NVLink) ----------------------- */

/* A communicator for hop traffic (NCCL 2.28, dlopen'ed from nccl_path; NULL =
 * "libnccl.so.2").  Rank 0 creates the 128-byte unique id, the host
 * distributes it (torch.distributed), every rank calls coe_comm_create. */
typedef struct coe_comm coe_comm;
int coe_comm_unique_id(const char *nccl_path, void *out128);
int coe_comm_create(const char *nccl_path, int rank, int world, const void *id128, coe_comm **out);
void coe_comm_destroy(coe_comm *c);
/* In-process transport for several runtimes on one device (one host thread each;
 * synchronise all runtimes and reset the hub between steps). */
typedef struct coe_local_hub coe_local_hub;
coe_local_hub *coe_local_hub_create(int world);
void coe_local_hub_destroy(coe_local_hub *hub);
void coe_local_hub_reset(coe_local_hub *hub);
int coe_comm_create_local(coe_local_hub *hub, int rank, coe_comm **out);
/* K4 on its own: one expert's bytes (or one W1 / W2 half), pinned host -> its HBM slot, on
 * the caller's copy-engine stream; done_event (may be NULL) is recorded after the copy.
 * Replaces CostModel.load_latency_from as charged by Simulation._start_load
 * (costmodel.py:69-73, engine.py:643-677); coe_runtime_step issues these itself. */
int coe_swap_in(void *dst_slot, const void *src_pinned, int64_t bytes, cudaStream_t copy_stream,
                cudaEvent_t done_event);
/* K5 on its own: all-to-all of follow-up activations with exact per-peer counts (bf16
 * elements): sendbuf / recvbuf hold world contiguous segments in rank order; the self
 * segment is a device copy, the rest one NCCL group of sends / receives (ring order) on
 * `stream`.  The follow-ups a batch_done epoch admits on other executors
 * (engine.py:751-753).  With an in-process hub communicator every rank calls it from its
 * own host thread.  coe_runtime_step fuses hops into K3 instead (peer mode) or groups its
 * own sends / receives per wave (NCCL mode). */
int coe_hop(coe_comm *comm, const void *sendbuf, const int64_t *send_counts, void *recvbuf,
            const int64_t *recv_counts, cudaStream_t stream);
/* Attach to a runtime (rank == the executor it serves); steps then exchange
 * hopped activations on a dedicated hop stream. */
int coe_runtime_attach_comm(coe_runtime *rt, coe_comm *comm);
/* (f3) Peer-GPU swap-in tier for executors of ONE process (one runtime each, stepped in
 * lockstep and synchronised between steps: runtime.step_executors).  A peer-tier LOAD of
 * expert e from executor j is copied from j's HBM (cudaMemcpyPeerAsync) when e was resident
 * on j when the previous step ended, is in j's initial placement and is not a victim of any
 * of j's LOADs in this plan -- so j never rewrites those bytes during the step; otherwise it
 * is served from the host tier (identical bytes, decisions unchanged).  peers[r] = the
 * runtime of executor r (world entries; peers[rank] is rt itself). */
int coe_runtime_attach_local_experts(coe_runtime *rt, coe_runtime *const *peers, int32_t world);
/* The same tier between PROCESSES (one executor per rank, CUDA IPC): export this runtime's
 * expert allocations (pooled slab, or one slab per shape; *count handles of 64 bytes), map a
 * peer rank's, and after every step hand each rank's end-of-step residency to the others
 * (per expert: slab << 40 | byte offset, -1 when not resident).  A qualifying peer-tier copy
 * waits for the source rank's step-end flag; a rank whose experts were read makes its next
 * step's copies wait for the readers' step end. */
int coe_runtime_ipc_export_experts(coe_runtime *rt, void *handles, int32_t *count);
int coe_runtime_ipc_open_experts(coe_runtime *rt, int32_t rank, const void *handles, int32_t count);
int coe_runtime_residency_codes(coe_runtime *rt, int64_t *codes /* [num_experts] */);
int coe_runtime_set_peer_residency(coe_runtime *rt, int32_t rank, const int64_t *codes);
/* scheduling knobs (see coe_runtime_config); reserve_sms < 0 keeps the current split */
int coe_runtime_set_knobs(coe_runtime *rt, int64_t wave_rows_cap, int64_t urgent_rows_cap, int32_t reserve_sms);

/* ---------------- seeded synthetic data ---------------------------------- */

/* Fill n bf16 values with the counter-based uniform generator shared with the
 * oracle (oracle/synth.py): value(i) = scale * (u(seed, i) - 0.5) * 2. */
int coe_fill_uniform_bf16(void *dst, int64_t n, uint64_t seed, float scale, cudaStream_t stream);
/* elements [start, start + n) of the same stream (e.g. one request's rows of the X buffer) */
int coe_fill_uniform_bf16_at(void *dst, int64_t start, int64_t n, uint64_t seed, float scale, cudaStream_t stream);

#ifdef __cplusplus
}
#endif

#endif /* COE_CUDA_H */
