/*
 * coe_planner.h -- C-ABI of the CoE serving planner (host, no CUDA).
 *
 * The planner is the *decide* half of the B200 serving path: it replays the
 * reference engine's admission -> step -> load -> batch -> follow-up cycle
 * (/root/reference/pkg/src/coesim/engine.py:588-758) on the float64 virtual
 * clock of the device document (costmodel.py:55-73) and emits
 *   - the reference trace (engine.py:555-565, event kinds in COE_EV_*),
 *   - the run metrics (engine.py:797-824),
 *   - a per-executor op log (LOAD / BATCH) that the GPU runtime executes,
 *   - one admission record per (request, stage) carrying the run-rank key
 *     that the GPU grouping kernel (coe_group_sort, coe_cuda.h) sorts by.
 *
 * Reference interfaces replaced (the drop-in seams of SURVEY.md §8b):
 *   coe_plan_run            <- engine.run(RunConfig)          engine.py:827-829
 *   policy fields           <- POLICIES / PolicySpec          engine.py:59-76
 *   assign / arrange        <- scheduler.assign, arrange_position   scheduler.py:72-108
 *   batch cap               <- scheduler.batch_cap            scheduler.py:111-118
 *   eviction                <- TwoStageEvictor.select / LruEvictor / FifoEvictor
 *                              expert_pool.py:96-148, baselines.py:20-73
 *   initial placement       <- initialize_pools               expert_pool.py:62-87
 *   host tier               <- _HostCache                     engine.py:289-330
 *
 * All pointers are host pointers owned by the caller for the duration of
 * coe_plan_create (the planner copies what it needs).  Every function returns
 * 0 on success or a COE_ERR_* code; coe_plan_last_error() gives the message.
 * Single-threaded, like the reference.
 */
#ifndef COE_PLANNER_H
#define COE_PLANNER_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  COE_OK = 0,
  COE_ERR_CONFIG = 2,      /* ConfigurationError (cli exit 2, cli.py:36-38) */
  COE_ERR_STARVATION = 3,  /* MemoryStarvationError (exit 3)               */
  COE_ERR_RUNTIME = 4,     /* RuntimeError: conservation (engine.py:783-795) */
  COE_ERR_VALUE = 5,       /* ValueError / KeyError from pool misuse       */
  COE_ERR_CUDA = 6         /* CUDA runtime failure (coe_cuda.h)            */
};

/* Trace event kinds, engine.py:555-565 */
enum {
  COE_EV_ARRIVAL = 0, COE_EV_ASSIGN = 1, COE_EV_EVICT = 2, COE_EV_LOAD = 3, COE_EV_LOAD_DONE = 4,
  COE_EV_BATCH_START = 5, COE_EV_BATCH_DONE = 6, COE_EV_FOLLOW_UP = 7, COE_EV_COMPLETE = 8
};

/* Op kinds of the physical op log */
enum { COE_OP_LOAD = 0, COE_OP_BATCH = 1 };

/* Tier ids (types.py:17); COE_TIER_PEER is the (f3) extension: an NVLink copy
 * from another GPU executor's HBM (RunConfig.peer_tier) */
enum { COE_TIER_DEVICE = 0, COE_TIER_HOST = 1, COE_TIER_SSD = 2, COE_TIER_PEER = 3 };

typedef struct coe_plan_config {
  /* experts, indexed densely in lexicographic order of their string ids so
   * integer tie-breaks equal the reference's string tie-breaks */
  int32_t num_experts;
  const int64_t *expert_bytes;      /* [E] param_bytes                        */
  const double *usage_prob;         /* [E]                                    */
  const int32_t *expert_arch;       /* [E] arch index                         */
  const int32_t *upstream_offsets;  /* [E+1] CSR of ExpertSpec.upstream       */
  const int32_t *upstream_index;    /* [nnz]                                  */
  const int32_t *desc_order;        /* [E] experts_by_descending_prob order   */

  /* per (arch, proc) tables, index = arch*2 + proc (proc 0 = gpu, 1 = cpu) */
  int32_t num_arches;
  const uint8_t *perf_valid;        /* PerfEntry present                      */
  const int32_t *perf_max_batch;
  const double *perf_k;
  const double *perf_b;
  const uint8_t *cost_valid;        /* ExecConstants present                  */
  const double *cost_k;
  const double *cost_b;
  const int64_t *cost_n_sat;
  const double *cost_gamma;
  const int64_t *cost_base_bytes;
  const int64_t *cost_per_item_bytes;

  /* memory tiers (costmodel.py:69-73) */
  int32_t numa;                     /* 1: numa (host tier exists), 0: uma    */
  double host_bw, host_overhead;
  double ssd_bw, ssd_overhead;
  int32_t host_mode;                /* -1 no host cache, 0 prob, 1 lru, 2 fifo */
  double host_cache_budget;

  /* executors, in engine.py:497-519 order */
  int32_t num_executors;
  const int32_t *exec_proc;
  const double *exec_expert_budget;
  const double *exec_inference_budget;
  const double *exec_k_scale;

  /* policy (engine.py:59-76) */
  int32_t assign_makespan;          /* 1 makespan, 0 round robin              */
  int32_t arrange;                  /* 1 arrange behind same-expert entries   */
  int32_t evict;                    /* 0 two_stage, 1 lru, 2 fifo             */

  /* requests in stream order; chains already resolved (routing.py:33-43) */
  int32_t num_requests;
  const int64_t *request_id;
  const double *arrival_s;
  const int32_t *chain_offsets;     /* [R+1]                                  */
  const int32_t *chain_experts;

  int32_t record_trace;             /* RunConfig.trace                        */
  int32_t record_ops;               /* emit op log + admission records        */

  /* (f3) peer-GPU swap-in tier (RunConfig.peer_tier): a load of an expert that
   * another GPU executor holds (and is not loading) copies it from that
   * executor at peer_bw / peer_overhead; the scheduler's switch-cost
   * predictions keep the reference's host/ssd tier (engine.py:583-586) */
  int32_t peer_enabled;
  double peer_bw, peer_overhead;
} coe_plan_config;

typedef struct coe_plan coe_plan;

typedef struct coe_plan_metrics {
  int64_t completed;
  int64_t follow_ups;               /* follow-ups completed                   */
  double makespan_s;                /* last completion time                   */
  int64_t evictions;
  int64_t stale_predictions;
  double sched_wall_s;
  int64_t sched_calls;
} coe_plan_metrics;

/* One op of the physical op log. */
typedef struct coe_op {
  int32_t executor;
  int32_t kind;        /* COE_OP_LOAD / COE_OP_BATCH                          */
  int32_t expert;
  int32_t count;       /* LOAD: #victims; BATCH: #members                    */
  int64_t offset;      /* into coe_plan_op_args (victims or member pairs)    */
  double time_s;       /* virtual start time                                  */
  int32_t tier;        /* LOAD: source tier                                   */
  int32_t seq;         /* BATCH: index of the batch within its executor;
                          LOAD: source executor for COE_TIER_PEER, else -1   */
} coe_op;

/* One admission (a request entering an executor queue for one stage). */
typedef struct coe_admission {
  int32_t executor;
  int32_t run_rank;    /* grouping key: run creation order within executor   */
  int32_t request;     /* request index in stream order                      */
  int32_t stage;       /* position in the request's chain                    */
} coe_admission;

int coe_plan_create(const coe_plan_config *cfg, coe_plan **out);
int coe_plan_run(coe_plan *plan);
void coe_plan_destroy(coe_plan *plan);
const char *coe_plan_last_error(void);

int coe_plan_metrics_get(const coe_plan *plan, coe_plan_metrics *out);
/* per executor: busy_s (float64) and switches (int64), [X] each */
int coe_plan_executor_stats(const coe_plan *plan, double *busy_s, int64_t *switches);

/* trace: parallel arrays of length n; executor/expert/request -1 == None */
int64_t coe_plan_trace_len(const coe_plan *plan);
int coe_plan_trace(const coe_plan *plan, double *time_s, int32_t *executor, int32_t *event,
                   int32_t *expert, int64_t *request_id);

/* initial residency (initialize_pools): expert per slot, per executor CSR */
int coe_plan_initial_residency(const coe_plan *plan, int32_t *offsets /*[X+1]*/, int32_t *experts /*[<=E*X]*/);

int64_t coe_plan_num_ops(const coe_plan *plan);
const coe_op *coe_plan_ops(const coe_plan *plan);
int64_t coe_plan_num_op_args(const coe_plan *plan);
const int32_t *coe_plan_op_args(const coe_plan *plan);   /* victims: expert ids; batch: (request, stage) pairs */
int64_t coe_plan_num_admissions(const coe_plan *plan);
const coe_admission *coe_plan_admissions(const coe_plan *plan);

/* Cross-executor follow-up hops in global (admission) order: the output of
 * `stage` of `request` moves src -> dst (engine.py:751-753 admits the
 * follow-up on another executor).  Returns the hop count; fills at most
 * `capacity` entries.  Requires record_ops. */
int64_t coe_plan_hops(const coe_plan *plan, int64_t capacity, int64_t *index, int32_t *src, int32_t *dst,
                      int32_t *request, int32_t *stage);

#ifdef __cplusplus
}
#endif

#endif /* COE_PLANNER_H */
