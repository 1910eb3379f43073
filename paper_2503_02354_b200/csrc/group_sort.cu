// group_sort.cu -- K1 (segmented stable radix sort by run-rank) and K2 (run /
// batch compaction), plus the seeded synthetic-data fill shared with the oracle.
//
// K1 replaces the reference's per-admission arrange_position backward scan +
// list.insert (scheduler.py:100-108, engine.py:251-254): an executor's queue
// is always the stable sort of its admissions by (run_rank, admission seq)
// (SURVEY.md §0.3), so sorting every admission of a step by the 32-bit key
// executor << rank_bits | run_rank (input already in admission order, LSD
// radix is stable) yields each executor's execution order in one pass over HBM.
// K2 replaces head_run / batch_cap / split_batch (engine.py:270-283,
// scheduler.py:111-137): batches are consecutive slices of that order; K2
// finds their offsets, gathers (request, stage) members for the grouped MLP,
// counts runs and flags any batch that would straddle two runs.
//
// Layout: SoA int32 arrays; 4096-key tiles (256 threads x 16; 1024-key tiles up to 1M keys).
// One read of (executor, run_rank) counts every pass's digits; then ONE kernel per 8-bit
// pass: a stable in-shared-memory ranking of each tile (warp match_any), the tile's
// per-digit offsets by decoupled look-back over its predecessors, and a coalesced
// digit-segment write-out.  The first pass builds the keys on the fly.  HBM-bound integer
// work at scale (8 B for the counting read + 16 B moved per key per pass); launch-latency-
// bound at serving size (a memset + 1 + passes launches).

#include <algorithm>
#include <cstdint>
#include <string>

#include <cuda_bf16.h>
#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "coe_cuda.h"
#include "common.cuh"

namespace {

constexpr int SORT_THREADS = 256;
// keys per thread per tile: 16 (4096-key tiles) at scale -- fewer, larger tiles shorten the
// look-back chains (measured at 16.8M keys: 2048-key tiles 16 % slower, 1024-key tiles 74 %) --
// and 4 (1024-key tiles) for serving-size steps, where more CTAs help
constexpr int ITEMS_LARGE = 16, ITEMS_SMALL = 4;
constexpr int64_t SMALL_SORT_MAX = 1 << 20;
constexpr int RADIX = 256;
constexpr int SORT_WARPS = SORT_THREADS / 32;

constexpr int MAX_PASSES = 4;
// decoupled look-back words: bits 31:30 = status (0 not ready, 1 tile aggregate, 2 inclusive
// prefix), bits 29:0 = count (n < 2^30)
constexpr uint32_t LB_AGG = 1u << 30, LB_INC = 2u << 30, LB_VAL = LB_AGG - 1u;

__device__ __forceinline__ uint32_t sort_key(const int32_t *exec, const int32_t *rank, int64_t i, int rank_bits) {
  return ((uint32_t)exec[i] << rank_bits) | (uint32_t)rank[i];
}

// Step 0: the global digit counts of EVERY pass in one read of (executor, run_rank) -- a
// digit's total does not depend on the order the keys are in.  Block-private shared
// histograms; each thread counts ITEMS consecutive keys and adds a digit's count once per run
// of equal digits (serving keys are nearly sorted: a thread's keys share their high digits),
// and a warp whose 32 x ITEMS keys all share one digit adds it with a single atomic.  Random
// keys cost one shared atomic per key and pass, with no warp-wide match (ncu, 16.8 M uniform
// 22-bit keys: 336 us with a match_any per key and pass, profiles/r2n7_*).
template <int ITEMS>
__global__ void __launch_bounds__(SORT_THREADS) radix_global_hist(const int32_t *exec, const int32_t *rank, int64_t n,
                                                                  int rank_bits, int num_passes, uint32_t *ghist) {
  constexpr int TILE = SORT_THREADS * ITEMS;
  __shared__ uint32_t h[MAX_PASSES][RADIX];
  for (int j = threadIdx.x; j < MAX_PASSES * RADIX; j += SORT_THREADS) (&h[0][0])[j] = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t stride = (int64_t)gridDim.x * TILE;
  uint32_t cur[ITEMS], nxt[ITEMS];
  auto load = [&](uint32_t *k, int64_t base) {
    const int64_t b = base + (int64_t)threadIdx.x * ITEMS;
#pragma unroll
    for (int r = 0; r < ITEMS; ++r) k[r] = b + r < n ? sort_key(exec, rank, b + r, rank_bits) : 0u;
  };
  int64_t base = (int64_t)blockIdx.x * TILE;
  if (base < n) load(cur, base);
  for (; base < n; base += stride) {  // uniform across the block
    if (base + stride < n) load(nxt, base + stride);  // next tile in flight while this one counts
    const int64_t b = base + (int64_t)threadIdx.x * ITEMS;
    const int nv = (int)(n - b >= ITEMS ? ITEMS : (n - b > 0 ? n - b : 0));  // valid keys of this thread
    for (int p = 0; p < num_passes; ++p) {
      const int sh = 8 * p;
      const uint32_t first = (cur[0] >> sh) & 255u;
      bool same = nv == ITEMS;
#pragma unroll
      for (int r = 1; r < ITEMS; ++r) same = same && ((cur[r] >> sh) & 255u) == first;
      const uint32_t lane0 = __shfl_sync(0xffffffffu, first, 0);  // every lane: no short-circuit around it
      if (__all_sync(0xffffffffu, same && first == lane0)) {
        if (lane == 0) atomicAdd(&h[p][first], 32u * ITEMS);
        continue;
      }
      uint32_t run = first, cnt = 0;
#pragma unroll
      for (int r = 0; r < ITEMS; ++r) {
        if (r < nv) {
          const uint32_t d = (cur[r] >> sh) & 255u;
          if (d != run) {
            atomicAdd(&h[p][run], cnt);
            run = d;
            cnt = 0;
          }
          ++cnt;
        }
      }
      if (cnt) atomicAdd(&h[p][run], cnt);
    }
#pragma unroll
    for (int r = 0; r < ITEMS; ++r) cur[r] = nxt[r];
  }
  __syncthreads();
  for (int j = threadIdx.x; j < num_passes * RADIX; j += SORT_THREADS) {
    const uint32_t c = (&h[0][0])[j];
    if (c) atomicAdd(&ghist[j], c);
  }
}

// One 8-bit pass, one kernel (single-pass "onesweep" scheme): tiles are numbered in the
// order their CTAs start (atomic counter), so a tile only ever waits on tiles that are
// already running.  Each CTA ranks its tile stably by digit in shared memory -- every warp
// walks its own contiguous chunk 32 keys at a time (match_any ranks + warp-private digit
// counters) -- publishes its per-digit counts, resolves its exclusive per-digit prefix by
// decoupled look-back over the preceding tiles' published aggregates / inclusive prefixes,
// then writes the locally sorted tile out so consecutive threads store consecutive
// addresses of a digit's output segment (coalesced).  The first pass builds the keys from
// (executor, run_rank) on the fly and its values are the admission indices.
// Exclusive scan of one value per thread over the 256-thread block: warp shuffles, then the
// eight warp totals (two barriers instead of a 16-barrier Hillis-Steele scan).
__device__ __forceinline__ uint32_t block_exclusive_scan256(uint32_t v, uint32_t *warp_tot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, off);
    if (lane >= off) x += y;
  }
  if (lane == 31) warp_tot[warp] = x;
  __syncthreads();
  uint32_t base = 0;
#pragma unroll
  for (int w = 0; w < SORT_WARPS; ++w) base += w < warp ? warp_tot[w] : 0u;
  return base + x - v;
}

// One 8-bit pass, one persistent kernel (single-pass "onesweep" scheme): each CTA claims
// tiles in order from an atomic counter, so a tile only ever waits on tiles that running
// CTAs already hold.  Each CTA ranks its tile stably by digit in shared memory -- every warp
// walks its own contiguous chunk 32 keys at a time (match_any ranks + warp-private digit
// counters) -- publishes its per-digit counts, resolves its exclusive per-digit prefix by
// decoupled look-back over the preceding tiles' published aggregates / inclusive prefixes,
// then writes the locally sorted tile out so consecutive threads store consecutive
// addresses of a digit's output segment (coalesced).  The digit bases (scan of the global
// counts) are computed once per CTA.  The first pass builds the keys from
// (executor, run_rank) on the fly and its values are the admission indices.
template <int ITEMS, bool FIRST>
__global__ void __launch_bounds__(SORT_THREADS, ITEMS >= 16 ? 3 : 6)
    onesweep_pass(const uint32_t *keys_in, const int32_t *vals_in, const int32_t *exec, const int32_t *rank,
                  int rank_bits, uint32_t *keys_out, int32_t *vals_out, const uint32_t *ghist, uint32_t *lookback,
                  uint32_t *tile_counter, int64_t n, int num_tiles, int shift) {
  constexpr int TILE = SORT_THREADS * ITEMS;
  constexpr int CHUNK = 32 * ITEMS;  // keys per warp
  __shared__ uint32_t sk[TILE];
  __shared__ int32_t sv[TILE];
  __shared__ uint32_t wcnt[SORT_WARPS][RADIX];  // per-warp digit counts, then per-warp tile offsets
  __shared__ uint32_t out_shift[RADIX];         // global start - tile-local start, per digit
  __shared__ uint32_t warp_tot[2][SORT_WARPS];
  __shared__ int tile_sh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t digit_base = block_exclusive_scan256(ghist[tid], warp_tot[0]);  // thread = digit
  const uint32_t lt_mask = (1u << lane) - 1u;
  volatile uint32_t *lb = lookback;
  for (;;) {
    if (tid == 0) tile_sh = (int)atomicAdd(tile_counter, 1u);
    for (int j = tid; j < SORT_WARPS * RADIX; j += SORT_THREADS) (&wcnt[0][0])[j] = 0;
    __syncthreads();  // also: the previous tile's write-out is done with sk / sv / out_shift
    const int tile = tile_sh;
    if (tile >= num_tiles) break;
    const int64_t base = (int64_t)tile * TILE;
    const int tile_n = (int)((n - base) < TILE ? (n - base) : TILE);
    uint32_t key[ITEMS], rnk[ITEMS];
    int32_t val[ITEMS];
#pragma unroll
    for (int r = 0; r < ITEMS; ++r) {  // all loads first: independent requests in flight
      const int i = warp * CHUNK + r * 32 + lane;
      if constexpr (FIRST) {
        key[r] = i < tile_n ? sort_key(exec, rank, base + i, rank_bits) : 0u;
        val[r] = (int32_t)(base + i);
      } else {
        key[r] = i < tile_n ? keys_in[base + i] : 0u;
        val[r] = i < tile_n ? vals_in[base + i] : 0;
      }
    }
    // warp walk: warp-local stable ranks
#pragma unroll
    for (int r = 0; r < ITEMS; ++r) {
      const int i = warp * CHUNK + r * 32 + lane;
      const bool valid = i < tile_n;
      const uint32_t digit = valid ? ((key[r] >> shift) & 255u) : 256u;
      const uint32_t same = __match_any_sync(0xffffffffu, digit);
      const uint32_t before = __popc(same & lt_mask);
      rnk[r] = valid ? wcnt[warp][digit] + before : 0u;
      __syncwarp();
      if (valid && before == 0) wcnt[warp][digit] += __popc(same);
      __syncwarp();
    }
    __syncthreads();
    // thread = digit: this tile's count, published at once; then the look-back
    uint32_t total = 0;
#pragma unroll
    for (int w = 0; w < SORT_WARPS; ++w) total += wcnt[w][tid];
    uint32_t prefix = 0;
    if (tile == 0) {
      lb[tid] = LB_INC | total;
    } else {
      lb[(int64_t)tile * RADIX + tid] = LB_AGG | total;
      for (int j = tile - 1;;) {
        const uint32_t v = lb[(int64_t)j * RADIX + tid];
        if ((v & (LB_AGG | LB_INC)) == 0) continue;  // predecessor still ranking: spin
        prefix += v & LB_VAL;
        if (v & LB_INC) break;
        --j;
      }
      lb[(int64_t)tile * RADIX + tid] = LB_INC | (prefix + total);
    }
    // tile-local digit starts, then per-(warp, digit) offsets
    uint32_t run = block_exclusive_scan256(total, warp_tot[1]);
    out_shift[tid] = digit_base + prefix - run;  // mod 2^32
#pragma unroll
    for (int w = 0; w < SORT_WARPS; ++w) {
      const uint32_t c = wcnt[w][tid];
      wcnt[w][tid] = run;
      run += c;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < ITEMS; ++r) {
      const int i = warp * CHUNK + r * 32 + lane;
      if (i < tile_n) {
        const uint32_t pos = wcnt[warp][(key[r] >> shift) & 255u] + rnk[r];
        sk[pos] = key[r];
        sv[pos] = val[r];
      }
    }
    __syncthreads();
    for (int k = tid; k < tile_n; k += SORT_THREADS) {
      const uint32_t kk = sk[k];
      const uint32_t g = out_shift[(kk >> shift) & 255u] + (uint32_t)k;
      keys_out[g] = kk;
      vals_out[g] = sv[k];
    }
  }
}

// K2 part 1: gather members, mark run starts / executor segment starts.  Each thread handles
// GATHER_ITEMS admissions (block-strided, so every load instruction stays coalesced) and issues
// all their perm / key loads before the dependent member gathers: several independent chains in
// flight per thread (one per thread left it latency-bound at ~2.6 TB/s, profiles/r2n9_*).
constexpr int GATHER_ITEMS = 4;

__global__ void __launch_bounds__(256) compact_gather(const int32_t *perm, const uint32_t *keys, const int32_t *adm_req,
                               const int32_t *adm_stage, const int32_t *adm_in, const int32_t *adm_out, int64_t n,
                               int rank_bits, int32_t *member_req, int32_t *member_stage, int32_t *member_in,
                               int32_t *member_out, int32_t *seg_start, int32_t *run_count) {
  const int64_t base = (int64_t)blockIdx.x * (blockDim.x * GATHER_ITEMS) + threadIdx.x;
  int32_t p[GATHER_ITEMS];
  uint32_t k[GATHER_ITEMS], kp[GATHER_ITEMS];
#pragma unroll
  for (int j = 0; j < GATHER_ITEMS; ++j) {
    const int64_t i = base + (int64_t)j * blockDim.x;
    if (i < n) {
      p[j] = perm[i];
      k[j] = keys[i];
      kp[j] = i > 0 ? keys[i - 1] : ~k[j];
    }
  }
  int starts = 0;
#pragma unroll
  for (int j = 0; j < GATHER_ITEMS; ++j) {
    const int64_t i = base + (int64_t)j * blockDim.x;
    if (i < n) {
      member_req[i] = adm_req[p[j]];
      member_stage[i] = adm_stage[p[j]];
      if (adm_in) {  // activation-row routes (coe_run_compact_routes)
        member_in[i] = adm_in[p[j]];
        member_out[i] = adm_out[p[j]];
      }
      if (i == 0 || kp[j] != k[j]) ++starts;
      if (i == 0 || (kp[j] >> rank_bits) != (k[j] >> rank_bits)) seg_start[k[j] >> rank_bits] = (int32_t)i;
    }
  }
  // block-reduce the run starts into one atomic
  for (int off = 16; off; off >>= 1) starts += __shfl_down_sync(0xffffffffu, starts, off);
  __shared__ int warp_sum[32];
  if ((threadIdx.x & 31) == 0) warp_sum[threadIdx.x >> 5] = starts;
  __syncthreads();
  if (threadIdx.x == 0) {
    int sum = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) sum += warp_sum[w];
    if (sum) atomicAdd(run_count, sum);
  }
}

// K2 part 2: batch offsets = executor segment start + exclusive scan of that executor's
// batch sizes in op order; three kernels so it scales with the batch count: per-block sums
// per executor, a scan of those sums, then per-block scans + offsets + the one-run check.
constexpr int BATCH_THREADS = 1024;

__device__ __forceinline__ int block_exclusive_scan(int v, int *warp_sums, int &total) {
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  int x = v;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    const int y = __shfl_up_sync(0xffffffffu, x, off);
    if (lane >= off) x += y;
  }
  if (lane == 31) warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    int w = warp_sums[lane];
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, w, off);
      if (lane >= off) w += y;
    }
    warp_sums[lane] = w;
  }
  __syncthreads();
  const int incl = x + (warp ? warp_sums[warp - 1] : 0);
  total = warp_sums[31];
  __syncthreads();
  return incl - v;
}

// Each thread owns BATCH_ITEMS consecutive batches (loads of several batches in flight per
// thread; the block's scan runs over the per-thread sums).
constexpr int BATCH_ITEMS = 4;
constexpr int BATCH_PER_BLOCK = BATCH_THREADS * BATCH_ITEMS;

__global__ void __launch_bounds__(BATCH_THREADS) batch_block_sums(const int32_t *batch_exec, const int32_t *batch_size,
                                                                  int num_batches, int num_executors,
                                                                  int32_t *block_sums) {
  __shared__ int warp_sums[32];
  const int b0 = blockIdx.x * BATCH_PER_BLOCK + threadIdx.x * BATCH_ITEMS;
  int x[BATCH_ITEMS], v[BATCH_ITEMS];
#pragma unroll
  for (int j = 0; j < BATCH_ITEMS; ++j) {
    x[j] = b0 + j < num_batches ? batch_exec[b0 + j] : -1;
    v[j] = b0 + j < num_batches ? batch_size[b0 + j] : 0;
  }
  for (int e = 0; e < num_executors; ++e) {
    int sum = 0, total;
#pragma unroll
    for (int j = 0; j < BATCH_ITEMS; ++j) sum += x[j] == e ? v[j] : 0;
    block_exclusive_scan(sum, warp_sums, total);
    if (threadIdx.x == 0) block_sums[(int64_t)blockIdx.x * num_executors + e] = total;
  }
}

__global__ void __launch_bounds__(BATCH_THREADS) scan_block_sums(int32_t *block_sums, int num_blocks,
                                                                 int num_executors) {
  __shared__ int warp_sums[32];
  __shared__ int carry;
  for (int e = 0; e < num_executors; ++e) {
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < num_blocks; base += BATCH_THREADS) {
      const int i = base + threadIdx.x;
      const int v = i < num_blocks ? block_sums[(int64_t)i * num_executors + e] : 0;
      int total;
      const int ex = block_exclusive_scan(v, warp_sums, total);
      if (i < num_blocks) block_sums[(int64_t)i * num_executors + e] = carry + ex;
      __syncthreads();
      if (threadIdx.x == 0) carry += total;
      __syncthreads();
    }
  }
}

__global__ void __launch_bounds__(BATCH_THREADS) compact_batches(const int32_t *batch_exec, const int32_t *batch_size,
                                                                 int num_batches, int num_executors,
                                                                 const int32_t *seg_start, const int32_t *block_sums,
                                                                 const uint32_t *keys, int64_t n, int rank_bits,
                                                                 int32_t *batch_off, int32_t *violations) {
  __shared__ int warp_sums[32];
  const int b0 = blockIdx.x * BATCH_PER_BLOCK + threadIdx.x * BATCH_ITEMS;
  int x[BATCH_ITEMS], v[BATCH_ITEMS], mine[BATCH_ITEMS];
#pragma unroll
  for (int j = 0; j < BATCH_ITEMS; ++j) {
    x[j] = b0 + j < num_batches ? batch_exec[b0 + j] : -1;
    v[j] = b0 + j < num_batches ? batch_size[b0 + j] : 0;
    mine[j] = 0;
  }
  for (int e = 0; e < num_executors; ++e) {
    int sum = 0, total;
#pragma unroll
    for (int j = 0; j < BATCH_ITEMS; ++j) sum += x[j] == e ? v[j] : 0;
    int run = block_exclusive_scan(sum, warp_sums, total);
    const int base = seg_start[e] + block_sums[(int64_t)blockIdx.x * num_executors + e];
#pragma unroll
    for (int j = 0; j < BATCH_ITEMS; ++j)
      if (x[j] == e) {
        mine[j] = base + run;
        run += v[j];
      }
  }
  int bad_count = 0;
#pragma unroll
  for (int j = 0; j < BATCH_ITEMS; ++j) {
    if (b0 + j < num_batches) {
      batch_off[b0 + j] = mine[j];
      const int64_t lo = mine[j], hi = lo + v[j] - 1;
      const bool bad = v[j] <= 0 || lo < 0 || hi >= n || keys[lo] != keys[hi] || (int)(keys[lo] >> rank_bits) != x[j];
      bad_count += bad ? 1 : 0;
    }
  }
  if (bad_count) atomicAdd(violations, bad_count);
}

// K1 + K2 fused for one executor's step at serving size (<= 32,768 admissions, <= 4,096
// batches): ONE block of 1,024 threads sorts (run_rank << idx_bits | admission) -- unique keys,
// so the order is the stable sort by run-rank -- in shared memory, gathers the members and
// their row routes, scans the batch sizes into offsets and checks the one-run-per-batch
// contract.  One launch instead of the counting pass, the radix passes, three memsets and the
// compaction kernels, which at this size are pure launch latency.
constexpr int FUSED_THREADS = 1024;
constexpr int FUSED_BATCH_IPT = 4;

template <int IPT>
__global__ void __launch_bounds__(FUSED_THREADS, 1)
    group_compact_block(const int32_t *run_rank, const int32_t *adm_req, const int32_t *adm_stage,
                        const int32_t *adm_in, const int32_t *adm_out, int n, int rank_bits, int idx_bits,
                        const int32_t *batch_size, int num_batches, int32_t *out_perm, int32_t *batch_off,
                        int32_t *member_req, int32_t *member_stage, int32_t *member_in, int32_t *member_out,
                        int32_t *flags) {
  using Sort = cub::BlockRadixSort<uint32_t, FUSED_THREADS, IPT>;
  using Reduce = cub::BlockReduce<int, FUSED_THREADS>;
  using Scan = cub::BlockScan<int, FUSED_THREADS>;
  extern __shared__ __align__(16) uint8_t fused_smem[];
  __shared__ typename Reduce::TempStorage red;
  __shared__ typename Scan::TempStorage scan;
  const int t = threadIdx.x;
  const uint32_t idx_mask = (1u << idx_bits) - 1u;
  const uint32_t pad = 1u << (rank_bits + idx_bits);  // sorts after every admission
  uint32_t keys[IPT];
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    const int i = t * IPT + k;
    keys[k] = i < n ? ((uint32_t)run_rank[i] << idx_bits) | (uint32_t)i : pad;
  }
  Sort(*reinterpret_cast<typename Sort::TempStorage *>(fused_smem)).Sort(keys, 0, rank_bits + idx_bits + 1);
  __syncthreads();  // the sort's storage now holds the sorted ranks
  int32_t *s_rank = reinterpret_cast<int32_t *>(fused_smem);
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    const int pos = t * IPT + k;
    if (pos < n) {
      const int32_t i = (int32_t)(keys[k] & idx_mask);
      s_rank[pos] = (int32_t)(keys[k] >> idx_bits);
      out_perm[pos] = i;
      member_req[pos] = adm_req[i];
      member_stage[pos] = adm_stage[i];
      if (adm_in) {
        member_in[pos] = adm_in[i];
        member_out[pos] = adm_out[i];
      }
    }
  }
  __syncthreads();
  int starts = 0;
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    const int pos = t * IPT + k;
    if (pos < n && (pos == 0 || s_rank[pos - 1] != s_rank[pos])) ++starts;
  }
  const int runs = Reduce(red).Sum(starts);
  int sizes[FUSED_BATCH_IPT], offs[FUSED_BATCH_IPT];
#pragma unroll
  for (int k = 0; k < FUSED_BATCH_IPT; ++k) {
    const int b = t * FUSED_BATCH_IPT + k;
    sizes[k] = b < num_batches ? batch_size[b] : 0;
  }
  Scan(scan).ExclusiveSum(sizes, offs);
  int bad = 0;
#pragma unroll
  for (int k = 0; k < FUSED_BATCH_IPT; ++k) {
    const int b = t * FUSED_BATCH_IPT + k;
    if (b < num_batches) {
      batch_off[b] = offs[k];
      const int lo = offs[k], hi = lo + sizes[k] - 1;
      bad += (sizes[k] <= 0 || hi >= n || s_rank[lo] != s_rank[hi]) ? 1 : 0;
    }
  }
  __syncthreads();
  const int violations = Reduce(red).Sum(bad);
  if (t == 0) {
    flags[0] = runs;
    flags[1] = violations;
  }
}

template <int IPT>
bool launch_fused(const int32_t *run_rank, const int32_t *adm_req, const int32_t *adm_stage, const int32_t *adm_in,
                  const int32_t *adm_out, int n, int rank_bits, int idx_bits, const int32_t *batch_size,
                  int num_batches, int32_t *out_perm, int32_t *out_batch_off, int32_t *member_req,
                  int32_t *member_stage, int32_t *member_in, int32_t *member_out, int32_t *flags,
                  cudaStream_t stream) {
  using Sort = cub::BlockRadixSort<uint32_t, FUSED_THREADS, IPT>;
  constexpr size_t smem = sizeof(typename Sort::TempStorage) > (size_t)FUSED_THREADS * IPT * 4
                              ? sizeof(typename Sort::TempStorage)
                              : (size_t)FUSED_THREADS * IPT * 4;
  static const bool configured =
      cudaFuncSetAttribute(group_compact_block<IPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) ==
      cudaSuccess;
  if (!configured) return false;
  group_compact_block<IPT><<<1, FUSED_THREADS, smem, stream>>>(run_rank, adm_req, adm_stage, adm_in, adm_out, n,
                                                                rank_bits, idx_bits, batch_size, num_batches, out_perm,
                                                                out_batch_off, member_req, member_stage, member_in,
                                                                member_out, flags);
  return coe_cuda_ok(cudaGetLastError(), "group_compact_block");
}

// counter-based uniform generator (splitmix64), mirrored in oracle/synth.py
__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void fill_uniform_bf16(__nv_bfloat16_raw *dst, int64_t start, int64_t n, uint64_t seed, float two_scale) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = splitmix64(seed + (uint64_t)(start + i + 1) * 0x9E3779B97F4A7C15ull);
    float u = __uint2float_rn((uint32_t)(z >> 40)) * (1.0f / 16777216.0f);
    float v = __fmul_rn(__fsub_rn(u, 0.5f), two_scale);
    uint32_t bits = __float_as_uint(v);
    bits += 0x7FFFu + ((bits >> 16) & 1u);  // round to nearest even
    __nv_bfloat16_raw r;
    r.x = (unsigned short)(bits >> 16);
    dst[i] = r;
  }
}

bool check(cudaError_t e, const char *what) { return coe_cuda_ok(e, what); }

// Persistent grid of one pass kernel: every SM slot it can occupy (queried once per
// instantiation), with a max shared-memory carve-out so registers bound occupancy.
template <int ITEMS, bool FIRST>
void launch_pass(const uint32_t *ki, const int32_t *vi, const int32_t *executor, const int32_t *run_rank,
                 int rank_bits, uint32_t *ko, int32_t *vo, const uint32_t *gh, uint32_t *lb, uint32_t *counter,
                 int64_t n, int num_tiles, int shift, cudaStream_t stream) {
  static const int resident = [] {
    auto kernel = onesweep_pass<ITEMS, FIRST>;
    cudaFuncSetAttribute(kernel, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    int per_sm = 0, sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, SORT_THREADS, 0);
    return std::max(1, sms * std::max(per_sm, 1));
  }();
  onesweep_pass<ITEMS, FIRST><<<std::min(num_tiles, resident), SORT_THREADS, 0, stream>>>(
      ki, vi, executor, run_rank, rank_bits, ko, vo, gh, lb, counter, n, num_tiles, shift);
}

}  // namespace

extern "C" {

int64_t coe_group_sort_scratch_bytes(int64_t n) {
  const int64_t tile = SORT_THREADS * (int64_t)ITEMS_SMALL;  // the smallest tile bounds the tile count
  int64_t tiles = (n + tile - 1) / tile;
  if (tiles < 1) tiles = 1;
  // ping-pong keys / values + per-pass look-back words + global digit counts + tile counters
  return 4 * 4 * (n + 16) + 4 * (int64_t)MAX_PASSES * RADIX * tiles + 4 * MAX_PASSES * RADIX + 64 + 1024;
}

int coe_group_sort(const int32_t *executor, const int32_t *run_rank, int64_t n, int rank_bits, int num_passes,
                   int32_t *out_perm, int32_t *out_keys, void *scratch, cudaStream_t stream) {
  if (n <= 0) return COE_CUDA_OK;
  if (num_passes < 1 || num_passes > MAX_PASSES || rank_bits < 1 || rank_bits > 31 || n >= (int64_t)LB_AGG) {
    coe_set_error("coe_group_sort: bad pass count / rank bits / size");
    return COE_CUDA_ERR_CONFIG;
  }
  const bool small = n <= SMALL_SORT_MAX;
  const int64_t tile = SORT_THREADS * (int64_t)(small ? ITEMS_SMALL : ITEMS_LARGE);
  const int num_tiles = (int)((n + tile - 1) / tile);
  char *s = static_cast<char *>(scratch);
  uint32_t *ka = reinterpret_cast<uint32_t *>(s);
  uint32_t *kb = ka + n + 16;
  int32_t *va = reinterpret_cast<int32_t *>(kb + n + 16);
  int32_t *vb = va + n + 16;
  // zeroed together: look-back words of every pass, global digit counts, tile counters
  uint32_t *lookback = reinterpret_cast<uint32_t *>(vb + n + 16);
  uint32_t *ghist = lookback + (int64_t)num_passes * RADIX * num_tiles;
  uint32_t *counters = ghist + MAX_PASSES * RADIX;
  const size_t zero_bytes = 4 * ((size_t)num_passes * RADIX * num_tiles + MAX_PASSES * RADIX + 16);
  if (!check(cudaMemsetAsync(lookback, 0, zero_bytes, stream), "coe_group_sort memset")) return COE_CUDA_ERR_CUDA;
  const int hist_grid = std::min(num_tiles, 148 * 8);
  if (small)
    radix_global_hist<ITEMS_SMALL><<<hist_grid, SORT_THREADS, 0, stream>>>(executor, run_rank, n, rank_bits,
                                                                            num_passes, ghist);
  else
    radix_global_hist<ITEMS_LARGE / 2><<<hist_grid, SORT_THREADS, 0, stream>>>(executor, run_rank, n, rank_bits,
                                                                                num_passes, ghist);
  const uint32_t *ki = nullptr;
  const int32_t *vi = nullptr;
  for (int p = 0; p < num_passes; ++p) {
    // the last pass scatters straight into the caller's arrays
    uint32_t *ko = p == num_passes - 1 ? reinterpret_cast<uint32_t *>(out_keys) : (p & 1 ? ka : kb);
    int32_t *vo = p == num_passes - 1 ? out_perm : (p & 1 ? va : vb);
    uint32_t *lb = lookback + (int64_t)p * RADIX * num_tiles;
    const uint32_t *gh = ghist + p * RADIX;
    if (small) p == 0 ? launch_pass<ITEMS_SMALL, true>(ki, vi, executor, run_rank, rank_bits, ko, vo, gh, lb,
                                                        counters + p, n, num_tiles, 8 * p, stream)
                      : launch_pass<ITEMS_SMALL, false>(ki, vi, executor, run_rank, rank_bits, ko, vo, gh, lb,
                                                         counters + p, n, num_tiles, 8 * p, stream);
    else p == 0 ? launch_pass<ITEMS_LARGE, true>(ki, vi, executor, run_rank, rank_bits, ko, vo, gh, lb, counters + p,
                                                 n, num_tiles, 8 * p, stream)
                : launch_pass<ITEMS_LARGE, false>(ki, vi, executor, run_rank, rank_bits, ko, vo, gh, lb, counters + p,
                                                  n, num_tiles, 8 * p, stream);
    ki = ko;
    vi = vo;
  }
  return check(cudaGetLastError(), "coe_group_sort") ? COE_CUDA_OK : COE_CUDA_ERR_CUDA;
}

int64_t coe_run_compact_scratch_bytes(int64_t n, int num_batches, int num_executors) {
  (void)n;
  const int64_t blocks = (num_batches + BATCH_PER_BLOCK - 1) / BATCH_PER_BLOCK;
  return 4 * ((int64_t)num_executors + 16) + 4 * (blocks + 1) * num_executors;
}

int coe_run_compact(const int32_t *perm, const int32_t *sorted_keys, const int32_t *adm_request,
                    const int32_t *adm_stage, int64_t n, int rank_bits, const int32_t *batch_exec,
                    const int32_t *batch_size, int num_batches, int num_executors, int32_t *out_batch_off,
                    int32_t *out_member_req, int32_t *out_member_stage, int32_t *out_run_count,
                    int32_t *out_violations, void *scratch, cudaStream_t stream) {
  return coe_run_compact_routes(perm, sorted_keys, adm_request, adm_stage, nullptr, nullptr, n, rank_bits, batch_exec,
                                batch_size, num_batches, num_executors, out_batch_off, out_member_req,
                                out_member_stage, nullptr, nullptr, out_run_count, out_violations, scratch, stream);
}

int coe_run_compact_routes(const int32_t *perm, const int32_t *sorted_keys, const int32_t *adm_request,
                           const int32_t *adm_stage, const int32_t *adm_in, const int32_t *adm_out, int64_t n,
                           int rank_bits, const int32_t *batch_exec, const int32_t *batch_size, int num_batches,
                           int num_executors, int32_t *out_batch_off, int32_t *out_member_req,
                           int32_t *out_member_stage, int32_t *out_member_in, int32_t *out_member_out,
                           int32_t *out_run_count, int32_t *out_violations, void *scratch, cudaStream_t stream) {
  if ((adm_in == nullptr) != (adm_out == nullptr) || (adm_in && (!out_member_in || !out_member_out))) {
    coe_set_error("coe_run_compact_routes: route arrays must be given in / out together");
    return COE_CUDA_ERR_CONFIG;
  }
  int32_t *seg_start = static_cast<int32_t *>(scratch);
  int32_t *block_sums = seg_start + num_executors + 16;
  if (!check(cudaMemsetAsync(seg_start, 0, 4 * (size_t)num_executors, stream), "compact memset") ||
      !check(cudaMemsetAsync(out_run_count, 0, 4, stream), "compact memset") ||
      !check(cudaMemsetAsync(out_violations, 0, 4, stream), "compact memset"))
    return COE_CUDA_ERR_CUDA;
  if (n > 0) {
    const int blocks = (int)((n + 256 * GATHER_ITEMS - 1) / (256 * GATHER_ITEMS));
    compact_gather<<<blocks, 256, 0, stream>>>(perm, reinterpret_cast<const uint32_t *>(sorted_keys), adm_request,
                                               adm_stage, adm_in, adm_out, n, rank_bits, out_member_req,
                                               out_member_stage, out_member_in, out_member_out, seg_start,
                                               out_run_count);
  }
  if (num_batches > 0) {
    const int blocks = (num_batches + BATCH_PER_BLOCK - 1) / BATCH_PER_BLOCK;
    if (blocks > 1) {
      batch_block_sums<<<blocks, BATCH_THREADS, 0, stream>>>(batch_exec, batch_size, num_batches, num_executors,
                                                             block_sums);
      scan_block_sums<<<1, BATCH_THREADS, 0, stream>>>(block_sums, blocks, num_executors);
    } else if (!check(cudaMemsetAsync(block_sums, 0, 4 * (size_t)num_executors, stream), "compact memset")) {
      return COE_CUDA_ERR_CUDA;
    }
    compact_batches<<<blocks, BATCH_THREADS, 0, stream>>>(batch_exec, batch_size, num_batches, num_executors,
                                                          seg_start, block_sums,
                                                          reinterpret_cast<const uint32_t *>(sorted_keys), n,
                                                          rank_bits, out_batch_off, out_violations);
  }
  return check(cudaGetLastError(), "coe_run_compact") ? COE_CUDA_OK : COE_CUDA_ERR_CUDA;
}

int coe_group_compact_fused(const int32_t *run_rank, const int32_t *adm_request, const int32_t *adm_stage,
                            const int32_t *adm_in, const int32_t *adm_out, int64_t n, int rank_bits,
                            const int32_t *batch_size, int num_batches, int32_t *out_perm, int32_t *out_batch_off,
                            int32_t *out_member_req, int32_t *out_member_stage, int32_t *out_member_in,
                            int32_t *out_member_out, int32_t *out_flags, cudaStream_t stream) {
  int idx_bits = 1;
  while ((1ll << idx_bits) < n) ++idx_bits;
  if (n < 1 || n > COE_FUSED_MAX_ADMISSIONS || num_batches > COE_FUSED_MAX_BATCHES || rank_bits + idx_bits + 1 > 32) {
    coe_set_error("coe_group_compact_fused: step too large for one block (use coe_group_sort + coe_run_compact)");
    return COE_CUDA_ERR_CONFIG;
  }
  const int ni = (int)n;
  bool good = ni <= FUSED_THREADS * 8
                  ? launch_fused<8>(run_rank, adm_request, adm_stage, adm_in, adm_out, ni, rank_bits, idx_bits,
                                    batch_size, num_batches, out_perm, out_batch_off, out_member_req,
                                    out_member_stage, out_member_in, out_member_out, out_flags, stream)
              : ni <= FUSED_THREADS * 16
                  ? launch_fused<16>(run_rank, adm_request, adm_stage, adm_in, adm_out, ni, rank_bits, idx_bits,
                                     batch_size, num_batches, out_perm, out_batch_off, out_member_req,
                                     out_member_stage, out_member_in, out_member_out, out_flags, stream)
                  : launch_fused<32>(run_rank, adm_request, adm_stage, adm_in, adm_out, ni, rank_bits, idx_bits,
                                     batch_size, num_batches, out_perm, out_batch_off, out_member_req,
                                     out_member_stage, out_member_in, out_member_out, out_flags, stream);
  return good ? COE_CUDA_OK : COE_CUDA_ERR_CUDA;
}

int coe_fill_uniform_bf16_at(void *dst, int64_t start, int64_t n, uint64_t seed, float scale, cudaStream_t stream) {
  if (n <= 0) return COE_CUDA_OK;
  if (start < 0) {
    coe_set_error("coe_fill_uniform_bf16_at: negative start");
    return COE_CUDA_ERR_CONFIG;
  }
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  fill_uniform_bf16<<<blocks, 256, 0, stream>>>(static_cast<__nv_bfloat16_raw *>(dst), start, n, seed,
                                                2.0f * scale);
  return check(cudaGetLastError(), "coe_fill_uniform_bf16") ? COE_CUDA_OK : COE_CUDA_ERR_CUDA;
}

int coe_fill_uniform_bf16(void *dst, int64_t n, uint64_t seed, float scale, cudaStream_t stream) {
  return coe_fill_uniform_bf16_at(dst, 0, n, seed, scale, stream);
}

}  // extern "C"
