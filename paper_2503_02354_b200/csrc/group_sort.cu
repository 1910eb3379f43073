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
// Layout: SoA int32 arrays; 2048-element tiles (256 threads x 8 rounds);
// per-tile digit histograms -> one-block exclusive scan -> stable scatter with
// warp match_any ranks.  Everything is HBM/latency-bound integer work.

#include <cstdint>
#include <string>

#include <cuda_bf16.h>

#include "coe_cuda.h"
#include "common.cuh"

namespace {

constexpr int SORT_THREADS = 256;
constexpr int ROUNDS = 8;
constexpr int TILE = SORT_THREADS * ROUNDS;
constexpr int RADIX = 256;

__global__ void make_keys(const int32_t *exec, const int32_t *rank, int64_t n, int rank_bits, uint32_t *keys,
                          int32_t *vals) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) {
    keys[i] = ((uint32_t)exec[i] << rank_bits) | (uint32_t)rank[i];
    vals[i] = (int32_t)i;
  }
}

__global__ void radix_hist(const uint32_t *keys, int64_t n, int shift, int num_tiles, uint32_t *hist) {
  __shared__ uint32_t h[RADIX];
  h[threadIdx.x] = 0;
  __syncthreads();
  int64_t base = (int64_t)blockIdx.x * TILE;
  for (int r = 0; r < ROUNDS; ++r) {
    int64_t i = base + r * SORT_THREADS + threadIdx.x;
    if (i < n) atomicAdd(&h[(keys[i] >> shift) & 255], 1u);
  }
  __syncthreads();
  hist[threadIdx.x * num_tiles + blockIdx.x] = h[threadIdx.x];
}

// single-block exclusive scan of m uint32 values in place
__global__ void exclusive_scan_1block(uint32_t *data, int64_t m) {
  __shared__ uint32_t partial[1024];
  const int t = threadIdx.x;
  const int64_t per = (m + blockDim.x - 1) / blockDim.x;
  const int64_t lo = t * per;
  const int64_t hi = lo + per < m ? lo + per : m;
  uint32_t sum = 0;
  for (int64_t i = lo; i < hi; ++i) sum += data[i];
  partial[t] = sum;
  __syncthreads();
  for (int off = 1; off < (int)blockDim.x; off <<= 1) {  // Hillis-Steele over thread totals
    uint32_t v = t >= off ? partial[t - off] : 0;
    __syncthreads();
    partial[t] += v;
    __syncthreads();
  }
  uint32_t run = partial[t] - sum;
  for (int64_t i = lo; i < hi; ++i) {
    uint32_t v = data[i];
    data[i] = run;
    run += v;
  }
}

__global__ void radix_scatter(const uint32_t *keys_in, const int32_t *vals_in, uint32_t *keys_out, int32_t *vals_out,
                              const uint32_t *offsets, int64_t n, int shift, int num_tiles) {
  __shared__ uint32_t run_base[RADIX];
  __shared__ uint32_t warp_cnt[SORT_THREADS / 32][RADIX];
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  run_base[tid] = offsets[tid * num_tiles + blockIdx.x];
  const uint32_t lt_mask = (1u << lane) - 1u;
  int64_t base = (int64_t)blockIdx.x * TILE;
  for (int r = 0; r < ROUNDS; ++r) {
    for (int j = tid; j < (SORT_THREADS / 32) * RADIX; j += SORT_THREADS) (&warp_cnt[0][0])[j] = 0;
    __syncthreads();
    int64_t i = base + r * SORT_THREADS + tid;
    bool valid = i < n;
    uint32_t key = valid ? keys_in[i] : 0u;
    uint32_t digit = valid ? ((key >> shift) & 255u) : 256u;
    uint32_t same = __match_any_sync(0xffffffffu, digit);
    uint32_t rank = __popc(same & lt_mask);
    if (valid && rank == 0) warp_cnt[warp][digit] = __popc(same);
    __syncthreads();
    if (valid) {
      uint32_t pos = run_base[digit] + rank;
      for (int w = 0; w < warp; ++w) pos += warp_cnt[w][digit];
      keys_out[pos] = key;
      vals_out[pos] = vals_in[i];
    }
    __syncthreads();
    uint32_t add = 0;
    for (int w = 0; w < SORT_THREADS / 32; ++w) add += warp_cnt[w][tid];
    run_base[tid] += add;
    __syncthreads();
  }
}

// K2 part 1: gather members, mark run starts / executor segment starts.
__global__ void compact_gather(const int32_t *perm, const uint32_t *keys, const int32_t *adm_req,
                               const int32_t *adm_stage, int64_t n, int rank_bits, int32_t *member_req,
                               int32_t *member_stage, int32_t *seg_start, int32_t *run_count) {
  int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  int starts = 0;
  if (i < n) {
    int32_t p = perm[i];
    member_req[i] = adm_req[p];
    member_stage[i] = adm_stage[p];
    uint32_t k = keys[i];
    bool new_run = i == 0 || keys[i - 1] != k;
    starts = new_run ? 1 : 0;
    if (i == 0 || (keys[i - 1] >> rank_bits) != (k >> rank_bits)) seg_start[k >> rank_bits] = (int32_t)i;
  }
  // block-reduce the run starts into one atomic
  for (int off = 16; off; off >>= 1) starts += __shfl_down_sync(0xffffffffu, starts, off);
  __shared__ int warp_sum[32];
  if ((threadIdx.x & 31) == 0) warp_sum[threadIdx.x >> 5] = starts;
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += warp_sum[w];
    if (s) atomicAdd(run_count, s);
  }
}

// K2 part 2: per-executor exclusive scan of batch sizes in op order (one block),
// then batch offsets = segment start + prefix; check single-run batches.
__global__ void compact_batches(const int32_t *batch_exec, const int32_t *batch_size, int num_batches,
                                int num_executors, const int32_t *seg_start, const uint32_t *keys, int64_t n,
                                int rank_bits, int32_t *batch_off, int32_t *violations) {
  __shared__ int32_t scan[1024];
  __shared__ int32_t carry;
  const int t = threadIdx.x;
  for (int x = 0; x < num_executors; ++x) {
    if (t == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < num_batches; base += blockDim.x) {
      int b = base + t;
      int v = (b < num_batches && batch_exec[b] == x) ? batch_size[b] : 0;
      scan[t] = v;
      __syncthreads();
      for (int off = 1; off < (int)blockDim.x; off <<= 1) {
        int add = t >= off ? scan[t - off] : 0;
        __syncthreads();
        scan[t] += add;
        __syncthreads();
      }
      if (b < num_batches && batch_exec[b] == x) batch_off[b] = seg_start[x] + carry + scan[t] - v;
      __syncthreads();
      if (t == blockDim.x - 1) carry += scan[t];
      __syncthreads();
    }
  }
  for (int b = t; b < num_batches; b += blockDim.x) {
    int lo = batch_off[b];
    int hi = lo + batch_size[b] - 1;
    bool bad = batch_size[b] <= 0 || lo < 0 || hi >= n || keys[lo] != keys[hi] ||
               (int)(keys[lo] >> rank_bits) != batch_exec[b];
    if (bad) atomicAdd(violations, 1);
  }
}

// counter-based uniform generator (splitmix64), mirrored in oracle/synth.py
__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void fill_uniform_bf16(__nv_bfloat16_raw *dst, int64_t n, uint64_t seed, float two_scale) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = splitmix64(seed + (uint64_t)(i + 1) * 0x9E3779B97F4A7C15ull);
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

}  // namespace

extern "C" {

int64_t coe_group_sort_scratch_bytes(int64_t n) {
  int64_t tiles = (n + TILE - 1) / TILE;
  if (tiles < 1) tiles = 1;
  return 4 * 4 * (n + 64) + 4 * RADIX * tiles + 1024;
}

int coe_group_sort(const int32_t *executor, const int32_t *run_rank, int64_t n, int rank_bits, int num_passes,
                   int32_t *out_perm, int32_t *out_keys, void *scratch, cudaStream_t stream) {
  if (n <= 0) return COE_CUDA_OK;
  if (num_passes < 1 || num_passes > 4 || rank_bits < 1 || rank_bits > 31) {
    coe_set_error("coe_group_sort: bad pass count / rank bits");
    return COE_CUDA_ERR_CONFIG;
  }
  const int num_tiles = (int)((n + TILE - 1) / TILE);
  char *s = static_cast<char *>(scratch);
  uint32_t *ka = reinterpret_cast<uint32_t *>(s);
  uint32_t *kb = ka + n + 16;
  int32_t *va = reinterpret_cast<int32_t *>(kb + n + 16);
  int32_t *vb = va + n + 16;
  uint32_t *hist = reinterpret_cast<uint32_t *>(vb + n + 16);
  const int blocks = (int)((n + 255) / 256);
  make_keys<<<blocks, 256, 0, stream>>>(executor, run_rank, n, rank_bits, ka, va);
  for (int p = 0; p < num_passes; ++p) {
    radix_hist<<<num_tiles, SORT_THREADS, 0, stream>>>(ka, n, 8 * p, num_tiles, hist);
    exclusive_scan_1block<<<1, 1024, 0, stream>>>(hist, (int64_t)RADIX * num_tiles);
    radix_scatter<<<num_tiles, SORT_THREADS, 0, stream>>>(ka, va, kb, vb, hist, n, 8 * p, num_tiles);
    std::swap(ka, kb);
    std::swap(va, vb);
  }
  if (!check(cudaMemcpyAsync(out_perm, va, n * 4, cudaMemcpyDeviceToDevice, stream), "sort perm copy")) return COE_CUDA_ERR_CUDA;
  if (!check(cudaMemcpyAsync(out_keys, ka, n * 4, cudaMemcpyDeviceToDevice, stream), "sort key copy")) return COE_CUDA_ERR_CUDA;
  return check(cudaGetLastError(), "coe_group_sort") ? COE_CUDA_OK : COE_CUDA_ERR_CUDA;
}

int64_t coe_run_compact_scratch_bytes(int64_t n, int num_batches, int num_executors) {
  (void)n;
  (void)num_batches;
  return 4 * (int64_t)(num_executors + 16);
}

int coe_run_compact(const int32_t *perm, const int32_t *sorted_keys, const int32_t *adm_request,
                    const int32_t *adm_stage, int64_t n, int rank_bits, const int32_t *batch_exec,
                    const int32_t *batch_size, int num_batches, int num_executors, int32_t *out_batch_off,
                    int32_t *out_member_req, int32_t *out_member_stage, int32_t *out_run_count,
                    int32_t *out_violations, void *scratch, cudaStream_t stream) {
  int32_t *seg_start = static_cast<int32_t *>(scratch);
  if (!check(cudaMemsetAsync(seg_start, 0, 4 * (size_t)num_executors, stream), "compact memset") ||
      !check(cudaMemsetAsync(out_run_count, 0, 4, stream), "compact memset") ||
      !check(cudaMemsetAsync(out_violations, 0, 4, stream), "compact memset"))
    return COE_CUDA_ERR_CUDA;
  if (n > 0) {
    const int blocks = (int)((n + 255) / 256);
    compact_gather<<<blocks, 256, 0, stream>>>(perm, reinterpret_cast<const uint32_t *>(sorted_keys), adm_request,
                                               adm_stage, n, rank_bits, out_member_req, out_member_stage, seg_start,
                                               out_run_count);
  }
  if (num_batches > 0)
    compact_batches<<<1, 1024, 0, stream>>>(batch_exec, batch_size, num_batches, num_executors, seg_start,
                                            reinterpret_cast<const uint32_t *>(sorted_keys), n, rank_bits,
                                            out_batch_off, out_violations);
  return check(cudaGetLastError(), "coe_run_compact") ? COE_CUDA_OK : COE_CUDA_ERR_CUDA;
}

int coe_fill_uniform_bf16(void *dst, int64_t n, uint64_t seed, float scale, cudaStream_t stream) {
  if (n <= 0) return COE_CUDA_OK;
  int blocks = (int)((n + 255) / 256);
  if (blocks > 148 * 16) blocks = 148 * 16;
  fill_uniform_bf16<<<blocks, 256, 0, stream>>>(static_cast<__nv_bfloat16_raw *>(dst), n, seed, 2.0f * scale);
  return check(cudaGetLastError(), "coe_fill_uniform_bf16") ? COE_CUDA_OK : COE_CUDA_ERR_CUDA;
}

}  // extern "C"
