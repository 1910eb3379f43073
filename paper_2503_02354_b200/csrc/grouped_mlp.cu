// grouped_mlp.cu -- K3: grouped expert MLP on tcgen05 / TMEM / TMA (sm_100a).
//
// Replaces the expert forward that the reference only *models*
// (CostModel.exec_latency as invoked by Simulation._start_batch,
// /root/reference/pkg/src/coesim/costmodel.py:55-64, engine.py:693-716).
// One launch runs one GEMM of a "wave" of planned batches (groups):
//
//   mode 0 (up):   H[g]   = gelu(X[g] . W1[slot_g]^T)   X rows gathered per request
//   mode 1 (down): Y[g]   = H[g] . W2[slot_g]^T          Y rows scattered per request
//
// Activations are [requests*T, d] row blocks: stage 0 reads the request
// inputs X, stage s > 0 reads ping-pong buffer P[(s-1)&1]; the output of stage
// s is written to P[s&1] (so X stays pristine across steps).  Which requests form a group comes from the GPU grouping
// (coe_group_sort / coe_run_compact): member_req/member_stage are the sorted
// admissions and batch_off the start of each planned batch inside them.
//
// Kernel shape: persistent, one CTA per SM, warp-specialised --
//   warp 0: TMA producer (A: per-request row boxes, B: one 3-D box of the
//           expert-slot weight tensor), 4-stage smem ring, mbarrier handshake;
//   warp 1: single-thread tcgen05.mma issuer, 128x256x16 bf16 -> f32 into a
//           double-buffered TMEM accumulator (2 x 256 columns);
//   warp 2: TMEM allocator;
//   warps 4-7: epilogue, tcgen05.ld 32x32b -> gelu/convert -> bf16 stores.
// Tiles are walked m-fastest inside (group, n-block) so concurrently running
// CTAs share the same weight tile through L2.

#include <cuda_bf16.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "coe_cuda.h"
#include "common.cuh"
#include "sm100.cuh"

namespace {

constexpr int BM = 128;
constexpr int BN = 256;
constexpr int BK = 64;
constexpr int STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;
constexpr int B_BYTES = BN * BK * 2;
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int TMEM_COLS = 512;  // 2 accumulator buffers x BN fp32 columns
constexpr int NUM_THREADS = 256;
constexpr int EPI_WARP0 = 4;
constexpr int MAX_GROUPS = 1024;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/ + MAX_GROUPS * 4;

struct GemmArgs {
  const coe_mlp_group *groups;
  int num_groups;
  int total_tiles;
  const int32_t *batch_off;
  const int32_t *member_req;
  const int32_t *member_stage;
  int T;
  int K;
  int N;
  int ld;  // row stride (elements) of the activation buffers X / P0 / P1
  int n_blocks;
  int mode;
  int a_box_rows;
  __nv_bfloat16 *out_h;
  __nv_bfloat16 *out_act0;
  __nv_bfloat16 *out_act1;
  int32_t *tile_counter;  // [next tile, CTAs done]: dynamic tile scheduler, self-resetting
  // fused follow-up hops (down pass): hop_dst[req * hop_stride + stage] = executor that runs
  // the request's next stage when it is not this one (-1 otherwise); those output rows are
  // stored straight into that executor's activation buffer (NVLink peer stores across GPUs)
  const int8_t *hop_dst;
  int hop_stride;
  __nv_bfloat16 *peer_act[COE_MAX_PEERS][2];
};

constexpr int TILE_RING = 4;  // tile indices handed from the producer to the MMA / epilogue warps

// A-operand source of a member at chain stage s: 0 = X, 1 = P0, 2 = P1.
__device__ __forceinline__ int a_source(int stage) { return stage == 0 ? 0 : 1 + ((stage - 1) & 1); }

__device__ __forceinline__ float gelu_tanh(float x) {
  float u = 0.7978845608028654f * (x + 0.044715f * x * x * x);
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(u));
  return 0.5f * x * (1.0f + t);
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t *>(&v);
}

struct TileCoord {
  int g, m_blk, n_blk;
};

__device__ __forceinline__ TileCoord decode_tile(int t, const int32_t *tile_start, int num_groups,
                                                 const coe_mlp_group *groups, int n_blocks) {
  int lo = 0, hi = num_groups - 1;
  while (lo < hi) {  // last group with tile_start <= t
    int mid = (lo + hi + 1) >> 1;
    if (tile_start[mid] <= t) lo = mid;
    else hi = mid - 1;
  }
  int local = t - tile_start[lo];
  int m_tiles = (groups[lo].rows + BM - 1) / BM;
  TileCoord c;
  c.g = lo;
  c.n_blk = local / m_tiles;
  c.m_blk = local - c.n_blk * m_tiles;
  (void)n_blocks;
  return c;
}

__global__ void __launch_bounds__(NUM_THREADS, 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap tm_a0, const __grid_constant__ CUtensorMap tm_a1,
                        const __grid_constant__ CUtensorMap tm_a2, const __grid_constant__ CUtensorMap tm_b,
                        GemmArgs args) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *stage_base = smem;
  uint64_t *full_bar = reinterpret_cast<uint64_t *>(smem + STAGES * STAGE_BYTES);
  uint64_t *empty_bar = full_bar + STAGES;
  uint64_t *tfull_bar = empty_bar + STAGES;
  uint64_t *tempty_bar = tfull_bar + 2;
  uint64_t *ring_full = tempty_bar + 2;
  uint64_t *ring_empty = ring_full + TILE_RING;
  int32_t *ring_tile = reinterpret_cast<int32_t *>(ring_empty + TILE_RING);
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(ring_tile + TILE_RING);
  int32_t *tile_start = reinterpret_cast<int32_t *>(smem + STAGES * STAGE_BYTES + 256);

  const uint32_t warp = sm100::warp_id();
  const uint32_t lane = sm100::lane_id();

  for (int i = threadIdx.x; i < args.num_groups; i += NUM_THREADS) tile_start[i] = args.groups[i].tile_start;
  if (warp == 0 && lane == 0) {
    sm100::prefetch_tmap(&tm_a0);
    sm100::prefetch_tmap(&tm_a1);
    sm100::prefetch_tmap(&tm_a2);
    sm100::prefetch_tmap(&tm_b);
    for (int s = 0; s < STAGES; ++s) {
      sm100::mbar_init(&full_bar[s], 1);
      sm100::mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      sm100::mbar_init(&tfull_bar[s], 1);
      sm100::mbar_init(&tempty_bar[s], 128);
    }
    for (int s = 0; s < TILE_RING; ++s) {
      sm100::mbar_init(&ring_full[s], 1);
      sm100::mbar_init(&ring_empty[s], 1 + 4);  // the MMA thread + one lane per epilogue warp
    }
    sm100::fence_mbar_init();
  }
  if (warp == 2) sm100::tmem_alloc<TMEM_COLS>(tmem_slot);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int k_blocks = args.K / BK;

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer =====
      int stage = 0;
      uint32_t phase = 0;
      // dynamic scheduler: tiles are claimed in (group, n-block, m-block) order, so CTAs
      // running at the same time share weight tiles through L2, and a CTA that starts late
      // (SMs held by another stream's kernel) simply claims fewer tiles.  The next claim is
      // issued before the current tile's loads so its latency hides behind them.
      // (tile_counter == nullptr: static round-robin, tile = blockIdx.x + i * gridDim.x)
      const bool dyn = args.tile_counter != nullptr;
      int claim = dyn ? atomicAdd(&args.tile_counter[0], 1) : (int)blockIdx.x;
      for (int i = 0;; ++i) {
        const int t = claim < args.total_tiles ? claim : -1;
        sm100::mbar_wait(&ring_empty[i % TILE_RING], ((i / TILE_RING) & 1) ^ 1);
        ring_tile[i % TILE_RING] = t;
        sm100::mbar_arrive(&ring_full[i % TILE_RING]);
        if (t < 0) break;
        claim = dyn ? atomicAdd(&args.tile_counter[0], 1) : claim + (int)gridDim.x;
        TileCoord c = decode_tile(t, tile_start, args.num_groups, args.groups, args.n_blocks);
        const coe_mlp_group grp = args.groups[c.g];
        int box_row[BM / 32];
        int box_par[BM / 32];
        int nboxes;
        uint32_t a_bytes;
        if (args.mode == 0) {
          const int boff = args.batch_off[grp.batch];
          const int rows_left = grp.rows - c.m_blk * BM;
          const int rows_here = rows_left < BM ? rows_left : BM;
          nboxes = (rows_here + args.a_box_rows - 1) / args.a_box_rows;
          for (int b = 0; b < nboxes; ++b) {
            int r = c.m_blk * BM + b * args.a_box_rows;
            int j = r / args.T;
            int req = args.member_req[boff + j];
            box_row[b] = req * args.T + (r - j * args.T);
            box_par[b] = a_source(args.member_stage[boff + j]);
          }
          a_bytes = (uint32_t)(nboxes * args.a_box_rows * BK * 2);
        } else {
          nboxes = 1;
          box_row[0] = grp.h_row + c.m_blk * BM;
          box_par[0] = 0;
          a_bytes = A_BYTES;
        }
        for (int kb = 0; kb < k_blocks; ++kb) {
          sm100::mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t *sa = stage_base + stage * STAGE_BYTES;
          uint8_t *sb = sa + A_BYTES;
          sm100::mbar_arrive_expect_tx(&full_bar[stage], a_bytes + B_BYTES);
          for (int b = 0; b < nboxes; ++b)
            sm100::tma_load_2d(sa + b * args.a_box_rows * 128,
                               box_par[b] == 0 ? &tm_a0 : (box_par[b] == 1 ? &tm_a1 : &tm_a2), &full_bar[stage],
                               kb * BK, box_row[b]);
          sm100::tma_load_3d(sb, &tm_b, &full_bar[stage], kb * BK, c.n_blk * BN, grp.slot);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ===== MMA issuer =====
      constexpr uint32_t idesc = sm100::make_idesc_bf16_f32(BM, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int i = 0;; ++i) {
        sm100::mbar_wait(&ring_full[i % TILE_RING], (i / TILE_RING) & 1);
        const int t = ring_tile[i % TILE_RING];
        sm100::mbar_arrive(&ring_empty[i % TILE_RING]);
        if (t < 0) break;
        sm100::mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        sm100::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < k_blocks; ++kb) {
          sm100::mbar_wait(&full_bar[stage], phase);
          sm100::tc_fence_after();
          const uint32_t sa = sm100::smem_u32(stage_base + stage * STAGE_BYTES);
          const uint32_t sb = sa + A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            uint64_t adesc = sm100::make_desc_k_sw128(sa + k * 32);
            uint64_t bdesc = sm100::make_desc_k_sw128(sb + k * 32);
            sm100::mma_bf16_ss(d_tmem, adesc, bdesc, idesc, (kb | k) != 0);
          }
          sm100::mma_commit(&empty_bar[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        sm100::mma_commit(&tfull_bar[acc]);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= EPI_WARP0) {
    // ===== epilogue =====
    const uint32_t quarter = warp & 3;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int i = 0;; ++i) {
      sm100::mbar_wait(&ring_full[i % TILE_RING], (i / TILE_RING) & 1);
      const int t = ring_tile[i % TILE_RING];
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&ring_empty[i % TILE_RING]);
      if (t < 0) break;
      TileCoord c = decode_tile(t, tile_start, args.num_groups, args.groups, args.n_blocks);
      const coe_mlp_group grp = args.groups[c.g];
      const int row = c.m_blk * BM + quarter * 32 + lane;
      const bool valid = row < grp.rows;
      __nv_bfloat16 *out_row = nullptr;
      if (valid) {
        if (args.mode == 0) {
          out_row = args.out_h + (size_t)(grp.h_row + row) * args.N;
        } else {
          const int boff = args.batch_off[grp.batch];
          const int j = row / args.T;
          const int req = args.member_req[boff + j];
          const int st = args.member_stage[boff + j];
          __nv_bfloat16 *dst = (st & 1) ? args.out_act1 : args.out_act0;
          if (args.hop_dst) {
            const int hd = args.hop_dst[(size_t)req * args.hop_stride + st];
            if (hd >= 0) dst = args.peer_act[hd][st & 1];
          }
          out_row = dst + ((size_t)req * args.T + (row - j * args.T)) * args.ld;
        }
        out_row += c.n_blk * BN;
      }
      sm100::mbar_wait(&tfull_bar[acc], acc_phase);
      sm100::tc_fence_after();
      const uint32_t taddr = tmem_base + ((quarter * 32) << 16) + acc * BN;
#pragma unroll 1
      for (int chunk = 0; chunk < BN / 32; ++chunk) {
        uint32_t v[32];
        sm100::tmem_ld_32x32b_x32(taddr + chunk * 32, v);
        sm100::tmem_ld_wait();
        if (valid) {
          uint32_t packed[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float lo = __uint_as_float(v[2 * i]);
            float hi = __uint_as_float(v[2 * i + 1]);
            if (args.mode == 0) {
              lo = gelu_tanh(lo);
              hi = gelu_tanh(hi);
            }
            packed[i] = pack_bf16(lo, hi);
          }
          uint4 *dst = reinterpret_cast<uint4 *>(out_row + chunk * 32);
#pragma unroll
          for (int i = 0; i < 4; ++i)
            dst[i] = make_uint4(packed[4 * i], packed[4 * i + 1], packed[4 * i + 2], packed[4 * i + 3]);
        }
      }
      sm100::tc_fence_before();
      sm100::mbar_arrive(&tempty_bar[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }

  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc<TMEM_COLS>(tmem_base);
  }
  if (threadIdx.x == 0 && args.tile_counter) {
    // every claim of this CTA precedes its arrival here; the last CTA out re-arms the
    // counter for the next launch on this stream (launches on a stream are ordered)
    if (atomicAdd(&args.tile_counter[1], 1) == (int)gridDim.x - 1) {
      args.tile_counter[0] = 0;
      args.tile_counter[1] = 0;
      __threadfence();
    }
  }
}

// ---- host side ---------------------------------------------------------------

using EncodeTiledFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                   const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  }
  return fn;
}

// 2-D bf16 row-major [rows, cols] map (row stride ld >= cols elements), box {64, box_rows},
// 128B swizzle.
bool make_map_2d(CUtensorMap *map, void *base, uint64_t rows, uint64_t cols, uint32_t box_rows, uint64_t ld = 0) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {(ld ? ld : cols) * 2};
  cuuint32_t box[2] = {BK, box_rows};
  cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 3-D bf16 map over expert slots: [slots][rows][cols], slot stride in bytes.
bool make_map_3d(CUtensorMap *map, void *base, uint64_t slots, uint64_t rows, uint64_t cols, uint64_t slot_stride) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {cols, rows, slots};
  cuuint64_t strides[2] = {cols * 2, slot_stride};
  cuuint32_t box[3] = {BK, BN, 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, base, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace

struct coe_mlp {
  coe_mlp_config cfg;
  CUtensorMap xmap, act0, act1, hmap, w1, w2;
  int num_sms;
  int a_box_rows;
  int32_t *tile_counter = nullptr;  // device [2]; one per instance = one per stream
  const int8_t *hop_dst = nullptr;   // fused hops (coe_mlp_set_hops)
  int hop_stride = 0;
  __nv_bfloat16 *peer_act[COE_MAX_PEERS][2] = {};
  bool dynamic = false;             // COE_K3_DYNAMIC=1: atomic tile claims instead of the static
                                    // round-robin (measured 3 % slower on full-GPU waves, r1)
};

extern "C" {

int coe_mlp_create(const coe_mlp_config *cfg, coe_mlp **out) {
  if (cfg->act_ld > 0 && (cfg->act_ld < cfg->d || cfg->act_ld % 8)) {
    coe_set_error("grouped MLP: act_ld must be >= d and a multiple of 8");
    return COE_CUDA_ERR_CONFIG;
  }
  if (cfg->d % BN || cfg->h % BN || cfg->d % BK || cfg->h % BK) {
    coe_set_error("grouped MLP needs d and h to be multiples of 256");
    return COE_CUDA_ERR_CONFIG;
  }
  if (!(cfg->T == 32 || cfg->T == 64 || cfg->T % 128 == 0)) {
    coe_set_error("grouped MLP needs rows-per-request T in {32, 64} or a multiple of 128");
    return COE_CUDA_ERR_CONFIG;
  }
  auto *m = new coe_mlp();
  m->cfg = *cfg;
  m->dynamic = getenv("COE_K3_DYNAMIC") && atoi(getenv("COE_K3_DYNAMIC")) != 0;
  m->a_box_rows = cfg->T < BM ? cfg->T : BM;
  bool ok = true;
  const uint64_t ld = cfg->act_ld > 0 ? (uint64_t)cfg->act_ld : (uint64_t)cfg->d;
  ok &= make_map_2d(&m->xmap, cfg->x, (uint64_t)cfg->act_rows, cfg->d, m->a_box_rows, ld);
  ok &= make_map_2d(&m->act0, cfg->act0, (uint64_t)cfg->act_rows, cfg->d, m->a_box_rows, ld);
  ok &= make_map_2d(&m->act1, cfg->act1, (uint64_t)cfg->act_rows, cfg->d, m->a_box_rows, ld);
  ok &= make_map_2d(&m->hmap, cfg->h_scratch, (uint64_t)cfg->h_rows, cfg->h, BM);
  // slot layout: [W1: h x d][W2: d x h]
  ok &= make_map_3d(&m->w1, cfg->slab, cfg->num_slots, cfg->h, cfg->d, cfg->slot_stride_bytes);
  ok &= make_map_3d(&m->w2, (char *)cfg->slab + (size_t)cfg->h * cfg->d * 2, cfg->num_slots, cfg->d, cfg->h,
                    cfg->slot_stride_bytes);
  if (!ok) {
    delete m;
    coe_set_error("cuTensorMapEncodeTiled failed (alignment / driver entry point)");
    return COE_CUDA_ERR_CUDA;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&m->num_sms, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e = cudaFuncSetAttribute(grouped_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
  if (e == cudaSuccess) e = cudaMalloc(&m->tile_counter, 2 * sizeof(int32_t));
  if (e == cudaSuccess) e = cudaMemset(m->tile_counter, 0, 2 * sizeof(int32_t));
  if (e != cudaSuccess) {
    if (m->tile_counter) cudaFree(m->tile_counter);
    delete m;
    coe_set_error(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    return COE_CUDA_ERR_CUDA;
  }
  *out = m;
  return COE_CUDA_OK;
}

void coe_mlp_destroy(coe_mlp *m) {
  if (!m) return;
  if (m->tile_counter) cudaFree(m->tile_counter);
  delete m;
}

int coe_mlp_max_groups(void) { return MAX_GROUPS; }

int coe_mlp_set_hops(coe_mlp *m, const int8_t *hop_dst, int hop_stride, void *const *peer_act, int world) {
  if (world > COE_MAX_PEERS) {
    coe_set_error("fused hops: more executors than COE_MAX_PEERS");
    return COE_CUDA_ERR_CONFIG;
  }
  m->hop_dst = hop_dst;
  m->hop_stride = hop_stride;
  for (int r = 0; r < COE_MAX_PEERS; ++r)
    for (int b = 0; b < 2; ++b)
      m->peer_act[r][b] = (hop_dst && r < world) ? static_cast<__nv_bfloat16 *>(peer_act[2 * r + b]) : nullptr;
  return COE_CUDA_OK;
}

int coe_grouped_mlp(coe_mlp *m, const coe_mlp_group *groups_up, const coe_mlp_group *groups_down, int num_groups,
                    int tiles_up, int tiles_down, const int32_t *batch_off, const int32_t *member_req,
                    const int32_t *member_stage, int which, int max_ctas, cudaStream_t stream) {
  if (num_groups <= 0) return COE_CUDA_OK;
  if (num_groups > MAX_GROUPS) {
    coe_set_error("too many groups in one wave");
    return COE_CUDA_ERR_CONFIG;
  }
  const coe_mlp_config &c = m->cfg;
  for (int pass = 0; pass < 2; ++pass) {
    if (!(which & (1 << pass))) continue;
    GemmArgs a{};
    a.groups = pass == 0 ? groups_up : groups_down;
    a.num_groups = num_groups;
    a.total_tiles = pass == 0 ? tiles_up : tiles_down;
    a.batch_off = batch_off;
    a.member_req = member_req;
    a.member_stage = member_stage;
    a.T = c.T;
    a.K = pass == 0 ? c.d : c.h;
    a.N = pass == 0 ? c.h : c.d;
    a.ld = c.act_ld > 0 ? c.act_ld : c.d;
    a.n_blocks = a.N / BN;
    a.mode = pass;
    a.a_box_rows = m->a_box_rows;
    a.out_h = reinterpret_cast<__nv_bfloat16 *>(c.h_scratch);
    a.out_act0 = reinterpret_cast<__nv_bfloat16 *>(c.act0);
    a.out_act1 = reinterpret_cast<__nv_bfloat16 *>(c.act1);
    a.tile_counter = m->dynamic ? m->tile_counter : nullptr;
    a.hop_dst = pass == 1 ? m->hop_dst : nullptr;
    a.hop_stride = m->hop_stride;
    std::memcpy(a.peer_act, m->peer_act, sizeof(a.peer_act));
    if (a.total_tiles <= 0) continue;
    int cap = (max_ctas > 0 && max_ctas < m->num_sms) ? max_ctas : m->num_sms;
    int grid = a.total_tiles < cap ? a.total_tiles : cap;
    if (pass == 0)
      grouped_gemm_kernel<<<grid, NUM_THREADS, SMEM_BYTES, stream>>>(m->xmap, m->act0, m->act1, m->w1, a);
    else
      grouped_gemm_kernel<<<grid, NUM_THREADS, SMEM_BYTES, stream>>>(m->hmap, m->hmap, m->hmap, m->w2, a);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
      coe_set_error(std::string("grouped_gemm_kernel launch: ") + cudaGetErrorString(e));
      return COE_CUDA_ERR_CUDA;
    }
  }
  return COE_CUDA_OK;
}

}  // extern "C"
