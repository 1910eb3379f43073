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
// Activations are [requests*T, ld] row blocks: stage 0 reads the request inputs X,
// stage s > 0 reads ping-pong buffer P[(s-1)&1]; the output of stage s is written to
// P[s&1] (so X stays pristine across steps) -- or, for a request whose next stage runs
// on another executor, straight into that executor's P (fused hop, coe_mlp_set_hops).
// Which requests form a group comes from the GPU grouping (coe_group_sort /
// coe_run_compact): member_req/member_stage are the sorted admissions and batch_off the
// start of each planned batch inside them.
//
// Kernel shape (default CG = 2): persistent, warp-specialised, CTA PAIRS -- a cluster of
// 2 CTAs on one TPC computes a 256 x 256 tile with tcgen05.mma.cta_group::2:
//   warp 0: TMA producer in each CTA: its own 128 A rows (per-request row boxes) and HALF
//           of B (128 rows of the expert-slot weight tensor), 6-stage 32 KB smem ring;
//           the .cta_group::2 loads complete on the LEADER CTA's mbarrier;
//   warp 1: leader only: single-thread issuer of 256x256x16 bf16 -> f32 MMAs into a
//           double-buffered TMEM accumulator (2 x 256 columns per CTA); multicast
//           commits free the stage / publish the accumulator in both CTAs;
//   warp 2: TMEM allocator (cta_group::2 in both CTAs); warp 3: tile-table scan;
//   warps 4-11: epilogue, two warps per TMEM lane quarter (half the columns each),
//           tcgen05.ld one 32-column chunk ahead -> gelu / bf16 -> stores; one lane per
//           warp signals the leader's TMEM-empty barrier.
// CG = 1 (COE_K3_CG=1) is the single-CTA 128 x 256 variant (4-stage 48 KB ring).
// Tiles are walked m-fastest inside (group, n-block) so concurrently running pairs share
// the same weight tile through L2.

#include <cuda_bf16.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "coe_cuda.h"
#include "common.cuh"
#include "sm100.cuh"

namespace {

constexpr int BM = 128;  // rows per CTA tile (TMEM lanes)
constexpr int BN = 256;  // output columns per tile (one 256-column TMEM accumulator)
constexpr int BK = 64;   // K per stage (one 128-byte swizzle row of bf16)
constexpr int TMEM_COLS = 512;  // 2 accumulator buffers x BN fp32 columns
constexpr int NUM_THREADS = 384;
constexpr int EPI_WARP0 = 4;
constexpr int EPI_WARPS = 8;  // two warps per TMEM lane quarter, each drains half the columns
constexpr int MAX_GROUPS = 1024;
constexpr int CRD_STAGES = 6;
constexpr int EPI_SCRATCH = 2048;  // per epilogue warp: one 32-row x 32-column bf16 chunk, staged for coalesced stores  // tile-coordinate ring (warp 3 -> TMA producer + epilogue warps)

// Per-tile coordinates resolved ahead by the coordinate warp (warp 3): the dependent global
// loads (group -> batch offset -> member routes) leave the TMA producer's and the epilogue's
// critical path.  One entry per tile of this CTA.
struct TileCrd {
  int32_t box_row[4];        // A: first row of each TMA box (per-request boxes in the up pass)
  int32_t box_par[4];        // A: which activation map (0 = X / H, 1, 2)
  int32_t nboxes, slot, b_row;
  uint32_t a_bytes;
  __nv_bfloat16 *qbase[4];   // epilogue: output row of the first row of each 32-row lane quarter
  int32_t qvalid[4];         // rows of the quarter inside the group
};
static_assert(sizeof(TileCrd) <= 128, "TileCrd exceeds its slot");

// CG = CTAs per MMA: 1 -- one CTA computes a 128 x 256 tile and loads A (128 x 64) and B
// (256 x 64) per stage; 2 -- a CTA pair (cluster of 2 on one TPC) computes a 256 x 256 tile
// with tcgen05.mma.cta_group::2: each CTA loads its own 128 A rows and HALF of B (128 x 64),
// so per-CTA operand traffic per stage drops from 48 KB to 32 KB for the same MMA work.
template <int CG>
struct Tiling {
  static constexpr int TILE_M = BM * CG;
  static constexpr int B_ROWS = BN / CG;
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = B_ROWS * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = CG == 1 ? 4 : 6;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/ + MAX_GROUPS * 4 +
                              CRD_STAGES * 128 + EPI_WARPS * EPI_SCRATCH;
};

struct GemmArgs {
  const coe_mlp_group *groups;
  int num_groups;
  int total_tiles;  // CG == 1: host-computed; CG == 2: recomputed in the prologue
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
  // fused follow-up hops (down pass): hop_dst[req * hop_stride + stage] = executor that runs
  // the request's next stage when it is not this one (-1 otherwise); those output rows are
  // stored straight into that executor's activation buffer (NVLink peer stores across GPUs)
  const int8_t *hop_dst;
  int hop_stride;
  __nv_bfloat16 *peer_act[COE_MAX_PEERS][2];
  // routed mode (coe_grouped_mlp_routed; member_in != nullptr): every member carries its own
  // activation rows -- in = (row << 1) | from_X, out = (row << 4) | kind with kind 0 the local
  // activation ring A, 1 the device output buffer Y, 2 the e2e output staging ring, 3 + r
  // executor r's A (a fused hop into its landing rows); rows count requests (T rows each)
  const int32_t *member_in;
  const int32_t *member_out;
  __nv_bfloat16 *out_y;
  __nv_bfloat16 *out_stage;
  int debug;  // experiments only (COE_K3_DEBUG): bit 0 skips the epilogue stores, bit 1 the gelu
};

// A-operand source of a member at chain stage s: 0 = X, 1 = P0, 2 = P1.
__device__ __forceinline__ int a_source(int stage) { return stage == 0 ? 0 : 1 + ((stage - 1) & 1); }

// gelu_tanh(x) = 0.5 x (1 + tanh(sqrt(2/pi) (x + 0.044715 x^3))), as 0.5x + 0.5x * tanh(x (c0 + c1 x^2)):
// 5 FP32 ops + 1 MUFU.  The epilogue warps share the SM sub-partitions with the single-thread
// TMA producer and MMA issuer, so fewer epilogue instructions leave them more issue slots.
__device__ __forceinline__ float gelu_tanh(float x) {
  const float x2 = x * x;
  const float u = x * fmaf(0.0356774081363001f, x2, 0.7978845608028654f);
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(u));
  const float h = 0.5f * x;
  return fmaf(h, t, h);
}

__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t *>(&v);
}

struct TileCoord {
  int g, m_blk, n_blk;  // m_blk in units of the (pair) tile height
};

template <int CG>
__device__ __forceinline__ TileCoord decode_tile(int t, const int32_t *tile_start, int num_groups,
                                                 const coe_mlp_group *groups) {
  int lo = 0, hi = num_groups - 1;
  while (lo < hi) {  // last group with tile_start <= t
    int mid = (lo + hi + 1) >> 1;
    if (tile_start[mid] <= t) lo = mid;
    else hi = mid - 1;
  }
  int local = t - tile_start[lo];
  int m_tiles = (groups[lo].rows + Tiling<CG>::TILE_M - 1) / Tiling<CG>::TILE_M;
  TileCoord c;
  c.g = lo;
  c.n_blk = local / m_tiles;
  c.m_blk = local - c.n_blk * m_tiles;
  return c;
}

template <int CG, bool CW>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap tm_a0, const __grid_constant__ CUtensorMap tm_a1,
                        const __grid_constant__ CUtensorMap tm_a2, const __grid_constant__ CUtensorMap tm_b,
                        GemmArgs args) {
  using TL = Tiling<CG>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t *stage_base = smem;
  uint64_t *full_bar = reinterpret_cast<uint64_t *>(smem + TL::STAGES * TL::STAGE_BYTES);
  uint64_t *empty_bar = full_bar + TL::STAGES;
  uint64_t *tfull_bar = empty_bar + TL::STAGES;
  uint64_t *tempty_bar = tfull_bar + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tempty_bar + 2);
  int32_t *total_slot = reinterpret_cast<int32_t *>(tmem_slot + 1);
  int32_t *tile_start = reinterpret_cast<int32_t *>(smem + TL::STAGES * TL::STAGE_BYTES + 256);
  TileCrd *crd = reinterpret_cast<TileCrd *>(smem + TL::STAGES * TL::STAGE_BYTES + 256 + MAX_GROUPS * 4);
  uint8_t *epi_scratch = smem + TL::STAGES * TL::STAGE_BYTES + 256 + MAX_GROUPS * 4 + CRD_STAGES * 128;
  uint64_t *crd_full = reinterpret_cast<uint64_t *>(tmem_slot + 2);  // after tmem_slot / total_slot, 8-aligned
  uint64_t *crd_empty = crd_full + CRD_STAGES;

  const uint32_t warp = sm100::warp_id();
  const uint32_t lane = sm100::lane_id();
  const uint32_t cta_rank = CG == 2 ? sm100::cluster_ctarank() : 0;  // 0 = leader (issues the MMAs)
  const int tile0 = blockIdx.x / CG, tile_step = gridDim.x / CG;

  if constexpr (CG == 1) {
    for (int i = threadIdx.x; i < args.num_groups; i += NUM_THREADS) tile_start[i] = args.groups[i].tile_start;
  } else if (warp == 3) {
    // pair tiles per group (256-row tiles): exclusive scan across the warp, chunk per lane
    const int per = (args.num_groups + 31) / 32;
    const int lo = min((int)lane * per, args.num_groups), hi = min(lo + per, args.num_groups);
    auto tiles_of = [&](int g) { return (args.groups[g].rows + TL::TILE_M - 1) / TL::TILE_M * args.n_blocks; };
    int sum = 0;
    for (int g = lo; g < hi; ++g) sum += tiles_of(g);
    int incl = sum;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, off);
      if ((int)lane >= off) incl += v;
    }
    int run = incl - sum;
    for (int g = lo; g < hi; ++g) {
      tile_start[g] = run;
      run += tiles_of(g);
    }
    if (lane == 31) *total_slot = incl;
  }
  if (warp == 0 && lane == 0) {
    sm100::prefetch_tmap(&tm_a0);
    sm100::prefetch_tmap(&tm_a1);
    sm100::prefetch_tmap(&tm_a2);
    sm100::prefetch_tmap(&tm_b);
    for (int s = 0; s < TL::STAGES; ++s) {
      sm100::mbar_init(&full_bar[s], 1);
      sm100::mbar_init(&empty_bar[s], 1);
    }
    for (int s = 0; s < CRD_STAGES; ++s) {
      sm100::mbar_init(&crd_full[s], 1);
      sm100::mbar_init(&crd_empty[s], 1 + EPI_WARPS);  // the TMA producer + one lane per epilogue warp
    }
    for (int s = 0; s < 2; ++s) {
      sm100::mbar_init(&tfull_bar[s], 1);
      // CG 1: every epilogue thread arrives; CG 2: one lane per epilogue warp of both CTAs
      sm100::mbar_init(&tempty_bar[s], CG == 1 ? 32 * EPI_WARPS : 2 * EPI_WARPS);
    }
    sm100::fence_mbar_init();
  }
  if (warp == 2) sm100::tmem_alloc<TMEM_COLS, CG>(tmem_slot);
  sm100::tc_fence_before();
  if constexpr (CG == 2) {
    sm100::cluster_sync();  // peer barriers initialised, TMEM allocated in both
    __syncthreads();        // (also a CTA barrier: compute-sanitizer racecheck does not model cluster barriers)
  } else {
    __syncthreads();
  }
  sm100::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int total_tiles = CG == 1 ? args.total_tiles : *total_slot;
  const int k_blocks = args.K / BK;

  if (warp == 0) {
    if (lane == 0) {
      if constexpr (CW) {
      // ===== TMA producer (both CTAs of a pair: own A rows, own half of B) =====
      int stage = 0;
      uint32_t phase = 0;
      int cs = 0;
      uint32_t cph = 0;
      for (int t = tile0; t < total_tiles; t += tile_step) {
        sm100::mbar_wait(&crd_full[cs], cph);
        const TileCrd &e = crd[cs];
        int box_row[BM / 32];
        int box_par[BM / 32];
        const int nboxes = e.nboxes;
#pragma unroll
        for (int b = 0; b < BM / 32; ++b) {
          box_row[b] = e.box_row[b];
          box_par[b] = e.box_par[b];
        }
        const uint32_t a_bytes = e.a_bytes;
        const int b_row = e.b_row, slot = e.slot;
        sm100::mbar_arrive(&crd_empty[cs]);
        if (++cs == CRD_STAGES) {
          cs = 0;
          cph ^= 1;
        }
        for (int kb = 0; kb < k_blocks; ++kb) {
          sm100::mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t *sa = stage_base + stage * TL::STAGE_BYTES;
          uint8_t *sb = sa + TL::A_BYTES;
          if constexpr (CG == 1) {
            sm100::mbar_arrive_expect_tx(&full_bar[stage], a_bytes + TL::B_BYTES);
#pragma unroll
            for (int b = 0; b < BM / 32; ++b)
              if (b < nboxes)
                sm100::tma_load_2d(sa + b * args.a_box_rows * 128,
                                 box_par[b] == 0 ? &tm_a0 : (box_par[b] == 1 ? &tm_a1 : &tm_a2), &full_bar[stage],
                                 kb * BK, box_row[b]);
            sm100::tma_load_3d(sb, &tm_b, &full_bar[stage], kb * BK, b_row, slot);
          } else {
            const uint32_t bar = sm100::mapa_shared(sm100::smem_u32(&full_bar[stage]), 0);
            if (cta_rank == 0) sm100::mbar_arrive_expect_tx(&full_bar[stage], 2 * TL::STAGE_BYTES);
#pragma unroll
            for (int b = 0; b < BM / 32; ++b)
              if (b < nboxes)
                sm100::tma_load_2d_pair(sa + b * args.a_box_rows * 128,
                                      box_par[b] == 0 ? &tm_a0 : (box_par[b] == 1 ? &tm_a1 : &tm_a2), bar, kb * BK,
                                      box_row[b]);
            sm100::tma_load_3d_pair(sb, &tm_b, bar, kb * BK, b_row, slot);
          }
          if (++stage == TL::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      } else {
      // ===== TMA producer (both CTAs of a pair: own A rows, own half of B) =====
      int stage = 0;
      uint32_t phase = 0;
      for (int t = tile0; t < total_tiles; t += tile_step) {
        TileCoord c = decode_tile<CG>(t, tile_start, args.num_groups, args.groups);
        const coe_mlp_group grp = args.groups[c.g];
        const int m0 = c.m_blk * TL::TILE_M + (int)cta_rank * BM;  // first row of this CTA's half
        int box_row[BM / 32];
        int box_par[BM / 32];
        int nboxes;
        uint32_t a_bytes;
        if (args.mode == 0) {
          const int boff = args.batch_off[grp.batch];
          const int members = grp.rows / args.T;
          if constexpr (CG == 1) {
            const int rows_here = min(grp.rows - m0, BM);
            nboxes = (rows_here + args.a_box_rows - 1) / args.a_box_rows;
          } else {
            nboxes = BM / args.a_box_rows;  // full boxes: the leader expects a fixed byte count
          }
#pragma unroll
          for (int b = 0; b < BM / 32; ++b) {
            if (b >= nboxes) break;
            const int r = m0 + b * args.a_box_rows;
            int j = r / args.T;
            const int within = r - j * args.T;
            j = min(j, members - 1);  // rows past the group (pair tail): any valid member, discarded
            if (args.member_in) {
              const int code = args.member_in[boff + j];
              box_row[b] = (code >> 1) * args.T + within;
              box_par[b] = (code & 1) ? 0 : 1;
            } else {
              box_row[b] = args.member_req[boff + j] * args.T + within;
              box_par[b] = a_source(args.member_stage[boff + j]);
            }
          }
          a_bytes = (uint32_t)(nboxes * args.a_box_rows * BK * 2);
        } else {
          nboxes = 1;
          box_row[0] = grp.h_row + m0;  // past the H scratch end TMA fills zeros (bytes still counted)
          box_par[0] = 0;
          a_bytes = TL::A_BYTES;
        }
        const int b_row = c.n_blk * BN + (int)cta_rank * TL::B_ROWS;
        for (int kb = 0; kb < k_blocks; ++kb) {
          sm100::mbar_wait(&empty_bar[stage], phase ^ 1);
          uint8_t *sa = stage_base + stage * TL::STAGE_BYTES;
          uint8_t *sb = sa + TL::A_BYTES;
          if constexpr (CG == 1) {
            sm100::mbar_arrive_expect_tx(&full_bar[stage], a_bytes + TL::B_BYTES);
#pragma unroll
            for (int b = 0; b < BM / 32; ++b)
              if (b < nboxes)
                sm100::tma_load_2d(sa + b * args.a_box_rows * 128,
                                 box_par[b] == 0 ? &tm_a0 : (box_par[b] == 1 ? &tm_a1 : &tm_a2), &full_bar[stage],
                                 kb * BK, box_row[b]);
            sm100::tma_load_3d(sb, &tm_b, &full_bar[stage], kb * BK, b_row, grp.slot);
          } else {
            const uint32_t bar = sm100::mapa_shared(sm100::smem_u32(&full_bar[stage]), 0);
            if (cta_rank == 0) sm100::mbar_arrive_expect_tx(&full_bar[stage], 2 * TL::STAGE_BYTES);
#pragma unroll
            for (int b = 0; b < BM / 32; ++b)
              if (b < nboxes)
                sm100::tma_load_2d_pair(sa + b * args.a_box_rows * 128,
                                      box_par[b] == 0 ? &tm_a0 : (box_par[b] == 1 ? &tm_a1 : &tm_a2), bar, kb * BK,
                                      box_row[b]);
            sm100::tma_load_3d_pair(sb, &tm_b, bar, kb * BK, b_row, grp.slot);
          }
          if (++stage == TL::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
    }
  } else if (CW && warp == 3) {
    // ===== coordinate warp: resolves each tile's A boxes, weight slot and output rows ahead
    // of the producer and the epilogue (lanes 0-3: one A box / one lane quarter each) =====
    int cs = 0;
    uint32_t cph = 0;
    for (int t = tile0; t < total_tiles; t += tile_step) {
      const TileCoord c = decode_tile<CG>(t, tile_start, args.num_groups, args.groups);
      const coe_mlp_group grp = args.groups[c.g];
      const int m0 = c.m_blk * TL::TILE_M + (int)cta_rank * BM;  // first row of this CTA's half
      const int boff = args.batch_off[grp.batch];
      int nboxes;
      if (args.mode == 0) {
        if constexpr (CG == 1) nboxes = (min(grp.rows - m0, BM) + args.a_box_rows - 1) / args.a_box_rows;
        else nboxes = BM / args.a_box_rows;  // full boxes: the leader expects a fixed byte count
      } else {
        nboxes = 1;
      }
      int brow = 0, bpar = 0;
      __nv_bfloat16 *qbase = nullptr;
      int qvalid = 0;
      if (lane < 4) {
        if (lane < nboxes) {
          if (args.mode == 0) {
            const int members = grp.rows / args.T;
            const int r = m0 + (int)lane * args.a_box_rows;
            int j = r / args.T;
            const int within = r - j * args.T;
            j = min(j, members - 1);  // rows past the group (pair tail): any valid member, discarded
            if (args.member_in) {
              const int code = args.member_in[boff + j];
              brow = (code >> 1) * args.T + within;
              bpar = (code & 1) ? 0 : 1;
            } else {
              brow = args.member_req[boff + j] * args.T + within;
              bpar = a_source(args.member_stage[boff + j]);
            }
          } else {
            brow = grp.h_row + m0;  // past the H scratch end TMA fills zeros (bytes still counted)
          }
        }
        const int row = m0 + (int)lane * 32;  // a 32-row quarter never straddles members (T % 32 == 0)
        qvalid = max(0, min(32, grp.rows - row));
        if (qvalid > 0) {
          if (args.mode == 0) {
            qbase = args.out_h + (size_t)(grp.h_row + row) * args.N;
          } else {
            const int j = row / args.T;
            if (args.member_out) {
              const int code = args.member_out[boff + j];
              const int kind = code & 15;
              __nv_bfloat16 *dst = kind == 0   ? args.out_act0
                                   : kind == 1 ? args.out_y
                                   : kind == 2 ? args.out_stage
                                               : args.peer_act[kind - 3][0];
              qbase = dst + ((size_t)(code >> 4) * args.T + (row - j * args.T)) * args.ld;
            } else {
              const int req = args.member_req[boff + j];
              const int st = args.member_stage[boff + j];
              __nv_bfloat16 *dst = (st & 1) ? args.out_act1 : args.out_act0;
              if (args.hop_dst) {
                const int hd = args.hop_dst[(size_t)req * args.hop_stride + st];
                if (hd >= 0) dst = args.peer_act[hd][st & 1];
              }
              qbase = dst + ((size_t)req * args.T + (row - j * args.T)) * args.ld;
            }
          }
          qbase += c.n_blk * BN;
        }
      }
      sm100::mbar_wait(&crd_empty[cs], cph ^ 1);
      TileCrd &e = crd[cs];
      if (lane < 4) {
        e.box_row[lane] = brow;
        e.box_par[lane] = bpar;
        e.qbase[lane] = qbase;
        e.qvalid[lane] = qvalid;
      }
      if (lane == 0) {
        e.nboxes = nboxes;
        e.slot = grp.slot;
        e.b_row = c.n_blk * BN + (int)cta_rank * TL::B_ROWS;
        e.a_bytes = args.mode == 0 ? (uint32_t)(nboxes * args.a_box_rows * BK * 2) : (uint32_t)TL::A_BYTES;
      }
      __syncwarp();
      if (lane == 0) sm100::mbar_arrive(&crd_full[cs]);
      if (++cs == CRD_STAGES) {
        cs = 0;
        cph ^= 1;
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && cta_rank == 0) {
      // ===== MMA issuer (the leader CTA of a pair issues for both) =====
      constexpr uint32_t idesc = sm100::make_idesc_bf16_f32(TL::TILE_M, BN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = tile0; t < total_tiles; t += tile_step) {
        sm100::mbar_wait(&tempty_bar[acc], acc_phase ^ 1);
        sm100::tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN;
        for (int kb = 0; kb < k_blocks; ++kb) {
          sm100::mbar_wait(&full_bar[stage], phase);
          sm100::tc_fence_after();
          const uint32_t sa = sm100::smem_u32(stage_base + stage * TL::STAGE_BYTES);
          const uint32_t sb = sa + TL::A_BYTES;
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            uint64_t adesc = sm100::make_desc_k_sw128(sa + k * 32);
            uint64_t bdesc = sm100::make_desc_k_sw128(sb + k * 32);
            if constexpr (CG == 1) sm100::mma_bf16_ss(d_tmem, adesc, bdesc, idesc, (kb | k) != 0);
            else sm100::mma_bf16_ss_pair(d_tmem, adesc, bdesc, idesc, (kb | k) != 0);
          }
          if constexpr (CG == 1) sm100::mma_commit(&empty_bar[stage]);
          else sm100::mma_commit_pair(&empty_bar[stage], 0x3);  // frees the stage in both CTAs
          if (++stage == TL::STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        if constexpr (CG == 1) sm100::mma_commit(&tfull_bar[acc]);
        else sm100::mma_commit_pair(&tfull_bar[acc], 0x3);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp >= EPI_WARP0) {
    // ===== epilogue (each CTA drains its own 128 TMEM lanes; warps w and w+4 share a lane
    // quarter and split its 256 columns; TMEM loads run one 32-column chunk ahead) =====
    const uint32_t quarter = warp & 3;
    const int chunk0 = (int)((warp - EPI_WARP0) >> 2) * (BN / 32 / 2);
    uint8_t *my_scratch = epi_scratch + (warp - EPI_WARP0) * EPI_SCRATCH;
    constexpr int CHUNKS = BN / 32 / 2;
    const uint32_t tempty_leader = CG == 2 ? sm100::mapa_shared(sm100::smem_u32(&tempty_bar[0]), 0) : 0;
    const size_t out_stride = args.mode == 0 ? (size_t)args.N : (size_t)args.ld;
    int acc = 0;
    uint32_t acc_phase = 0;
    int cs = 0;
    uint32_t cph = 0;
    for (int t = tile0; t < total_tiles; t += tile_step) {
      bool valid;
      __nv_bfloat16 *out_row = nullptr;
      if constexpr (CW) {
        sm100::mbar_wait(&crd_full[cs], cph);
        valid = (int)lane < crd[cs].qvalid[quarter];
        if (valid) out_row = crd[cs].qbase[quarter] + lane * out_stride;
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive(&crd_empty[cs]);
        if (++cs == CRD_STAGES) {
          cs = 0;
          cph ^= 1;
        }
      } else {
      TileCoord c = decode_tile<CG>(t, tile_start, args.num_groups, args.groups);
      const coe_mlp_group grp = args.groups[c.g];
      const int row = c.m_blk * TL::TILE_M + (int)cta_rank * BM + quarter * 32 + lane;
      valid = row < grp.rows;
      if (valid) {
        if (args.mode == 0) {
          out_row = args.out_h + (size_t)(grp.h_row + row) * args.N;
        } else {
          const int boff = args.batch_off[grp.batch];
          const int j = row / args.T;
          if (args.member_out) {
            const int code = args.member_out[boff + j];
            const int kind = code & 15;
            __nv_bfloat16 *dst = kind == 0   ? args.out_act0
                                 : kind == 1 ? args.out_y
                                 : kind == 2 ? args.out_stage
                                             : args.peer_act[kind - 3][0];
            out_row = dst + ((size_t)(code >> 4) * args.T + (row - j * args.T)) * args.ld;
          } else {
            const int req = args.member_req[boff + j];
            const int st = args.member_stage[boff + j];
            __nv_bfloat16 *dst = (st & 1) ? args.out_act1 : args.out_act0;
            if (args.hop_dst) {
              const int hd = args.hop_dst[(size_t)req * args.hop_stride + st];
              if (hd >= 0) dst = args.peer_act[hd][st & 1];
            }
            out_row = dst + ((size_t)req * args.T + (row - j * args.T)) * args.ld;
          }
        }
        out_row += c.n_blk * BN;
      }
      }
      sm100::mbar_wait(&tfull_bar[acc], acc_phase);
      sm100::tc_fence_after();
      // coalesced stores: each lane holds one row's 32 columns (64 B); the chunk is staged in the
      // warp's scratch (16 B units XOR-swizzled by row: conflict-free both ways) and written back
      // as 8 rows x 64 B per store instruction -- full 32 B sectors instead of 32 rows x 16 B
      if (!valid) out_row = nullptr;
      uint64_t row_ptr[4];  // rows it * 8 + lane / 4 of this quarter (null: outside the group)
#pragma unroll
      for (int it = 0; it < 4; ++it)
        row_ptr[it] = __shfl_sync(0xffffffffu, reinterpret_cast<uint64_t>(out_row), it * 8 + (int)(lane >> 2));
      const uint32_t piece = lane & 3;
      const uint32_t taddr = tmem_base + ((quarter * 32) << 16) + acc * BN;
      uint32_t v[2][32];
      sm100::tmem_ld_32x32b_x32(taddr + chunk0 * 32, v[0]);
      sm100::tmem_ld_wait_regs(v[0]);
#pragma unroll
      for (int k = 0; k < CHUNKS; ++k) {
        uint32_t(&cur)[32] = v[k & 1];
        if (k + 1 < CHUNKS) sm100::tmem_ld_32x32b_x32(taddr + (chunk0 + k + 1) * 32, v[(k + 1) & 1]);
        if (!(args.debug & 1)) {
          uint32_t packed[16];
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            float lo = __uint_as_float(cur[2 * i]);
            float hi = __uint_as_float(cur[2 * i + 1]);
            if (args.mode == 0 && !(args.debug & 2)) {
              lo = gelu_tanh(lo);
              hi = gelu_tanh(hi);
            }
            packed[i] = pack_bf16(lo, hi);
          }
          const uint32_t sw = (lane >> 1) & 3;
#pragma unroll
          for (int i = 0; i < 4; ++i)
            *reinterpret_cast<uint4 *>(my_scratch + lane * 64 + ((i ^ sw) << 4)) =
                make_uint4(packed[4 * i], packed[4 * i + 1], packed[4 * i + 2], packed[4 * i + 3]);
          __syncwarp();
#pragma unroll
          for (int it = 0; it < 4; ++it) {
            const uint32_t rr = it * 8 + (lane >> 2);
            if (row_ptr[it]) {
              const uint4 val = *reinterpret_cast<const uint4 *>(my_scratch + rr * 64 + ((piece ^ ((rr >> 1) & 3)) << 4));
              reinterpret_cast<uint4 *>(reinterpret_cast<__nv_bfloat16 *>(row_ptr[it]) + (chunk0 + k) * 32)[piece] = val;
            }
          }
          __syncwarp();
        }
        if (k + 1 < CHUNKS) sm100::tmem_ld_wait_regs(v[(k + 1) & 1]);
      }
      sm100::tc_fence_before();
      if constexpr (CG == 1) {
        sm100::mbar_arrive(&tempty_bar[acc]);
      } else {
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive_cluster(tempty_leader + acc * 8);  // the leader's tempty[acc]
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
  }

  sm100::tc_fence_before();
  if constexpr (CG == 2) sm100::cluster_sync();  // no CTA leaves while its peer may still signal it
  else __syncthreads();
  if (warp == 2) {
    sm100::tc_fence_after();
    sm100::tmem_dealloc<TMEM_COLS, CG>(tmem_base);
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
bool make_map_3d(CUtensorMap *map, void *base, uint64_t slots, uint64_t rows, uint64_t cols, uint64_t slot_stride,
                 uint32_t box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[3] = {cols, rows, slots};
  cuuint64_t strides[2] = {cols * 2, slot_stride};
  cuuint32_t box[3] = {BK, box_rows, 1};
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
  int cg = 2;                        // CTAs per MMA (COE_K3_CG=1 selects the single-CTA kernel)
  int cw = -1;  // coordinate warp: -1 auto (up passes with K <= 2048: +6-10 %; elsewhere -1-3 %,
                // profiles/r2o_k3_coord_ab.json), 0 / 1 forced by COE_K3_COORD
  CUtensorMap xmap_alt;              // stage-0 inputs from a second X buffer (coe_mlp_set_input)
  const void *x_alt = nullptr;
  bool use_alt = false;
  const int8_t *hop_dst = nullptr;   // fused hops (coe_mlp_set_hops)
  int hop_stride = 0;
  __nv_bfloat16 *peer_act[COE_MAX_PEERS][2] = {};
  __nv_bfloat16 *out_y = nullptr, *out_stage = nullptr;  // routed mode (coe_mlp_set_outputs)
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
  if (const char *v = getenv("COE_K3_CG")) m->cg = atoi(v) == 1 ? 1 : 2;
  if (const char *v = getenv("COE_K3_COORD")) m->cw = atoi(v) != 0 ? 1 : 0;
  m->a_box_rows = cfg->T < BM ? cfg->T : BM;
  bool ok = true;
  const uint64_t ld = cfg->act_ld > 0 ? (uint64_t)cfg->act_ld : (uint64_t)cfg->d;
  const uint64_t x_rows = cfg->x_rows > 0 ? (uint64_t)cfg->x_rows : (uint64_t)cfg->act_rows;
  ok &= make_map_2d(&m->xmap, cfg->x, x_rows, cfg->d, m->a_box_rows, ld);
  ok &= make_map_2d(&m->act0, cfg->act0, (uint64_t)cfg->act_rows, cfg->d, m->a_box_rows, ld);
  ok &= make_map_2d(&m->act1, cfg->act1, (uint64_t)cfg->act_rows, cfg->d, m->a_box_rows, ld);
  ok &= make_map_2d(&m->hmap, cfg->h_scratch, (uint64_t)cfg->h_rows, cfg->h, BM);
  // slot layout: [W1: h x d][W2: d x h]
  // B box: the whole 256-column n-block (1 CTA) or each pair CTA's half of it
  const uint32_t b_rows = (uint32_t)(BN / m->cg);
  ok &= make_map_3d(&m->w1, cfg->slab, cfg->num_slots, cfg->h, cfg->d, cfg->slot_stride_bytes, b_rows);
  ok &= make_map_3d(&m->w2, (char *)cfg->slab + (size_t)cfg->h * cfg->d * 2, cfg->num_slots, cfg->d, cfg->h,
                    cfg->slot_stride_bytes, b_rows);
  if (!ok) {
    delete m;
    coe_set_error("cuTensorMapEncodeTiled failed (alignment / driver entry point)");
    return COE_CUDA_ERR_CUDA;
  }
  int dev = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&m->num_sms, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e = cudaSuccess;
  for (cudaError_t r : {cudaFuncSetAttribute(grouped_gemm_kernel<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             Tiling<1>::SMEM),
                        cudaFuncSetAttribute(grouped_gemm_kernel<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             Tiling<1>::SMEM),
                        cudaFuncSetAttribute(grouped_gemm_kernel<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             Tiling<2>::SMEM),
                        cudaFuncSetAttribute(grouped_gemm_kernel<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             Tiling<2>::SMEM)})
    if (r != cudaSuccess) e = r;
  if (e != cudaSuccess) {
    delete m;
    coe_set_error(std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
    return COE_CUDA_ERR_CUDA;
  }
  *out = m;
  return COE_CUDA_OK;
}

void coe_mlp_destroy(coe_mlp *m) { delete m; }

int coe_mlp_set_input(coe_mlp *m, void *x) {
  if (!x || x == m->cfg.x) {
    m->use_alt = false;
    return COE_CUDA_OK;
  }
  if (x != m->x_alt) {
    const uint64_t ld = m->cfg.act_ld > 0 ? (uint64_t)m->cfg.act_ld : (uint64_t)m->cfg.d;
    const uint64_t x_rows = m->cfg.x_rows > 0 ? (uint64_t)m->cfg.x_rows : (uint64_t)m->cfg.act_rows;
    if (!make_map_2d(&m->xmap_alt, x, x_rows, m->cfg.d, m->a_box_rows, ld)) {
      coe_set_error("coe_mlp_set_input: cuTensorMapEncodeTiled failed");
      return COE_CUDA_ERR_CUDA;
    }
    m->x_alt = x;
  }
  m->use_alt = true;
  return COE_CUDA_OK;
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
      m->peer_act[r][b] = (peer_act && r < world) ? static_cast<__nv_bfloat16 *>(peer_act[2 * r + b]) : nullptr;
  return COE_CUDA_OK;
}

int coe_mlp_set_outputs(coe_mlp *m, void *y, void *out_stage) {
  m->out_y = static_cast<__nv_bfloat16 *>(y);
  m->out_stage = static_cast<__nv_bfloat16 *>(out_stage);
  return COE_CUDA_OK;
}

static int launch_grouped(coe_mlp *m, const coe_mlp_group *groups_up, const coe_mlp_group *groups_down, int num_groups,
                          int tiles_up, int tiles_down, const int32_t *batch_off, const int32_t *member_req,
                          const int32_t *member_stage, const int32_t *member_in, const int32_t *member_out,
                          int which, int max_ctas, cudaStream_t stream);

int coe_grouped_mlp(coe_mlp *m, const coe_mlp_group *groups_up, const coe_mlp_group *groups_down, int num_groups,
                    int tiles_up, int tiles_down, const int32_t *batch_off, const int32_t *member_req,
                    const int32_t *member_stage, int which, int max_ctas, cudaStream_t stream) {
  return launch_grouped(m, groups_up, groups_down, num_groups, tiles_up, tiles_down, batch_off, member_req,
                        member_stage, nullptr, nullptr, which, max_ctas, stream);
}

int coe_grouped_mlp_routed(coe_mlp *m, const coe_mlp_group *groups_up, const coe_mlp_group *groups_down,
                           int num_groups, int tiles_up, int tiles_down, const int32_t *batch_off,
                           const int32_t *member_in, const int32_t *member_out, int which, int max_ctas,
                           cudaStream_t stream) {
  if (!member_in || !member_out) {
    coe_set_error("coe_grouped_mlp_routed: member routes required");
    return COE_CUDA_ERR_CONFIG;
  }
  return launch_grouped(m, groups_up, groups_down, num_groups, tiles_up, tiles_down, batch_off, nullptr, nullptr,
                        member_in, member_out, which, max_ctas, stream);
}

static int launch_grouped(coe_mlp *m, const coe_mlp_group *groups_up, const coe_mlp_group *groups_down, int num_groups,
                          int tiles_up, int tiles_down, const int32_t *batch_off, const int32_t *member_req,
                          const int32_t *member_stage, const int32_t *member_in, const int32_t *member_out,
                          int which, int max_ctas, cudaStream_t stream) {
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
    a.hop_dst = (pass == 1 && !member_in) ? m->hop_dst : nullptr;
    a.hop_stride = m->hop_stride;
    std::memcpy(a.peer_act, m->peer_act, sizeof(a.peer_act));
    a.member_in = member_in;
    a.member_out = member_out;
    a.out_y = m->out_y;
    a.out_stage = m->out_stage;
    a.debug = getenv("COE_K3_DEBUG") ? atoi(getenv("COE_K3_DEBUG")) : 0;
    if (a.total_tiles <= 0) continue;
    int cap = (max_ctas > 0 && max_ctas < m->num_sms) ? max_ctas : m->num_sms;
    const CUtensorMap &ta0 = pass == 0 ? (m->use_alt ? m->xmap_alt : m->xmap) : m->hmap, &ta1 = pass == 0 ? m->act0 : m->hmap,
                      &ta2 = pass == 0 ? (member_in ? m->act0 : m->act1) : m->hmap, &tb = pass == 0 ? m->w1 : m->w2;
    cudaError_t e;
    const bool cw = m->cw >= 0 ? m->cw == 1 : (pass == 0 && a.K <= 2048);
    if (m->cg == 1) {
      const int grid = a.total_tiles < cap ? a.total_tiles : cap;
      if (cw) grouped_gemm_kernel<1, true><<<grid, NUM_THREADS, Tiling<1>::SMEM, stream>>>(ta0, ta1, ta2, tb, a);
      else grouped_gemm_kernel<1, false><<<grid, NUM_THREADS, Tiling<1>::SMEM, stream>>>(ta0, ta1, ta2, tb, a);
      e = cudaGetLastError();
    } else {
      // pairs: at most one per 128-row tile (the kernel recounts 256-row pair tiles itself)
      const int pairs = std::max(1, std::min(cap / 2, a.total_tiles));
      cudaLaunchConfig_t lc{};
      lc.gridDim = dim3(2 * pairs);
      lc.blockDim = dim3(NUM_THREADS);
      lc.dynamicSmemBytes = Tiling<2>::SMEM;
      lc.stream = stream;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = 2;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      lc.attrs = attr;
      lc.numAttrs = 1;
      e = cw ? cudaLaunchKernelEx(&lc, grouped_gemm_kernel<2, true>, ta0, ta1, ta2, tb, a)
                : cudaLaunchKernelEx(&lc, grouped_gemm_kernel<2, false>, ta0, ta1, ta2, tb, a);
    }
    if (e != cudaSuccess) {
      coe_set_error(std::string("grouped_gemm_kernel launch: ") + cudaGetErrorString(e));
      return COE_CUDA_ERR_CUDA;
    }
  }
  return COE_CUDA_OK;
}

}  // extern "C"
