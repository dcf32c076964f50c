// F1 -- B200 fp32 SIMT family (KP_FAMILY_SIMT): the paper's 640-config parameter
// space (dataset.py:41-46) re-instantiated B200-first.
//
// What a config means here (same 5-tuple, same per-work-item contract):
//   * each thread (work item) owns an R x C output tile and accumulates it in
//     registers, stepping k by A: per step it reads an R x A LHS fragment (R vector
//     loads of width A along k) and an A x C RHS fragment (A vector loads of width
//     min(C,4) along n) -- from shared memory instead of global memory;
//   * the CTA is the work group: wg_rows x wg_cols threads, CTA tile
//     BM = R*wg_rows by BN = C*wg_cols, grid = work_items() geometry
//     (dataset.py:312-316) with the m-groups in gridDim.x.
// B200-specific choices (not tunables; derived from the tuple at compile time):
//   * global -> shared staging with cp.async (LDGSTS) 16-byte zero-filling copies
//     (4-byte copies when a row is not 16-byte aligned, e.g. k = 27 or 147), in a
//     STAGES-deep ring (2..4) sized so the occupancy target below fits in 227 KB;
//   * stage depth BK in {32,16,8}: the largest that fits two stages in the budget;
//   * warp tiling: lanes form a WTR x WTC patch of the work group chosen to minimise
//     the per-warp operand footprint WTR*R + WTC*C, so shared-memory reads are
//     broadcast across the patch and conflict-free (padded LHS rows, RHS columns
//     interleaved in float4 groups);
//   * tails by zero-fill: out-of-range rows/cols/k land as zeros in shared memory and
//     contribute fma(0, 0, acc) == acc exactly.
// Every output element is the sequential fp32 fma chain over k = 0..K-1, so F1 is
// bit-identical to F0 and to the oracle (oracle/gemm_ref.c).
#pragma once

#include <cooperative_groups.h>
#include <cuda.h>

#include <cstring>

#include "common.cuh"
#include "families.h"

namespace kp {

// ---- TMA staging (bulk tensor copies + mbarrier) -----------------------------
// The operand tensor maps of one launch (unused by the cp.async path).
struct F1Maps {
  CUtensorMap a, b;
  FastDiv cw, ch, cc;  // implicit conv: division by the image width, height and channels
};

__device__ __forceinline__ uint32_t f1_smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void f1_mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(f1_smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void f1_mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(f1_smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void f1_mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "KP_F1_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra KP_F1_WAIT_%=;\n"
      "}\n" ::"r"(f1_smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void f1_tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y,
                                               int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::
          "r"(f1_smem_u32(dst)),
      "l"(map), "r"(f1_smem_u32(bar)), "r"(x), "r"(y), "r"(z)
      : "memory");
}

// TMA im2col copy: pixelsPerColumn consecutive output pixels (w fastest, then h, then
// image) starting at base pixel (w, h, n) of the map's bounding box, each contributing
// channelsPerPixel channels from c of input pixel (w + dx, h + dy); zero outside.
__device__ __forceinline__ void f1_tma_im2col_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c, int w,
                                                 int h, int n, uint16_t dx, uint16_t dy) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, "
      "%6}], [%2], {%7, %8};" ::"r"(f1_smem_u32(dst)),
      "l"(map), "r"(f1_smem_u32(bar)), "r"(c), "r"(w), "r"(h), "r"(n), "h"(dx), "h"(dy)
      : "memory");
}

constexpr int f1_pick_wtc(int R, int C, int WGR, int WGC) {
  int best = -1, best_cost = 1 << 30;
  for (int wtc = 1; wtc <= 32; wtc *= 2) {
    const int wtr = 32 / wtc;
    if (WGC % wtc != 0 || WGR % wtr != 0) continue;
    const int cost = wtr * R + wtc * C;
    if (cost <= best_cost) {  // ties go to the wider (store-coalescing) patch
      best_cost = cost;
      best = wtc;
    }
  }
  return best;
}

template <int R, int A, int C, int WGR, int WGC>
struct F1Cfg {
  static constexpr int NT = WGR * WGC;
  static constexpr int BM = R * WGR;
  static constexpr int BN = C * WGC;
  static constexpr int VC = C < 4 ? C : 4;
  static constexpr int PADA = 4;
  // Occupancy target: >= 16 resident warps per SM (4 per scheduler) so FFMA2 issue
  // hides LDS latency.  MIN_BLOCKS feeds __launch_bounds__ (caps registers at
  // 65536 / (MIN_BLOCKS * NT)) and the per-CTA shared-memory budget.
#ifndef KP_F1_WARPS
#define KP_F1_WARPS 16
#endif
  static constexpr int MIN_BLOCKS = (KP_F1_WARPS * 32 / NT) > 1 ? (KP_F1_WARPS * 32 / NT) : 1;
  static constexpr int stage_floats(int bk) { return BM * (bk + PADA) + bk * BN; }
  // Stage depth BK comes from a budget of up to 4 CTAs per SM; 64-thread work groups then
  // take the 8-CTA budget (their full 16-warp target) when two stages of that BK still fit
  // in it -- measured +2..17 % on those configs, while shrinking BK to fit 8 CTAs lost up
  // to 2x (profiles/r2/occupancy_budget_ab.md).
  static constexpr int budget_for(int ctas) {
    return (227 * 1024) / (MIN_BLOCKS < ctas ? MIN_BLOCKS : ctas) - 1024;
  }
  static constexpr int kBudget4 = budget_for(4);
#ifndef KP_F1_MAX_BK
#define KP_F1_MAX_BK 32
#endif
  static constexpr int BK = (KP_F1_MAX_BK >= 32 && 2 * 4 * stage_floats(32) <= kBudget4)   ? 32
                            : (KP_F1_MAX_BK >= 16 && 2 * 4 * stage_floats(16) <= kBudget4) ? 16
                                                                                         : 8;
#ifndef KP_F1_MAX_CTAS
#define KP_F1_MAX_CTAS 8
#endif
  static constexpr int kBudget =
      2 * 4 * stage_floats(BK) <= budget_for(KP_F1_MAX_CTAS) ? budget_for(KP_F1_MAX_CTAS) : kBudget4;
  static constexpr int SA = BK + PADA;  // LHS smem row stride (floats)
  static constexpr int SB = BN;         // RHS smem row stride (floats)
  static constexpr int STAGE = stage_floats(BK);
  static constexpr int STAGES_FIT = kBudget / (4 * STAGE);
  static constexpr int STAGES = STAGES_FIT < 2 ? 2 : (STAGES_FIT > 4 ? 4 : STAGES_FIT);
  static constexpr int SMEM_BYTES = STAGES * STAGE * 4;
  // k-sliced launches park the fp32 partial tile (row stride SP) in shared memory.
  // (padded, and keeping each thread's VC-wide stores aligned).
  static constexpr int SP = BN % 4 == 0 ? BN + 4 : (BN % 2 == 0 ? BN + 2 : BN + 1);
  static constexpr int SLICE_SMEM_BYTES = SMEM_BYTES > BM * SP * 4 ? SMEM_BYTES : BM * SP * 4;
  static constexpr int WTC = f1_pick_wtc(R, C, WGR, WGC);
  static constexpr int WTR = 32 / WTC;
  static constexpr int WPC = WGC / WTC;  // warps across the work-group columns
  // Shared-memory wavefronts (measured): an LDS.64/128 costs half
  // when each pair of adjacent lanes reads the same address.  Only one operand can be
  // pair-shared in an outer-product warp tile, so pair the lanes on the operand with
  // more floats per thread per k-step: the LHS (R floats, if read as >= 2-wide vectors)
  // or the RHS (C floats, if VC >= 2).
  static constexpr int COST_PAIR_A = (A >= 2 && WTC >= 2 ? R : 2 * R) + 2 * C;  // in half-wavefronts
  static constexpr int COST_PAIR_B = 2 * R + (VC >= 2 && WTR >= 2 ? C : 2 * C);
  // Measured: only worth it for LDS.128 RHS fragments (VC == 4); with 8-byte RHS reads
  // the row-fastest lane order costs more in the epilogue than it saves.
  static constexpr bool PAIR_B = VC == 4 && COST_PAIR_B < COST_PAIR_A;
  static constexpr bool B_CHUNKS = (BN % 4) == 0;
  // TMA staging variant: the same smem layout (LHS rows padded to SA floats, RHS rows
  // of BN floats) written by bulk tensor copies -- the LHS box is SA = BK + 4 floats
  // wide, so the pad columns arrive as the next k-tile's first floats (never read) and
  // the padded layout needs no swizzle.  Boxes are <= 256 rows; the RHS box is one
  // BN-wide row block, so TMA staging needs BN <= 256 and BN % 4 == 0.
  static constexpr int A_BOX_ROWS = BM < 256 ? BM : 256;
  static constexpr int A_BOXES = (BM + A_BOX_ROWS - 1) / A_BOX_ROWS;
  static constexpr int T_B_OFF = (BM * SA + 31) / 32 * 32;  // floats; 128-byte aligned RHS
  static constexpr int T_STAGE = (T_B_OFF + BK * BN + 31) / 32 * 32;
  static constexpr int T_TX_BYTES = 4 * (A_BOXES * A_BOX_ROWS * SA + BK * BN);
  static constexpr bool TMA_OK = B_CHUNKS && BN <= 256;
  // full barriers and arrival counters sit past both the ring and the sliced launches'
  // partial tile (which reuses the ring); +128 bytes to align the dynamic base
  static constexpr int T_BAR_OFF = ((STAGES * T_STAGE > BM * SP ? STAGES * T_STAGE : BM * SP) * 4 + 15) / 16 * 16;
  static constexpr int T_SMEM_BYTES = T_BAR_OFF + STAGES * 12 + 128;
  static_assert(WTC > 0, "work group not tileable by warps");
  static_assert(NT % 32 == 0, "work group must be whole warps");
  static_assert(BK % A == 0, "stage depth must be a multiple of A");
  static_assert(SMEM_BYTES <= 227 * 1024, "shared memory");
};

// Cluster reduction of a k-sliced tile: CTA rank z of the (1, 1, kslices) cluster
// owns elements [z*chunk, (z+1)*chunk) of the BM x BN tile (flat, row-major) and sums
// them over every rank's shared-memory partial (DSMEM loads) in rank order.
template <int BM, int BN, int SP, int NT>
__device__ __forceinline__ void f1_slice_reduce(const GemmArgs& p, float* smem, float* Cb, int64_t m0, int64_t n0) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();  // every slice's partial is in place
  const int S = p.kslices;
  const int z = static_cast<int>(cl.block_rank());
  // rank s's partial tile, as a generic pointer into its shared memory (mapa)
  auto part = [&](int s) -> const float* { return cl.map_shared_rank(smem, s); };
  const int m = p.m, n = p.n;
  if constexpr (BN % 4 == 0) {
    constexpr int Q = BN / 4, TOT = BM * Q;
    const int chunk = (TOT + S - 1) / S;
    const int end = min(TOT, (z + 1) * chunk);
    for (int i = z * chunk + static_cast<int>(threadIdx.x); i < end; i += NT) {
      const int r = i / Q, c = (i - r * Q) * 4;
      const int64_t row = m0 + r, col = n0 + c;
      if (row >= m || col >= n) continue;
      float4 v = *reinterpret_cast<const float4*>(part(0) + r * SP + c);
      for (int s = 1; s < S; ++s) {
        const float4 w = *reinterpret_cast<const float4*>(part(s) + r * SP + c);
        v.x = v.x + w.x; v.y = v.y + w.y; v.z = v.z + w.z; v.w = v.w + w.w;
      }
      float o[4] = {v.x, v.y, v.z, v.w};
      float* out = Cb + row * p.ldc + col;
      if (p.bias || p.relu) epilogue_run<4>(p, o, col);
      if (p.c_vec4 && col + 4 <= n) {
        stg_vec<4>(out, o);
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (col + e < n) out[e] = o[e];
      }
    }
  } else {
    constexpr int TOT = BM * BN;
    const int chunk = (TOT + S - 1) / S;
    const int end = min(TOT, (z + 1) * chunk);
    for (int i = z * chunk + static_cast<int>(threadIdx.x); i < end; i += NT) {
      const int r = i / BN, c = i - r * BN;
      const int64_t row = m0 + r, col = n0 + c;
      if (row >= m || col >= n) continue;
      float v = part(0)[r * SP + c];
      for (int s = 1; s < S; ++s) v = v + part(s)[r * SP + c];
      if (p.bias || p.relu) v = epilogue(p, v, col);
      Cb[row * p.ldc + col] = v;
    }
  }
  cl.sync();  // keep this CTA's partial alive until every rank has read it
}

// TMA = false: every thread stages its share of each k-tile with cp.async and the CTA
// syncs once per k-tile.  TMA = true (16-byte-aligned operand rows, BN <= 256): bulk
// tensor copies fill the same layout; each stage has a full mbarrier (the copies'
// transaction bytes) and an arrival counter -- every warp waits on the stage's barrier,
// runs its outer products, and its lane 0 counts the stage as consumed; the warp that
// completes the count refills the stage with the k-tile STAGES ahead.  No CTA-wide
// barrier and no per-thread copy address math in the main loop.
// MODE: 0 = cp.async staging, 1 = TMA staging, 2 = TMA staging of an implicit conv (the
// im2col issue code is compiled only into this instance, so the GEMM instances keep their
// register allocation)
template <int R, int A, int C, int WGR, int WGC, int MODE>
__global__ void __launch_bounds__(WGR * WGC, F1Cfg<R, A, C, WGR, WGC>::MIN_BLOCKS)
    f1_kernel(GemmArgs p, int groups_n, const __grid_constant__ F1Maps maps) {
  using Cfg = F1Cfg<R, A, C, WGR, WGC>;
  constexpr bool TMA = MODE != 0, CONV = MODE == 2;
  constexpr int NT = Cfg::NT, BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK;
  constexpr int SA = Cfg::SA, SB = Cfg::SB, STAGES = Cfg::STAGES, VC = Cfg::VC;
  extern __shared__ __align__(16) float smem_dyn[];
  float* smem = smem_dyn;
  if constexpr (TMA) {  // bulk tensor copies need 128-byte-aligned destinations
    const uint32_t s0 = f1_smem_u32(smem_dyn);
    smem = smem_dyn + (((s0 + 127u) & ~127u) - s0) / 4;
  }

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  // lane -> (row, col) inside the warp tile: adjacent lanes share the paired operand
  const int lr = Cfg::PAIR_B ? lane % Cfg::WTR : lane / Cfg::WTC;
  const int lc = Cfg::PAIR_B ? lane / Cfg::WTR : lane % Cfg::WTC;
  // Warp-blocked ownership: warp (wy, wx) owns the contiguous R*WTR x C*WTC block at
  // (wrow0, wcol0); inside it lane (lr, lc) takes rows wrow0 + r*WTR + lr and float-vector
  // columns wcol0 + cv*WTC*VC + lc*VC.  Same shared-memory access pattern as a strided
  // mapping (consecutive rows / consecutive vectors across the patch), but a tail tile's
  // rows or columns beyond the problem land in whole warps, which then skip the math.
  const int wrow0 = (warp / Cfg::WPC) * (R * Cfg::WTR);
  const int wcol0 = (warp % Cfg::WPC) * (C * Cfg::WTC);
  auto trow = [&](int r) { return wrow0 + r * Cfg::WTR + lr; };
  auto tcol = [&](int cv) { return wcol0 + cv * Cfg::WTC * VC + lc * VC; };

  const int64_t gm = blockIdx.x / groups_n;
  const int gn = blockIdx.x - static_cast<int>(gm * groups_n);
  const int b = blockIdx.y;
  const int m = p.m, k = p.k, n = p.n;
  const int64_t m0 = gm * BM;
  const int64_t n0 = static_cast<int64_t>(gn) * BN;
  const bool warp_live = wrow0 < m - m0 && wcol0 < n - n0;

  const float* __restrict__ Ab = static_cast<const float*>(p.A) + b * p.sA;
  const float* __restrict__ Bb = static_cast<const float*>(p.B) + b * p.sB;
  float* __restrict__ Cb = static_cast<float*>(p.C) + b * p.sC;
  const int64_t lda = p.lda, ldb = p.ldb;
  const bool a16 = p.a_vec, b16 = Cfg::B_CHUNKS && p.b_vec;

  auto load_tile = [&](int stage, int kt) {
    float* as = smem + stage * Cfg::STAGE;
    float* bs = as + BM * SA;
    const int k0 = kt * BK;
    if (a16) {
      constexpr int CPR = BK / 4, CH = BM * CPR;
#pragma unroll
      for (int j = 0; j < (CH + NT - 1) / NT; ++j) {
        const int c = tid + j * NT;
        if (CH % NT == 0 || c < CH) {
          const int r = c / CPR, q = c - r * CPR;
          const int64_t gr = m0 + r;
          const int gk = k0 + q * 4;
          const bool ok = gr < m && gk < k;
          cp_async16(as + r * SA + q * 4, ok ? Ab + gr * lda + gk : Ab, ok ? 16 : 0);
        }
      }
    } else {
      constexpr int EL = BM * BK;
#pragma unroll 4
      for (int j = 0; j < (EL + NT - 1) / NT; ++j) {
        const int e = tid + j * NT;
        if (EL % NT == 0 || e < EL) {
          const int r = e / BK, q = e - r * BK;
          const int64_t gr = m0 + r;
          const int gk = k0 + q;
          const bool ok = gr < m && gk < k;
          cp_async4(as + r * SA + q, ok ? Ab + gr * lda + gk : Ab, ok ? 4 : 0);
        }
      }
    }
    if (b16) {
      constexpr int CPR = BN / 4 > 0 ? BN / 4 : 1, CH = BK * CPR;
#pragma unroll
      for (int j = 0; j < (CH + NT - 1) / NT; ++j) {
        const int c = tid + j * NT;
        if (CH % NT == 0 || c < CH) {
          const int r = c / CPR, q = c - r * CPR;
          const int gk = k0 + r;
          const int64_t gc = n0 + q * 4;
          const bool ok = gk < k && gc < n;
          cp_async16(bs + r * SB + q * 4, ok ? Bb + static_cast<int64_t>(gk) * ldb + gc : Bb, ok ? 16 : 0);
        }
      }
    } else {
      constexpr int EL = BK * BN;
#pragma unroll 4
      for (int j = 0; j < (EL + NT - 1) / NT; ++j) {
        const int e = tid + j * NT;
        if (EL % NT == 0 || e < EL) {
          const int r = e / BN, q = e - r * BN;
          const int gk = k0 + r;
          const int64_t gc = n0 + q;
          const bool ok = gk < k && gc < n;
          cp_async4(bs + r * SB + q, ok ? Bb + static_cast<int64_t>(gk) * ldb + gc : Bb, ok ? 4 : 0);
        }
      }
    }
  };

  // Accumulators as column pairs: the outer product a[r] * w[c:c+2] maps onto one
  // FFMA2 (sm_100 packed fp32 FMA, scalar-broadcast first operand) -- half the issue
  // slots of scalar FFMA and the same per-lane IEEE fma, so results stay bit-exact.
  constexpr int CP = (C + 1) / 2;
  float2 acc[R][CP];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < CP; ++c) acc[r][c] = make_float2(0.0f, 0.0f);

  // This CTA's k-tiles: all of them, or slice blockIdx.z of a k-sliced launch.
  const int KTall = (k + BK - 1) / BK;
  const int kt0 = static_cast<int>(blockIdx.z) * p.kt_per_slice;
  const int KT = min(KTall - kt0, p.kt_per_slice);

  // The outer products of one staged k-tile (both staging paths share the layout).
  auto tile_math = [&](const float* as, const float* bs) {
#pragma unroll
    for (int kk = 0; kk < BK; kk += A) {
      float a[R][A];
#pragma unroll
      for (int r = 0; r < R; ++r) lds_vec<A>(as + trow(r) * SA + kk, a[r]);
#pragma unroll
      for (int i = 0; i < A; ++i) {
        float w[C];
#pragma unroll
        for (int cv = 0; cv < C / VC; ++cv) lds_vec<VC>(bs + (kk + i) * SB + tcol(cv), w + cv * VC);
        if constexpr (C == 1) {
#pragma unroll
          for (int r = 0; r < R; ++r) acc[r][0].x = __fmaf_rn(a[r][i], w[0], acc[r][0].x);
        } else {
#pragma unroll
          for (int r = 0; r < R; ++r)
#pragma unroll
            for (int c = 0; c < CP; ++c)
              acc[r][c] = __ffma2_rn(make_float2(a[r][i], a[r][i]), make_float2(w[2 * c], w[2 * c + 1]), acc[r][c]);
        }
      }
    }
  };

  if constexpr (TMA) {
    constexpr int NW = NT / 32;
    uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<char*>(smem) + Cfg::T_BAR_OFF);
    int* consumed = reinterpret_cast<int*>(full + STAGES);
    const int za = (p.batch > 1 && p.sA != 0) ? b : 0;
    const int zb = (p.batch > 1 && p.sB != 0) ? b : 0;
    auto issue = [&](int stage, int kt) {  // one thread: the k-tile's boxes into a stage
      float* as = smem + stage * Cfg::T_STAGE;
      f1_mbar_expect_tx(&full[stage], Cfg::T_TX_BYTES);
      if constexpr (CONV) {
        // implicit conv: k-tile kt lies inside one filter tap (conv_c % BK == 0)
        // (host-built reciprocals: no integer division on the issuing lane)
        const int k0 = kt * BK, tap = maps.cc.div(k0), c0 = k0 - tap * p.conv_c;
        const uint16_t dy = static_cast<uint16_t>(tap / 3), dx = static_cast<uint16_t>(tap - 3 * (tap / 3));
#pragma unroll
        for (int i = 0; i < Cfg::A_BOXES; ++i) {
          const int r = static_cast<int>(m0) + i * Cfg::A_BOX_ROWS;
          const int t = maps.cw.div(r), w = r - t * p.conv_w;
          const int img = maps.ch.div(t), h = t - img * p.conv_h;
          f1_tma_im2col_4d(as + i * Cfg::A_BOX_ROWS * SA, &maps.a, &full[stage], c0, w - 1, h - 1, img, dx, dy);
        }
      } else {
#pragma unroll
        for (int i = 0; i < Cfg::A_BOXES; ++i)
          f1_tma_load_3d(as + i * Cfg::A_BOX_ROWS * SA, &maps.a, &full[stage], kt * BK,
                         static_cast<int>(m0) + i * Cfg::A_BOX_ROWS, za);
      }
      f1_tma_load_3d(as + Cfg::T_B_OFF, &maps.b, &full[stage], static_cast<int>(n0), kt * BK, zb);
    };
    if (tid == 0) {
#pragma unroll
      for (int s = 0; s < STAGES; ++s) {
        f1_mbar_init(&full[s], 1);
        consumed[s] = 0;
      }
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    if (tid == 0) {
      for (int s = 0; s < STAGES && s < KT; ++s) issue(s, kt0 + s);
    }
    for (int kt = 0; kt < KT; ++kt) {
      const int s = kt % STAGES;
      f1_mbar_wait(&full[s], (kt / STAGES) & 1);
      const float* as = smem + s * Cfg::T_STAGE;
      if (warp_live) tile_math(as, as + Cfg::T_B_OFF);
      __syncwarp();
      if (lane == 0) {
        __threadfence_block();  // this warp's reads of the stage happen before the count
        const int prior = atomicAdd(&consumed[s], 1);
        if ((prior + 1) % NW == 0 && kt + STAGES < KT) {  // last consumer refills the stage
          __threadfence_block();
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          issue(s, kt0 + kt + STAGES);
        }
      }
    }
    __syncthreads();  // every stage consumed (no copy in flight) before smem is reused
  } else {
#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
      if (s < KT) load_tile(s, kt0 + s);
      cp_async_commit();
    }
    for (int kt = 0; kt < KT; ++kt) {
      cp_async_wait<STAGES - 2>();
      __syncthreads();
      {
        const int nk = kt + STAGES - 1;
        if (nk < KT) load_tile(nk % STAGES, kt0 + nk);
        cp_async_commit();
      }
      const float* as = smem + (kt % STAGES) * Cfg::STAGE;
      if (warp_live) tile_math(as, as + BM * SA);  // else: the warp's block lies outside the problem
    }
    cp_async_wait<0>();
  }

  if (p.kslices > 1) {
    // k-sliced: park the partial tile in this CTA's shared memory, then each CTA of
    // the cluster sums 1/kslices of the tile over the slices in rank order 0, 1, ...
    // (a fixed order, so the result is deterministic: ((p0 + p1) + p2) + ...).
    __syncthreads();
    constexpr int SP = Cfg::SP;
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int cv = 0; cv < C / VC; ++cv) {
        float v[VC];
#pragma unroll
        for (int e = 0; e < VC; ++e) {
          const float2 pr = acc[r][(cv * VC + e) / 2];
          v[e] = ((cv * VC + e) & 1) ? pr.y : pr.x;
        }
        stg_vec<VC>(smem + trow(r) * SP + tcol(cv), v);
      }
    f1_slice_reduce<BM, BN, SP, NT>(p, smem, Cb, m0, n0);
    return;
  }

  // the thread's C bias values, fetched once up front (independent loads) instead of one
  // dependent load per output element; epilogue() order: + bias, then ReLU
  float bcol[C];
#pragma unroll
  for (int cv = 0; cv < C / VC; ++cv) {
    const int64_t col = n0 + tcol(cv);
#pragma unroll
    for (int e = 0; e < VC; ++e) bcol[cv * VC + e] = (p.bias && col + e < n) ? __ldg(p.bias + col + e) : 0.0f;
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t row = m0 + trow(r);
    if (row >= m) continue;
    float* out = Cb + row * p.ldc;
#pragma unroll
    for (int cv = 0; cv < C / VC; ++cv) {
      const int64_t col = n0 + tcol(cv);
      float v[VC];
#pragma unroll
      for (int e = 0; e < VC; ++e) {
        const float2 pr = acc[r][(cv * VC + e) / 2];
        v[e] = ((cv * VC + e) & 1) ? pr.y : pr.x;
        if (p.bias) v[e] = v[e] + bcol[cv * VC + e];
        if (p.relu) v[e] = fmaxf(v[e], 0.0f);
      }
      if (p.c_vec && col + VC <= n) {
        stg_vec<VC>(out + col, v);
      } else {
#pragma unroll
        for (int e = 0; e < VC; ++e)
          if (col + e < n) out[col + e] = v[e];
      }
    }
  }
}

template <int R, int A, int C, int WGR, int WGC>
cudaError_t f1_set_attributes() {
  using Cfg = F1Cfg<R, A, C, WGR, WGC>;
  static bool attr_set = false;  // benign race: idempotent attribute writes
  if (!attr_set) {
    for (auto fn : {f1_kernel<R, A, C, WGR, WGC, 0>, f1_kernel<R, A, C, WGR, WGC, 1>, f1_kernel<R, A, C, WGR, WGC, 2>}) {
      const int bytes = fn == f1_kernel<R, A, C, WGR, WGC, 0> ? Cfg::SLICE_SMEM_BYTES : Cfg::T_SMEM_BYTES;
      cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
      if (e != cudaSuccess) return e;
      e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      if (e != cudaSuccess) return e;
    }
    attr_set = true;
  }
  return cudaSuccess;
}

template <int R, int A, int C, int WGR, int WGC>
int f1_cluster_fit(int slices) {
  using Cfg = F1Cfg<R, A, C, WGR, WGC>;
  if (f1_set_attributes<R, A, C, WGR, WGC>() != cudaSuccess) return -1;
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(1, 1, slices);
  lc.blockDim = dim3(Cfg::NT);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = slices;
  lc.attrs = at;
  lc.numAttrs = 1;
  // the planner does not know the operands' alignment: report the smaller fit of the
  // two staging paths
  int best = -1;
  for (int t = 0; t < 2; ++t) {
    int n = 0;
    lc.dynamicSmemBytes = t ? Cfg::T_SMEM_BYTES : Cfg::SLICE_SMEM_BYTES;
    const cudaError_t e = t ? cudaOccupancyMaxActiveClusters(&n, f1_kernel<R, A, C, WGR, WGC, 1>, &lc)
                            : cudaOccupancyMaxActiveClusters(&n, f1_kernel<R, A, C, WGR, WGC, 0>, &lc);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return -1;
    }
    best = best < 0 ? n : (n < best ? n : best);
  }
  return best;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda symbol
// needed at this call site).
using F1EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
inline F1EncodeFn f1_encode_fn() {
  static F1EncodeFn fn = [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<F1EncodeFn>(ptr);
    return static_cast<F1EncodeFn>(nullptr);
  }();
  return fn;
}

// A 3-d fp32 tensor map (inner dim0, rows dim1, batch dim2) with an unswizzled box.
// A zero batch stride (broadcast operand) becomes a batch extent of 1.
inline bool f1_encode(CUtensorMap* map, const void* base, int64_t d0, int64_t d1, int64_t ld, int64_t sbatch,
                      int batch, int box0, int box1) {
  F1EncodeFn enc = f1_encode_fn();
  if (!enc) return false;
  const bool batched = batch > 1 && sbatch != 0;
  cuuint64_t dims[3] = {static_cast<cuuint64_t>(d0), static_cast<cuuint64_t>(d1),
                        static_cast<cuuint64_t>(batched ? batch : 1)};
  cuuint64_t strides[2] = {static_cast<cuuint64_t>(ld) * 4,
                           static_cast<cuuint64_t>(batched ? sbatch : (ld * d1 + 3) / 4 * 4) * 4};
  cuuint32_t box[3] = {static_cast<cuuint32_t>(box0), static_cast<cuuint32_t>(box1), 1};
  cuuint32_t es[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// The im2col map of a 3x3 / stride 1 / pad 1 convolution over an NHWC activation of
// `imgs` images: bounding box corners -1 / -1 (base pixel = output pixel - 1 in w and h),
// tap offsets (dx, dy) in 0..2 passed per copy.
using F1EncodeIm2colFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                      const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                                      const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                      CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
inline bool f1_encode_im2col(CUtensorMap* map, const void* x, int imgs, int H, int W, int Cin, int channels,
                             int pixels) {
  static F1EncodeIm2colFn enc = [] {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      return reinterpret_cast<F1EncodeIm2colFn>(ptr);
    return static_cast<F1EncodeIm2colFn>(nullptr);
  }();
  if (!enc) return false;
  cuuint64_t dims[4] = {static_cast<cuuint64_t>(Cin), static_cast<cuuint64_t>(W), static_cast<cuuint64_t>(H),
                        static_cast<cuuint64_t>(imgs)};
  cuuint64_t strides[3] = {static_cast<cuuint64_t>(Cin) * 4, static_cast<cuuint64_t>(W) * Cin * 4,
                           static_cast<cuuint64_t>(H) * W * Cin * 4};
  const int lower[2] = {-1, -1}, upper[2] = {-1, -1};
  cuuint32_t es[4] = {1, 1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<void*>(x), dims, strides, lower, upper,
             static_cast<cuuint32_t>(channels), static_cast<cuuint32_t>(pixels), es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int R, int A, int C, int WGR, int WGC>
cudaError_t f1_launch(const GemmArgs& p0, cudaStream_t s) {
  using Cfg = F1Cfg<R, A, C, WGR, WGC>;
  if (cudaError_t e = f1_set_attributes<R, A, C, WGR, WGC>(); e != cudaSuccess) return e;
  GemmArgs p = p0;
  auto aligned = [](const void* ptr, int bytes) { return (reinterpret_cast<uintptr_t>(ptr) % bytes) == 0; };
  p.a_vec = (p.k % 4 == 0) && (p.lda % 4 == 0) && (p.sA % 4 == 0) && aligned(p.A, 16);
  p.b_vec = (p.n % 4 == 0) && (p.ldb % 4 == 0) && (p.sB % 4 == 0) && aligned(p.B, 16);
  p.c_vec = (p.ldc % Cfg::VC == 0) && (p.sC % Cfg::VC == 0) && aligned(p.C, 4 * Cfg::VC);
  p.c_vec4 = (p.ldc % 4 == 0) && (p.sC % 4 == 0) && aligned(p.C, 16);
  const int64_t groups_m = (p.m + Cfg::BM - 1) / Cfg::BM;
  const int64_t groups_n = (p.n + Cfg::BN - 1) / Cfg::BN;
  const int64_t gx = groups_m * groups_n;
  if (gx > 0x7fffffffLL || p.batch > 65535) return cudaErrorInvalidConfiguration;
  if (p.kslices <= 1) {
    p.kslices = 1;
    p.kt_per_slice = (p.k + Cfg::BK - 1) / Cfg::BK;
  } else if (p.kslices > kMaxKSlices) {
    return cudaErrorInvalidConfiguration;
  }
  // TMA staging: rows 16-byte aligned in both operands (the tensor maps' stride rule;
  // k and n themselves may be ragged -- the boxes zero-fill past them), coordinates
  // within int range.
  const bool conv = p.conv_c > 0;
  if (conv && !(Cfg::TMA_OK && p.conv_c % Cfg::BK == 0 && p.k == 9 * p.conv_c && p.batch == 1 &&
                p.m % (p.conv_h * p.conv_w) == 0 && aligned(p.A, 16) && aligned(p.B, 16) && p.ldb % 4 == 0))
    return cudaErrorInvalidValue;
  const bool tma = conv || (Cfg::TMA_OK && g_f1_tma_staging.load(std::memory_order_relaxed) != 0 && aligned(p.A, 16) && aligned(p.B, 16) && p.lda % 4 == 0 &&
                   p.ldb % 4 == 0 && (p.batch == 1 || ((p.sA % 4 == 0) && (p.sB % 4 == 0))) &&
                   p.m < (1LL << 31) - Cfg::BM && p.k < (1 << 30));
  F1Maps maps;
  if (tma) {
    // one-entry cache per instantiation and host thread: sweeps and layer loops re-launch
    // the same operands, and encoding costs ~1 us of host time
    struct Key {
      const void *pa, *pb;
      int64_t m, k, n, batch, lda, ldb, sA, sB, ch, cw, cc;
      bool operator==(const Key& o) const { return std::memcmp(this, &o, sizeof(Key)) == 0; }
    };
    thread_local Key last_key;
    thread_local F1Maps last_maps;
    thread_local bool have = false;
    Key key;
    std::memset(&key, 0, sizeof(key));
    key.pa = p.A; key.pb = p.B; key.m = p.m; key.k = p.k; key.n = p.n; key.batch = p.batch;
    key.lda = p.lda; key.ldb = p.ldb; key.sA = p.sA; key.sB = p.sB;
    key.ch = p.conv_h; key.cw = p.conv_w; key.cc = p.conv_c;
    if (!(have && key == last_key)) {
      const bool a_ok =
          conv ? f1_encode_im2col(&last_maps.a, p.A, p.m / (p.conv_h * p.conv_w), p.conv_h, p.conv_w, p.conv_c,
                                  Cfg::SA, Cfg::A_BOX_ROWS)
               : f1_encode(&last_maps.a, p.A, p.k, p.m, p.lda, p.sA, p.batch, Cfg::SA, Cfg::A_BOX_ROWS);
      if (!a_ok ||
          !f1_encode(&last_maps.b, p.B, p.n, p.k, p.ldb, p.sB, p.batch, Cfg::BN, Cfg::BK)) {
        have = false;
        return cudaErrorInvalidValue;
      }
      last_key = key;
      have = true;
    }
    maps = last_maps;
    if (conv) {
      maps.cw = FastDiv(static_cast<uint32_t>(p.conv_w));
      maps.ch = FastDiv(static_cast<uint32_t>(p.conv_h));
      maps.cc = FastDiv(static_cast<uint32_t>(p.conv_c));
    }
  } else {
    std::memset(&maps, 0, sizeof(maps));
  }
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(static_cast<unsigned>(gx), p.batch, p.kslices);
  lc.blockDim = dim3(Cfg::NT);
  lc.dynamicSmemBytes = tma ? Cfg::T_SMEM_BYTES : (p.kslices > 1 ? Cfg::SLICE_SMEM_BYTES : Cfg::SMEM_BYTES);
  lc.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = p.kslices;
  lc.attrs = at;
  lc.numAttrs = p.kslices > 1 ? 1 : 0;
  const int gn = static_cast<int>(groups_n);
  if (!tma) return cudaLaunchKernelEx(&lc, f1_kernel<R, A, C, WGR, WGC, 0>, p, gn, maps);
  return p.conv_c > 0 ? cudaLaunchKernelEx(&lc, f1_kernel<R, A, C, WGR, WGC, 2>, p, gn, maps)
                      : cudaLaunchKernelEx(&lc, f1_kernel<R, A, C, WGR, WGC, 1>, p, gn, maps);
}

}  // namespace kp
