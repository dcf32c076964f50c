// F1 v2 (experimental layout of the SIMT family; selected with -DKP_F1_V2=1):
// the LHS tile is stored k-major in shared memory (transposed on the fly by 4-byte
// cp.async, one LHS row per thread-lane so the smem writes are conflict-free), so a
// per-k LHS fragment is R contiguous rows -> LDS.128 quads, and the FFMA2 pair operand
// is a pair of ROWS (adjacent registers) times a scalar RHS column value.  Per step a
// thread loads an R x A LHS fragment (A loads of width R) and an A x C RHS fragment
// (A loads of width C) -- the paper's per-step tile semantics -- then issues R*A*C FMAs.
// Accumulation is still the sequential fp32 fma chain over k, so results stay
// bit-identical to the oracle.
#pragma once

#include "common.cuh"
#include "f1_simt.cuh"

namespace kp {

template <int R, int A, int C, int WGR, int WGC>
struct F1v2Cfg {
  static constexpr int NT = WGR * WGC;
  static constexpr int BM = R * WGR;
  static constexpr int BN = C * WGC;
  static constexpr int VR = R < 4 ? R : 4;  // LHS read width (rows)
  static constexpr int VC = C < 4 ? C : 4;  // RHS read width (cols)
  static constexpr int PADM = 4;
  static constexpr int MIN_BLOCKS = (KP_F1_WARPS * 32 / NT) > 1 ? (KP_F1_WARPS * 32 / NT) : 1;
  static constexpr int kBudget = (227 * 1024) / (MIN_BLOCKS < 4 ? MIN_BLOCKS : 4) - 1024;
  static constexpr int stage_floats(int bk) { return bk * (BM + PADM) + bk * BN; }
  static constexpr int BK = (KP_F1_MAX_BK >= 32 && 3 * 4 * stage_floats(32) <= kBudget)   ? 32
                            : (KP_F1_MAX_BK >= 16 && 2 * 4 * stage_floats(16) <= kBudget) ? 16
                                                                                        : 8;
  static constexpr int SA = BM + PADM;  // LHS smem row (one k) stride, floats
  static constexpr int SB = BN;
  static constexpr int STAGE = stage_floats(BK);
  static constexpr int STAGES_FIT = kBudget / (4 * STAGE);
  static constexpr int STAGES = STAGES_FIT < 2 ? 2 : (STAGES_FIT > 4 ? 4 : STAGES_FIT);
  static constexpr int SMEM_BYTES = STAGES * STAGE * 4;
  static constexpr int WTC = f1_pick_wtc(R, C, WGR, WGC);
  static constexpr int WTR = 32 / WTC;
  static constexpr int WPC = WGC / WTC;
  static constexpr bool ROW_PAIRS = R >= 2;  // FFMA2 pair operand: two rows (else two cols)
  static constexpr bool B_CHUNKS = (BN % 4) == 0;
  static_assert(BK % A == 0, "stage depth must be a multiple of A");
  static_assert(SMEM_BYTES <= 227 * 1024, "shared memory");
};

template <int R, int A, int C, int WGR, int WGC>
__global__ void __launch_bounds__(WGR * WGC, F1v2Cfg<R, A, C, WGR, WGC>::MIN_BLOCKS)
    f1v2_kernel(GemmArgs p, int groups_n) {
  using Cfg = F1v2Cfg<R, A, C, WGR, WGC>;
  constexpr int NT = Cfg::NT, BM = Cfg::BM, BN = Cfg::BN, BK = Cfg::BK;
  constexpr int SA = Cfg::SA, SB = Cfg::SB, STAGES = Cfg::STAGES, VR = Cfg::VR, VC = Cfg::VC;
  extern __shared__ __align__(16) float smem[];

  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  // adjacent lanes share the LHS rows (pair-broadcast LDS), lanes differ in columns
  const int ty = (warp / Cfg::WPC) * Cfg::WTR + lane / Cfg::WTC;
  const int tx = (warp % Cfg::WPC) * Cfg::WTC + lane % Cfg::WTC;

  const int64_t gm = blockIdx.x / groups_n;
  const int gn = blockIdx.x - static_cast<int>(gm * groups_n);
  const int b = blockIdx.y;
  const int m = p.m, k = p.k, n = p.n;
  const int64_t m0 = gm * BM;
  const int64_t n0 = static_cast<int64_t>(gn) * BN;
  const float* __restrict__ Ab = static_cast<const float*>(p.A) + b * p.sA;
  const float* __restrict__ Bb = static_cast<const float*>(p.B) + b * p.sB;
  float* __restrict__ Cb = static_cast<float*>(p.C) + b * p.sC;
  const int64_t lda = p.lda, ldb = p.ldb;
  const bool b16 = Cfg::B_CHUNKS && p.b_vec;

  auto load_tile = [&](int stage, int kt) {
    float* as = smem + stage * Cfg::STAGE;
    float* bs = as + BK * SA;
    const int k0 = kt * BK;
    // LHS: element e -> (row = e % BM, kk = e / BM); consecutive lanes take consecutive
    // rows, so the transposed smem writes As[kk][row] are conflict-free; each lane
    // walks its row along k, the L1 serving the re-reads of a row's 128-byte line.
    constexpr int EL = BM * BK;
#pragma unroll 4
    for (int j = 0; j < (EL + NT - 1) / NT; ++j) {
      const int e = tid + j * NT;
      if (EL % NT == 0 || e < EL) {
        const int row = e % BM, kk = e / BM;
        const int64_t gr = m0 + row;
        const int gk = k0 + kk;
        const bool ok = gr < m && gk < k;
        cp_async4(as + kk * SA + row, ok ? Ab + gr * lda + gk : Ab, ok ? 4 : 0);
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
      constexpr int EL2 = BK * BN;
#pragma unroll 4
      for (int j = 0; j < (EL2 + NT - 1) / NT; ++j) {
        const int e = tid + j * NT;
        if (EL2 % NT == 0 || e < EL2) {
          const int r = e / BN, q = e - r * BN;
          const int gk = k0 + r;
          const int64_t gc = n0 + q;
          const bool ok = gk < k && gc < n;
          cp_async4(bs + r * SB + q, ok ? Bb + static_cast<int64_t>(gk) * ldb + gc : Bb, ok ? 4 : 0);
        }
      }
    }
  };

  // accumulators: ROW_PAIRS -> acc[r/2][c] = (row r, row r+1) at column c
  constexpr int PR = Cfg::ROW_PAIRS ? R / 2 : R;
  constexpr int PC = Cfg::ROW_PAIRS ? C : (C + 1) / 2;
  float2 acc[PR][PC];
#pragma unroll
  for (int i = 0; i < PR; ++i)
#pragma unroll
    for (int j = 0; j < PC; ++j) acc[i][j] = make_float2(0.0f, 0.0f);

  // thread's rows: quads of VR rows interleaved across the work group; cols likewise
  auto row_off = [&](int r) { return (r / VR) * (WGR * VR) + ty * VR + (r % VR); };
  auto col_off = [&](int c) { return (c / VC) * (WGC * VC) + tx * VC + (c % VC); };

  const int KT = (k + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < KT) load_tile(s, s);
    cp_async_commit();
  }
  for (int kt = 0; kt < KT; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nk = kt + STAGES - 1;
      if (nk < KT) load_tile(nk % STAGES, nk);
      cp_async_commit();
    }
    const float* as = smem + (kt % STAGES) * Cfg::STAGE;
    const float* bs = as + BK * SA;
#pragma unroll
    for (int kk = 0; kk < BK; kk += A) {
      float a[A][R];
      float w[A][C];
#pragma unroll
      for (int i = 0; i < A; ++i) {
#pragma unroll
        for (int rv = 0; rv < R / VR; ++rv) lds_vec<VR>(as + (kk + i) * SA + row_off(rv * VR), a[i] + rv * VR);
#pragma unroll
        for (int cv = 0; cv < C / VC; ++cv) lds_vec<VC>(bs + (kk + i) * SB + col_off(cv * VC), w[i] + cv * VC);
      }
#pragma unroll
      for (int i = 0; i < A; ++i) {
        if constexpr (Cfg::ROW_PAIRS) {
#pragma unroll
          for (int rp = 0; rp < PR; ++rp)
#pragma unroll
            for (int cc = 0; cc < C; ++cc) {
              const int c = (rp & 1) ? C - 1 - cc : cc;  // serpentine: share the row pair
              acc[rp][c] = __ffma2_rn(make_float2(a[i][2 * rp], a[i][2 * rp + 1]), make_float2(w[i][c], w[i][c]),
                                      acc[rp][c]);
            }
        } else if constexpr (C >= 2) {
#pragma unroll
          for (int cp = 0; cp < PC; ++cp)
            acc[0][cp] = __ffma2_rn(make_float2(a[i][0], a[i][0]), make_float2(w[i][2 * cp], w[i][2 * cp + 1]),
                                    acc[0][cp]);
        } else {
          acc[0][0].x = __fmaf_rn(a[i][0], w[i][0], acc[0][0].x);
        }
      }
    }
  }
  cp_async_wait<0>();

  auto value = [&](int r, int c) -> float {
    if constexpr (Cfg::ROW_PAIRS) {
      const float2 v = acc[r / 2][c];
      return (r & 1) ? v.y : v.x;
    } else {
      const float2 v = acc[0][c / 2];
      return (c & 1) ? v.y : v.x;
    }
  };
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int64_t row = m0 + row_off(r);
    if (row >= m) continue;
    float* out = Cb + row * p.ldc;
#pragma unroll
    for (int cv = 0; cv < C / VC; ++cv) {
      const int64_t col = n0 + col_off(cv * VC);
      float v[VC];
#pragma unroll
      for (int e = 0; e < VC; ++e) {
        v[e] = value(r, cv * VC + e);
        if (p.bias || p.relu) v[e] = (col + e < n) ? epilogue(p, v[e], col + e) : v[e];
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
cudaError_t f1v2_launch(const GemmArgs& p0, cudaStream_t s) {
  using Cfg = F1v2Cfg<R, A, C, WGR, WGC>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(f1v2_kernel<R, A, C, WGR, WGC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Cfg::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  GemmArgs p = p0;
  auto aligned = [](const void* ptr, int bytes) { return (reinterpret_cast<uintptr_t>(ptr) % bytes) == 0; };
  p.b_vec = (p.n % 4 == 0) && (p.ldb % 4 == 0) && (p.sB % 4 == 0) && aligned(p.B, 16);
  p.c_vec = (p.ldc % Cfg::VC == 0) && (p.sC % Cfg::VC == 0) && aligned(p.C, 4 * Cfg::VC);
  const int64_t groups_m = (p.m + Cfg::BM - 1) / Cfg::BM;
  const int64_t groups_n = (p.n + Cfg::BN - 1) / Cfg::BN;
  const int64_t gx = groups_m * groups_n;
  if (gx > 0x7fffffffLL || p.batch > 65535) return cudaErrorInvalidConfiguration;
  f1v2_kernel<R, A, C, WGR, WGC><<<dim3(static_cast<unsigned>(gx), p.batch), Cfg::NT, Cfg::SMEM_BYTES, s>>>(
      p, static_cast<int>(groups_n));
  return cudaGetLastError();
}

}  // namespace kp
