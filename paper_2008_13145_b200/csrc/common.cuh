// Shared device helpers and launch-parameter structs for the kpgemm families.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "kpgemm.h"

namespace kp {

// Launch parameters common to every fp32 family.  Dims follow the reference's
// ProblemSize order (m, k, n, batch), dataset.py:61-74.
// Division by a runtime constant d >= 1 for dividends in [0, 2^31): q = umulhi(n, mul) >> shr
// (round-up reciprocal, mul = ceil(2^(31 + ceil(log2 d)) / d), shr = ceil(log2 d) - 1; d == 1
// is the identity).  Host-built; replaces ~20-instruction integer divisions in the SIMT
// implicit-conv issue path (carried in F1Maps, so GemmArgs -- and the GEMM instances'
// code -- are unchanged).
struct FastDiv {
  uint32_t d, mul, shr;
  __host__ __device__ FastDiv() : d(1), mul(0), shr(0) {}
  __host__ explicit FastDiv(uint32_t divisor) : d(divisor), mul(0), shr(0) {
    if (divisor > 1) {
      uint32_t lg = 0;
      while ((1ull << lg) < divisor) ++lg;  // ceil(log2 d)
      const uint64_t p = 31 + lg;
      mul = static_cast<uint32_t>(((1ull << p) + divisor - 1) / divisor);
      shr = static_cast<uint32_t>(p - 32);
    }
  }
  __device__ __forceinline__ int div(int n) const {
    return d == 1 ? n : static_cast<int>(__umulhi(static_cast<uint32_t>(n), mul) >> shr);
  }
};

struct GemmArgs {
  int m, k, n, batch;
  const void* A;
  int64_t lda, sA;
  const void* B;
  int64_t ldb, sB;
  void* C;
  int64_t ldc, sC;
  // Host-computed alignment facts (uniform across the grid).
  int a_vec;  // rows of A may be read with the family's vector width along k
  int b_vec;  // rows of B may be read with the family's vector width along n
  int c_vec;  // rows of C may be written with the family's vector width along n
  int c_vec4;  // rows of C may be written as float4 (k-sliced reduction stores)
  // Fused epilogue (kp_gemm_ex): C = act(A*B + bias[col]); bias may be null.
  const float* bias;
  int relu;
  // Tensor-core families only (KP_EPI_BF16_OUT): C is bf16, the epilogue result rounded
  // to nearest even -- the operand the next BF16 layer reads, no separate cast pass.
  int c_bf16;
  // k-slicing (SIMT family, planned by capi.cu): the k-tiles are cut into kslices
  // consecutive ranges of kt_per_slice tiles; slice z is computed by the CTA at
  // blockIdx.z of a (1, 1, kslices) thread-block cluster and the partial tiles are
  // summed in slice order through distributed shared memory.  kslices == 1 is the
  // plain single-chain kernel.
  int kslices;
  int kt_per_slice;
  // Tensor-core families only: the last tail_tiles output tiles (a partial last wave of
  // the persistent kernel) run as a second, k-sliced launch with tail_slices slices.
  int tail_tiles;
  int tail_slices;
  // Implicit-GEMM 3x3 / stride 1 / pad 1 convolution (SIMT TMA staging only): when
  // conv_c > 0, A is the NHWC activation (batch = m / (conv_h * conv_w) images of
  // conv_h x conv_w x conv_c) and row r / column k of the GEMM operand is the im2col
  // patch value kp_im2col3x3_nhwc would write, gathered by TMA im2col copies.
  int conv_h, conv_w, conv_c;
};

// Epilogue of every family: bias add (fp32, round-to-nearest) then ReLU.  Applied
// after the fma chain, so the result equals oracle_chain + bias -> max(0, .) exactly.
__device__ __forceinline__ float epilogue(const GemmArgs& p, float v, int64_t col) {
  if (p.bias) v = v + __ldg(p.bias + col);
  if (p.relu) v = fmaxf(v, 0.0f);
  return v;
}

// The same epilogue over N consecutive columns [col, col + N) of one row (col warp-
// uniform, N % 4 == 0): the bias values are fetched up front -- float4 loads when the run
// is in range and 16-byte aligned -- so the N loads overlap instead of each add waiting
// on its own load (the per-element form serialised N global-load latencies per run and
// made bias + ReLU tiles 2-4x slower than plain ones).  Columns >= n get bias 0 and are
// never stored.  Same values as epilogue() per element.
template <int N>
__device__ __forceinline__ void epilogue_run(const GemmArgs& p, float* v, int64_t col) {
  static_assert(N % 4 == 0, "runs of whole float4s");
  const float* bias = p.bias;
  if (bias) {
    float bv[N];
    if (col + N <= p.n && ((reinterpret_cast<uintptr_t>(bias + col) & 15) == 0)) {
#pragma unroll
      for (int q = 0; q < N / 4; ++q) {
        const float4 t = __ldg(reinterpret_cast<const float4*>(bias + col) + q);
        bv[4 * q] = t.x; bv[4 * q + 1] = t.y; bv[4 * q + 2] = t.z; bv[4 * q + 3] = t.w;
      }
    } else {
#pragma unroll
      for (int e = 0; e < N; ++e) bv[e] = col + e < p.n ? __ldg(bias + col + e) : 0.0f;
    }
#pragma unroll
    for (int e = 0; e < N; ++e) v[e] = v[e] + bv[e];
  }
  if (p.relu) {
#pragma unroll
    for (int e = 0; e < N; ++e) v[e] = fmaxf(v[e], 0.0f);
  }
}

// Two fp32 values rounded to nearest even and packed as bf16 (lo in the low half).
__device__ __forceinline__ unsigned pack_bf16x2(float lo, float hi) {
  const __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<const unsigned*>(&v);
}

// ---- vector load / store of N consecutive floats (N in {1,2,4,8}) ---------
template <int N>
__device__ __forceinline__ void ldg_vec(const float* __restrict__ p, float* out) {
  if constexpr (N == 1) {
    out[0] = __ldg(p);
  } else if constexpr (N == 2) {
    float2 v = __ldg(reinterpret_cast<const float2*>(p));
    out[0] = v.x; out[1] = v.y;
  } else if constexpr (N == 4) {
    float4 v = __ldg(reinterpret_cast<const float4*>(p));
    out[0] = v.x; out[1] = v.y; out[2] = v.z; out[3] = v.w;
  } else {
    static_assert(N == 8, "vector width");
    float4 v0 = __ldg(reinterpret_cast<const float4*>(p));
    float4 v1 = __ldg(reinterpret_cast<const float4*>(p + 4));
    out[0] = v0.x; out[1] = v0.y; out[2] = v0.z; out[3] = v0.w;
    out[4] = v1.x; out[5] = v1.y; out[6] = v1.z; out[7] = v1.w;
  }
}

template <int N>
__device__ __forceinline__ void lds_vec(const float* p, float* out) {
  if constexpr (N == 1) {
    out[0] = p[0];
  } else if constexpr (N == 2) {
    float2 v = *reinterpret_cast<const float2*>(p);
    out[0] = v.x; out[1] = v.y;
  } else if constexpr (N == 4) {
    float4 v = *reinterpret_cast<const float4*>(p);
    out[0] = v.x; out[1] = v.y; out[2] = v.z; out[3] = v.w;
  } else {
    static_assert(N == 8, "vector width");
    float4 v0 = *reinterpret_cast<const float4*>(p);
    float4 v1 = *reinterpret_cast<const float4*>(p + 4);
    out[0] = v0.x; out[1] = v0.y; out[2] = v0.z; out[3] = v0.w;
    out[4] = v1.x; out[5] = v1.y; out[6] = v1.z; out[7] = v1.w;
  }
}

template <int N>
__device__ __forceinline__ void stg_vec(float* p, const float* v) {
  if constexpr (N == 1) {
    p[0] = v[0];
  } else if constexpr (N == 2) {
    *reinterpret_cast<float2*>(p) = make_float2(v[0], v[1]);
  } else if constexpr (N == 4) {
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
  } else {
    static_assert(N == 8, "vector width");
    *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    *reinterpret_cast<float4*>(p + 4) = make_float4(v[4], v[5], v[6], v[7]);
  }
}

// ---- cp.async (LDGSTS) with zero fill ------------------------------------
// src_bytes == 0 writes zeros and reads nothing.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, int src_bytes) {
  unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

}  // namespace kp
