// Micro-benchmark (dev tool, not product): where does the F1 8x8 inner loop lose FMA
// throughput?  Three variants of the same 8x8-per-thread FFMA2 outer product, 128-thread
// CTAs at 4 CTAs/SM (the (8,x,8,16,8) launch shape), timed with CUDA events:
//   REG  -- fragments rotate through registers (no shared memory): the issue/dependency
//           ceiling of the FFMA2 stream itself;
//   LDS  -- fragments read from a shared tile with F1's access pattern (A: 2x LDS.128 per
//           row per 8 k, pair-shared lanes; B: 2x LDS.128 per k), no global traffic, one
//           __syncthreads per 32 k (the per-stage barrier);
//   LDS0 -- LDS without the barrier;
//   REGS / LDSS -- REG / LDS with scalar FFMA instead of FFMA2.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o f1_inner f1_inner.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int R = 8, C = 8, CP = C / 2, BK = 32, BM = 128, BN = 64, SA = BK + 4;

template <int MODE>
__global__ void __launch_bounds__(128, 4) inner(float* out, int iters) {
  __shared__ __align__(16) float as[BM * SA];
  __shared__ __align__(16) float bs[BK * BN];
  for (int i = threadIdx.x; i < BM * SA; i += 128) as[i] = 1e-3f * (i & 31);
  for (int i = threadIdx.x; i < BK * BN; i += 128) bs[i] = 1e-3f * (i & 15);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int lr = lane / 8, lc = lane % 8;               // 4 x 8 warp patch
  const int wrow0 = warp * (R * 4), wcol0 = 0;          // WPC = 1
  float2 acc[R][CP];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < CP; ++c) acc[r][c] = make_float2(0.f, 0.f);
  float ra[R], rw[C];
#pragma unroll
  for (int r = 0; r < R; ++r) ra[r] = 1e-3f * (r + lane);
#pragma unroll
  for (int c = 0; c < C; ++c) rw[c] = 1e-3f * (c + lane);
  for (int it = 0; it < iters; ++it) {
    if (MODE == 1 || MODE == 4) __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; kk += 8) {
      float a[R][8];
      if (MODE == 0 || MODE == 3) {
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int i = 0; i < 8; ++i) a[r][i] = ra[r];
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const float4* p = reinterpret_cast<const float4*>(as + (wrow0 + r * 4 + lr) * SA + kk);
          float4 v0 = p[0], v1 = p[1];
          a[r][0] = v0.x; a[r][1] = v0.y; a[r][2] = v0.z; a[r][3] = v0.w;
          a[r][4] = v1.x; a[r][5] = v1.y; a[r][6] = v1.z; a[r][7] = v1.w;
        }
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float w[C];
        if (MODE == 0 || MODE == 3) {
#pragma unroll
          for (int c = 0; c < C; ++c) w[c] = rw[c];
        } else {
#pragma unroll
          for (int cv = 0; cv < 2; ++cv) {
            float4 v = *reinterpret_cast<const float4*>(bs + (kk + i) * BN + wcol0 + cv * 32 + lc * 4);
            w[cv * 4] = v.x; w[cv * 4 + 1] = v.y; w[cv * 4 + 2] = v.z; w[cv * 4 + 3] = v.w;
          }
        }
        if (MODE >= 3) {
#pragma unroll
          for (int r = 0; r < R; ++r)
#pragma unroll
            for (int c = 0; c < CP; ++c) {
              acc[r][c].x = __fmaf_rn(a[r][i], w[2 * c], acc[r][c].x);
              acc[r][c].y = __fmaf_rn(a[r][i], w[2 * c + 1], acc[r][c].y);
            }
        } else {
#pragma unroll
          for (int r = 0; r < R; ++r)
#pragma unroll
            for (int c = 0; c < CP; ++c)
              acc[r][c] = __ffma2_rn(make_float2(a[r][i], a[r][i]), make_float2(w[2 * c], w[2 * c + 1]), acc[r][c]);
        }
      }
    }
  }
  float s = 0.f;
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < CP; ++c) s += acc[r][c].x + acc[r][c].y;
  if (s == 1234.5f) out[threadIdx.x] = s;
}

template <int MODE>
double run(int sms, int iters) {
  float* out;
  cudaMalloc(&out, 4096);
  const int blocks = sms * 4 * 8;  // 8 waves of 4 CTAs/SM
  inner<MODE><<<blocks, 128>>>(out, 10);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  inner<MODE><<<blocks, 128>>>(out, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaFree(out);
  const double flops = 2.0 * R * C * BK * double(iters) * 128.0 * blocks;
  return flops / (ms * 1e-3) / 1e12;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 4000;
  printf("{\"REG\": %.2f, \"LDS\": %.2f, \"REGS\": %.2f, \"LDSS\": %.2f}\n", run<0>(sms, iters),
         run<1>(sms, iters), run<3>(sms, iters), run<4>(sms, iters));
  return 0;
}
