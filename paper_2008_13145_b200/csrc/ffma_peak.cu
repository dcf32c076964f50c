// FP32 FFMA peak probe: 16 independent register-resident FFMA chains per thread
// (scalar FFMA, or FFMA2 pairs when packed),
// unrolled 8 deep, on sms*8 CTAs of 256 threads.  Its TFLOP/s is the measured FP32
// SIMT peak that the SIMT families' roofline fraction is quoted against.
#include "families.h"

namespace kp {
namespace {

template <bool kPacked>
__global__ void __launch_bounds__(256) ffma_peak_kernel(float* sink, int iters, float s, float t) {
  float x[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) x[j] = static_cast<float>(threadIdx.x + j);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if constexpr (kPacked) {
#pragma unroll
        for (int j = 0; j < 16; j += 2) {
          float2 v = __ffma2_rn(make_float2(s, s), make_float2(x[j], x[j + 1]), make_float2(t, t));
          x[j] = v.x;
          x[j + 1] = v.y;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) x[j] = __fmaf_rn(x[j], s, t);
      }
  }
  float acc = 0.f;
#pragma unroll
  for (int j = 0; j < 16; ++j) acc += x[j];
  if (acc == 1234.5f) sink[threadIdx.x] = acc;  // keep the chains live
}

}  // namespace

cudaError_t ffma_peak_launch(float* sink, int blocks, int threads, int iters, bool packed, cudaStream_t s) {
  if (packed)
    ffma_peak_kernel<true><<<blocks, threads, 0, s>>>(sink, iters, 0.999f, 0.001f);
  else
    ffma_peak_kernel<false><<<blocks, threads, 0, s>>>(sink, iters, 0.999f, 0.001f);
  return cudaGetLastError();
}

}  // namespace kp
