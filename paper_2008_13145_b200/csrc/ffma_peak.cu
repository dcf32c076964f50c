// FP32 FFMA peak probe: 16 independent register-resident FFMA chains per thread,
// unrolled 8 deep, on sms*8 CTAs of 256 threads.  Its TFLOP/s is the measured FP32
// SIMT peak that the SIMT families' roofline fraction is quoted against.
#include "families.h"

namespace kp {
namespace {

__global__ void __launch_bounds__(256) ffma_peak_kernel(float* sink, int iters, float s, float t) {
  float x[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) x[j] = static_cast<float>(threadIdx.x + j);
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u)
#pragma unroll
      for (int j = 0; j < 16; ++j) x[j] = __fmaf_rn(x[j], s, t);
  }
  float acc = 0.f;
#pragma unroll
  for (int j = 0; j < 16; ++j) acc += x[j];
  if (acc == 1234.5f) sink[threadIdx.x] = acc;  // keep the chains live
}

}  // namespace

cudaError_t ffma_peak_launch(float* sink, int blocks, int threads, int iters, cudaStream_t s) {
  ffma_peak_kernel<<<blocks, threads, 0, s>>>(sink, iters, 0.999f, 0.001f);
  return cudaGetLastError();
}

}  // namespace kp
