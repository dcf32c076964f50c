// Conv-as-GEMM helpers for VGG16 inference (BASELINE.json configs[2]), NHWC fp32.
//
// The paper evaluates its selected kernels inside a VGG16 network
// where SYCL-DNN lowers convolutions to matmuls.  Here a 3x3 / stride 1 / pad 1
// convolution becomes im2col (this kernel) + one tree-dispatched GEMM with the bias
// and ReLU fused into the GEMM epilogue (kp_gemm_ex); pooling is a separate HBM-bound
// pass.  NHWC keeps the GEMM output (B*H*W) x Cout equal to the next layer's input.
#include "families.h"

#include <cuda_bf16.h>

namespace kp {
namespace {

// One thread per output element; consecutive threads walk k = (dy*3 + dx)*C + c, so
// both the gather (contiguous channels of one tap) and the store are coalesced.
__global__ void im2col3x3_nhwc_kernel(const float* __restrict__ x, int B, int H, int W, int C,
                                      float* __restrict__ out, int64_t ldo) {
  const int64_t K = 9LL * C;
  const int64_t total = static_cast<int64_t>(B) * H * W * K;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = i / K;
    const int kk = static_cast<int>(i - row * K);
    const int tap = kk / C, c = kk - tap * C;
    const int dy = tap / 3 - 1, dx = tap % 3 - 1;
    const int w = static_cast<int>(row % W);
    const int64_t bh = row / W;
    const int h = static_cast<int>(bh % H);
    const int b = static_cast<int>(bh / H);
    const int hy = h + dy, wx = w + dx;
    float v = 0.0f;
    if (hy >= 0 && hy < H && wx >= 0 && wx < W) v = __ldg(x + ((static_cast<int64_t>(b) * H + hy) * W + wx) * C + c);
    out[row * ldo + kk] = v;
  }
}

// Vectorised im2col for C % 4 == 0 (every VGG16 layer but conv1_1): one thread per
// float4 of one tap of one output pixel, 32-bit index math (the 64-bit divisions of
// the scalar kernel made it integer-bound, not HBM-bound).  Consecutive threads walk the
// channels of a tap, then the taps, so loads and stores stay coalesced 16-byte accesses.
__global__ void im2col3x3_nhwc_vec4_kernel(const float4* __restrict__ x, int B, int H, int W, int C4,
                                           float4* __restrict__ out, int64_t ldo4, unsigned total) {
  const unsigned K4 = 9u * C4;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const unsigned row = i / K4;
    const unsigned kk = i - row * K4;
    const unsigned tap = kk / C4, c4 = kk - tap * C4;
    const int dy = static_cast<int>(tap / 3) - 1, dx = static_cast<int>(tap % 3) - 1;
    const unsigned bh = row / W;
    const int w = static_cast<int>(row - bh * W);
    const unsigned b = bh / H;
    const int h = static_cast<int>(bh - b * H);
    const int hy = h + dy, wx = w + dx;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (hy >= 0 && hy < H && wx >= 0 && wx < W)
      v = __ldg(x + ((static_cast<int64_t>(b) * H + hy) * W + wx) * C4 + c4);
    out[static_cast<int64_t>(row) * ldo4 + kk] = v;
  }
}

// im2col into rows padded to kpad >= 9C columns (zeros beyond 9C), one thread per float4
// of a row, 32-bit index math.  For conv1_1 (C = 3, 9C = 27): 28-float rows are 16-byte
// aligned, so the GEMM takes the vector / TMA operand paths, and the zero column times a
// zero weight row adds fma(0, 0, acc) == acc -- the chain over the 27 real taps.
__global__ void im2col3x3_nhwc_pad_kernel(const float* __restrict__ x, int B, int H, int W, int C, int kpad,
                                          float4* __restrict__ out, unsigned total4) {
  const unsigned q4 = kpad / 4, K = 9u * C;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < total4; i += gridDim.x * blockDim.x) {
    const unsigned row = i / q4, k0 = (i - row * q4) * 4;
    const unsigned bh = row / W;
    const int w = static_cast<int>(row - bh * W);
    const unsigned b = bh / H;
    const int h = static_cast<int>(bh - b * H);
    float v[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const unsigned kk = k0 + e;
      v[e] = 0.0f;
      if (kk < K) {
        const unsigned tap = kk / C, c = kk - tap * C;
        const int hy = h + static_cast<int>(tap / 3) - 1, wx = w + static_cast<int>(tap % 3) - 1;
        if (hy >= 0 && hy < H && wx >= 0 && wx < W) v[e] = __ldg(x + ((static_cast<int64_t>(b) * H + hy) * W + wx) * C + c);
      }
    }
    out[i] = make_float4(v[0], v[1], v[2], v[3]);
  }
}

// conv1_1 (C = 3): one thread per output pixel builds its whole padded row -- the 27
// patch values from 9 three-float pixel reads (compile-time channel count, no integer
// division per element), zeros up to kpad <= 32 -- and writes it as float4s (fp32 rows) or
// 16-byte groups of 8 bf16 (round to nearest even).  Same values as the generic kernels.
template <bool BF16>
__global__ void im2col3x3_c3_kernel(const float* __restrict__ x, int B, int H, int W, int kpad, void* __restrict__ out,
                                    unsigned rows) {
  for (unsigned row = blockIdx.x * blockDim.x + threadIdx.x; row < rows; row += gridDim.x * blockDim.x) {
    const unsigned bh = row / W;
    const int w = static_cast<int>(row - bh * W);
    const unsigned b = bh / H;
    const int h = static_cast<int>(bh - b * H);
    float v[32];
#pragma unroll
    for (int e = 27; e < 32; ++e) v[e] = 0.0f;
#pragma unroll
    for (int tap = 0; tap < 9; ++tap) {
      const int hy = h + tap / 3 - 1, wx = w + tap % 3 - 1;
      const bool in = hy >= 0 && hy < H && wx >= 0 && wx < W;
      const float* src = x + ((static_cast<int64_t>(b) * H + hy) * W + wx) * 3;
#pragma unroll
      for (int c = 0; c < 3; ++c) v[tap * 3 + c] = in ? __ldg(src + c) : 0.0f;
    }
    if constexpr (BF16) {
      uint4* o = static_cast<uint4*>(out) + static_cast<int64_t>(row) * (kpad / 8);
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (q < kpad / 8)
          o[q] = make_uint4(pack_bf16x2(v[8 * q], v[8 * q + 1]), pack_bf16x2(v[8 * q + 2], v[8 * q + 3]),
                            pack_bf16x2(v[8 * q + 4], v[8 * q + 5]), pack_bf16x2(v[8 * q + 6], v[8 * q + 7]));
    } else {
      float4* o = static_cast<float4*>(out) + static_cast<int64_t>(row) * (kpad / 4);
#pragma unroll
      for (int q = 0; q < 8; ++q)
        if (q < kpad / 4) o[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
  }
}

// bf16 operands for the BF16 tensor-core family: im2col of fp32 NHWC activations into
// kpad-wide bf16 rows (zeros beyond 9C), one thread per 8 columns (one 16-byte store);
// the 8 columns are one tap's contiguous channels when C % 8 == 0 (two float4 loads),
// else gathered one by one (conv1_1, C = 3).
__global__ void im2col3x3_nhwc_bf16_kernel(const float* __restrict__ x, int B, int H, int W, int C, int kpad,
                                           uint4* __restrict__ out, unsigned total8) {
  const unsigned q8 = kpad / 8, K = 9u * C;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < total8; i += gridDim.x * blockDim.x) {
    const unsigned row = i / q8, k0 = (i - row * q8) * 8;
    const unsigned bh = row / W;
    const int w = static_cast<int>(row - bh * W);
    const unsigned b = bh / H;
    const int h = static_cast<int>(bh - b * H);
    float v[8];
    if (C % 8 == 0 && k0 + 8 <= K) {
      const unsigned tap = k0 / C, c = k0 - tap * C;
      const int hy = h + static_cast<int>(tap / 3) - 1, wx = w + static_cast<int>(tap % 3) - 1;
      if (hy >= 0 && hy < H && wx >= 0 && wx < W) {
        const float4* src = reinterpret_cast<const float4*>(x + ((static_cast<int64_t>(b) * H + hy) * W + wx) * C + c);
        const float4 a = __ldg(src), d = __ldg(src + 1);
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = d.x; v[5] = d.y; v[6] = d.z; v[7] = d.w;
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) v[e] = 0.0f;
      }
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const unsigned kk = k0 + e;
        v[e] = 0.0f;
        if (kk < K) {
          const unsigned tap = kk / C, c = kk - tap * C;
          const int hy = h + static_cast<int>(tap / 3) - 1, wx = w + static_cast<int>(tap % 3) - 1;
          if (hy >= 0 && hy < H && wx >= 0 && wx < W)
            v[e] = __ldg(x + ((static_cast<int64_t>(b) * H + hy) * W + wx) * C + c);
        }
      }
    }
    uint4 o;
    o.x = pack_bf16x2(v[0], v[1]);
    o.y = pack_bf16x2(v[2], v[3]);
    o.z = pack_bf16x2(v[4], v[5]);
    o.w = pack_bf16x2(v[6], v[7]);
    out[i] = o;
  }
}

// fp32 -> bf16 (round to nearest even), 8 elements per thread (n % 8 == 0, 16-byte aligned).
__global__ void cast_bf16_kernel(const float4* __restrict__ x, uint4* __restrict__ out, unsigned total8) {
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < total8; i += gridDim.x * blockDim.x) {
    const float4 a = __ldg(x + 2 * i), d = __ldg(x + 2 * i + 1);
    out[i] = make_uint4(pack_bf16x2(a.x, a.y), pack_bf16x2(a.z, a.w), pack_bf16x2(d.x, d.y), pack_bf16x2(d.z, d.w));
  }
}

// 2x2 / stride 2 max pool, float4 over channels (C % 4 == 0), 32-bit index math.
__global__ void maxpool2_nhwc_vec4_kernel(const float4* __restrict__ x, int B, int H, int W, int C4,
                                          float4* __restrict__ out, unsigned total) {
  const unsigned Ho = H / 2, Wo = W / 2;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const unsigned c4 = i % C4;
    unsigned r = i / C4;
    const unsigned wo = r % Wo;
    r /= Wo;
    const unsigned ho = r % Ho;
    const unsigned b = r / Ho;
    const float4* base = x + ((static_cast<int64_t>(b) * H + 2 * ho) * W + 2 * wo) * C4 + c4;
    const float4 a0 = __ldg(base), a1 = __ldg(base + C4);
    const float4 a2 = __ldg(base + static_cast<int64_t>(W) * C4), a3 = __ldg(base + static_cast<int64_t>(W) * C4 + C4);
    out[i] = make_float4(fmaxf(fmaxf(a0.x, a1.x), fmaxf(a2.x, a3.x)), fmaxf(fmaxf(a0.y, a1.y), fmaxf(a2.y, a3.y)),
                         fmaxf(fmaxf(a0.z, a1.z), fmaxf(a2.z, a3.z)), fmaxf(fmaxf(a0.w, a1.w), fmaxf(a2.w, a3.w)));
  }
}

// 2x2 / stride 2 max pool of bf16 NHWC activations (BF16 family, written by the GEMM
// epilogue with KP_EPI_BF16_OUT), 8 channels per thread (C % 8 == 0).  The max of four
// bf16 values is one of them, so the result is exact.
__device__ __forceinline__ unsigned max_bf16x2(unsigned a, unsigned b) {
  __nv_bfloat162 x = *reinterpret_cast<const __nv_bfloat162*>(&a), y = *reinterpret_cast<const __nv_bfloat162*>(&b);
  const __nv_bfloat162 r = __hmax2(x, y);
  return *reinterpret_cast<const unsigned*>(&r);
}

__global__ void maxpool2_nhwc_bf16_kernel(const uint4* __restrict__ x, int B, int H, int W, int C8,
                                          uint4* __restrict__ out, unsigned total) {
  const unsigned Ho = H / 2, Wo = W / 2;
  for (unsigned i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const unsigned c8 = i % C8;
    unsigned r = i / C8;
    const unsigned wo = r % Wo;
    r /= Wo;
    const unsigned ho = r % Ho;
    const unsigned b = r / Ho;
    const uint4* base = x + ((static_cast<int64_t>(b) * H + 2 * ho) * W + 2 * wo) * C8 + c8;
    const uint4 a0 = __ldg(base), a1 = __ldg(base + C8);
    const uint4 a2 = __ldg(base + static_cast<int64_t>(W) * C8), a3 = __ldg(base + static_cast<int64_t>(W) * C8 + C8);
    out[i] = make_uint4(max_bf16x2(max_bf16x2(a0.x, a1.x), max_bf16x2(a2.x, a3.x)),
                        max_bf16x2(max_bf16x2(a0.y, a1.y), max_bf16x2(a2.y, a3.y)),
                        max_bf16x2(max_bf16x2(a0.z, a1.z), max_bf16x2(a2.z, a3.z)),
                        max_bf16x2(max_bf16x2(a0.w, a1.w), max_bf16x2(a2.w, a3.w)));
  }
}

// 2x2 / stride 2 max pool; one thread per output element (channel fastest).
__global__ void maxpool2_nhwc_kernel(const float* __restrict__ x, int B, int H, int W, int C, float* __restrict__ out) {
  const int Ho = H / 2, Wo = W / 2;
  const int64_t total = static_cast<int64_t>(B) * Ho * Wo * C;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int c = static_cast<int>(i % C);
    int64_t r = i / C;
    const int wo = static_cast<int>(r % Wo);
    r /= Wo;
    const int ho = static_cast<int>(r % Ho);
    const int64_t b = r / Ho;
    const float* base = x + ((b * H + 2 * ho) * W + 2 * wo) * C + c;
    const float a0 = __ldg(base), a1 = __ldg(base + C);
    const float a2 = __ldg(base + static_cast<int64_t>(W) * C), a3 = __ldg(base + static_cast<int64_t>(W) * C + C);
    out[i] = fmaxf(fmaxf(a0, a1), fmaxf(a2, a3));
  }
}

int grid_for(int64_t total, int threads) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t want = (total + threads - 1) / threads;
  const int64_t cap = static_cast<int64_t>(sms) * 32;  // grid-stride beyond 32 CTAs/SM
  return static_cast<int>(want < cap ? (want > 0 ? want : 1) : cap);
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }


// Row repack for operands TMA cannot address (row pitch not a multiple of 16 bytes, e.g.
// raw k = 27 im2col rows): copies `rows` x `cols` elements of each batch into rows
// pitched to `ldd` (a multiple of 16 bytes).  One thread per destination 16-byte chunk;
// the pad elements past `cols` are written as zeros (the tensor maps never read them).
template <typename T>
__global__ void repack_rows_kernel(const T* __restrict__ src, int64_t ld, int64_t sbatch, int rows, int cols,
                                   T* __restrict__ dst, int64_t ldd, int64_t chunks_per_row, int64_t total) {
  constexpr int V = 16 / sizeof(T);
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t rq = i / chunks_per_row;
    const int q = static_cast<int>(i - rq * chunks_per_row);
    const int64_t b = rq / rows;
    const int64_t r = rq - b * rows;
    const T* in = src + b * sbatch + r * ld;
    T v[V];
#pragma unroll
    for (int e = 0; e < V; ++e) {
      const int c = q * V + e;
      v[e] = c < cols ? in[c] : T(0);
    }
    *reinterpret_cast<uint4*>(dst + (b * rows + r) * ldd + static_cast<int64_t>(q) * V) =
        *reinterpret_cast<const uint4*>(v);
  }
}
}  // namespace

cudaError_t im2col3x3_nhwc_launch(const float* x, int B, int H, int W, int C, float* out, int64_t ldo,
                                  cudaStream_t s) {
  const int64_t total = static_cast<int64_t>(B) * H * W * 9 * C;
  if (C % 4 == 0 && ldo % 4 == 0 && aligned16(x) && aligned16(out) && total / 4 < 0x7fffffffLL) {
    const unsigned t4 = static_cast<unsigned>(total / 4);
    im2col3x3_nhwc_vec4_kernel<<<grid_for(t4, 256), 256, 0, s>>>(reinterpret_cast<const float4*>(x), B, H, W, C / 4,
                                                                   reinterpret_cast<float4*>(out), ldo / 4, t4);
    return cudaGetLastError();
  }
  im2col3x3_nhwc_kernel<<<grid_for(total, 256), 256, 0, s>>>(x, B, H, W, C, out, ldo);
  return cudaGetLastError();
}

cudaError_t im2col3x3_nhwc_pad_launch(const float* x, int B, int H, int W, int C, float* out, int kpad,
                                      cudaStream_t s) {
  const int64_t total4 = static_cast<int64_t>(B) * H * W * (kpad / 4);
  if (kpad % 4 != 0 || kpad < 9 * C || !aligned16(out) || total4 >= 0x7fffffffLL) return cudaErrorInvalidValue;
  if (C == 3 && kpad <= 32) {
    const int64_t rows = static_cast<int64_t>(B) * H * W;
    im2col3x3_c3_kernel<false><<<grid_for(rows, 256), 256, 0, s>>>(x, B, H, W, kpad, out, static_cast<unsigned>(rows));
    return cudaGetLastError();
  }
  im2col3x3_nhwc_pad_kernel<<<grid_for(total4, 256), 256, 0, s>>>(x, B, H, W, C, kpad, reinterpret_cast<float4*>(out),
                                                                   static_cast<unsigned>(total4));
  return cudaGetLastError();
}

cudaError_t im2col3x3_nhwc_bf16_launch(const float* x, int B, int H, int W, int C, void* out, int kpad,
                                       cudaStream_t s) {
  const int64_t total8 = static_cast<int64_t>(B) * H * W * (kpad / 8);
  if (kpad % 8 != 0 || kpad < 9 * C || !aligned16(out) || total8 >= 0x7fffffffLL ||
      (C % 8 == 0 && !aligned16(x)))
    return cudaErrorInvalidValue;
  if (C == 3 && kpad <= 32) {
    const int64_t rows = static_cast<int64_t>(B) * H * W;
    im2col3x3_c3_kernel<true><<<grid_for(rows, 256), 256, 0, s>>>(x, B, H, W, kpad, out, static_cast<unsigned>(rows));
    return cudaGetLastError();
  }
  im2col3x3_nhwc_bf16_kernel<<<grid_for(total8, 256), 256, 0, s>>>(x, B, H, W, C, kpad, reinterpret_cast<uint4*>(out),
                                                                    static_cast<unsigned>(total8));
  return cudaGetLastError();
}

cudaError_t cast_bf16_launch(const float* x, int64_t n, void* out, cudaStream_t s) {
  if (n % 8 != 0 || !aligned16(x) || !aligned16(out) || n / 8 >= 0x7fffffffLL) return cudaErrorInvalidValue;
  cast_bf16_kernel<<<grid_for(n / 8, 256), 256, 0, s>>>(reinterpret_cast<const float4*>(x), reinterpret_cast<uint4*>(out),
                                                         static_cast<unsigned>(n / 8));
  return cudaGetLastError();
}

cudaError_t maxpool2_nhwc_launch(const float* x, int B, int H, int W, int C, float* out, cudaStream_t s) {
  const int64_t total = static_cast<int64_t>(B) * (H / 2) * (W / 2) * C;
  if (C % 4 == 0 && aligned16(x) && aligned16(out) && total / 4 < 0x7fffffffLL) {
    const unsigned t4 = static_cast<unsigned>(total / 4);
    maxpool2_nhwc_vec4_kernel<<<grid_for(t4, 256), 256, 0, s>>>(reinterpret_cast<const float4*>(x), B, H, W, C / 4,
                                                                  reinterpret_cast<float4*>(out), t4);
    return cudaGetLastError();
  }
  maxpool2_nhwc_kernel<<<grid_for(total, 256), 256, 0, s>>>(x, B, H, W, C, out);
  return cudaGetLastError();
}

cudaError_t maxpool2_nhwc_bf16_launch(const void* x, int B, int H, int W, int C, void* out, cudaStream_t s) {
  const int64_t total = static_cast<int64_t>(B) * (H / 2) * (W / 2) * C;
  if (C % 8 != 0 || !aligned16(x) || !aligned16(out) || total / 8 >= 0x7fffffffLL) return cudaErrorInvalidValue;
  const unsigned t8 = static_cast<unsigned>(total / 8);
  if (t8 == 0) return cudaSuccess;
  maxpool2_nhwc_bf16_kernel<<<grid_for(t8, 256), 256, 0, s>>>(static_cast<const uint4*>(x), B, H, W, C / 8,
                                                                static_cast<uint4*>(out), t8);
  return cudaGetLastError();
}

cudaError_t repack_rows_launch(const void* src, int64_t ld, int64_t sbatch, int rows, int cols, int batch, int es,
                               void* dst, int64_t ldd, cudaStream_t s) {
  if ((es != 2 && es != 4) || !aligned16(dst) || (ldd * es) % 16 != 0 || ldd < cols) return cudaErrorInvalidValue;
  const int64_t chunks = ldd * es / 16;
  const int64_t total = static_cast<int64_t>(batch) * rows * chunks;
  if (total == 0) return cudaSuccess;
  if (es == 2)
    repack_rows_kernel<uint16_t><<<grid_for(total, 256), 256, 0, s>>>(
        static_cast<const uint16_t*>(src), ld, sbatch, rows, cols, static_cast<uint16_t*>(dst), ldd, chunks, total);
  else
    repack_rows_kernel<uint32_t><<<grid_for(total, 256), 256, 0, s>>>(
        static_cast<const uint32_t*>(src), ld, sbatch, rows, cols, static_cast<uint32_t*>(dst), ldd, chunks, total);
  return cudaGetLastError();
}

}  // namespace kp
