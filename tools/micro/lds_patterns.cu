// Micro-benchmark (dev tool, not product): shared-memory wavefronts per LDS for
// lane -> address patterns.  Run under ncu --set full and read the source page.
#include <cstdio>
#include <cuda_runtime.h>

template <int PAT>
__device__ __forceinline__ int addr_of(int lane) {
  switch (PAT) {
    case 0: return 0;                    // full broadcast
    case 1: return lane >> 2;            // 8 distinct, 4 consecutive lanes share
    case 2: return lane & 3;             // 4 distinct, strided sharing
    case 3: return lane >> 3;            // 4 distinct, 8 consecutive share
    case 4: return lane & 7;             // 8 distinct, strided
    case 5: return lane >> 1;            // 16 distinct, pairs
    case 6: return lane;                 // 32 distinct
    case 7: return lane >> 4;            // 2 distinct, half warps
    case 8: return (lane & 3) + 4 * (lane >> 4);  // 8 distinct: (lane%4, half)
    case 9: return lane & 15;            // 16 distinct strided
    default: return 0;
  }
}

template <int PAT>
__global__ void k128(float* out, int iters) {
  __shared__ float4 s[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) s[i] = make_float4(i, i + 1, i + 2, i + 3);
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float4 acc = make_float4(0, 0, 0, 0);
  const int base = w * 64;
  for (int it = 0; it < iters; ++it) {
    float4 v = s[(base + addr_of<PAT>(lane) + it) & 1023];
    acc.x += v.x; acc.y += v.y; acc.z += v.z; acc.w += v.w;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y + acc.z + acc.w;
}

template <int PAT>
__global__ void k64(float* out, int iters) {
  __shared__ float2 s[2048];
  for (int i = threadIdx.x; i < 2048; i += blockDim.x) s[i] = make_float2(i, i + 1);
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  float2 acc = make_float2(0, 0);
  const int base = w * 64;
  for (int it = 0; it < iters; ++it) {
    float2 v = s[(base + addr_of<PAT>(lane) + it) & 2047];
    acc.x += v.x; acc.y += v.y;
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc.x + acc.y;
}

template <int PAT>
void run(float* d) {
  k128<PAT><<<148, 256>>>(d, 4096);
  k64<PAT><<<148, 256>>>(d, 4096);
}

int main() {
  float* d;
  cudaMalloc(&d, 148 * 256 * 4);
  run<0>(d); run<1>(d); run<2>(d); run<3>(d); run<4>(d);
  run<5>(d); run<6>(d); run<7>(d); run<8>(d); run<9>(d);
  cudaDeviceSynchronize();
  printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
