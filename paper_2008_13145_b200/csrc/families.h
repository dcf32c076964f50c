// Internal interface between the C ABI (capi.cu) and the kernel families.
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"

namespace kp {

// Work-group pairs in DEFAULT_WG_PAIRS order (dataset.py:19-31); the config index
// of (R, A, C, wg) is ((log2 R * 4 + log2 A) * 4 + log2 C) * 10 + wg_index, i.e.
// enumerate_configs() order (dataset.py:173-196: R slowest, wg pair fastest).
constexpr int kNumWgPairs = 10;
constexpr int kWgPairs[kNumWgPairs][2] = {{1, 64}, {1, 128}, {8, 8},  {8, 16}, {8, 32},
                                          {16, 8}, {16, 16}, {32, 8}, {64, 1}, {128, 1}};
constexpr int kPaperConfigs = 640;

using GemmLaunchFn = cudaError_t (*)(const GemmArgs&, cudaStream_t);

// F0 (family PAPER): any (R,A,C) in {1,2,4,8}^3, any block shape <= 1024 threads.
cudaError_t f0_launch(const KernelChoice& ch, GemmArgs p, cudaStream_t s);

// F1 (family SIMT): table of 640 launchers in enumerate_configs order, filled by
// the ten per-work-group translation units (f1_simt_inst.cu compiled ten times).
void f1_fill_wg0(GemmLaunchFn* table);
void f1_fill_wg1(GemmLaunchFn* table);
void f1_fill_wg2(GemmLaunchFn* table);
void f1_fill_wg3(GemmLaunchFn* table);
void f1_fill_wg4(GemmLaunchFn* table);
void f1_fill_wg5(GemmLaunchFn* table);
void f1_fill_wg6(GemmLaunchFn* table);
void f1_fill_wg7(GemmLaunchFn* table);
void f1_fill_wg8(GemmLaunchFn* table);
void f1_fill_wg9(GemmLaunchFn* table);

// Conv-as-GEMM helpers (nn_ops.cu).
cudaError_t im2col3x3_nhwc_launch(const float* x, int B, int H, int W, int C, float* out, int64_t ldo,
                                  cudaStream_t s);
cudaError_t maxpool2_nhwc_launch(const float* x, int B, int H, int W, int C, float* out, cudaStream_t s);

// FFMA peak probe.
cudaError_t ffma_peak_launch(float* sink, int blocks, int threads, int iters, bool packed, cudaStream_t s);

}  // namespace kp
