// Internal interface between the C ABI (capi.cu) and the kernel families.
#pragma once

#include <cuda_runtime.h>

#include <atomic>

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

// One F1 instantiation: its launcher plus the compile-time tile facts the k-slice
// planner (capi.cu) needs.  bm x bn is the CTA output tile, bk the k-tile depth, occ
// the resident-CTA target per SM (__launch_bounds__ min blocks).
struct F1Entry {
  GemmLaunchFn launch;
  int bm, bn, bk, occ;
  int tma_ok;  // TMA staging applies (16-byte-aligned rows assumed): CTA tile <= 256 columns
  // cudaOccupancyMaxActiveClusters for a (1, 1, slices) cluster launch (< 0: error)
  int (*cluster_fit)(int slices);
};
// SIMT operand staging mode (kp_set_simt_staging): 1 = TMA where eligible, 0 = cp.async.
extern std::atomic<int> g_f1_tma_staging;

constexpr int kMaxKSlices = 16;      // non-portable thread-block-cluster limit on sm_100
constexpr int kDefaultKSlices = 16;  // cap of kp_set_max_k_slices; the planner's rules pick S
constexpr int kPortableKSlices = 8;  // tensor-core families: portable clusters measured faster than 9..16

// F0 (family PAPER): any (R,A,C) in {1,2,4,8}^3, any block shape <= 1024 threads.
cudaError_t f0_launch(const KernelChoice& ch, GemmArgs p, cudaStream_t s);

// F1 (family SIMT): table of 640 entries in enumerate_configs order, filled by
// the ten per-work-group translation units (f1_simt_inst.cu compiled ten times).
void f1_fill_wg0(F1Entry* table);
void f1_fill_wg1(F1Entry* table);
void f1_fill_wg2(F1Entry* table);
void f1_fill_wg3(F1Entry* table);
void f1_fill_wg4(F1Entry* table);
void f1_fill_wg5(F1Entry* table);
void f1_fill_wg6(F1Entry* table);
void f1_fill_wg7(F1Entry* table);
void f1_fill_wg8(F1Entry* table);
void f1_fill_wg9(F1Entry* table);

// Conv-as-GEMM helpers (nn_ops.cu).
cudaError_t im2col3x3_nhwc_launch(const float* x, int B, int H, int W, int C, float* out, int64_t ldo,
                                  cudaStream_t s);
cudaError_t maxpool2_nhwc_launch(const float* x, int B, int H, int W, int C, float* out, cudaStream_t s);
cudaError_t im2col3x3_nhwc_pad_launch(const float* x, int B, int H, int W, int C, float* out, int kpad,
                                      cudaStream_t s);
cudaError_t im2col3x3_nhwc_bf16_launch(const float* x, int B, int H, int W, int C, void* out, int kpad,
                                       cudaStream_t s);
cudaError_t maxpool2_nhwc_bf16_launch(const void* x, int B, int H, int W, int C, void* out, cudaStream_t s);
cudaError_t cast_bf16_launch(const float* x, int64_t n, void* out, cudaStream_t s);
// Copy batch x rows x cols elements (es bytes each; source pitch ld, batch stride sbatch)
// into rows pitched to ldd (a multiple of 16 bytes), batch stride rows * ldd.
cudaError_t repack_rows_launch(const void* src, int64_t ld, int64_t sbatch, int rows, int cols, int batch, int es,
                               void* dst, int64_t ldd, cudaStream_t s);

// FFMA peak probe.
cudaError_t ffma_peak_launch(float* sink, int blocks, int threads, int iters, bool packed, cudaStream_t s);

}  // namespace kp
