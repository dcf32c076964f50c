// F0 -- the paper-faithful fp32 SIMT matmul family (KP_FAMILY_PAPER).
//
// Semantics follow the kernel the paper benchmarks and the
// reference's description of a config (dataset.py:41-46): each work item owns an
// R x C output tile and, per step, loads an R x A tile of the LHS and an A x C tile
// of the RHS straight from global memory as vectors of width A and C
// (dataset.py:33: "tile sizes double as vector load widths"), accumulating into
// registers.  There is no shared memory.  The work-group shape
// (wg_rows, wg_cols) is a launch-time choice (blockDim), so the 640-config space is
// 64 template instantiations x 10 runtime block shapes.
//
// Launch geometry is exactly work_items() (dataset.py:312-316):
//   blockDim = (wg_cols, wg_rows)
//   gridDim  = (ceil(m/(R*wg_rows)) * ceil(n/(C*wg_cols)), batch)
// The m-groups sit in gridDim.x (2^31-1 limit), never gridDim.y (65535), because
// VGG conv1 at batch 64 folds to m = 3.2M rows (hard part 2).
//
// Accumulation order: every output element is a single fp32 fma chain over
// k = 0..K-1 in order starting from +0, so the result is bit-identical to the
// oracle's sequential fmaf chain (oracle/gemm_ref.c) and to family SIMT.
#include "common.cuh"
#include "families.h"

namespace kp {
namespace {

template <int R, int A, int C>
__global__ void f0_kernel(GemmArgs p, int groups_n) {
  const int wgR = blockDim.y, wgC = blockDim.x;
  const int64_t gm = blockIdx.x / groups_n;
  const int gn = blockIdx.x - static_cast<int>(gm * groups_n);
  const int b = blockIdx.y;
  const int64_t row0 = (gm * wgR + threadIdx.y) * R;
  const int64_t col0 = (static_cast<int64_t>(gn) * wgC + threadIdx.x) * C;
  const int m = p.m, k = p.k, n = p.n;
  if (row0 >= m || col0 >= n) return;  // no smem, no barriers: early exit is safe

  const float* __restrict__ Ab = static_cast<const float*>(p.A) + b * p.sA;
  const float* __restrict__ Bb = static_cast<const float*>(p.B) + b * p.sB;
  float* __restrict__ Cb = static_cast<float*>(p.C) + b * p.sC;

  float acc[R][C];
#pragma unroll
  for (int r = 0; r < R; ++r)
#pragma unroll
    for (int c = 0; c < C; ++c) acc[r][c] = 0.0f;

  const bool rows_full = row0 + R <= m;
  const bool cols_full = col0 + C <= n;
  int kk = 0;

  if (p.a_vec && p.b_vec && cols_full) {
    // Vector path: R loads of width A from the LHS, A loads of width C from the RHS.
    const int kfull = k - (k % A);
    for (; kk < kfull; kk += A) {
      float a[R][A];
      float w[A][C];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (rows_full || row0 + r < m) {
          ldg_vec<A>(Ab + (row0 + r) * p.lda + kk, a[r]);
        } else {
#pragma unroll
          for (int i = 0; i < A; ++i) a[r][i] = 0.0f;
        }
      }
#pragma unroll
      for (int i = 0; i < A; ++i) ldg_vec<C>(Bb + static_cast<int64_t>(kk + i) * p.ldb + col0, w[i]);
#pragma unroll
      for (int i = 0; i < A; ++i)
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int c = 0; c < C; ++c) acc[r][c] = __fmaf_rn(a[r][i], w[i][c], acc[r][c]);
    }
  }
  // Scalar, bounds-checked path: k tails, ragged n, unaligned operands.  Padding
  // lanes contribute fma(0, 0, acc) == acc exactly.
  for (; kk < k; kk += A) {
    float a[R][A];
    float w[A][C];
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int i = 0; i < A; ++i)
        a[r][i] = (row0 + r < m && kk + i < k) ? __ldg(Ab + (row0 + r) * p.lda + kk + i) : 0.0f;
#pragma unroll
    for (int i = 0; i < A; ++i)
#pragma unroll
      for (int c = 0; c < C; ++c)
        w[i][c] = (kk + i < k && col0 + c < n) ? __ldg(Bb + static_cast<int64_t>(kk + i) * p.ldb + col0 + c)
                                               : 0.0f;
#pragma unroll
    for (int i = 0; i < A; ++i)
#pragma unroll
      for (int r = 0; r < R; ++r)
#pragma unroll
        for (int c = 0; c < C; ++c) acc[r][c] = __fmaf_rn(a[r][i], w[i][c], acc[r][c]);
  }

  if (p.bias || p.relu) {
#pragma unroll
    for (int r = 0; r < R; ++r)
#pragma unroll
      for (int c = 0; c < C; ++c)
        if (col0 + c < n) acc[r][c] = epilogue(p, acc[r][c], col0 + c);
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    if (!rows_full && row0 + r >= m) break;
    float* out = Cb + (row0 + r) * p.ldc + col0;
    if (cols_full && p.c_vec) {
      stg_vec<C>(out, acc[r]);
    } else {
#pragma unroll
      for (int c = 0; c < C; ++c)
        if (col0 + c < n) out[c] = acc[r][c];
    }
  }
}

template <int R, int A, int C>
cudaError_t launch_one(const KernelChoice& ch, const GemmArgs& p, cudaStream_t s) {
  const int64_t groups_m = (p.m + static_cast<int64_t>(R) * ch.wg_rows - 1) / (static_cast<int64_t>(R) * ch.wg_rows);
  const int64_t groups_n = (p.n + static_cast<int64_t>(C) * ch.wg_cols - 1) / (static_cast<int64_t>(C) * ch.wg_cols);
  const int64_t gx = groups_m * groups_n;
  if (gx > 0x7fffffffLL || p.batch > 65535) return cudaErrorInvalidConfiguration;
  dim3 block(ch.wg_cols, ch.wg_rows);
  dim3 grid(static_cast<unsigned>(gx), p.batch);
  f0_kernel<R, A, C><<<grid, block, 0, s>>>(p, static_cast<int>(groups_n));
  return cudaGetLastError();
}

using LaunchFn = cudaError_t (*)(const KernelChoice&, const GemmArgs&, cudaStream_t);

template <int RI, int AI, int CI>
constexpr LaunchFn pick() {
  return &launch_one<(1 << RI), (1 << AI), (1 << CI)>;
}

// Table indexed by (log2 R, log2 A, log2 C).
#define KP_F0_ROW(RI, AI) pick<RI, AI, 0>(), pick<RI, AI, 1>(), pick<RI, AI, 2>(), pick<RI, AI, 3>()
#define KP_F0_BLOCK(RI) KP_F0_ROW(RI, 0), KP_F0_ROW(RI, 1), KP_F0_ROW(RI, 2), KP_F0_ROW(RI, 3)
const LaunchFn kTable[64] = {KP_F0_BLOCK(0), KP_F0_BLOCK(1), KP_F0_BLOCK(2), KP_F0_BLOCK(3)};
#undef KP_F0_BLOCK
#undef KP_F0_ROW

int ilog2_tile(int v) {
  switch (v) {
    case 1: return 0;
    case 2: return 1;
    case 4: return 2;
    case 8: return 3;
    default: return -1;
  }
}

}  // namespace

bool f0_alignment(const KernelChoice& ch, GemmArgs* p) {
  auto aligned = [](const void* ptr, int bytes) { return (reinterpret_cast<uintptr_t>(ptr) % bytes) == 0; };
  const int va = ch.tile_acc < 4 ? ch.tile_acc : 4;
  const int vc = ch.tile_cols < 4 ? ch.tile_cols : 4;
  p->a_vec = (p->lda % va == 0) && (p->sA % va == 0) && aligned(p->A, 4 * va);
  p->b_vec = (p->ldb % vc == 0) && (p->sB % vc == 0) && aligned(p->B, 4 * vc);
  p->c_vec = (p->ldc % vc == 0) && (p->sC % vc == 0) && aligned(p->C, 4 * vc);
  return true;
}

cudaError_t f0_launch(const KernelChoice& ch, GemmArgs p, cudaStream_t s) {
  const int ri = ilog2_tile(ch.tile_rows), ai = ilog2_tile(ch.tile_acc), ci = ilog2_tile(ch.tile_cols);
  if (ri < 0 || ai < 0 || ci < 0) return cudaErrorInvalidValue;
  f0_alignment(ch, &p);
  return kTable[ri * 16 + ai * 4 + ci](ch, p, s);
}

}  // namespace kp
