/*
 * gemm_ref.c -- CPU ORACLE for the kernel family.  TEST INFRASTRUCTURE ONLY: linked
 * by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * leg as the checker or the CPU reference timing; never by the product path.
 *
 * Restates the paper's matmul kernel (kernelprune dataset.py:41-46):
 * work items own an R x C output tile, step k by A, loading an R x A LHS tile and an
 * A x C RHS tile and accumulating in fp32.  Work groups of wg_rows x wg_cols items
 * tile the output exactly as work_items() describes (dataset.py:312-316).  The
 * reference ships no GEMM -- its numeric engine is numpy -- so
 * this port is pinned by construction: every output element is the sequential fp32
 * fused-multiply-add chain acc = fmaf(a[i][kk], b[kk][j], acc) over kk = 0..K-1
 * starting from +0.0f, the arithmetic the GPU families F0/F1 perform; they must
 * match it BIT-EXACTLY.  kp_ref_gemm_f64 is the float64 product (np.matmul on float64
 * operands) that tolerance checks and the TF32/BF16 families are judged against.
 *
 * Build: make -C oracle   ->  oracle/libgemmref.so (OpenMP over work groups).
 */
#include <math.h>
#include <omp.h>
#include <stdint.h>
#include <string.h>

/* OpenMP team size for the oracle (n > 0 sets it; launchers such as torchrun export
 * OMP_NUM_THREADS=1); returns the size now in effect. */
int kp_ref_threads(int n) {
  if (n > 0) omp_set_num_threads(n);
  return omp_get_max_threads();
}

/* Hardware FMA when the host has it (fmaf is correctly rounded either way, so the
 * clones are bit-identical); the default clone keeps the .so loadable anywhere. */
#define KP_CLONES __attribute__((target_clones("arch=x86-64-v3", "default")))

/* Paper-order tiled emulation: returns the number of work items launched. */
KP_CLONES int64_t kp_ref_gemm_tiled(int R, int A, int C, int wg_rows, int wg_cols, int m, int k, int n, int batch,
                          const float* Am, int64_t lda, int64_t sA, const float* Bm, int64_t ldb, int64_t sB,
                          float* Cm, int64_t ldc, int64_t sC) {
  const int64_t groups_m = (m + (int64_t)R * wg_rows - 1) / ((int64_t)R * wg_rows);
  const int64_t groups_n = (n + (int64_t)C * wg_cols - 1) / ((int64_t)C * wg_cols);
  const int64_t groups = groups_m * groups_n * batch;
#pragma omp parallel for schedule(dynamic, 16)
  for (int64_t g = 0; g < groups; ++g) {
    const int64_t b = g / (groups_m * groups_n);
    const int64_t rem = g % (groups_m * groups_n);
    const int64_t gm = rem / groups_n, gn = rem % groups_n;
    const float* Ab = Am + b * sA;
    const float* Bb = Bm + b * sB;
    float* Cb = Cm + b * sC;
    float acc[64];
    for (int wy = 0; wy < wg_rows; ++wy)
      for (int wx = 0; wx < wg_cols; ++wx) {
        const int64_t row0 = (gm * wg_rows + wy) * R, col0 = (gn * wg_cols + wx) * C;
        if (row0 >= m || col0 >= n) continue;
        for (int t = 0; t < R * C; ++t) acc[t] = 0.0f;
        for (int64_t kk = 0; kk < k; kk += A) {
          for (int i = 0; i < A; ++i) {
            if (kk + i >= k) break; /* the GPU's zero padding adds fmaf(0,0,acc) == acc */
            for (int r = 0; r < R; ++r) {
              if (row0 + r >= m) break;
              const float a = Ab[(row0 + r) * lda + kk + i];
              for (int c = 0; c < C; ++c) {
                if (col0 + c >= n) break;
                acc[r * C + c] = fmaf(a, Bb[(kk + i) * ldb + col0 + c], acc[r * C + c]);
              }
            }
          }
        }
        for (int r = 0; r < R && row0 + r < m; ++r)
          for (int c = 0; c < C && col0 + c < n; ++c) Cb[(row0 + r) * ldc + col0 + c] = acc[r * C + c];
      }
  }
  return groups * wg_rows * wg_cols;
}

/* A block of up to 8 output rows x 256 columns of the sequential fmaf chain: each B
 * row segment is loaded once per block and applied to every row (cache blocking
 * only -- every element still accumulates kk = 0..K-1 in order from +0).  Cloned so
 * the inner loop becomes packed hardware FMA where the host has it. */
#define KP_RB 8
#define KP_JB 256
KP_CLONES void kp_ref_chain_block(int rows, int k, int jn, const float* restrict A0, int64_t lda,
                                  const float* restrict B0, int64_t ldb, float* restrict C0, int64_t ldc) {
  float acc[KP_RB][KP_JB];
  for (int r = 0; r < rows; ++r)
    for (int j = 0; j < jn; ++j) acc[r][j] = 0.0f;
  for (int kk = 0; kk < k; ++kk) {
    const float* restrict brow = B0 + (int64_t)kk * ldb;
    for (int r = 0; r < rows; ++r) {
      const float a = A0[(int64_t)r * lda + kk];
      float* restrict c = acc[r];
      for (int j = 0; j < jn; ++j) c[j] = fmaf(a, brow[j], c[j]);
    }
  }
  for (int r = 0; r < rows; ++r)
    for (int j = 0; j < jn; ++j) C0[(int64_t)r * ldc + j] = acc[r][j];
}

/* Sequential fmaf chain per element, parallel over (batch, row block, column block). */
void kp_ref_gemm_chain(int m, int k, int n, int batch, const float* Am, int64_t lda, int64_t sA, const float* Bm,
                       int64_t ldb, int64_t sB, float* Cm, int64_t ldc, int64_t sC) {
  const int64_t rb = (m + KP_RB - 1) / KP_RB, jb = (n + KP_JB - 1) / KP_JB;
  const int64_t tasks = (int64_t)batch * rb * jb;
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t t = 0; t < tasks; ++t) {
    const int64_t b = t / (rb * jb), rem = t % (rb * jb);
    const int64_t i0 = (rem / jb) * KP_RB, j0 = (rem % jb) * KP_JB;
    const int rows = (int)(m - i0 < KP_RB ? m - i0 : KP_RB);
    const int jn = (int)(n - j0 < KP_JB ? n - j0 : KP_JB);
    kp_ref_chain_block(rows, k, jn, Am + b * sA + i0 * lda, lda, Bm + b * sB + j0, ldb, Cm + b * sC + i0 * ldc + j0,
                       ldc);
  }
}

/* k-sliced variant (the SIMT family's plan when a launch cannot fill the GPU, see
 * kp_gemm_plan in include/kpgemm.h): k is cut into consecutive slices of k_per_slice
 * (the last one shorter); each slice is the sequential fmaf chain from +0 over its k
 * range and the slices are summed in order, out = ((p0 + p1) + p2) + ...
 * k_per_slice >= k is the plain chain. */
void kp_ref_gemm_sliced(int m, int k, int n, int batch, int k_per_slice, const float* Am, int64_t lda, int64_t sA,
                        const float* Bm, int64_t ldb, int64_t sB, float* Cm, int64_t ldc, int64_t sC) {
  if (k_per_slice <= 0 || k_per_slice >= k) {
    kp_ref_gemm_chain(m, k, n, batch, Am, lda, sA, Bm, ldb, sB, Cm, ldc, sC);
    return;
  }
  const int64_t rb = (m + KP_RB - 1) / KP_RB, jb = (n + KP_JB - 1) / KP_JB;
  const int64_t tasks = (int64_t)batch * rb * jb;
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t t = 0; t < tasks; ++t) {
    const int64_t b = t / (rb * jb), rem = t % (rb * jb);
    const int64_t i0 = (rem / jb) * KP_RB, j0 = (rem % jb) * KP_JB;
    const int rows = (int)(m - i0 < KP_RB ? m - i0 : KP_RB);
    const int jn = (int)(n - j0 < KP_JB ? n - j0 : KP_JB);
    float part[KP_RB * KP_JB];
    float* out = Cm + b * sC + i0 * ldc + j0;
    for (int k0 = 0; k0 < k; k0 += k_per_slice) {
      const int kl = k - k0 < k_per_slice ? k - k0 : k_per_slice;
      kp_ref_chain_block(rows, kl, jn, Am + b * sA + i0 * lda + k0, lda, Bm + b * sB + (int64_t)k0 * ldb + j0, ldb,
                         part, KP_JB);
      for (int r = 0; r < rows; ++r)
        for (int j = 0; j < jn; ++j) {
          float* o = out + (int64_t)r * ldc + j;
          *o = k0 == 0 ? part[r * KP_JB + j] : *o + part[r * KP_JB + j];
        }
    }
  }
}

/* float64 product of the fp32 operands, plus the |A||B| magnitude for the
 * per-element error bound |C - C64| <= 2 k u (|A||B|)_ij. */
KP_CLONES void kp_ref_gemm_f64(int m, int k, int n, int batch, const float* Am, int64_t lda, int64_t sA, const float* Bm,
                     int64_t ldb, int64_t sB, double* Cm, double* Mag, int64_t ldc, int64_t sC) {
#pragma omp parallel for collapse(2) schedule(static)
  for (int b = 0; b < batch; ++b)
    for (int i = 0; i < m; ++i) {
      const float* arow = Am + b * sA + (int64_t)i * lda;
      const float* Bb = Bm + b * sB;
      double* crow = Cm + b * sC + (int64_t)i * ldc;
      double* mrow = Mag + b * sC + (int64_t)i * ldc;
      for (int j = 0; j < n; ++j) crow[j] = mrow[j] = 0.0;
      for (int kk = 0; kk < k; ++kk) {
        const double a = arow[kk];
        const float* brow = Bb + (int64_t)kk * ldb;
        for (int j = 0; j < n; ++j) {
          crow[j] += a * (double)brow[j];
          mrow[j] += fabs(a) * fabs((double)brow[j]);
        }
      }
    }
}
