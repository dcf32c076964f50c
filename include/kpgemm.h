/*
 * kpgemm.h -- C ABI of the B200 (sm_100a) tiled-GEMM kernel family behind the
 * kernelprune benchmark/selection path (arXiv 2008.13145).
 *
 * The reference package (`kernelprune`, /root/reference/pkg) is host-only: it
 * consumes a benchmark table and emits a selector, but the kernel, the timing
 * harness and the launcher sit outside it. This header is the boundary those
 * missing pieces plug into. Every entry point below names the reference
 * interface it serves:
 *
 *   KernelChoice ............ the struct the emitted `select_kernel(...)` returns
 *                             (codegen.py:185-194; the reference never defines it)
 *                             and the 5-tuple of KernelConfig (dataset.py:39-58).
 *   kp_gemm ................. "matmul-with-config": the kernel the paper times
 *                             (dataset.py:41-46 tile semantics,
 *                             dataset.py:312-316 launch geometry for family PAPER).
 *   kp_bench ................ the benchmark harness that produces one cell of the
 *                             CSV `m,k,n,batch,R,A,C,wgR,wgC,gflops`
 *                             (dataset.py:36, replacing synth_generate
 *                             dataset.py:319-347 as the PerfMatrix producer).
 *   kp_dispatch_* ........... the runtime selector: predict_tree (classify.py:230-237)
 *                             walked over a kptree v1 model (codegen.py:36-51) with the
 *                             same strict '<' comparison (codegen.py:188).
 *   kp_gemm_auto ............ select_kernel + launch in one call.
 *
 * Conventions
 *   - Problem dims are passed in the reference's ProblemSize order (m, k, n, batch)
 *     (dataset.py:61-74).  C[b] = A[b] * B[b]; A is m x k, B is k x n, C is m x n,
 *     all row-major with leading dimensions lda/ldb/ldc (elements) and batch strides
 *     sA/sB/sC (elements; sB == 0 broadcasts one weight matrix over the batch).
 *   - Element types by family: PAPER/SIMT/TF32: A,B,C fp32. BF16: A,B bf16, C fp32.
 *   - Every call returns 0 on success or a negative status (KP_E*) and records a
 *     thread-local message readable with kp_last_error().  The Python shim maps
 *     KP_EINVAL -> ValueError, KP_ENOENT -> KeyError/ValueError, KP_EIO -> RuntimeError
 *     (errors.py:1-49 taxonomy).  There is no CPU fallback anywhere.
 *   - The caller owns all device memory; no entry point allocates or frees device
 *     buffers.  `stream` is a cudaStream_t (NULL = legacy default stream).
 */
#ifndef KPGEMM_H_
#define KPGEMM_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KPGEMM_ABI_VERSION 1

/* Status codes (negated errno values). */
#define KP_OK 0
#define KP_ENOENT (-2)  /* unknown variant / no dispatch table */
#define KP_EIO (-5)     /* CUDA launch or runtime error */
#define KP_EINVAL (-22) /* bad config, shape, stride or alignment */

/* Kernel families.  Each family has its own config list and its own benchmark
 * table: the oracle-best denominator spans every column of a table
 * (evaluate.py:81), so families are never mixed in one table silently. */
#define KP_FAMILY_PAPER 0 /* F0: paper-faithful fp32 SIMT, no shared memory */
#define KP_FAMILY_SIMT 1  /* F1: B200 fp32 SIMT, TMA/mbarrier (or cp.async) smem ring, warp tiles   */
#define KP_FAMILY_TF32 2  /* F2: tcgen05 kind::tf32, fp32 in / fp32 out                            */
#define KP_FAMILY_BF16 3  /* F3: tcgen05 kind::f16, bf16 in / fp32 out                              */
#define KP_NUM_FAMILIES 4

/* Field order is the emitted selector's (codegen.py:191-192).  PAPER / SIMT families:
 * the paper's meaning below (dataset.py:39-58).  TF32 / BF16 families: (BM = 128, or 256
 * for CTA-pair configs, BK = elements per 128-byte k slab, BN, smem stages, 192 threads). */
typedef struct KernelChoice {
  int32_t tile_rows; /* R: output rows per work item              */
  int32_t tile_acc;  /* A: accumulation depth per step / k vector */
  int32_t tile_cols; /* C: output cols per work item              */
  int32_t wg_rows;   /* work-group rows                           */
  int32_t wg_cols;   /* work-group cols                           */
} KernelChoice;

/* ---- library / registry ------------------------------------------------ */
int kp_abi_version(void);
const char* kp_last_error(void);
int kp_num_variants(void);
/* Variant id of (family, choice), or KP_ENOENT. */
int kp_find_variant(int family, KernelChoice choice);
/* Registry entry of a variant id. */
int kp_variant_info(int id, KernelChoice* choice, int* family);
/* Number of configs of a family; their order is the family's canonical column
 * order (enumerate_configs order, dataset.py:173-196, for PAPER and SIMT). */
int kp_family_size(int family);
int kp_family_variant(int family, int index);

/* ---- GEMM ("matmul-with-config") --------------------------------------- */
int kp_gemm(int id, int m, int k, int n, int batch,
            const void* A, int64_t lda, int64_t sA,
            const void* B, int64_t ldb, int64_t sB,
            void* C, int64_t ldc, int64_t sC, void* stream);

/* Fused epilogue variant (VGG16 conv/fc layers):
 *   C = act(A * B + bias[col]), bias may be NULL, act = ReLU when flags & KP_EPI_RELU.
 * The bias add and ReLU follow the fp32 accumulation chain, so SIMT results stay
 * bit-exact against oracle_chain + bias -> max(0, .).
 * KP_EPI_BF16_OUT (TF32 and BF16 variants only, else KP_EINVAL): C is bf16, the fp32
 * epilogue result rounded to nearest even -- a BF16 layer's output written directly as
 * the next layer's operand (equal to fp32 C followed by kp_cast_bf16). */
#define KP_EPI_RELU 1
#define KP_EPI_BF16_OUT 2
int kp_gemm_ex(int id, int m, int k, int n, int batch,
               const void* A, int64_t lda, int64_t sA,
               const void* B, int64_t ldb, int64_t sB,
               void* C, int64_t ldc, int64_t sC,
               const float* bias, int flags, void* stream);

/* ---- k-slicing (SIMT, TF32 and BF16 families) ----------------------------
 * A launch whose output tiles leave SMs idle or end in a partial wave cuts k into S
 * consecutive slices, computed by the CTAs of one (1, 1, S) thread-block cluster per
 * output tile and summed in slice order ((p0 + p1) + p2) + ... through distributed
 * shared memory -- deterministic for a given (config, shape, device).
 *   SIMT:   u = output tiles / SMs; S = 16 (u < 0.15, a non-portable cluster), 8 (u < 0.5),
 *           4 (u < 2), 2 (u < 6), else 1,
 *           halved while the sliced grid exceeds 4 waves of resident CTAs, and never
 *           shallower than 64 in k (a rule fitted on measured forced-S data).
 *   TF32/BF16 (persistent 1-CTA/SM kernel): grids filling at most half the SMs,
 *           S = min(8, SMs / tiles, k / 768), lowered until every tile's cluster is
 *           co-resident in one wave (cudaOccupancyMaxActiveClusters); and for grids of
 *           more than one wave with long tiles (BN*k >= 1.72e6, TF32 0.86e6) whose
 *           partial last wave fills at most half the SMs, those tail tiles only, as a
 *           second sliced launch after the persistent one (kp_gemm_plan then reports
 *           the tail launch's S and depth).
 *   PAPER:  never (the paper's launch geometry).
 * kp_gemm_plan reports the plan kp_gemm would use: *k_slices = S and *k_per_slice =
 * the depth of every slice but the last (= k when S == 1).  num_sms <= 0 means the
 * current device's SM count and cluster limits (num_sms > 0 plans for a hypothetical
 * device with that many SMs and no cluster limit).  kp_set_max_k_slices caps S
 * (1 disables slicing: every SIMT output is then the single fp32 fma chain over k,
 * bit-identical to the PAPER family, and the tensor-core families run persistent);
 * returns the previous cap (default 16, range 1..16; the tensor-core rules never exceed 8). */
int kp_set_max_k_slices(int max_slices);
int kp_gemm_plan(int id, int m, int k, int n, int batch, int num_sms, int* k_slices, int* k_per_slice);

/* SIMT-family operand staging (a launch detail; results are bit-identical either way):
 * 1 = TMA bulk tensor copies + mbarriers wherever the operand rows are 16-byte
 * aligned and the CTA tile is <= 256 columns wide (default), 0 = per-thread cp.async
 * copies with one CTA barrier per k-tile everywhere.  Returns the previous mode; any
 * other value is -EINVAL. */
int kp_set_simt_staging(int mode);

/* Operands whose rows TMA cannot address (row pitch or base not 16-byte aligned, e.g. raw
 * k = 27 im2col rows) on the TMA-staged families (SIMT configs that stage with TMA, TF32,
 * BF16) are either copied into a 16-byte-pitched stream-ordered scratch first -- one
 * HBM-bound pass -- and then take the TMA path, or staged in-kernel (SIMT: 4-byte
 * cp.async; TF32/BF16: LSU loads into the swizzled ring).  mode 1 (default) repacks when
 * the copy pays for itself (tensor cores: unaligned operands >= 4 MB or k > 4 k-tiles;
 * SIMT: unaligned operands at least as large as the output), 2 always, 0 never.  Results
 * are identical either way (SIMT: bit-identical).  Returns the previous mode; any other
 * value is -EINVAL. */
int kp_set_operand_repack(int mode);

/* ---- benchmark harness ---------------------------------------------------
 * warmup untimed launches, then one launch timed alone to size the loop, then
 * max(min_iters, ceil(min_ms / t1)) (capped at max_iters) back-to-back launches
 * bracketed by CUDA events on `stream`.  *mean_ms = elapsed / iters.  When
 * min_iters <= 1 and the single launch already took >= min_ms it is the measurement
 * (*iters = 1). */
int kp_bench(int id, int m, int k, int n, int batch,
             const void* A, int64_t lda, int64_t sA,
             const void* B, int64_t ldb, int64_t sB,
             void* C, int64_t ldc, int64_t sC,
             int warmup, int min_iters, int max_iters, double min_ms,
             double* mean_ms, int* iters, void* stream);

/* The sweep protocol: like kp_bench, but launch i uses operand set i mod
 * n_sets (A[i], B[i], C[i]; same shape and strides) -- rotating through more data than
 * L2 holds keeps small problems from being timed with a warm cache -- and the timed loop
 * runs `repeats` times; *median_ms is the median of the per-launch means. */
int kp_bench_sets(int id, int m, int k, int n, int batch, int n_sets,
                  const void* const* A, int64_t lda, int64_t sA,
                  const void* const* B, int64_t ldb, int64_t sB,
                  void* const* C, int64_t ldc, int64_t sC,
                  int warmup, int min_iters, int max_iters, double min_ms, int repeats,
                  double* median_ms, int* iters, void* stream);

/* Peak FP32 throughput probe: register-resident FMA chains on every SM, scalar
 * FFMA (packed = 0) or sm_100 packed FFMA2 (packed = 1); returns TFLOP/s in *tflops
 * (the measured FP32 SIMT peak the SIMT families' roofline fraction uses). */
int kp_ffma_peak(int packed, double* tflops, void* stream);

/* ---- runtime dispatch table (tree -> variant id) ------------------------
 * A flattened CART tree in preorder (classify.py:56-77): internal nodes carry
 * feature in [0,4) and threshold; leaves carry leaf_class >= 0.  class_to_variant
 * maps the subset-local class (label_best_in_subset, classify.py:32-34) to a
 * variant id.  Returns a table handle >= 0.  Tables are immutable once loaded; load,
 * free and selection are thread-safe (a walk holds its table alive even if another
 * thread frees the handle meanwhile). */
int kp_dispatch_load(int n_nodes, const int32_t* feature, const double* threshold,
                     const int32_t* left, const int32_t* right, const int32_t* leaf_class,
                     int n_classes, const int32_t* class_to_variant);
int kp_dispatch_free(int handle);
/* Walk with features log2(m), log2(k), log2(n), log2(batch) supplied by the caller
 * (the Python shim computes them with np.log2, classify.py:27-29).  Returns the
 * subset-local class (>= 0) or a negative status. */
int kp_dispatch_class_feats(int handle, const double* feats4);
/* Same, returning the variant id. */
int kp_dispatch_select_feats(int handle, const double* feats4);
/* Convenience: features from the C library's log2 (exact parity caveat in DESIGN.md). */
int kp_dispatch_select(int handle, int m, int k, int n, int batch);
/* select + kp_gemm; *variant_out (may be NULL) receives the launched variant. */
int kp_gemm_auto(int handle, int m, int k, int n, int batch,
                 const void* A, int64_t lda, int64_t sA,
                 const void* B, int64_t ldb, int64_t sB,
                 void* C, int64_t ldc, int64_t sC, void* stream, int* variant_out);
int kp_gemm_auto_ex(int handle, int m, int k, int n, int batch,
                    const void* A, int64_t lda, int64_t sA,
                    const void* B, int64_t ldb, int64_t sB,
                    void* C, int64_t ldc, int64_t sC,
                    const float* bias, int flags, void* stream, int* variant_out);

/* ---- conv-as-GEMM helpers for VGG16 inference (NHWC fp32) ----------------
 * im2col of a 3x3, stride 1, pad 1 convolution: x is (B, H, W, C); out row
 * r = (b*H + h)*W + w holds the 9*C patch values ordered (dy, dx, c) -- the k order of
 * the (9*C) x Cout weight matrix -- with zeros outside the image; ldo >= 9*C. */
int kp_im2col3x3_nhwc(const float* x, int B, int H, int W, int C, float* out, int64_t ldo, void* stream);
/* Same patches into rows of kpad >= 9*C floats (kpad % 4 == 0, out 16-byte aligned),
 * zeros in columns 9*C..kpad-1: e.g. conv1_1 (C = 3) as 28-wide rows, which the GEMM
 * families read with their vector / TMA paths (pair it with a zero-padded weight row:
 * fma(0, 0, acc) == acc, so the fp32 chain is unchanged). */
int kp_im2col3x3_nhwc_pad(const float* x, int B, int H, int W, int C, float* out, int kpad, void* stream);
/* bf16 operands for the BF16 family: the same patches as bf16 rows of kpad columns
 * (kpad % 8 == 0, >= 9*C; zeros beyond 9*C; round to nearest even), and an fp32 -> bf16
 * cast of n elements (n % 8 == 0, 16-byte-aligned pointers). */
int kp_im2col3x3_nhwc_bf16(const float* x, int B, int H, int W, int C, void* out, int kpad, void* stream);
int kp_cast_bf16(const float* x, int64_t n, void* out, void* stream);
/* Implicit-GEMM 3x3 / stride 1 / pad 1 convolution: the GEMM that kp_im2col3x3_nhwc
 * (or kp_im2col3x3_nhwc_bf16) + kp_gemm_ex would run (m = B*H*W, k = 9*C, n = Cout,
 * weights (9*C) x Cout row-major, out (B*H*W) x Cout = NHWC fp32) with the patch rows
 * gathered straight from x by TMA im2col copies -- no im2col buffer in HBM.  Same launch
 * plan (k-slices) and accumulation order as the explicit path, so the output is
 * bit-identical.  Element types follow kp_gemm: x and w are fp32 for SIMT/TF32 variants
 * and bf16 for BF16 variants; out is fp32, or bf16 with flags & KP_EPI_BF16_OUT
 * (tensor-core variants, as kp_gemm_ex).
 * kp_conv3x3_supported(id, C, Cout) returns 1 when variant id can run it (SIMT variant
 * with TMA staging, i.e. CTA tile <= 256 columns, C a multiple of its k-tile depth,
 * Cout % 4 == 0; a TF32 variant with C % 32 == 0 and Cout % 4 == 0; a BF16 variant with
 * C % 64 == 0 and Cout % 8 == 0 -- the tensor-core producers load 128-byte-swizzled
 * im2col boxes into the tcgen05 ring, 1-CTA or CTA-pair kernel), 0 when not (PAPER), < 0 for a bad
 * id.  x, w and out must be 16-byte aligned. */
int kp_conv3x3_supported(int id, int C, int Cout);
int kp_conv3x3_nhwc_ex(int id, const void* x, int B, int H, int W, int C, const void* w, int Cout, void* out,
                       const float* bias, int flags, void* stream);
/* 2x2 / stride 2 max pooling, NHWC: (B, H, W, C) -> (B, H/2, W/2, C). */
int kp_maxpool2x2_nhwc(const float* x, int B, int H, int W, int C, float* out, void* stream);
/* The same pooling of bf16 activations (the BF16 family's KP_EPI_BF16_OUT layer outputs;
 * C % 8 == 0, x and out 16-byte aligned).  Exact: the max is one of its inputs, and
 * rounding is monotonic, so it equals pooling in fp32 and rounding afterwards. */
int kp_maxpool2x2_nhwc_bf16(const void* x, int B, int H, int W, int C, void* out, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* KPGEMM_H_ */
