// F2 (TF32) and F3 (BF16) -- tcgen05 tensor-core families (KP_FAMILY_TF32/BF16).
//
// Extra candidates beside the paper's SIMT space (BASELINE.json north_star): same
// operator contract as kp_gemm (C[b] = A[b] * B[b], row-major, fp32 out), computed
// on the 5th-generation tensor cores:
//   * TMA (cp.async.bulk.tensor) loads 128-byte-swizzled tiles into a STAGES-deep
//     shared-memory ring, signalling full/empty mbarriers;
//   * one elected thread issues tcgen05.mma (M=128, N=BN, K=32 bytes per instruction)
//     with A K-major and B MN-major (B is row-major K x N, so no transpose pass; for
//     tf32 the MN-major tile uses the 32-byte-atom 128B swizzle, the only MN-major
//     32-bit layout UMMA accepts),
//     accumulating in TMEM (BN fp32 columns x 128 lanes);
//   * tcgen05.commit frees each smem stage and finally signals the epilogue warps,
//     which drain TMEM with tcgen05.ld (32x32b) and store fp32 rows.
// Warp roles (192 threads): warp 0 = TMA producer, warp 1 = TMEM allocator + MMA
// issuer, warps 2..5 = epilogue (warp % 4 selects the TMEM lane quadrant).  The grid
// is persistent (one CTA per SM) with two TMEM accumulators so each tile's epilogue
// overlaps the next tile's MMAs.
//
// Config 5-tuple of these families (include/kpgemm.h KernelChoice), documented in
// (tile_rows, tile_acc, tile_cols, wg_rows, wg_cols) =
//   (BM = 128, or 256 for CTA pairs, BK = elements per 128-byte K slab, BN, STAGES,
//    threads per CTA = 192).
//
// Operands whose rows are not 16-byte aligned (TMA's requirement; e.g. VGG conv1_1
// k = 27, ResNet conv1 k = 147) are staged by the epilogue warps with ordinary loads
// into the identical swizzled layout, so every family runs every shape (the grid
// must be complete, dataset.py:259-264).
//
// Numerics: BF16 operands are exact bf16 inputs, fp32 accumulation.  TF32 reads fp32
// operands and uses their top 19 bits (truncation), fp32 accumulation; tolerances in
// tests/test_tc_gpu.py: |C - C64| <= (2*eps_in + 2*k*2^-24) * (|A||B|)_ij.
#include <cooperative_groups.h>
#include <cuda.h>

#include <cstdio>
#include <cstring>
#include <type_traits>

#include "families.h"
#include "tc_families.h"

namespace kp {
namespace {

constexpr int kThreads = 192;
constexpr int kTmaStoreMaxK = 2048;
constexpr int BM = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "KP_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra KP_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
      : "memory");
}

// TMA im2col load (implicit-GEMM 3x3 convolution): BM consecutive output pixels (w fastest,
// then h, then image) from base pixel (w, h, n) of the map's bounding box, each contributing
// the map's channelsPerPixel channels from c of input pixel (w + dx, h + dy); zero outside
// the image.  The rows land 128B-swizzled exactly as the tiled A box would.
__device__ __forceinline__ void tma_im2col_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c, int w, int h,
                                              int n, uint16_t dx, uint16_t dy) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.im2col.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, "
      "%6}], [%2], {%7, %8};" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c), "r"(w), "r"(h), "r"(n), "h"(dx), "h"(dy)
      : "memory");
}

// TMA store of a 32 x 32 fp32 box (128B-swizzled smem) to C at (x = col, y = row, z = batch).
// Implicit-conv producer state: the tile's base output pixel (w, h, img) and the k-tile's
// (channel block c0, filter tap dx/dy), advanced one k-tile at a time.
struct ConvCursor {
  int w = 0, h = 0, img = 0, c0 = 0, dx = 0, dy = 0;
  __device__ __forceinline__ void start(const GemmArgs& p, int m0, int k0) {
    const int tr = m0 / p.conv_w;
    w = m0 - tr * p.conv_w;
    img = tr / p.conv_h;
    h = tr - img * p.conv_h;
    const int tap = k0 / p.conv_c;
    c0 = k0 - tap * p.conv_c;
    dy = tap / 3;
    dx = tap - 3 * dy;
  }
  __device__ __forceinline__ void next(int conv_c, int bk) {
    c0 += bk;
    if (c0 == conv_c) {
      c0 = 0;
      if (++dx == 3) {
        dx = 0;
        ++dy;
      }
    }
  }
};

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int x, int y, int z) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(map),
               "r"(smem_u32(src)), "r"(x), "r"(y), "r"(z)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// Shared-memory matrix descriptor, version 1 (sm_100).  layout 2 = SWIZZLE_128B
// (16-byte chunks XOR row%8 over 1024-byte atoms), layout 1 = SWIZZLE_128B_BASE32B
// (32-byte chunks XOR row%4 over 512-byte atoms) -- the only MN-major layout the
// tensor core accepts for 32-bit (tf32) operands.
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr, uint32_t lbo_bytes, uint32_t sbo_bytes,
                                              uint32_t layout = 2) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((addr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo_bytes >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo_bytes >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // version
  d |= static_cast<uint64_t>(layout) << 61;
  return d;
}

template <bool kTF32>
__device__ __forceinline__ void mma_issue(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accum) {
  if constexpr (kTF32) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
  } else {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
  }
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float* v) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

template <bool kTF32, int BN, int STAGES>
struct TcCfg {
  static constexpr int ES = kTF32 ? 4 : 2;          // operand element size
  static constexpr int BK = 128 / ES;               // elements per 128-byte K slab
  static constexpr int UK = 32 / ES;                // K per tcgen05.mma (32 bytes)
  static constexpr int NATOM = 128 / ES;            // N elements per 128-byte swizzle atom
  static constexpr int A_BYTES = BM * 128;          // one stage of A (K-major)
  static constexpr int B_BYTES = BK * BN * ES;      // one stage of B (MN-major atoms)
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // two accumulators (double-buffered TMEM), power-of-two column allocation
  static constexpr int TMEM_COLS = 2 * BN <= 32 ? 32 : 2 * BN <= 64 ? 64 : 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;
  // k-sliced launches park the fp32 partial tile (row stride BN + 4) in the ring
  static constexpr int PART_STRIDE = BN + 4;
  static constexpr int PART_BYTES = BM * PART_STRIDE * 4;
  static constexpr int RING_BYTES = STAGES * STAGE_BYTES;
  static constexpr int SLICED_RING_BYTES = RING_BYTES > PART_BYTES ? RING_BYTES : PART_BYTES;
  // persistent launches stage the epilogue through smem for TMA stores: per epilogue
  // warp two 32 x 32 fp32 boxes (128B swizzle), 32 KB in all, after the barriers
  static constexpr int EPI_OFFSET = RING_BYTES + 1024;  // 1024-aligned (swizzle atoms)
  static constexpr int EPI_BYTES = 4 * 2 * 32 * 32 * 4;
  static constexpr int SMEM_BYTES = EPI_OFFSET + EPI_BYTES + 1024 /*align*/;
  static constexpr int SLICED_SMEM_BYTES = SLICED_RING_BYTES + 1024 + 256;
  static_assert(2 * BN <= 512, "two accumulators must fit TMEM");
  static constexpr uint32_t IDESC = (1u << 4)                      // D = f32
                                    | ((kTF32 ? 2u : 1u) << 7)     // A = tf32 / bf16
                                    | ((kTF32 ? 2u : 1u) << 10)    // B = tf32 / bf16
                                    | (0u << 15)                   // A K-major
                                    | (1u << 16)                   // B MN-major
                                    | (static_cast<uint32_t>(BN >> 3) << 17) | (static_cast<uint32_t>(BM >> 4) << 24);
  static_assert(BN % NATOM == 0 && BN >= 16 && BN <= 256, "tile N");
  static_assert(SLICED_SMEM_BYTES <= 227 * 1024 && SMEM_BYTES <= 227 * 1024, "smem");
};

// LSU staging (operands whose rows are not 16-byte aligned, e.g. k = 27 or 147, so
// TMA cannot address them): the four epilogue warps load the stage with ordinary
// loads, write the same 128-byte-swizzled layout TMA would produce (16-byte chunk c of
// row r lands at chunk c ^ (r % 8) of its 1024-byte atom), make the generic-proxy
// writes visible to the tensor core with fence.proxy.async, and arrive on the stage's
// full barrier (128 arrivals instead of one transaction count).
template <bool kTF32, int BN>
__device__ __forceinline__ void lsu_stage(uint8_t* sa, uint8_t* sb, const GemmArgs& p, int b, int m0, int n0, int k0,
                                          int t) {
  using Elem = typename std::conditional<kTF32, uint32_t, uint16_t>::type;
  constexpr int ES = sizeof(Elem), BK = 128 / ES, NATOM = 128 / ES;
  const Elem* A = static_cast<const Elem*>(p.A) + static_cast<int64_t>(b) * p.sA;
  const Elem* B = static_cast<const Elem*>(p.B) + static_cast<int64_t>(b) * p.sB;
  // 8 independent loads in flight per thread before their shared-memory stores (a
  // load-store-load chain leaves the 128 staging threads latency-bound)
  constexpr int kBatch = 8;
  static_assert((BM * BK / 128) % kBatch == 0 && (BK * BN / 128) % kBatch == 0, "LSU batches");
#pragma unroll 1
  for (int base = 0; base < BM * BK / 128; base += kBatch) {
    Elem v[kBatch];
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
      const int e = t + (base + j) * 128, row = e / BK, kc = e - row * BK;
      const int gr = m0 + row, gk = k0 + kc;
      v[j] = (gr < p.m && gk < p.k) ? A[static_cast<int64_t>(gr) * p.lda + gk] : Elem(0);
    }
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
      const int e = t + (base + j) * 128, row = e / BK, kc = e - row * BK;
      const int byte = kc * ES;
      *reinterpret_cast<Elem*>(sa + (row >> 3) * 1024 + (row & 7) * 128 + (((byte >> 4) ^ (row & 7)) << 4) +
                               (byte & 15)) = v[j];
    }
  }
#pragma unroll 1
  for (int base = 0; base < BK * BN / 128; base += kBatch) {
    Elem v[kBatch];
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
      const int e = t + (base + j) * 128, kr = e / BN, nc = e - kr * BN;
      const int gk = k0 + kr, gn = n0 + nc;
      v[j] = (gk < p.k && gn < p.n) ? B[static_cast<int64_t>(gk) * p.ldb + gn] : Elem(0);
    }
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
      const int e = t + (base + j) * 128, kr = e / BN, nc = e - kr * BN;
      const int jj = nc / NATOM, byte = (nc - jj * NATOM) * ES;
      const int off = kTF32 ? (kr * 128 + (((byte >> 5) ^ (kr & 3)) << 5) + (byte & 31))  // 128B_BASE32B
                            : ((kr >> 3) * 1024 + (kr & 7) * 128 + (((byte >> 4) ^ (kr & 7)) << 4) + (byte & 15));
      *reinterpret_cast<Elem*>(sb + jj * (BK * 128) + off) = v[j];
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Tile order inside one batch: bands of kGroupM m-tiles; within a band n-major with m
// fastest, so the ~148 tiles in flight share a few A panels and a few B panels in L2
// (plain m-fastest order streams all of A once per n column).
constexpr int kGroupM = 16;
template <int BN>
__device__ __forceinline__ void tile_coords(int t, int tiles_m, int tiles_n, int& b, int& m0, int& n0) {
  const int per_batch = tiles_m * tiles_n;
  b = t / per_batch;
  const int r = t - b * per_batch;
  const int band = r / (kGroupM * tiles_n);
  const int first = band * kGroupM;
  const int rows = tiles_m - first < kGroupM ? tiles_m - first : kGroupM;
  const int local = r - band * kGroupM * tiles_n;
  m0 = (first + local % rows) * BM;
  n0 = (local / rows) * BN;
}

// Cluster reduction of a k-sliced launch (grid = (#tiles, 1, S), cluster (1, 1, S), one
// tile per CTA): CTA rank z sums elements [z*chunk, (z+1)*chunk) of the 128 x BN tile
// over every rank's shared-memory partial (DSMEM) in rank order, then applies the
// epilogue and stores.  Same slice order as the SIMT family: ((p0 + p1) + p2) + ...
template <int BN>
__device__ __forceinline__ void tc_slice_reduce(const GemmArgs& p, float* part, int tiles_m, int tiles_n,
                                                int tile_begin) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  cl.sync();
  int b, m0, n0;
  tile_coords<BN>(tile_begin + static_cast<int>(blockIdx.x), tiles_m, tiles_n, b, m0, n0);
  constexpr int PS = BN + 4, Q = BN / 4, TOT = BM * Q;
  const int S = p.kslices, z = static_cast<int>(cl.block_rank());
  const int chunk = (TOT + S - 1) / S, end = min(TOT, (z + 1) * chunk);
  float* Cb = static_cast<float*>(p.C) + static_cast<int64_t>(b) * p.sC;
  for (int i = z * chunk + static_cast<int>(threadIdx.x); i < end; i += kThreads) {
    const int r = i / Q, c = (i - r * Q) * 4;
    const int row = m0 + r, col = n0 + c;
    if (row >= p.m || col >= p.n) continue;
    float4 v = *reinterpret_cast<const float4*>(cl.map_shared_rank(part, 0) + r * PS + c);
    for (int s = 1; s < S; ++s) {
      const float4 w = *reinterpret_cast<const float4*>(cl.map_shared_rank(part, s) + r * PS + c);
      v.x = v.x + w.x; v.y = v.y + w.y; v.z = v.z + w.z; v.w = v.w + w.w;
    }
    float o[4] = {v.x, v.y, v.z, v.w};
    if (p.bias || p.relu) epilogue_run<4>(p, o, col);
    if (p.c_bf16) {
      __nv_bfloat16* ob = static_cast<__nv_bfloat16*>(p.C) + static_cast<int64_t>(b) * p.sC +
                          static_cast<int64_t>(row) * p.ldc + col;
      if (p.c_vec && col + 4 <= p.n) {
        *reinterpret_cast<uint2*>(ob) = make_uint2(pack_bf16x2(o[0], o[1]), pack_bf16x2(o[2], o[3]));
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (col + e < p.n) ob[e] = __float2bfloat16_rn(o[e]);
      }
      continue;
    }
    float* out = Cb + static_cast<int64_t>(row) * p.ldc + col;
    if (p.c_vec && col + 4 <= p.n) {
      *reinterpret_cast<float4*>(out) = make_float4(o[0], o[1], o[2], o[3]);
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (col + e < p.n) out[e] = o[e];
    }
  }
  cl.sync();  // keep this CTA's partial alive until every rank has read it
}

// Persistent: gridDim.x = min(#tiles, #SMs) CTAs walk the tile list (tile_coords
// order, then batch) with stride gridDim.x.  The smem ring runs continuously across tiles
// and TMEM holds two accumulators, so the epilogue of tile i overlaps the MMAs of
// tile i+1 (tmem_full / tmem_empty mbarrier pairs).
template <bool kTF32, int BN, int STAGES, bool kLsu, bool kSliced>
__global__ void __launch_bounds__(kThreads, 1)
    tc_gemm_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                   const __grid_constant__ CUtensorMap mapC, GemmArgs p, int tiles_m, int tiles_n, int a_batched,
                   int b_batched, int tma_store, int tile_begin, int tile_count) {
  using Cfg = TcCfg<kTF32, BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (kSliced ? Cfg::SLICED_RING_BYTES : Cfg::RING_BYTES));
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;  // [2]
  uint64_t* tmem_empty = tmem_full + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // this CTA's k-tiles: all of them, or slice blockIdx.z of a k-sliced launch
  // (kSliced is a separate instantiation so the persistent kernel keeps its own code)
  const int kt0 = kSliced ? static_cast<int>(blockIdx.z) * p.kt_per_slice : 0;
  const int KT = kSliced ? min((p.k + Cfg::BK - 1) / Cfg::BK - kt0, p.kt_per_slice) : (p.k + Cfg::BK - 1) / Cfg::BK;
  constexpr bool sliced = kSliced;
  const int per_batch = tiles_m * tiles_n;
  const int n_tiles = tile_count;  // this launch's tiles: [tile_begin, tile_begin + tile_count)
  (void)per_batch;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], kLsu ? 128 : 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tmem_full[a], 1);
      mbar_init(&tmem_empty[a], 4);  // one arrival per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (!kLsu) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&mapB) : "memory");
    }
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(Cfg::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0 && lane == 0 && !kLsu) {
    // ---------------- TMA producer ----------------
    int it = 0;  // global k-iteration counter (ring position across tiles)
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
      int b, m0, n0;
      tile_coords<BN>(tile_begin + t, tiles_m, tiles_n, b, m0, n0);
      const int za = a_batched ? b : 0, zb = b_batched ? b : 0;
      // implicit conv: the tile's base pixel once per tile, then (channel block, tap)
      // stepped per k-tile (conv_c % BK == 0) -- no integer division in the k loop, whose
      // single issuing thread bounds the launch (per-k-tile divisions measured up to 1.4x)
      ConvCursor cc;
      if (p.conv_c > 0) cc.start(p, m0, kt0 * Cfg::BK);
      for (int kt = 0; kt < KT; ++kt, ++it) {
        const int s = it % STAGES;
        mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);  // fresh barrier: passes
        uint8_t* sa = smem + s * Cfg::STAGE_BYTES;
        uint8_t* sb = sa + Cfg::A_BYTES;
        mbar_expect_tx(&full[s], Cfg::STAGE_BYTES);
        if (p.conv_c > 0) {
          tma_im2col_4d(sa, &mapA, &full[s], cc.c0, cc.w - 1, cc.h - 1, cc.img, static_cast<uint16_t>(cc.dx),
                        static_cast<uint16_t>(cc.dy));
          cc.next(p.conv_c, Cfg::BK);
        } else {
          tma_load_3d(sa, &mapA, &full[s], (kt0 + kt) * Cfg::BK, m0, za);
        }
#pragma unroll
        for (int j = 0; j < BN / Cfg::NATOM; ++j)
          tma_load_3d(sb + j * (Cfg::BK * 128), &mapB, &full[s], n0 + j * Cfg::NATOM, (kt0 + kt) * Cfg::BK, zb);
      }
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer ----------------
    int it = 0, i = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
      const int a = i & 1;
      mbar_wait(&tmem_empty[a], ((i >> 1) & 1) ^ 1);  // epilogue drained this accumulator
      tc_fence_after();
      const uint32_t dtmem = tmem_base + a * BN;
      for (int kt = 0; kt < KT; ++kt, ++it) {
        const int s = it % STAGES;
        mbar_wait(&full[s], (it / STAGES) & 1);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + s * Cfg::STAGE_BYTES);
        const uint32_t sb = sa + Cfg::A_BYTES;
#pragma unroll
        for (int kk = 0; kk < Cfg::BK / Cfg::UK; ++kk) {
          const uint64_t adesc = smem_desc(sa + kk * 32, 16, 1024);
          const uint64_t bdesc = kTF32 ? smem_desc(sb + kk * Cfg::UK * 128, Cfg::BK * 128, 512, 1)
                                       : smem_desc(sb + kk * Cfg::UK * 128, Cfg::BK * 128, 1024, 2);
          mma_issue<kTF32>(dtmem, adesc, bdesc, Cfg::IDESC, (kt | kk) != 0);
        }
        mma_commit(&empty[s]);
      }
      mma_commit(&tmem_full[a]);
    }
  } else if (warp >= 2) {
    // ---------------- epilogue (and LSU producer for unaligned operands) ----------------
    const int quad = warp & 3;
    int it = 0, i = 0, epi_box = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++i) {
      int b, m0, n0;
      tile_coords<BN>(tile_begin + t, tiles_m, tiles_n, b, m0, n0);
      if constexpr (kLsu) {
        const int tid = threadIdx.x - 64;
        for (int kt = 0; kt < KT; ++kt, ++it) {
          const int s = it % STAGES;
          mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
          uint8_t* sa = smem + s * Cfg::STAGE_BYTES;
          lsu_stage<kTF32, BN>(sa, sa + Cfg::A_BYTES, p, b, m0, n0, (kt0 + kt) * Cfg::BK, tid);
          asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[s])) : "memory");
        }
      }
      const int a = i & 1;
      mbar_wait(&tmem_full[a], (i >> 1) & 1);
      tc_fence_after();
      const int row = m0 + quad * 32 + lane;
      float* out = static_cast<float*>(p.C) + static_cast<int64_t>(b) * p.sC + static_cast<int64_t>(row) * p.ldc;
      // k-sliced: the accumulator goes to this CTA's partial tile in shared memory (the
      // ring is idle: tmem_full means every MMA, and so every smem read, has finished)
      float* part = reinterpret_cast<float*>(smem) + (quad * 32 + lane) * Cfg::PART_STRIDE;
      if (!sliced && tma_store) {
        // TMEM -> registers -> 128B-swizzled smem box (lane = row, conflict-free float4
        // stores) -> one TMA store per 32 x 32 box; two boxes per warp in flight
        uint8_t* stage = smem + Cfg::EPI_OFFSET + quad * (2 * 32 * 32 * 4);
#pragma unroll 1
        for (int c = 0; c < BN; c += 32, ++epi_box) {
          float v[32];
          tmem_ld16(tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + a * BN + c, v);
          tmem_ld16(tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + a * BN + c + 16, v + 16);
          if (p.bias || p.relu) epilogue_run<32>(p, v, n0 + c);
          uint8_t* box = stage + (epi_box & 1) * (32 * 32 * 4);
          if (lane == 0) bulk_wait_read<1>();  // the store that last used this box has read it
          __syncwarp();
          if (p.c_bf16) {
            // bf16 box: 64-byte rows, 64B swizzle (16-byte chunk j of row r at j ^ ((r >> 1) & 3))
#pragma unroll
            for (int j = 0; j < 4; ++j)
              *reinterpret_cast<uint4*>(box + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4)) =
                  make_uint4(pack_bf16x2(v[8 * j], v[8 * j + 1]), pack_bf16x2(v[8 * j + 2], v[8 * j + 3]),
                             pack_bf16x2(v[8 * j + 4], v[8 * j + 5]), pack_bf16x2(v[8 * j + 6], v[8 * j + 7]));
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              *reinterpret_cast<float4*>(box + lane * 128 + ((j ^ (lane & 7)) << 4)) =
                  make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            tma_store_3d(&mapC, box, n0 + c, m0 + quad * 32, b);
            bulk_commit();
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tmem_empty[a])) : "memory");
        continue;
      }
#pragma unroll 1
      for (int c = 0; c < BN; c += 16) {
        float v[16];
        tmem_ld16(tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + a * BN + c, v);
        if constexpr (sliced) {
#pragma unroll
          for (int q = 0; q < 4; ++q)
            *reinterpret_cast<float4*>(part + c + 4 * q) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
        } else if (row < p.m) {
          const int col = n0 + c;
          if (p.bias || p.relu) epilogue_run<16>(p, v, col);
          if (p.c_bf16) {
            __nv_bfloat16* ob = static_cast<__nv_bfloat16*>(p.C) + static_cast<int64_t>(b) * p.sC +
                                static_cast<int64_t>(row) * p.ldc + col;
            if (p.c_vec && col + 16 <= p.n) {
              uint32_t w[8];
#pragma unroll
              for (int q = 0; q < 8; ++q) w[q] = pack_bf16x2(v[2 * q], v[2 * q + 1]);
              reinterpret_cast<uint4*>(ob)[0] = make_uint4(w[0], w[1], w[2], w[3]);
              reinterpret_cast<uint4*>(ob)[1] = make_uint4(w[4], w[5], w[6], w[7]);
            } else {
#pragma unroll
              for (int e = 0; e < 16; ++e)
                if (col + e < p.n) ob[e] = __float2bfloat16_rn(v[e]);
            }
          } else if (p.c_vec && col + 16 <= p.n) {
#pragma unroll
            for (int q = 0; q < 4; ++q)
              *reinterpret_cast<float4*>(out + col + 4 * q) =
                  make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
          } else {
#pragma unroll
            for (int e = 0; e < 16; ++e)
              if (col + e < p.n) out[col + e] = v[e];
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&tmem_empty[a])) : "memory");
    }
  }
  if (warp >= 2 && lane == 0 && !sliced && tma_store) bulk_wait_all();  // staged boxes written out
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(Cfg::TMEM_COLS));
  }
  if constexpr (sliced) tc_slice_reduce<BN>(p, reinterpret_cast<float*>(smem), tiles_m, tiles_n, tile_begin);
}

// ------------------------------------------------------- CTA pairs (2-CTA MMA) --
// tcgen05.mma.cta_group::2: a (2, 1, 1) cluster -- two SMs of one TPC -- computes a
// 256 x BN tile.  Each CTA stages its own 128 rows of A and its own BN/2 columns of B
// (so each operand byte is loaded by one SM only and each SM's shared memory feeds
// half the B panel), the leader CTA issues M = 256 MMAs that read both CTAs' stages,
// and each CTA's TMEM receives its 128 rows x BN fp32 accumulator.  Barriers:
//   full[s]       leader only: one arrive.expect_tx for both CTAs' bytes; both CTAs'
//                 TMA copies complete_tx on it (.cta_group::2 signalling);
//   empty[s]      both CTAs: the leader's tcgen05.commit multicasts to both;
//   tmem_full[a]  both CTAs: commit multicast, each CTA's epilogue waits on its own;
//   tmem_empty[a] leader only: 8 arrivals (4 epilogue warps per CTA, the peer's remote).
// Persistent over tile pairs; TMA operands only (the launcher falls back to the 1-CTA
// kernel for LSU staging and k-sliced launches).
constexpr int BM2 = 256;

template <bool kTF32, int BN, int STAGES>
struct Tc2Cfg {
  using Base = TcCfg<kTF32, BN, 2>;  // stage-independent facts (BK, UK, NATOM, TMEM columns)
  static constexpr int ES = Base::ES, BK = Base::BK, UK = Base::UK, NATOM = Base::NATOM;
  static constexpr int BNH = BN / 2;                     // B columns staged per CTA
  static constexpr int A_BYTES = BM * 128;               // this CTA's 128 rows of A
  static constexpr int B_BYTES = BK * BNH * ES;          // this CTA's half of B
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int TMEM_COLS = Base::TMEM_COLS;
  static constexpr int RING_BYTES = STAGES * STAGE_BYTES;
  static constexpr int EPI_OFFSET = RING_BYTES + 1024;
  static constexpr int EPI_BYTES = 4 * 2 * 32 * 32 * 4;
  static constexpr int SMEM_BYTES = EPI_OFFSET + EPI_BYTES + 1024;
  static constexpr uint32_t IDESC = (1u << 4) | ((kTF32 ? 2u : 1u) << 7) | ((kTF32 ? 2u : 1u) << 10) | (0u << 15) |
                                    (1u << 16) | (static_cast<uint32_t>(BN >> 3) << 17) |
                                    (static_cast<uint32_t>(BM2 >> 4) << 24);
  static_assert(BNH % NATOM == 0, "each CTA stages whole swizzle atoms of B");
  static_assert(SMEM_BYTES <= 227 * 1024, "smem");
};

// mbarrier wait that traps after ~2^28 polls (seconds) instead of hanging the GPU if a
// pair's protocol ever loses an arrival: a trapped kernel fails its launch cleanly.
__device__ __forceinline__ void mbar_wait_pair(uint64_t* bar, uint32_t parity) {
  uint32_t done = 0;
  for (uint32_t polls = 0; !done; ++polls) {
    asm volatile(
        "{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
    if (polls > (1u << 28)) __trap();
  }
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of this CTA's variable at `p` as seen in CTA `rank`
__device__ __forceinline__ uint32_t map_rank(const void* p, uint32_t rank) {
  uint32_t out;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(out) : "r"(smem_u32(p)), "r"(rank));
  return out;
}
__device__ __forceinline__ void tma_load_3d_pair(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int x, int y,
                                                 int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
      "%5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(bar_cluster), "r"(x), "r"(y), "r"(z)
      : "memory");
}
// TMA im2col load into the pair's shared::cluster space, completion on the leader's barrier
__device__ __forceinline__ void tma_im2col_4d_pair(void* dst, const CUtensorMap* map, uint32_t bar_cluster, int c,
                                                   int w, int h, int n, uint16_t dx, uint16_t dy) {
  asm volatile(
      "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.im2col.mbarrier::complete_tx::bytes [%0], [%1, "
      "{%3, %4, %5, %6}], [%2], {%7, %8};" ::"r"(smem_u32(dst)),
      "l"(map), "r"(bar_cluster), "r"(c), "r"(w), "r"(h), "r"(n), "h"(dx), "h"(dy)
      : "memory");
}
template <bool kTF32>
__device__ __forceinline__ void mma_issue_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                               uint32_t accum) {
  if constexpr (kTF32) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
  } else {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
  }
}
__device__ __forceinline__ void mma_commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"(static_cast<uint16_t>(3))
      : "memory");
}

__device__ __forceinline__ void tile_coords_pair(int t, int tiles_m, int tiles_n, int bn, int& b, int& m0, int& n0) {
  const int per_batch = tiles_m * tiles_n;
  b = t / per_batch;
  const int r = t - b * per_batch;
  const int band = r / (kGroupM * tiles_n);
  const int first = band * kGroupM;
  const int rows = tiles_m - first < kGroupM ? tiles_m - first : kGroupM;
  const int local = r - band * kGroupM * tiles_n;
  m0 = (first + local % rows) * BM2;
  n0 = (local / rows) * bn;
}

template <bool kTF32, int BN, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    tc2_gemm_kernel(const __grid_constant__ CUtensorMap mapA, const __grid_constant__ CUtensorMap mapB,
                    const __grid_constant__ CUtensorMap mapC, GemmArgs p, int tiles_m, int tiles_n, int a_batched,
                    int b_batched, int tma_store) {
  using Cfg = Tc2Cfg<kTF32, BN, STAGES>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + Cfg::RING_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tmem_full = empty + STAGES;  // [2]
  uint64_t* tmem_empty = tmem_full + 2;  // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int KT = (p.k + Cfg::BK - 1) / Cfg::BK;
  const int n_tiles = tiles_m * tiles_n * p.batch;  // 256-row tiles
  const int pair = static_cast<int>(blockIdx.x) >> 1, pairs = static_cast<int>(gridDim.x) >> 1;

  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tmem_full[a], 1);
      mbar_init(&tmem_empty[a], 8);  // 4 epilogue warps in each CTA of the pair
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&mapB) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(Cfg::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();  // barriers initialised and TMEM allocated in both CTAs
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer (both CTAs; completions land on the leader) ----------------
    int it = 0;
    for (int t = pair; t < n_tiles; t += pairs) {
      int b, m0, n0;
      tile_coords_pair(t, tiles_m, tiles_n, BN, b, m0, n0);
      const int za = a_batched ? b : 0, zb = b_batched ? b : 0;
      ConvCursor cc;
      if (p.conv_c > 0) cc.start(p, m0 + static_cast<int>(rank) * BM, 0);
      for (int kt = 0; kt < KT; ++kt, ++it) {
        const int s = it % STAGES;
        mbar_wait_pair(&empty[s], ((it / STAGES) & 1) ^ 1);
        uint8_t* sa = smem + s * Cfg::STAGE_BYTES;
        uint8_t* sb = sa + Cfg::A_BYTES;
        const uint32_t fbar = map_rank(&full[s], 0);
        if (leader) mbar_expect_tx(&full[s], 2 * Cfg::STAGE_BYTES);
        if (p.conv_c > 0) {
          // implicit conv: this CTA's 128 pixels of the 256-row tile, one filter tap per k-tile
          tma_im2col_4d_pair(sa, &mapA, fbar, cc.c0, cc.w - 1, cc.h - 1, cc.img, static_cast<uint16_t>(cc.dx),
                             static_cast<uint16_t>(cc.dy));
          cc.next(p.conv_c, Cfg::BK);
        } else {
          tma_load_3d_pair(sa, &mapA, fbar, kt * Cfg::BK, m0 + static_cast<int>(rank) * BM, za);
        }
#pragma unroll
        for (int j = 0; j < Cfg::BNH / Cfg::NATOM; ++j)
          tma_load_3d_pair(sb + j * (Cfg::BK * 128), &mapB, fbar, n0 + static_cast<int>(rank) * Cfg::BNH + j * Cfg::NATOM,
                           kt * Cfg::BK, zb);
      }
    }
  } else if (warp == 1 && lane == 0 && leader) {
    // ---------------- MMA issuer (leader only; M = 256 over both CTAs' stages) ----------------
    int it = 0, i = 0;
    for (int t = pair; t < n_tiles; t += pairs, ++i) {
      const int a = i & 1;
      mbar_wait_pair(&tmem_empty[a], ((i >> 1) & 1) ^ 1);
      tc_fence_after();
      const uint32_t dtmem = tmem_base + a * BN;
      for (int kt = 0; kt < KT; ++kt, ++it) {
        const int s = it % STAGES;
        mbar_wait_pair(&full[s], (it / STAGES) & 1);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + s * Cfg::STAGE_BYTES);
        const uint32_t sb = sa + Cfg::A_BYTES;
#pragma unroll
        for (int kk = 0; kk < Cfg::BK / Cfg::UK; ++kk) {
          const uint64_t adesc = smem_desc(sa + kk * 32, 16, 1024);
          const uint64_t bdesc = kTF32 ? smem_desc(sb + kk * Cfg::UK * 128, Cfg::BK * 128, 512, 1)
                                       : smem_desc(sb + kk * Cfg::UK * 128, Cfg::BK * 128, 1024, 2);
          mma_issue_pair<kTF32>(dtmem, adesc, bdesc, Cfg::IDESC, (kt | kk) != 0);
        }
        mma_commit_pair(&empty[s]);
      }
      mma_commit_pair(&tmem_full[a]);
    }
  } else if (warp >= 2) {
    // ---------------- epilogue: this CTA's 128 rows of each 256-row tile ----------------
    const int quad = warp & 3;
    const uint32_t empty_bar0 = map_rank(&tmem_empty[0], 0), empty_bar1 = map_rank(&tmem_empty[1], 0);
    int i = 0, epi_box = 0;
    for (int t = pair; t < n_tiles; t += pairs, ++i) {
      int b, m0, n0;
      tile_coords_pair(t, tiles_m, tiles_n, BN, b, m0, n0);
      m0 += static_cast<int>(rank) * BM;
      const int a = i & 1;
      mbar_wait_pair(&tmem_full[a], (i >> 1) & 1);
      tc_fence_after();
      const int row = m0 + quad * 32 + lane;
      float* out = static_cast<float*>(p.C) + static_cast<int64_t>(b) * p.sC + static_cast<int64_t>(row) * p.ldc;
      if (tma_store) {
        uint8_t* stage = smem + Cfg::EPI_OFFSET + quad * (2 * 32 * 32 * 4);
#pragma unroll 1
        for (int c = 0; c < BN; c += 32, ++epi_box) {
          float v[32];
          tmem_ld16(tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + a * BN + c, v);
          tmem_ld16(tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + a * BN + c + 16, v + 16);
          if (p.bias || p.relu) epilogue_run<32>(p, v, n0 + c);
          uint8_t* box = stage + (epi_box & 1) * (32 * 32 * 4);
          if (lane == 0) bulk_wait_read<1>();
          __syncwarp();
          if (p.c_bf16) {
            // bf16 box: 64-byte rows, 64B swizzle (16-byte chunk j of row r at j ^ ((r >> 1) & 3))
#pragma unroll
            for (int j = 0; j < 4; ++j)
              *reinterpret_cast<uint4*>(box + lane * 64 + ((j ^ ((lane >> 1) & 3)) << 4)) =
                  make_uint4(pack_bf16x2(v[8 * j], v[8 * j + 1]), pack_bf16x2(v[8 * j + 2], v[8 * j + 3]),
                             pack_bf16x2(v[8 * j + 4], v[8 * j + 5]), pack_bf16x2(v[8 * j + 6], v[8 * j + 7]));
          } else {
#pragma unroll
            for (int j = 0; j < 8; ++j)
              *reinterpret_cast<float4*>(box + lane * 128 + ((j ^ (lane & 7)) << 4)) =
                  make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            tma_store_3d(&mapC, box, n0 + c, m0 + quad * 32, b);
            bulk_commit();
          }
        }
      } else {
#pragma unroll 1
        for (int c = 0; c < BN; c += 16) {
          float v[16];
          tmem_ld16(tmem_base + (static_cast<uint32_t>(quad * 32) << 16) + a * BN + c, v);
          if (row < p.m) {
            const int col = n0 + c;
            if (p.bias || p.relu) epilogue_run<16>(p, v, col);
            if (p.c_bf16) {
              __nv_bfloat16* ob = static_cast<__nv_bfloat16*>(p.C) + static_cast<int64_t>(b) * p.sC +
                                  static_cast<int64_t>(row) * p.ldc + col;
              if (p.c_vec && col + 16 <= p.n) {
                uint32_t w[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) w[q] = pack_bf16x2(v[2 * q], v[2 * q + 1]);
                reinterpret_cast<uint4*>(ob)[0] = make_uint4(w[0], w[1], w[2], w[3]);
                reinterpret_cast<uint4*>(ob)[1] = make_uint4(w[4], w[5], w[6], w[7]);
              } else {
#pragma unroll
                for (int e = 0; e < 16; ++e)
                  if (col + e < p.n) ob[e] = __float2bfloat16_rn(v[e]);
              }
            } else if (p.c_vec && col + 16 <= p.n) {
#pragma unroll
              for (int q = 0; q < 4; ++q)
                *reinterpret_cast<float4*>(out + col + 4 * q) =
                    make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
            } else {
#pragma unroll
              for (int e = 0; e < 16; ++e)
                if (col + e < p.n) out[col + e] = v[e];
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0)
        asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(a ? empty_bar1 : empty_bar0)
                     : "memory");
    }
  }
  if (warp >= 2 && lane == 0 && tma_store) bulk_wait_all();
  tc_fence_before();
  cluster_sync_all();  // both CTAs done with TMEM and with each other's barriers
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(Cfg::TMEM_COLS));
  }
}

// ---------------------------------------------------------------- host side --
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

using EncodeIm2colFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                    const cuuint64_t*, const int*, const int*, cuuint32_t, cuuint32_t,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeIm2colFn encode_im2col_fn() {
  static EncodeIm2colFn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeIm2col", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeIm2colFn>(ptr);
  }
  return fn;
}

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    void* ptr = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(ptr);
  }
  return fn;
}

thread_local char g_reason[256] = "";

int num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

struct TcConfig {
  bool tf32;
  int bn, stages;
  int cg;  // 1: one CTA per 128-row tile; 2: CTA pairs (cta_group::2) per 256-row tile
};

// The family config lists (index order = the family's canonical column order; the
// first eight are round 1's, later entries append so measured tables keep their columns).
constexpr TcConfig kTf32Configs[] = {{true, 32, 4, 1},  {true, 64, 4, 1},  {true, 128, 4, 1}, {true, 256, 4, 1},
                                     {true, 64, 8, 1},  {true, 128, 6, 1}, {true, 256, 3, 1}, {true, 192, 4, 1},
                                     {true, 96, 4, 1},  {true, 160, 4, 1}, {true, 256, 6, 2}, {true, 128, 8, 2},
                                     {true, 192, 6, 2}};
constexpr TcConfig kBf16Configs[] = {{false, 64, 4, 1},  {false, 128, 4, 1}, {false, 256, 4, 1}, {false, 64, 8, 1},
                                     {false, 128, 6, 1}, {false, 256, 3, 1}, {false, 128, 2, 1}, {false, 192, 4, 1},
                                     {false, 256, 6, 2}, {false, 128, 8, 2}, {false, 256, 4, 2}};
constexpr int kNumTf32 = sizeof(kTf32Configs) / sizeof(kTf32Configs[0]);
constexpr int kNumBf16 = sizeof(kBf16Configs) / sizeof(kBf16Configs[0]);

const TcConfig* config_of(int family, int index) {
  if (family == KP_FAMILY_TF32) return (index >= 0 && index < kNumTf32) ? &kTf32Configs[index] : nullptr;
  if (family == KP_FAMILY_BF16) return (index >= 0 && index < kNumBf16) ? &kBf16Configs[index] : nullptr;
  return nullptr;
}

bool tma_ok(const GemmArgs& p, int es) {
  auto aligned = [](const void* ptr, int bytes) { return (reinterpret_cast<uintptr_t>(ptr) % bytes) == 0; };
  return aligned(p.A, 16) && aligned(p.B, 16) && (p.lda * es) % 16 == 0 && (p.ldb * es) % 16 == 0 &&
         (p.batch == 1 || ((p.sA * es) % 16 == 0 && (p.sB * es) % 16 == 0));
}

// A persistent CTA-pair launch over 256-row tiles (tc2_gemm_kernel).
template <bool kTF32, int BN, int STAGES>
cudaError_t launch_pair(const GemmArgs& p, const CUtensorMap& ma, const CUtensorMap& mb, const CUtensorMap& mc,
                        int a_batched, int b_batched, int tma_store, cudaStream_t s) {
  using Cfg = Tc2Cfg<kTF32, BN, STAGES>;
  static int fit = 0;  // co-resident pairs (cudaOccupancyMaxActiveClusters), per instantiation
  cudaLaunchConfig_t lc = {};
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  lc.blockDim = dim3(kThreads);
  lc.dynamicSmemBytes = Cfg::SMEM_BYTES;
  lc.stream = s;
  lc.attrs = at;
  lc.numAttrs = 1;
  if (!fit) {
    cudaError_t e = cudaFuncSetAttribute(tc2_gemm_kernel<kTF32, BN, STAGES>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    lc.gridDim = dim3(2);
    int n = 0;
    e = cudaOccupancyMaxActiveClusters(&n, tc2_gemm_kernel<kTF32, BN, STAGES>, &lc);
    if (e != cudaSuccess) return e;
    if (n < 1) return cudaErrorInvalidConfiguration;
    fit = n;
  }
  const int tiles_m = (p.m + BM2 - 1) / BM2, tiles_n = (p.n + BN - 1) / BN;
  const int64_t n_tiles = static_cast<int64_t>(tiles_m) * tiles_n * p.batch;
  if (n_tiles > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  const int pairs = static_cast<int>(n_tiles < fit ? n_tiles : fit);
  lc.gridDim = dim3(static_cast<unsigned>(2 * pairs));
  return cudaLaunchKernelEx(&lc, tc2_gemm_kernel<kTF32, BN, STAGES>, ma, mb, mc, p, tiles_m, tiles_n, a_batched,
                            b_batched, tma_store);
}

// PAIR_STAGES > 0: a CTA-pair config -- persistent TMA launches run tc2_gemm_kernel with
// that ring depth; LSU staging and k-sliced plans run the 1-CTA kernel (STAGES deep).
template <bool kTF32, int BN, int STAGES, int PAIR_STAGES = 0>
cudaError_t launch_tc(const GemmArgs& p0, cudaStream_t s) {
  using Cfg = TcCfg<kTF32, BN, STAGES>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaSuccess;
    for (auto fn : {tc_gemm_kernel<kTF32, BN, STAGES, false, false>, tc_gemm_kernel<kTF32, BN, STAGES, true, false>})
      if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
    for (auto fn : {tc_gemm_kernel<kTF32, BN, STAGES, false, true>, tc_gemm_kernel<kTF32, BN, STAGES, true, true>}) {
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SLICED_SMEM_BYTES);
      if (e == cudaSuccess) e = cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    }
    if (e != cudaSuccess) return e;
    attr = true;
  }
  GemmArgs p = p0;
  auto aligned = [](const void* ptr, int bytes) { return (reinterpret_cast<uintptr_t>(ptr) % bytes) == 0; };
  p.c_vec = p.c_bf16 ? (p.ldc % 8 == 0) && (p.sC % 8 == 0) && aligned(p.C, 16)
                     : (p.ldc % 4 == 0) && (p.sC % 4 == 0) && aligned(p.C, 16);
  const int tiles_m = (p.m + BM - 1) / BM, tiles_n = (p.n + BN - 1) / BN;
  const int64_t n_tiles = static_cast<int64_t>(tiles_m) * tiles_n * p.batch;
  if (n_tiles > 0x7fffffffLL) return cudaErrorInvalidConfiguration;
  const int KT = (p.k + Cfg::BK - 1) / Cfg::BK;
  if (p.kslices <= 1) {
    p.kslices = 1;
    p.kt_per_slice = KT;
  } else if (p.kslices > kMaxKSlices || n_tiles * p.kslices > 0x7fffffffLL) {
    return cudaErrorInvalidConfiguration;  // sliced launches run one (tile, slice) per CTA
  }
  // tail split (planner, capi.cu): the last tail_tiles tiles run as a second, sliced launch
  int tail = 0, tail_s = 1;
  if (p.kslices == 1 && p.tail_slices > 1 && p.tail_tiles > 0 && p.tail_tiles < n_tiles &&
      p.tail_slices <= kMaxKSlices) {
    tail = p.tail_tiles;
    tail_s = p.tail_slices;
  }
  EncodeFn enc = encode_fn();
  if (!enc) return cudaErrorNotSupported;
  // C as a TMA store target: persistent launches with 16-byte-aligned C rows and a short
  // k, where the epilogue is a large share of the tile (measured: 16384x64x16384 2.2x,
  // 6272x1152x256 +15 %); with long k the stores compete with the operand loads for the
  // TMA unit and direct stores measured slightly faster (profiles/r1_tc_epilogue.md)
  CUtensorMap mc;
  std::memset(&mc, 0, sizeof(mc));
  int tma_store = 0;
  // (bf16 C, KP_EPI_BF16_OUT: 32 x 32 boxes of 64-byte rows, 64B swizzle)
  if (p.kslices <= 1 && p.c_vec && p.k <= kTmaStoreMaxK) {
    const int ces = p.c_bf16 ? 2 : 4;
    cuuint64_t dims[3] = {static_cast<cuuint64_t>(p.n), static_cast<cuuint64_t>(p.m),
                          static_cast<cuuint64_t>(p.batch)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(p.ldc) * ces,
                             static_cast<cuuint64_t>(p.batch > 1 ? p.sC : p.ldc * p.m) * ces};
    if (p.batch == 1) strides[1] = (strides[1] + 15) / 16 * 16;
    cuuint32_t box[3] = {32, 32, 1};
    cuuint32_t es[3] = {1, 1, 1};
    tma_store = enc(&mc, p.c_bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, p.C, dims,
                    strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    p.c_bf16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
  }
  const bool lsu = !tma_ok(p, Cfg::ES);
  const int a_batched = (p.batch > 1 && p.sA != 0), b_batched = (p.batch > 1 && p.sB != 0);
  CUtensorMap ma, mb;
  std::memset(&ma, 0, sizeof(ma));
  std::memset(&mb, 0, sizeof(mb));
  if (!lsu) {
    const CUtensorMapDataType dt = kTF32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    {
      cuuint64_t dims[3] = {static_cast<cuuint64_t>(p.k), static_cast<cuuint64_t>(p.m),
                            static_cast<cuuint64_t>(a_batched ? p.batch : 1)};
      cuuint64_t strides[2] = {static_cast<cuuint64_t>(p.lda) * Cfg::ES,
                               static_cast<cuuint64_t>(a_batched ? p.sA : p.lda * p.m) * Cfg::ES};
      if (!a_batched) strides[1] = (strides[1] + 15) / 16 * 16;
      cuuint32_t box[3] = {static_cast<cuuint32_t>(Cfg::BK), static_cast<cuuint32_t>(BM), 1};
      cuuint32_t es[3] = {1, 1, 1};
      if (p.conv_c > 0) {
        // implicit conv: A is the NHWC activation; im2col boxes of BK channels x BM pixels,
        // bounding box corners -1 / -1 (base pixel = output pixel - 1 in w and h)
        EncodeIm2colFn enc2 = encode_im2col_fn();
        const int imgs = p.m / (p.conv_h * p.conv_w);
        cuuint64_t idims[4] = {static_cast<cuuint64_t>(p.conv_c), static_cast<cuuint64_t>(p.conv_w),
                               static_cast<cuuint64_t>(p.conv_h), static_cast<cuuint64_t>(imgs)};
        cuuint64_t istrides[3] = {static_cast<cuuint64_t>(p.conv_c) * Cfg::ES,
                                  static_cast<cuuint64_t>(p.conv_w) * p.conv_c * Cfg::ES,
                                  static_cast<cuuint64_t>(p.conv_h) * p.conv_w * p.conv_c * Cfg::ES};
        const int lower[2] = {-1, -1}, upper[2] = {-1, -1};
        cuuint32_t ies[4] = {1, 1, 1, 1};
        if (!enc2 || enc2(&ma, dt, 4, const_cast<void*>(p.A), idims, istrides, lower, upper,
                          static_cast<cuuint32_t>(Cfg::BK), static_cast<cuuint32_t>(BM), ies,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
          return cudaErrorInvalidValue;
      } else if (enc(&ma, dt, 3, const_cast<void*>(p.A), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        return cudaErrorInvalidValue;
      }
    }
    {
      cuuint64_t dims[3] = {static_cast<cuuint64_t>(p.n), static_cast<cuuint64_t>(p.k),
                            static_cast<cuuint64_t>(b_batched ? p.batch : 1)};
      cuuint64_t strides[2] = {static_cast<cuuint64_t>(p.ldb) * Cfg::ES,
                               static_cast<cuuint64_t>(b_batched ? p.sB : p.ldb * p.k) * Cfg::ES};
      if (!b_batched) strides[1] = (strides[1] + 15) / 16 * 16;
      cuuint32_t box[3] = {static_cast<cuuint32_t>(Cfg::NATOM), static_cast<cuuint32_t>(Cfg::BK), 1};
      cuuint32_t es[3] = {1, 1, 1};
      if (enc(&mb, dt, 3, const_cast<void*>(p.B), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              kTF32 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return cudaErrorInvalidValue;
    }
  }
  if constexpr (PAIR_STAGES > 0) {
    // CTA pairs for persistent TMA launches (no tail split: the pair kernel runs every tile)
    if (!lsu && p.kslices <= 1)
      return launch_pair<kTF32, BN, PAIR_STAGES>(p, ma, mb, mc, a_batched, b_batched, tma_store, s);
    tail = 0;
  }
  // one launch over tiles [t0, t0 + count): persistent (slices == 1, grid <= SMs) or
  // k-sliced (grid (count, 1, slices) in (1, 1, slices) clusters)
  auto go = [&](GemmArgs q, int t0, int count, int slices) -> cudaError_t {
    if (slices > 1) {  // no empty slice: every CTA must accumulate at least one k-tile
      const int per = (KT + slices - 1) / slices;
      slices = (KT + per - 1) / per;
    }
    cudaLaunchConfig_t lc = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 1;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = slices;
    lc.gridDim = slices > 1 ? dim3(static_cast<unsigned>(count), 1, slices)
                            : dim3(static_cast<unsigned>(count < num_sms() ? count : num_sms()));
    lc.blockDim = dim3(kThreads);
    lc.dynamicSmemBytes = slices > 1 ? Cfg::SLICED_SMEM_BYTES : Cfg::SMEM_BYTES;
    lc.stream = s;
    lc.attrs = at;
    lc.numAttrs = slices > 1 ? 1 : 0;
    if (slices > 1) {
      q.kslices = slices;
      q.kt_per_slice = (KT + slices - 1) / slices;
      return lsu ? cudaLaunchKernelEx(&lc, tc_gemm_kernel<kTF32, BN, STAGES, true, true>, ma, mb, mc, q, tiles_m,
                                      tiles_n, 0, 0, 0, t0, count)
                 : cudaLaunchKernelEx(&lc, tc_gemm_kernel<kTF32, BN, STAGES, false, true>, ma, mb, mc, q, tiles_m,
                                      tiles_n, a_batched, b_batched, 0, t0, count);
    }
    q.kslices = 1;
    q.kt_per_slice = KT;
    return lsu ? cudaLaunchKernelEx(&lc, tc_gemm_kernel<kTF32, BN, STAGES, true, false>, ma, mb, mc, q, tiles_m,
                                    tiles_n, 0, 0, tma_store, t0, count)
               : cudaLaunchKernelEx(&lc, tc_gemm_kernel<kTF32, BN, STAGES, false, false>, ma, mb, mc, q, tiles_m,
                                    tiles_n, a_batched, b_batched, tma_store, t0, count);
  };
  const int total = static_cast<int>(n_tiles);
  if (p.kslices > 1) return go(p, 0, total, p.kslices);  // the whole grid sliced
  if (tail > 0) {
    cudaError_t e = go(p, 0, total - tail, 1);
    if (e != cudaSuccess) return e;
    return go(p, total - tail, tail, tail_s);
  }
  return go(p, 0, total, 1);
}

// cudaOccupancyMaxActiveClusters of a (1, 1, slices) cluster launch (< 0: error).
template <bool kTF32, int BN, int STAGES>
int cluster_fit_tc(int slices) {
  using Cfg = TcCfg<kTF32, BN, STAGES>;
  for (auto fn : {tc_gemm_kernel<kTF32, BN, STAGES, false, true>, tc_gemm_kernel<kTF32, BN, STAGES, true, true>})
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SLICED_SMEM_BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
      cudaGetLastError();
      return -1;
    }
  cudaLaunchConfig_t lc = {};
  lc.gridDim = dim3(1, 1, slices);
  lc.blockDim = dim3(kThreads);
  lc.dynamicSmemBytes = Cfg::SLICED_SMEM_BYTES;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 1;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = slices;
  lc.attrs = at;
  lc.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, tc_gemm_kernel<kTF32, BN, STAGES, false, true>, &lc) != cudaSuccess) {
    cudaGetLastError();
    return -1;
  }
  return n;
}

// 1-CTA (BN, STAGES) of a config: pair configs fall back to their 1-CTA twin (the
// deepest ring that fits one SM) for LSU staging and k-sliced launches.
constexpr int twin_stages(const TcConfig& c) {
  return c.cg == 1 ? c.stages : (c.bn == 256 ? 3 : c.bn == 192 ? 4 : 6);
}

template <bool kTF32>
int dispatch_fit(const TcConfig& c, int slices) {
  switch (c.bn * 16 + twin_stages(c)) {
    case 32 * 16 + 4:
      if constexpr (kTF32) return cluster_fit_tc<kTF32, 32, 4>(slices);
      return -1;
    case 64 * 16 + 4: return cluster_fit_tc<kTF32, 64, 4>(slices);
    case 96 * 16 + 4:
      if constexpr (kTF32) return cluster_fit_tc<kTF32, 96, 4>(slices);
      return -1;
    case 128 * 16 + 4: return cluster_fit_tc<kTF32, 128, 4>(slices);
    case 160 * 16 + 4:
      if constexpr (kTF32) return cluster_fit_tc<kTF32, 160, 4>(slices);
      return -1;
    case 256 * 16 + 4: return cluster_fit_tc<kTF32, 256, 4>(slices);
    case 64 * 16 + 8: return cluster_fit_tc<kTF32, 64, 8>(slices);
    case 128 * 16 + 6: return cluster_fit_tc<kTF32, 128, 6>(slices);
    case 256 * 16 + 3: return cluster_fit_tc<kTF32, 256, 3>(slices);
    case 128 * 16 + 2:
      if constexpr (!kTF32) return cluster_fit_tc<kTF32, 128, 2>(slices);
      return -1;
    case 192 * 16 + 4: return cluster_fit_tc<kTF32, 192, 4>(slices);
    default: return -1;
  }
}

template <bool kTF32>
cudaError_t dispatch(const TcConfig& c, const GemmArgs& p, cudaStream_t s) {
  if (c.cg == 2) {
    switch (c.bn * 16 + c.stages) {
      case 256 * 16 + 6: return launch_tc<kTF32, 256, 3, 6>(p, s);
      case 128 * 16 + 8: return launch_tc<kTF32, 128, 6, 8>(p, s);
      case 256 * 16 + 4:
        if constexpr (!kTF32) return launch_tc<kTF32, 256, 3, 4>(p, s);
        return cudaErrorInvalidValue;
      case 192 * 16 + 6:
        if constexpr (kTF32) return launch_tc<kTF32, 192, 4, 6>(p, s);
        return cudaErrorInvalidValue;
      default: return cudaErrorInvalidValue;
    }
  }
  switch (c.bn * 16 + c.stages) {
    case 32 * 16 + 4:
      if constexpr (kTF32) return launch_tc<kTF32, 32, 4>(p, s);
      return cudaErrorInvalidValue;
    case 64 * 16 + 4: return launch_tc<kTF32, 64, 4>(p, s);
    case 96 * 16 + 4:
      if constexpr (kTF32) return launch_tc<kTF32, 96, 4>(p, s);
      return cudaErrorInvalidValue;
    case 128 * 16 + 4: return launch_tc<kTF32, 128, 4>(p, s);
    case 160 * 16 + 4:
      if constexpr (kTF32) return launch_tc<kTF32, 160, 4>(p, s);
      return cudaErrorInvalidValue;
    case 256 * 16 + 4: return launch_tc<kTF32, 256, 4>(p, s);
    case 64 * 16 + 8: return launch_tc<kTF32, 64, 8>(p, s);
    case 128 * 16 + 6: return launch_tc<kTF32, 128, 6>(p, s);
    case 256 * 16 + 3: return launch_tc<kTF32, 256, 3>(p, s);
    case 128 * 16 + 2:
      if constexpr (!kTF32) return launch_tc<kTF32, 128, 2>(p, s);
      return cudaErrorInvalidValue;
    case 192 * 16 + 4: return launch_tc<kTF32, 192, 4>(p, s);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace

int tc_family_size(int family) {
  return family == KP_FAMILY_TF32 ? kNumTf32 : family == KP_FAMILY_BF16 ? kNumBf16 : 0;
}

KernelChoice tc_family_choice(int family, int index) {
  const TcConfig* c = config_of(family, index);
  if (!c) return KernelChoice{0, 0, 0, 0, 0};
  return KernelChoice{BM * c->cg, c->tf32 ? 32 : 64, c->bn, c->stages, kThreads};
}

const char* tc_last_reason() { return g_reason; }

int tc_check(int family, int index, const GemmArgs& p) {
  (void)p;  // every shape runs: TMA when rows are 16-byte aligned, LSU staging otherwise
  if (!config_of(family, index)) {
    snprintf(g_reason, sizeof(g_reason), "no tensor-core config %d in family %d", index, family);
    return KP_ENOENT;
  }
  return KP_OK;
}

int tc_tile_n(int family, int index) {
  const TcConfig* c = config_of(family, index);
  return c ? c->bn : -1;
}

int tc_tile_k(int family) { return family == KP_FAMILY_TF32 ? 32 : 64; }

int tc_cluster_fit(int family, int index, int slices) {
  const TcConfig* c = config_of(family, index);
  if (!c) return -1;
  return c->tf32 ? dispatch_fit<true>(*c, slices) : dispatch_fit<false>(*c, slices);
}

cudaError_t tc_launch(int family, int index, const GemmArgs& p, cudaStream_t s) {
  const TcConfig* c = config_of(family, index);
  if (!c) return cudaErrorInvalidValue;
  return c->tf32 ? dispatch<true>(*c, p, s) : dispatch<false>(*c, p, s);
}

}  // namespace kp
