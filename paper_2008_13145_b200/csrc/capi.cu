// The C ABI of libkpgemm.so (include/kpgemm.h): variant registry, GEMM launch,
// benchmark harness, FFMA peak probe and the tree -> variant dispatch tables.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "families.h"
#include "kpgemm.h"
#include "tc_families.h"

std::atomic<int> kp::g_f1_tma_staging{1};  // kp_set_simt_staging
std::atomic<int> g_operand_repack{1};      // kp_set_operand_repack

namespace {

thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_last_error = buf;
  return code;
}

int cuda_fail(cudaError_t e, const char* what) {
  return fail(KP_EIO, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

// ---------------------------------------------------------------- registry --
struct Variant {
  int family;
  KernelChoice choice;
  int index;  // position inside the family's canonical config list
};

struct Registry {
  std::vector<Variant> variants;
  int family_begin[KP_NUM_FAMILIES + 1];
  kp::F1Entry f1[kp::kPaperConfigs];

  Registry() {
    std::memset(f1, 0, sizeof(f1));
    kp::f1_fill_wg0(f1);
    kp::f1_fill_wg1(f1);
    kp::f1_fill_wg2(f1);
    kp::f1_fill_wg3(f1);
    kp::f1_fill_wg4(f1);
    kp::f1_fill_wg5(f1);
    kp::f1_fill_wg6(f1);
    kp::f1_fill_wg7(f1);
    kp::f1_fill_wg8(f1);
    kp::f1_fill_wg9(f1);
    const int tiles[4] = {1, 2, 4, 8};
    for (int fam = 0; fam < KP_NUM_FAMILIES; ++fam) {
      family_begin[fam] = static_cast<int>(variants.size());
      if (fam == KP_FAMILY_PAPER || fam == KP_FAMILY_SIMT) {
        int idx = 0;
        for (int r : tiles)
          for (int a : tiles)
            for (int c : tiles)
              for (int w = 0; w < kp::kNumWgPairs; ++w) {
                KernelChoice ch{r, a, c, kp::kWgPairs[w][0], kp::kWgPairs[w][1]};
                variants.push_back(Variant{fam, ch, idx++});
              }
      } else {
        const int count = kp::tc_family_size(fam);
        for (int i = 0; i < count; ++i) variants.push_back(Variant{fam, kp::tc_family_choice(fam, i), i});
      }
    }
    family_begin[KP_NUM_FAMILIES] = static_cast<int>(variants.size());
  }
};

Registry& registry() {
  static Registry r;
  return r;
}

bool same(const KernelChoice& a, const KernelChoice& b) {
  return a.tile_rows == b.tile_rows && a.tile_acc == b.tile_acc && a.tile_cols == b.tile_cols &&
         a.wg_rows == b.wg_rows && a.wg_cols == b.wg_cols;
}

int check_problem(int id, int m, int k, int n, int batch, const void* A, int64_t lda, int64_t sA, const void* B,
                  int64_t ldb, int64_t sB, void* C, int64_t ldc, int64_t sC) {
  Registry& reg = registry();
  if (id < 0 || id >= static_cast<int>(reg.variants.size())) return fail(KP_ENOENT, "unknown variant id %d", id);
  if (m < 1 || k < 1 || n < 1 || batch < 1)
    return fail(KP_EINVAL, "dims must be >= 1 (m=%d k=%d n=%d batch=%d)", m, k, n, batch);
  if (!A || !B || !C) return fail(KP_EINVAL, "null operand pointer");
  if (lda < k || ldb < n || ldc < n) return fail(KP_EINVAL, "leading dimension smaller than the row length");
  if (sA < 0 || sB < 0 || sC < 0) return fail(KP_EINVAL, "negative batch stride");
  if (batch > 1 && sC < static_cast<int64_t>(m) * ldc) return fail(KP_EINVAL, "output batch stride overlaps");
  if (batch > 65535) return fail(KP_EINVAL, "batch > 65535");
  return KP_OK;
}

// ------------------------------------------------------------- k-slicing --
// When a launch's output tiles leave SMs idle or end in a partial wave, the k-tiles are
// cut into S consecutive slices computed by the S CTAs of a (1, 1, S) cluster and
// summed in slice order through distributed shared memory (f1_simt.cuh, tc_gemm.cu);
// plan_slices below holds the rules (include/kpgemm.h documents them).  The plan is a
// pure function of (config, shape, device), so results are deterministic on a given GPU
// model and the oracle reproduces the SIMT ones from kp_gemm_plan.
std::atomic<int> g_max_kslices{kp::kDefaultKSlices};
constexpr int kMinSliceK = 64;     // never cut k into slices shallower than this (SIMT)
constexpr int kMinSliceKTc = 768;  // tensor cores: shallower slices lose to the fixed costs

int num_sms_current() {
  static std::mutex mu;
  static std::vector<int> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  std::lock_guard<std::mutex> lock(mu);
  if (dev >= static_cast<int>(cache.size())) cache.resize(dev + 1, 0);
  if (cache[dev] == 0) {
    int sms = 0;
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms < 1) return -1;
    cache[dev] = sms;
  }
  return cache[dev];
}

// Tile facts of a sliceable variant: CTA tile bm x bn, k-tile bk, resident CTAs per SM.
struct SliceTile {
  int bm, bn, bk, occ;
};

bool slice_tile(const Variant& v, SliceTile* t) {
  if (v.family == KP_FAMILY_SIMT) {
    const kp::F1Entry& e = registry().f1[v.index];
    *t = SliceTile{e.bm, e.bn, e.bk, e.occ};
    return true;
  }
  if (v.family == KP_FAMILY_TF32 || v.family == KP_FAMILY_BF16) {
    // persistent 1-CTA/SM kernel; slicing only when at most half the SMs get a tile
    *t = SliceTile{128, kp::tc_tile_n(v.family, v.index), kp::tc_tile_k(v.family), 1};
    return t->bn > 0;
  }
  return false;  // PAPER: the paper's geometry, never sliced
}

int cluster_fit(const Variant& v, int slices) {
  if (v.family == KP_FAMILY_SIMT) return registry().f1[v.index].cluster_fit(slices);
  return kp::tc_cluster_fit(v.family, v.index, slices);
}

// Largest cluster size s <= want for which the device can co-schedule `clusters`
// (1, 1, s) clusters of this variant at once (cudaOccupancyMaxActiveClusters), so a
// sliced launch stays a single wave; cached per (variant, size).
int fit_slices(int id, const Variant& v, int want, int64_t clusters) {
  static std::mutex mu;
  static std::vector<int> fit;  // [id][slices]: max active clusters, -2 = not queried yet
  std::lock_guard<std::mutex> lock(mu);
  const size_t row = kp::kMaxKSlices + 1;
  if (fit.empty()) fit.assign(registry().variants.size() * row, -2);
  for (int s = want; s > 1; --s) {
    int& f = fit[id * row + s];
    if (f == -2) f = cluster_fit(v, s);
    if (f >= clusters) return s;
  }
  return 1;
}

// The k-slice plan of variant id on (m, k, n, batch): S slices of kt_per_slice k-tiles
// (S == 1: kt_per_slice = all k-tiles).  sms > 0 with device == false plans for a
// hypothetical device (no cluster-occupancy query).
struct TailPlan {
  int tail_tiles = 0, tail_slices = 0, kt_per_slice_tail = 0;
};

void plan_slices(int id, int m, int k, int n, int batch, int sms, bool device, int* slices, int* kt_per_slice,
                 int* bk, TailPlan* tail_out = nullptr) {
  const Variant& v = registry().variants[id];
  SliceTile t{1, 1, k, 1};
  const int max_slices = g_max_kslices.load(std::memory_order_relaxed);
  int s = 1;
  if (slice_tile(v, &t) && max_slices > 1) {
    const int64_t tiles = ((m + t.bm - 1) / t.bm) * static_cast<int64_t>((n + t.bn - 1) / t.bn) * batch;
    if (v.family == KP_FAMILY_SIMT) {
      // Tiles per SM -> slices, fitted on 673 measured (shape, config) cells with every
      // forced S (profiles/r1_kslicing.md): u < 0.5 -> 8, < 2 -> 4, < 6 -> 2, else 1;
      // halved while the sliced grid would exceed 4 waves of resident CTAs, and never
      // shallower than 64 in k.  Round 2 (TMA staging, 784 cells x S in 1..8,10,12,16,
      // profiles/r2/kslice_refit.md): grids under 0.15 tiles per SM take 16-CTA
      // (non-portable) clusters -- 0.952 -> 0.974 of the per-cell best S.
      const double u = static_cast<double>(tiles) / sms;
      s = u < 0.15 ? 16 : u < 0.5 ? 8 : u < 2.0 ? 4 : u < 6.0 ? 2 : 1;
      while (s > 1 && tiles * s > 4LL * sms * t.occ) s /= 2;
      if (s > max_slices) s = max_slices;
      if (s > k / kMinSliceK) s = k / kMinSliceK;
      if (s < 1) s = 1;
      if (device && s > 1) s = fit_slices(id, v, s, 1);
    } else if (2 * tiles <= static_cast<int64_t>(sms) * t.occ) {
      // persistent tensor-core kernel: slice only grids that fill at most half the SMs,
      // in one wave of clusters (a second wave of non-persistent CTAs loses to it)
      const int64_t want = static_cast<int64_t>(sms) * t.occ / tiles;
      const int cap = max_slices < kp::kPortableKSlices ? max_slices : kp::kPortableKSlices;
      s = static_cast<int>(want < cap ? want : cap);
      const int by_k = k / kMinSliceKTc;
      if (s > by_k) s = by_k;
      if (s < 1) s = 1;
      if (device && s > 1) s = fit_slices(id, v, s, tiles);
    } else if (tail_out && tiles > sms) {
      // more than one wave: the persistent kernel keeps the full waves; a partial last
      // wave filling at most half the SMs runs as a separate k-sliced launch
      // Only for long tiles (>= ~40 us of MMA: BN*k >= 1.72e6 for BF16, half that for TF32
      // at half the rate): the second launch, its pipeline fill and the DSMEM reduction
      // cost ~10 us, so shorter tails measured slower (profiles/r1_tc_epilogue.md).
      const int64_t r = tiles % sms;
      const int64_t work = static_cast<int64_t>(t.bn) * k * (v.family == KP_FAMILY_TF32 ? 2 : 1);
      if (r > 0 && 2 * r <= sms && k >= 2 * kMinSliceKTc && work >= 1720000) {
        const int cap = max_slices < kp::kPortableKSlices ? max_slices : kp::kPortableKSlices;
        int ts = static_cast<int>(sms / r < cap ? sms / r : cap);
        if (ts > k / kMinSliceKTc) ts = k / kMinSliceKTc;
        if (device && ts > 1) ts = fit_slices(id, v, ts, r);
        if (ts > 1) {
          const int kt = (k + t.bk - 1) / t.bk;
          tail_out->tail_tiles = static_cast<int>(r);
          tail_out->tail_slices = ts;
          tail_out->kt_per_slice_tail = (kt + ts - 1) / ts;
        }
      }
    }
  }
  const int kt = (k + t.bk - 1) / t.bk;
  int per = (kt + s - 1) / s;
  s = (kt + per - 1) / per;  // no empty slices
  if (s == 1) per = kt;
  *slices = s;
  *kt_per_slice = per;
  *bk = t.bk;
}

// ------------------------------------------------------- operand repacking --
// TMA needs 16-byte-aligned operand rows.  Operands whose rows are not (raw k = 27 or
// 147 im2col rows, n = 27, ...) are first copied into a 16-byte-pitched scratch copy --
// one HBM-bound pass -- and the launch then takes the TMA path (the tensor-core families'
// LSU staging measured 8 % of the HBM roofline on such rows; profiles/r2/repack.md).
// Scratch is stream-ordered, from a library-owned pool per device that keeps up to 1 GiB
// cached between launches (the process's default pool is left alone).
cudaError_t scratch_alloc(void** ptr, size_t bytes, cudaStream_t s) {
  static std::mutex mu;
  static std::vector<cudaMemPool_t> pools;
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  if (cudaError_t e = cudaStreamIsCapturing(s, &cap); e != cudaSuccess) return e;
  if (cap != cudaStreamCaptureStatusNone) return cudaMallocAsync(ptr, bytes, s);  // a graph memory node
  int dev = 0;
  if (cudaError_t e = cudaGetDevice(&dev); e != cudaSuccess) return e;
  cudaMemPool_t pool = nullptr;
  {
    std::lock_guard<std::mutex> lock(mu);
    if (dev >= static_cast<int>(pools.size())) pools.resize(dev + 1, nullptr);
    if (!pools[dev]) {
      cudaMemPoolProps props = {};
      props.allocType = cudaMemAllocationTypePinned;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = dev;
      if (cudaError_t e = cudaMemPoolCreate(&pools[dev], &props); e != cudaSuccess) return e;
      uint64_t keep = 1ull << 30;
      cudaMemPoolSetAttribute(pools[dev], cudaMemPoolAttrReleaseThreshold, &keep);
    }
    pool = pools[dev];
  }
  return cudaMallocFromPoolAsync(ptr, bytes, pool, s);
}

struct Repacked {
  void* buf[2] = {nullptr, nullptr};
  cudaStream_t s = nullptr;
  ~Repacked() {
    for (void* b : buf)
      if (b) cudaFreeAsync(b, s);  // stream-ordered: after the GEMM that reads it
  }
};

// Repack A and/or B of p (element size es) whose rows TMA cannot address, when the
// copy pays for itself (measured, profiles/r2/repack.md):
//   * tensor-core families: the in-kernel LSU staging runs at 8-30 % of the TMA path, so
//     repack unless the unaligned operands are small (< 4 MB) and k spans at most 4 k-tiles
//     (there the fixed cost of the extra pass loses: 12544 x 27 x 64 5.1 -> 3.8 TF/s);
//   * SIMT: 4-byte cp.async staging is close to TMA when the output dominates the traffic
//     (conv1_1: 20.8 TF/s in-kernel vs 19.4 with the repack pass), far behind it when the
//     operands do (32 x 12321 x 27: 0.23 -> 0.56 TF/s), so repack only when the unaligned
//     operands are at least as large as the output.
cudaError_t repack_unaligned(kp::GemmArgs& p, int es, bool tensor_core, int bk, bool always, Repacked& rp,
                             cudaStream_t s) {
  auto rows_ok = [&](const void* ptr, int64_t ld, int64_t sb) {
    return reinterpret_cast<uintptr_t>(ptr) % 16 == 0 && (ld * es) % 16 == 0 &&
           (p.batch == 1 || sb == 0 || (sb * es) % 16 == 0);
  };
  const bool a_bad = !rows_ok(p.A, p.lda, p.sA), b_bad = !rows_ok(p.B, p.ldb, p.sB);
  if (!a_bad && !b_bad) return cudaSuccess;
  const int64_t nba = (p.batch > 1 && p.sA != 0) ? p.batch : 1, nbb = (p.batch > 1 && p.sB != 0) ? p.batch : 1;
  const double bad_bytes = (a_bad ? static_cast<double>(nba) * p.m * p.k * es : 0.0) +
                           (b_bad ? static_cast<double>(nbb) * p.k * p.n * es : 0.0);
  const double out_bytes = static_cast<double>(p.batch) * p.m * p.n * 4.0;
  const bool pays = tensor_core ? (bad_bytes >= 4.0 * (1 << 20) || p.k > 4 * bk) : bad_bytes >= out_bytes;
  if (!pays && !always) return cudaSuccess;
  rp.s = s;
  const int al = 16 / es;
  struct Op {
    const void** ptr;
    int64_t *ld, *sb;
    int rows, cols;
  } ops[2] = {{&p.A, &p.lda, &p.sA, p.m, p.k}, {&p.B, &p.ldb, &p.sB, p.k, p.n}};
  for (int i = 0; i < 2; ++i) {
    Op& o = ops[i];
    if (rows_ok(*o.ptr, *o.ld, *o.sb)) continue;
    const int nb = (p.batch > 1 && *o.sb != 0) ? p.batch : 1;
    const int64_t ldd = (static_cast<int64_t>(o.cols) + al - 1) / al * al;
    if (cudaError_t e = scratch_alloc(&rp.buf[i], static_cast<size_t>(nb) * o.rows * ldd * es, s); e != cudaSuccess) {
      rp.buf[i] = nullptr;
      return e;
    }
    if (cudaError_t e = kp::repack_rows_launch(*o.ptr, *o.ld, *o.sb, o.rows, o.cols, nb, es, rp.buf[i], ldd, s);
        e != cudaSuccess)
      return e;
    *o.ptr = rp.buf[i];
    *o.ld = ldd;
    *o.sb = nb > 1 ? static_cast<int64_t>(o.rows) * ldd : 0;
  }
  return cudaSuccess;
}

int launch(int id, const kp::GemmArgs& p0, cudaStream_t s) {
  Registry& reg = registry();
  const Variant& v = reg.variants[id];
  cudaError_t e = cudaSuccess;
  kp::GemmArgs p = p0;
  switch (v.family) {
    case KP_FAMILY_PAPER:
      e = kp::f0_launch(v.choice, p, s);
      break;
    case KP_FAMILY_SIMT:
    default: {
      if (v.family != KP_FAMILY_SIMT) {
        const int rc = kp::tc_check(v.family, v.index, p);
        if (rc != KP_OK) return fail(rc, "variant %d cannot run this problem: %s", id, kp::tc_last_reason());
      }
      if (g_max_kslices.load(std::memory_order_relaxed) > 1) {
        const int sms = num_sms_current();
        if (sms < 1) return fail(KP_EIO, "cannot query the SM count of the current device");
        int bk = 0;
        TailPlan tail;
        plan_slices(id, p.m, p.k, p.n, p.batch, sms, true, &p.kslices, &p.kt_per_slice, &bk, &tail);
        p.tail_tiles = tail.tail_tiles;
        p.tail_slices = tail.tail_slices;
        static const int forced = [] {  // dev-only override for planner experiments
          const char* e = std::getenv("KPGEMM_FORCE_SLICES");
          return e ? std::atoi(e) : 0;
        }();
        if (forced > 0) {
          const int kt = (p.k + bk - 1) / bk;
          p.kt_per_slice = (kt + forced - 1) / forced;
          p.kslices = (kt + p.kt_per_slice - 1) / p.kt_per_slice;
        }
      }
      // TMA-staged families: repack operand rows TMA cannot address (SIMT: only when this
      // config stages with TMA; the implicit-conv path has its own operand contract)
      Repacked rp;
      const bool simt_tma = v.family == KP_FAMILY_SIMT && reg.f1[v.index].tma_ok && p.conv_c == 0 &&
                            kp::g_f1_tma_staging.load(std::memory_order_relaxed) != 0;
      if ((simt_tma || (v.family != KP_FAMILY_SIMT && p.conv_c == 0)) &&
          g_operand_repack.load(std::memory_order_relaxed) != 0) {
        const bool tc = v.family != KP_FAMILY_SIMT;
        const int bk = tc ? kp::tc_tile_k(v.family) : reg.f1[v.index].bk;
        e = repack_unaligned(p, v.family == KP_FAMILY_BF16 ? 2 : 4, tc, bk,
                             g_operand_repack.load(std::memory_order_relaxed) == 2, rp, s);
        if (e != cudaSuccess) return cuda_fail(e, "operand repack");
      }
      e = v.family == KP_FAMILY_SIMT ? reg.f1[v.index].launch(p, s) : kp::tc_launch(v.family, v.index, p, s);
      break;
    }
  }
  if (e != cudaSuccess) return cuda_fail(e, "kernel launch");
  return KP_OK;
}

kp::GemmArgs make_args(int m, int k, int n, int batch, const void* A, int64_t lda, int64_t sA, const void* B,
                       int64_t ldb, int64_t sB, void* C, int64_t ldc, int64_t sC) {
  kp::GemmArgs p;
  p.m = m; p.k = k; p.n = n; p.batch = batch;
  p.A = A; p.lda = lda; p.sA = sA;
  p.B = B; p.ldb = ldb; p.sB = sB;
  p.C = C; p.ldc = ldc; p.sC = sC;
  p.a_vec = p.b_vec = p.c_vec = p.c_vec4 = 0;
  p.kslices = 1;
  p.kt_per_slice = 0;
  p.tail_tiles = p.tail_slices = 0;
  p.conv_h = p.conv_w = p.conv_c = 0;
  p.bias = nullptr;
  p.relu = 0;
  p.c_bf16 = 0;
  return p;
}

// ---------------------------------------------------------- dispatch tables --
// Tables are immutable once loaded and held by shared_ptr: a lookup copies the pointer
// under the lock, so a concurrent load (vector growth) or free cannot invalidate a walk
// already in progress.
struct Table {
  std::vector<int32_t> feature, left, right, leaf_class, class_to_variant;
  std::vector<double> threshold;
};
std::mutex g_tables_mu;
std::vector<std::shared_ptr<const Table>> g_tables;

std::shared_ptr<const Table> get_table(int handle) {
  std::lock_guard<std::mutex> lock(g_tables_mu);
  if (handle < 0 || handle >= static_cast<int>(g_tables.size())) return nullptr;
  return g_tables[handle];
}

// predict_tree (classify.py:230-237): left iff x[f] < thr, strictly.
int walk(const Table& t, const double* x) {
  int node = 0;
  for (size_t steps = 0; steps <= t.feature.size(); ++steps) {
    const int cls = t.leaf_class[node];
    if (cls >= 0) return cls;
    node = (x[t.feature[node]] < t.threshold[node]) ? t.left[node] : t.right[node];
  }
  return fail(KP_EINVAL, "tree walk did not terminate");
}

}  // namespace

// ====================================================================== ABI ==
extern "C" {

int kp_abi_version(void) { return KPGEMM_ABI_VERSION; }

const char* kp_last_error(void) { return g_last_error.c_str(); }

int kp_num_variants(void) { return static_cast<int>(registry().variants.size()); }

int kp_family_size(int family) {
  if (family < 0 || family >= KP_NUM_FAMILIES) return fail(KP_EINVAL, "unknown family %d", family);
  Registry& reg = registry();
  return reg.family_begin[family + 1] - reg.family_begin[family];
}

int kp_family_variant(int family, int index) {
  const int size = kp_family_size(family);
  if (size < 0) return size;
  if (index < 0 || index >= size) return fail(KP_ENOENT, "family %d has no config index %d", family, index);
  return registry().family_begin[family] + index;
}

int kp_find_variant(int family, KernelChoice choice) {
  if (family < 0 || family >= KP_NUM_FAMILIES) return fail(KP_EINVAL, "unknown family %d", family);
  Registry& reg = registry();
  for (int i = reg.family_begin[family]; i < reg.family_begin[family + 1]; ++i)
    if (same(reg.variants[i].choice, choice)) return i;
  return fail(KP_ENOENT, "family %d has no config (%d,%d,%d,%d,%d)", family, choice.tile_rows, choice.tile_acc,
              choice.tile_cols, choice.wg_rows, choice.wg_cols);
}

int kp_variant_info(int id, KernelChoice* choice, int* family) {
  Registry& reg = registry();
  if (id < 0 || id >= static_cast<int>(reg.variants.size())) return fail(KP_ENOENT, "unknown variant id %d", id);
  if (choice) *choice = reg.variants[id].choice;
  if (family) *family = reg.variants[id].family;
  return KP_OK;
}

int kp_gemm(int id, int m, int k, int n, int batch, const void* A, int64_t lda, int64_t sA, const void* B,
            int64_t ldb, int64_t sB, void* C, int64_t ldc, int64_t sC, void* stream) {
  int rc = check_problem(id, m, k, n, batch, A, lda, sA, B, ldb, sB, C, ldc, sC);
  if (rc != KP_OK) return rc;
  return launch(id, make_args(m, k, n, batch, A, lda, sA, B, ldb, sB, C, ldc, sC), static_cast<cudaStream_t>(stream));
}

// Epilogue flags of kp_gemm_ex / kp_conv3x3_nhwc_ex into p (id already validated).
int apply_epilogue(int id, const float* bias, int flags, kp::GemmArgs& p) {
  if (flags & ~(KP_EPI_RELU | KP_EPI_BF16_OUT)) return fail(KP_EINVAL, "unknown epilogue flags 0x%x", flags);
  if (flags & KP_EPI_BF16_OUT) {
    const int fam = registry().variants[id].family;
    if (fam != KP_FAMILY_TF32 && fam != KP_FAMILY_BF16)
      return fail(KP_EINVAL, "KP_EPI_BF16_OUT needs a tensor-core variant (TF32 or BF16), variant %d is not", id);
    p.c_bf16 = 1;
  }
  p.bias = bias;
  p.relu = (flags & KP_EPI_RELU) != 0;
  return KP_OK;
}

int kp_gemm_ex(int id, int m, int k, int n, int batch, const void* A, int64_t lda, int64_t sA, const void* B,
               int64_t ldb, int64_t sB, void* C, int64_t ldc, int64_t sC, const float* bias, int flags,
               void* stream) {
  int rc = check_problem(id, m, k, n, batch, A, lda, sA, B, ldb, sB, C, ldc, sC);
  if (rc != KP_OK) return rc;
  kp::GemmArgs p = make_args(m, k, n, batch, A, lda, sA, B, ldb, sB, C, ldc, sC);
  rc = apply_epilogue(id, bias, flags, p);
  if (rc != KP_OK) return rc;
  return launch(id, p, static_cast<cudaStream_t>(stream));
}

int kp_conv3x3_supported(int id, int C, int Cout) {
  Registry& reg = registry();
  if (id < 0 || id >= static_cast<int>(reg.variants.size())) return fail(KP_ENOENT, "unknown variant id %d", id);
  const Variant& v = reg.variants[id];
  if (C < 1 || Cout < 1) return 0;
  // TF32 (fp32 activations): im2col boxes of 32 channels = one 128-byte K slab
  if (v.family == KP_FAMILY_TF32) return (C % kp::tc_tile_k(v.family) == 0 && Cout % 4 == 0) ? 1 : 0;
  // BF16 (bf16 activations and weights): 64 channels = one 128-byte K slab; weight rows of
  // Cout bf16 must be 16-byte pitched for the B tensor map
  if (v.family == KP_FAMILY_BF16) return (C % kp::tc_tile_k(v.family) == 0 && Cout % 8 == 0) ? 1 : 0;
  if (v.family != KP_FAMILY_SIMT) return 0;  // PAPER: the paper's kernel
  const kp::F1Entry& e = reg.f1[v.index];
  return (e.tma_ok && C % e.bk == 0 && Cout % 4 == 0) ? 1 : 0;
}

int kp_conv3x3_nhwc_ex(int id, const void* x, int B, int H, int W, int C, const void* w, int Cout, void* out,
                       const float* bias, int flags, void* stream) {
  if (B < 1 || H < 1 || W < 1 || C < 1 || Cout < 1) return fail(KP_EINVAL, "conv dims must be >= 1");
  if (static_cast<int64_t>(B) * H * W > 0x7fffffffLL || 9LL * C > 0x7fffffffLL)
    return fail(KP_EINVAL, "conv too large for 32-bit GEMM dims");
  const int rc = kp_conv3x3_supported(id, C, Cout);
  if (rc < 0) return rc;
  if (rc == 0) return fail(KP_EINVAL, "variant %d cannot run an implicit conv with C = %d, Cout = %d", id, C, Cout);
  if (!x || !w || !out) return fail(KP_EINVAL, "null operand pointer");
  auto aligned = [](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) % 16) == 0; };
  if (!aligned(x) || !aligned(w) || !aligned(out)) return fail(KP_EINVAL, "x, w and out must be 16-byte aligned");
  const int m = B * H * W, k = 9 * C;
  kp::GemmArgs p = make_args(m, k, Cout, 1, x, k, 0, w, Cout, 0, out, Cout, 0);
  const int erc = apply_epilogue(id, bias, flags, p);
  if (erc != KP_OK) return erc;
  p.conv_h = H;
  p.conv_w = W;
  p.conv_c = C;
  return launch(id, p, static_cast<cudaStream_t>(stream));
}

int kp_set_max_k_slices(int max_slices) {
  if (max_slices < 1 || max_slices > kp::kMaxKSlices)
    return fail(KP_EINVAL, "max k-slices must be in [1, %d], got %d", kp::kMaxKSlices, max_slices);
  return g_max_kslices.exchange(max_slices);
}

int kp_set_simt_staging(int mode) {
  if (mode != 0 && mode != 1) return fail(KP_EINVAL, "staging mode must be 0 (cp.async) or 1 (TMA), got %d", mode);
  return kp::g_f1_tma_staging.exchange(mode);
}

int kp_set_operand_repack(int mode) {
  if (mode < 0 || mode > 2)
    return fail(KP_EINVAL, "repack mode must be 0 (never), 1 (when it pays) or 2 (always), got %d", mode);
  return g_operand_repack.exchange(mode);
}

int kp_gemm_plan(int id, int m, int k, int n, int batch, int num_sms, int* k_slices, int* k_per_slice) {
  Registry& reg = registry();
  if (id < 0 || id >= static_cast<int>(reg.variants.size())) return fail(KP_ENOENT, "unknown variant id %d", id);
  if (m < 1 || k < 1 || n < 1 || batch < 1) return fail(KP_EINVAL, "dims must be >= 1");
  if (!k_slices || !k_per_slice) return fail(KP_EINVAL, "null output pointer");
  const bool device = num_sms <= 0;
  if (device && g_max_kslices.load(std::memory_order_relaxed) > 1) {
    num_sms = num_sms_current();
    if (num_sms < 1) return fail(KP_EIO, "cannot query the SM count of the current device");
  }
  int s = 1, per = 0, bk = 1;
  TailPlan tail;
  plan_slices(id, m, k, n, batch, num_sms > 0 ? num_sms : 1, device, &s, &per, &bk, &tail);
  if (s == 1 && tail.tail_slices > 1) {  // tensor cores: the partial last wave's launch
    const int kt = (k + bk - 1) / bk;
    per = tail.kt_per_slice_tail;
    s = (kt + per - 1) / per;
  }
  *k_slices = s;
  const int64_t depth = static_cast<int64_t>(per) * bk;
  *k_per_slice = s == 1 ? k : static_cast<int>(depth < k ? depth : k);
  return KP_OK;
}

int kp_bench_sets(int id, int m, int k, int n, int batch, int n_sets, const void* const* A, int64_t lda, int64_t sA,
                  const void* const* B, int64_t ldb, int64_t sB, void* const* C, int64_t ldc, int64_t sC, int warmup,
                  int min_iters, int max_iters, double min_ms, int repeats, double* median_ms, int* iters,
                  void* stream) {
  if (n_sets < 1 || !A || !B || !C) return fail(KP_EINVAL, "need at least one operand set");
  if (repeats < 1 || repeats > 64) return fail(KP_EINVAL, "repeats must be in [1, 64]");
  if (!median_ms || !iters) return fail(KP_EINVAL, "null output pointer");
  if (min_iters < 1 || max_iters < min_iters) return fail(KP_EINVAL, "bad iteration bounds");
  std::vector<kp::GemmArgs> sets;
  for (int i = 0; i < n_sets; ++i) {
    int rc = check_problem(id, m, k, n, batch, A[i], lda, sA, B[i], ldb, sB, C[i], ldc, sC);
    if (rc != KP_OK) return rc;
    sets.push_back(make_args(m, k, n, batch, A[i], lda, sA, B[i], ldb, sB, C[i], ldc, sC));
  }
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int rc = KP_OK;
  for (int i = 0; i < warmup; ++i)
    if ((rc = launch(id, sets[i % n_sets], s)) != KP_OK) return rc;
  cudaEvent_t e0, e1;
  cudaError_t e;
  if ((e = cudaEventCreate(&e0)) != cudaSuccess) return cuda_fail(e, "cudaEventCreate");
  if ((e = cudaEventCreate(&e1)) != cudaSuccess) {
    cudaEventDestroy(e0);
    return cuda_fail(e, "cudaEventCreate");
  }
  int next = 0;  // launches rotate through the operand sets
  auto timed = [&](int count, float* ms) -> int {
    cudaEventRecord(e0, s);
    for (int i = 0; i < count; ++i) {
      int r = launch(id, sets[next], s);
      next = (next + 1) % n_sets;
      if (r != KP_OK) return r;
    }
    cudaEventRecord(e1, s);
    cudaError_t err = cudaEventSynchronize(e1);
    if (err != cudaSuccess) return cuda_fail(err, "kernel execution");
    err = cudaEventElapsedTime(ms, e0, e1);
    if (err != cudaSuccess) return cuda_fail(err, "cudaEventElapsedTime");
    return KP_OK;
  };
  float t1 = 0.f;
  rc = timed(1, &t1);
  int count = min_iters;
  std::vector<double> means;
  if (rc == KP_OK) {
    if (repeats == 1 && min_iters <= 1 && t1 >= min_ms) {
      means.push_back(t1);  // a launch that alone fills the time budget is its own measurement
      count = 1;
    } else {
      const double want = t1 > 0.f ? std::ceil(min_ms / t1) : static_cast<double>(max_iters);
      count = static_cast<int>(want < min_iters ? min_iters : (want > max_iters ? max_iters : want));
      for (int r = 0; r < repeats && rc == KP_OK; ++r) {
        float tn = 0.f;
        rc = timed(count, &tn);
        means.push_back(static_cast<double>(tn) / count);
      }
    }
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (rc != KP_OK) return rc;
  std::sort(means.begin(), means.end());
  *median_ms = means[means.size() / 2];
  *iters = count;
  return KP_OK;
}

int kp_bench(int id, int m, int k, int n, int batch, const void* A, int64_t lda, int64_t sA, const void* B,
             int64_t ldb, int64_t sB, void* C, int64_t ldc, int64_t sC, int warmup, int min_iters, int max_iters,
             double min_ms, double* mean_ms, int* iters, void* stream) {
  return kp_bench_sets(id, m, k, n, batch, 1, &A, lda, sA, &B, ldb, sB, &C, ldc, sC, warmup, min_iters, max_iters,
                       min_ms, 1, mean_ms, iters, stream);
}

int kp_ffma_peak(int packed, double* tflops, void* stream) {
  if (!tflops) return fail(KP_EINVAL, "null output pointer");
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  float* sink = nullptr;
  cudaError_t e = cudaMalloc(&sink, sizeof(float) * 1024 * 1024);
  if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int threads = 256, blocks = sms * 8, iters = 1 << 14;
  e = kp::ffma_peak_launch(sink, blocks, threads, 256, packed != 0, s);  // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0, s);
  if (e == cudaSuccess) e = kp::ffma_peak_launch(sink, blocks, threads, iters, packed != 0, s);
  cudaEventRecord(e1, s);
  if (e == cudaSuccess) e = cudaEventSynchronize(e1);
  float ms = 0.f;
  if (e == cudaSuccess) e = cudaEventElapsedTime(&ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(sink);
  if (e != cudaSuccess) return cuda_fail(e, "ffma peak probe");
  // 16 independent FFMA chains x 8 unrolled steps per iteration, 2 flops each.
  const double flops = 2.0 * 16.0 * 8.0 * iters * static_cast<double>(threads) * blocks;
  *tflops = flops / (ms * 1e-3) / 1e12;
  return KP_OK;
}

int kp_im2col3x3_nhwc(const float* x, int B, int H, int W, int C, float* out, int64_t ldo, void* stream) {
  if (!x || !out) return fail(KP_EINVAL, "null pointer");
  if (B < 1 || H < 1 || W < 1 || C < 1) return fail(KP_EINVAL, "bad activation shape");
  if (ldo < 9LL * C) return fail(KP_EINVAL, "ldo smaller than 9*C");
  cudaError_t e = kp::im2col3x3_nhwc_launch(x, B, H, W, C, out, ldo, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? KP_OK : cuda_fail(e, "im2col launch");
}

int kp_im2col3x3_nhwc_pad(const float* x, int B, int H, int W, int C, float* out, int kpad, void* stream) {
  if (!x || !out) return fail(KP_EINVAL, "null pointer");
  if (B < 1 || H < 1 || W < 1 || C < 1) return fail(KP_EINVAL, "bad activation shape");
  if (kpad < 9 * C || kpad % 4 != 0) return fail(KP_EINVAL, "kpad must be a multiple of 4 and >= 9*C");
  if ((reinterpret_cast<uintptr_t>(out) & 15) != 0) return fail(KP_EINVAL, "out must be 16-byte aligned");
  cudaError_t e = kp::im2col3x3_nhwc_pad_launch(x, B, H, W, C, out, kpad, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? KP_OK : cuda_fail(e, "im2col (padded) launch");
}

int kp_im2col3x3_nhwc_bf16(const float* x, int B, int H, int W, int C, void* out, int kpad, void* stream) {
  if (!x || !out) return fail(KP_EINVAL, "null pointer");
  if (B < 1 || H < 1 || W < 1 || C < 1) return fail(KP_EINVAL, "bad activation shape");
  if (kpad < 9 * C || kpad % 8 != 0) return fail(KP_EINVAL, "kpad must be a multiple of 8 and >= 9*C");
  cudaError_t e = kp::im2col3x3_nhwc_bf16_launch(x, B, H, W, C, out, kpad, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? KP_OK : cuda_fail(e, "im2col (bf16) launch");
}

int kp_cast_bf16(const float* x, int64_t n, void* out, void* stream) {
  if (!x || !out || n < 1) return fail(KP_EINVAL, "bad cast arguments");
  cudaError_t e = kp::cast_bf16_launch(x, n, out, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? KP_OK : cuda_fail(e, "bf16 cast launch (n % 8 == 0, 16-byte aligned)");
}

int kp_maxpool2x2_nhwc(const float* x, int B, int H, int W, int C, float* out, void* stream) {
  if (!x || !out) return fail(KP_EINVAL, "null pointer");
  if (B < 1 || H < 2 || W < 2 || C < 1) return fail(KP_EINVAL, "bad activation shape");
  cudaError_t e = kp::maxpool2_nhwc_launch(x, B, H, W, C, out, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? KP_OK : cuda_fail(e, "maxpool launch");
}

int kp_maxpool2x2_nhwc_bf16(const void* x, int B, int H, int W, int C, void* out, void* stream) {
  if (!x || !out) return fail(KP_EINVAL, "null pointer");
  if (B < 1 || H < 2 || W < 2 || C < 1 || C % 8 != 0) return fail(KP_EINVAL, "bad activation shape (C % 8 == 0)");
  if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(out)) & 15)
    return fail(KP_EINVAL, "x and out must be 16-byte aligned");
  cudaError_t e = kp::maxpool2_nhwc_bf16_launch(x, B, H, W, C, out, static_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? KP_OK : cuda_fail(e, "maxpool (bf16) launch");
}

int kp_dispatch_load(int n_nodes, const int32_t* feature, const double* threshold, const int32_t* left,
                     const int32_t* right, const int32_t* leaf_class, int n_classes,
                     const int32_t* class_to_variant) {
  if (n_nodes < 1 || !feature || !threshold || !left || !right || !leaf_class)
    return fail(KP_EINVAL, "empty tree or null array");
  if (n_classes < 1 || !class_to_variant) return fail(KP_EINVAL, "no classes");
  const int nv = kp_num_variants();
  for (int c = 0; c < n_classes; ++c)
    if (class_to_variant[c] < 0 || class_to_variant[c] >= nv)
      return fail(KP_ENOENT, "class %d maps to unknown variant %d", c, class_to_variant[c]);
  // Structural checks mirror import_model (codegen.py:116-145).
  std::vector<int> seen(n_nodes, 0);
  std::vector<int> stack{0};
  int visited = 0;
  while (!stack.empty()) {
    const int v = stack.back();
    stack.pop_back();
    if (seen[v]) return fail(KP_EINVAL, "node %d reachable twice; not a tree", v);
    seen[v] = 1;
    ++visited;
    if (leaf_class[v] >= 0) {
      if (leaf_class[v] >= n_classes) return fail(KP_EINVAL, "leaf class %d outside %d classes", leaf_class[v], n_classes);
      continue;
    }
    if (feature[v] < 0 || feature[v] >= 4) return fail(KP_EINVAL, "feature index %d out of range", feature[v]);
    if (std::isnan(threshold[v])) return fail(KP_EINVAL, "NaN threshold at node %d", v);
    for (int child : {left[v], right[v]}) {
      if (child < 0 || child >= n_nodes) return fail(KP_EINVAL, "child id %d out of range", child);
      stack.push_back(child);
    }
  }
  if (visited != n_nodes) return fail(KP_EINVAL, "unreachable nodes in tree");
  auto tp = std::make_shared<Table>();
  Table& t = *tp;
  t.feature.assign(feature, feature + n_nodes);
  t.threshold.assign(threshold, threshold + n_nodes);
  t.left.assign(left, left + n_nodes);
  t.right.assign(right, right + n_nodes);
  t.leaf_class.assign(leaf_class, leaf_class + n_nodes);
  t.class_to_variant.assign(class_to_variant, class_to_variant + n_classes);
  std::lock_guard<std::mutex> lock(g_tables_mu);
  g_tables.push_back(std::move(tp));
  return static_cast<int>(g_tables.size()) - 1;
}

int kp_dispatch_free(int handle) {
  std::lock_guard<std::mutex> lock(g_tables_mu);
  if (handle < 0 || handle >= static_cast<int>(g_tables.size()) || !g_tables[handle])
    return fail(KP_ENOENT, "unknown dispatch table %d", handle);
  g_tables[handle].reset();  // walks holding the table keep it alive until they return
  return KP_OK;
}

int kp_dispatch_class_feats(int handle, const double* feats4) {
  const std::shared_ptr<const Table> t = get_table(handle);
  if (!t) return fail(KP_ENOENT, "unknown dispatch table %d", handle);
  if (!feats4) return fail(KP_EINVAL, "null feature vector");
  return walk(*t, feats4);
}

int kp_dispatch_select_feats(int handle, const double* feats4) {
  const std::shared_ptr<const Table> t = get_table(handle);  // one lookup for class and variant
  if (!t) return fail(KP_ENOENT, "unknown dispatch table %d", handle);
  if (!feats4) return fail(KP_EINVAL, "null feature vector");
  const int cls = walk(*t, feats4);
  if (cls < 0) return cls;
  return t->class_to_variant[cls];
}

int kp_dispatch_select(int handle, int m, int k, int n, int batch) {
  if (m < 1 || k < 1 || n < 1 || batch < 1) return fail(KP_EINVAL, "dims must be >= 1");
  const double f[4] = {std::log2(static_cast<double>(m)), std::log2(static_cast<double>(k)),
                       std::log2(static_cast<double>(n)), std::log2(static_cast<double>(batch))};
  return kp_dispatch_select_feats(handle, f);
}

int kp_gemm_auto(int handle, int m, int k, int n, int batch, const void* A, int64_t lda, int64_t sA, const void* B,
                 int64_t ldb, int64_t sB, void* C, int64_t ldc, int64_t sC, void* stream, int* variant_out) {
  return kp_gemm_auto_ex(handle, m, k, n, batch, A, lda, sA, B, ldb, sB, C, ldc, sC, nullptr, 0, stream,
                         variant_out);
}

int kp_gemm_auto_ex(int handle, int m, int k, int n, int batch, const void* A, int64_t lda, int64_t sA,
                    const void* B, int64_t ldb, int64_t sB, void* C, int64_t ldc, int64_t sC, const float* bias,
                    int flags, void* stream, int* variant_out) {
  const int id = kp_dispatch_select(handle, m, k, n, batch);
  if (id < 0) return id;
  if (variant_out) *variant_out = id;
  return kp_gemm_ex(id, m, k, n, batch, A, lda, sA, B, ldb, sB, C, ldc, sC, bias, flags, stream);
}

}  // extern "C"
