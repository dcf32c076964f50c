// Instantiates the 64 (R, A, C) F1 kernels of ONE work-group pair.  The Makefile
// compiles this file ten times with -DKP_WG_INDEX=0..9 (DEFAULT_WG_PAIRS order,
// dataset.py:19-31) so the 640 kernels build in parallel.
#include "families.h"
#include "f1_simt.cuh"

#ifndef KP_WG_INDEX
#error "compile with -DKP_WG_INDEX=<0..9>"
#endif

#define KP_CAT2(a, b) a##b
#define KP_CAT(a, b) KP_CAT2(a, b)

namespace kp {
namespace {

constexpr int WGR = kWgPairs[KP_WG_INDEX][0];
constexpr int WGC = kWgPairs[KP_WG_INDEX][1];

template <int RI, int AI, int CI>
void put(F1Entry* table) {
  constexpr int R = 1 << RI, A = 1 << AI, C = 1 << CI;
  using Cfg = F1Cfg<R, A, C, WGR, WGC>;
  const int cfg = ((RI * 4 + AI) * 4 + CI) * kNumWgPairs + KP_WG_INDEX;
  table[cfg] = F1Entry{&f1_launch<R, A, C, WGR, WGC>, Cfg::BM, Cfg::BN, Cfg::BK, Cfg::MIN_BLOCKS, Cfg::TMA_OK ? 1 : 0,
                       &f1_cluster_fit<R, A, C, WGR, WGC>};
}

template <int RI, int AI>
void put_row(F1Entry* t) {
  put<RI, AI, 0>(t);
  put<RI, AI, 1>(t);
  put<RI, AI, 2>(t);
  put<RI, AI, 3>(t);
}

template <int RI>
void put_block(F1Entry* t) {
  put_row<RI, 0>(t);
  put_row<RI, 1>(t);
  put_row<RI, 2>(t);
  put_row<RI, 3>(t);
}

}  // namespace

void KP_CAT(f1_fill_wg, KP_WG_INDEX)(F1Entry* table) {
  put_block<0>(table);
  put_block<1>(table);
  put_block<2>(table);
  put_block<3>(table);
}

}  // namespace kp
