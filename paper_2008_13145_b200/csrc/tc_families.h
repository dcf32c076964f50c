// Internal interface to the tcgen05 tensor-core families (TF32 = F2, BF16 = F3).
#pragma once

#include <cuda_runtime.h>

#include "common.cuh"

namespace kp {

int tc_family_size(int family);
KernelChoice tc_family_choice(int family, int index);
// KP_OK when (family, index) can run problem p, else KP_EINVAL (reason in tc_last_reason()).
int tc_check(int family, int index, const GemmArgs& p);
const char* tc_last_reason();
cudaError_t tc_launch(int family, int index, const GemmArgs& p, cudaStream_t s);
// Tile facts for the k-slice planner (capi.cu): BN of a config, BK of a family (BM = 128).
int tc_tile_n(int family, int index);
int tc_tile_k(int family);
// cudaOccupancyMaxActiveClusters of a (1, 1, slices) cluster launch (< 0: error).
int tc_cluster_fit(int family, int index, int slices);

}  // namespace kp
