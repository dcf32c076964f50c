// Placeholder until the tcgen05 families land: both tensor-core families are empty.
#include "tc_families.h"

namespace kp {
int tc_family_size(int) { return 0; }
KernelChoice tc_family_choice(int, int) { return KernelChoice{0, 0, 0, 0, 0}; }
int tc_check(int, int, const GemmArgs&) { return KP_EINVAL; }
const char* tc_last_reason() { return "tensor-core families not built"; }
cudaError_t tc_launch(int, int, const GemmArgs&, cudaStream_t) { return cudaErrorInvalidValue; }
}  // namespace kp
