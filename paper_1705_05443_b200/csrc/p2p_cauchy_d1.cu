// Explicit instantiation of the P2P launchers for SMASH_KERNEL_CAUCHY, 1-D points.
#include "p2p_kernels.cuh"

namespace smash {
namespace mv {
SMASH_P2P_INSTANTIATE(SMASH_KERNEL_CAUCHY, 1)
}  // namespace mv
}  // namespace smash
