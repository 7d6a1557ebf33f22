// Explicit instantiation of the P2P launchers for SMASH_KERNEL_EXP, 2-D points
// (split per kernel / dimension so the instantiations compile in parallel).
#include "p2p_kernels.cuh"

namespace smash {
namespace mv {
SMASH_P2P_INSTANTIATE(SMASH_KERNEL_EXP, 2)
}  // namespace mv
}  // namespace smash
