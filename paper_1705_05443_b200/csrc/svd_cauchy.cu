// K5 k_svd instantiations for one kernel kind (see svd_kernels.cuh); one unit per kind so they compile in parallel
#include "svd_kernels.cuh"

namespace smash {
namespace svdk {
template void svd_launch<SMASH_KERNEL_CAUCHY>(int, const SvdLaunch&);
}  // namespace svdk
}  // namespace smash
