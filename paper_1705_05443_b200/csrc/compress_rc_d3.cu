// Register-column compression kernels for 3-D points (explicit instantiation;
// one translation unit per dimension for parallel compilation).
#include "compress_rc.cuh"

namespace smash {
template void launch_compress_rc_dim<3>(const CompressArgs&, const RcVariant&, int, size_t, cudaStream_t);
}  // namespace smash
