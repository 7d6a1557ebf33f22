// K5: HSS nearfield SVD (placeholder until the batched Jacobi kernel lands).
#include "svd.cuh"

namespace smash {

int hss_level_svd(MatrixImpl* M, int side, int level, NearSets* near, int nmax, SvdWorkspace& ws,
                  cudaStream_t s) {
  (void)M; (void)side; (void)level; (void)near; (void)nmax; (void)ws; (void)s;
  throw Error(SMASH_ERR_INVALID, "HSS construction is not available in this build yet");
}

}  // namespace smash
