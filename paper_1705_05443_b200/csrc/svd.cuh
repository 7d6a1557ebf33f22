// K5: HSS nearfield block-row assembly + batched truncated SVD (see svd.cu).
#pragma once

#include "smash_impl.cuh"

namespace smash {

struct SvdWorkspace {
  DBuf<int> keep;       // per BFS node: number of kept singular vectors
  DBuf<int64_t> sv_off; // per BFS node: offset of S (nib x keep, row-major)
  DBuf<double> sv;      // kept left singular vectors
  DBuf<double> gws;     // per-node workspaces of the chunked (split) launches: one fixed-size block
};

// For every node of level l on `side`, assemble the nearfield block row
// (hss.py:281-285 / 292-296), compute its truncated SVD (lowrank.py:265-276)
// and leave S in ws.  Returns the level's maximum keep count.
int hss_level_svd(MatrixImpl* M, int side, int level, NearSets* near, int nmax, SvdWorkspace& ws,
                  cudaStream_t s, int sub_lb = -1, int sub_le = -1);

}  // namespace smash
