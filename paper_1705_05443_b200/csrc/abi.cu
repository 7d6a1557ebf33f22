// extern "C" entry points (include/smash_b200.h).  Each wraps the C++
// implementation, converts exceptions into status codes and records the
// message for smash_last_error().
#include "smash_impl.cuh"

namespace smash {
static thread_local std::string g_last_error;
void set_last_error(const std::string& msg) { g_last_error = msg; }
void matvec_release_plan(const MatrixImpl* m);
}  // namespace smash

struct smash_tree_s {
  smash::TreeImpl* impl;
};
struct smash_matrix_s {
  smash::MatrixImpl* impl;
};
struct smash_ulv_s {
  smash::UlvImpl* impl;
};

namespace {

template <typename F>
int guarded(F f) {
  try {
    f();
    return SMASH_OK;
  } catch (const smash::Error& e) {
    smash::set_last_error(e.what());
    return e.code;
  } catch (const std::exception& e) {
    smash::set_last_error(e.what());
    return SMASH_ERR_CUDA;
  } catch (...) {
    smash::set_last_error("unknown error");
    return SMASH_ERR_CUDA;
  }
}

inline cudaStream_t st(void* s) { return reinterpret_cast<cudaStream_t>(s); }

}  // namespace

extern "C" {

int smash_abi_version(void) { return 1; }

const char* smash_last_error(void) { return smash::g_last_error.c_str(); }

int smash_tree_build(const double* X, int64_t nx, const double* Y, int64_t ny, int32_t dim,
                     int32_t nu0, int32_t mode, void* stream, smash_tree_t* out) {
  return guarded([&] {
    SMASH_CHECK(out != nullptr, SMASH_ERR_INVALID, "out is NULL");
    SMASH_CHECK(X != nullptr || nx == 0, SMASH_ERR_INVALID, "X is NULL");
    smash::TreeImpl* t = smash::tree_build(X, nx, Y, ny, dim, nu0, mode, st(stream));
    *out = new smash_tree_s{t};
  });
}

int smash_tree_sizes(smash_tree_t t, int64_t* n_nodes, int32_t* n_levels, int64_t* n_row,
                     int64_t* n_col, int32_t* dim, int32_t* shared_points) {
  return guarded([&] {
    SMASH_CHECK(t && t->impl, SMASH_ERR_INVALID, "null tree");
    if (n_nodes) *n_nodes = t->impl->n_nodes;
    if (n_levels) *n_levels = t->impl->n_levels;
    if (n_row) *n_row = t->impl->nx;
    if (n_col) *n_col = t->impl->ny;
    if (dim) *dim = t->impl->dim;
    if (shared_points) *shared_points = t->impl->shared ? 1 : 0;
  });
}

int smash_tree_export(smash_tree_t t, int64_t* level, int64_t* parent, int64_t* child_ptr,
                      int64_t* child_idx, double* lo, double* hi, int64_t* row_start,
                      int64_t* row_stop, int64_t* col_start, int64_t* col_stop,
                      int64_t* perm_row, int64_t* perm_col, double* points_row,
                      double* points_col, void* stream) {
  return guarded([&] {
    SMASH_CHECK(t && t->impl, SMASH_ERR_INVALID, "null tree");
    smash::tree_export(t->impl, level, parent, child_ptr, child_idx, lo, hi, row_start, row_stop,
                       col_start, col_stop, perm_row, perm_col, points_row, points_col,
                       st(stream));
    smash::sync(st(stream));
  });
}

int smash_tree_free(smash_tree_t t) {
  return guarded([&] {
    if (!t) return;
    delete t->impl;
    delete t;
  });
}

int smash_leaf_sets(smash_tree_t t, double tau, int32_t structure, void* stream, int64_t* n_L,
                    int64_t* n_Lm) {
  return guarded([&] {
    SMASH_CHECK(t && t->impl, SMASH_ERR_INVALID, "null tree");
    smash::PairLists* P = smash::get_pairs(t->impl, tau, structure, st(stream));
    smash::sync(st(stream));
    if (n_L) *n_L = P->nL;
    if (n_Lm) *n_Lm = P->nLm;
  });
}

int smash_leaf_sets_export(smash_tree_t t, double tau, int32_t structure, int64_t* L, int64_t* Lm,
                           void* stream) {
  return guarded([&] {
    SMASH_CHECK(t && t->impl, SMASH_ERR_INVALID, "null tree");
    smash::PairLists* P = smash::get_pairs(t->impl, tau, structure, st(stream));
    smash::pairs_export(t->impl, P, L, Lm, st(stream));
  });
}

int smash_nearfield_export(smash_tree_t t, double tau, int64_t* ptr, int64_t* idx, void* stream) {
  return guarded([&] {
    SMASH_CHECK(t && t->impl, SMASH_ERR_INVALID, "null tree");
    smash::NearSets* N = smash::get_near(t->impl, tau, st(stream));
    smash::near_export(t->impl, N, ptr, idx, st(stream));
  });
}

int smash_nearfield(smash_tree_t t, double tau, void* stream, int64_t* total) {
  return guarded([&] {
    SMASH_CHECK(t && t->impl, SMASH_ERR_INVALID, "null tree");
    smash::NearSets* N = smash::get_near(t->impl, tau, st(stream));
    smash::sync(st(stream));
    if (total) *total = N->total;
  });
}

int smash_matrix_build(smash_tree_t t, const smash_build_params* p, void* stream,
                       smash_matrix_t* out) {
  return guarded([&] {
    SMASH_CHECK(t && t->impl && p && out, SMASH_ERR_INVALID, "null argument");
    smash::MatrixImpl* m = smash::matrix_build(t->impl, *p, st(stream));
    *out = new smash_matrix_s{m};
  });
}

int smash_matrix_import(smash_tree_t t, const smash_build_params* p, int32_t nsides,
                        const int64_t* const* rank, const int64_t* const* perm_ptr,
                        const int64_t* const* perm, const int64_t* const* skel_ptr,
                        const int64_t* const* skel, const int64_t* const* g_ptr,
                        const double* const* G, void* stream, smash_matrix_t* out) {
  return guarded([&] {
    SMASH_CHECK(t && t->impl && p && out && rank && perm_ptr && perm && skel_ptr && skel && g_ptr &&
                G, SMASH_ERR_INVALID, "null argument");
    SMASH_CHECK(nsides == 1 || nsides == 2, SMASH_ERR_INVALID, "nsides must be 1 or 2");
    smash::ImportSide sd[2];
    for (int k = 0; k < nsides; ++k) {
      SMASH_CHECK(rank[k] && perm_ptr[k] && skel_ptr[k] && g_ptr[k], SMASH_ERR_INVALID,
                  "null factor array");
      sd[k] = smash::ImportSide{rank[k], perm_ptr[k], perm[k], skel_ptr[k], skel[k], g_ptr[k], G[k]};
    }
    smash::MatrixImpl* m = smash::matrix_import(t->impl, *p, sd, nsides, st(stream));
    *out = new smash_matrix_s{m};
  });
}

int smash_matrix_build_local(smash_tree_t t, const smash_build_params* p, int32_t rank,
                             int32_t world, int32_t cut_level, void* stream, smash_matrix_t* out) {
  return guarded([&] {
    SMASH_CHECK(t && t->impl && p && out, SMASH_ERR_INVALID, "null argument");
    smash::MatrixImpl* m = smash::matrix_build_local(t->impl, *p, rank, world, cut_level, nullptr, 1,
                                                     st(stream));
    *out = new smash_matrix_s{m};
  });
}

int smash_matrix_build_sharded(smash_tree_t t, const smash_build_params* p, int32_t rank,
                               int32_t world, smash_exchange_fn fn, void* ctx, void* stream,
                               smash_matrix_t* out) {
  return guarded([&] {
    SMASH_CHECK(t && t->impl && p && out, SMASH_ERR_INVALID, "null argument");
    smash::MatrixImpl* m = smash::matrix_build_sharded(t->impl, *p, rank, world, fn, ctx, st(stream));
    *out = new smash_matrix_s{m};
  });
}

int smash_matrix_build_local_w(smash_tree_t t, const smash_build_params* p, int32_t rank,
                               int32_t world, int32_t cut_level, const double* cut_weight,
                               int32_t replicate, void* stream, smash_matrix_t* out) {
  return guarded([&] {
    SMASH_CHECK(t && t->impl && p && out, SMASH_ERR_INVALID, "null argument");
    smash::MatrixImpl* m = smash::matrix_build_local(t->impl, *p, rank, world, cut_level, cut_weight,
                                                     replicate, st(stream));
    *out = new smash_matrix_s{m};
  });
}

int smash_matrix_shard_cut(smash_tree_t t, int32_t world, int32_t cut_level, int32_t* cut) {
  return guarded([&] {
    SMASH_CHECK(t && t->impl && cut && world >= 1, SMASH_ERR_INVALID, "bad argument");
    const smash::TreeImpl* ti = t->impl;
    const int L = ti->n_levels;
    int c = L;
    for (int l = 2; l <= L; ++l)
      if (ti->level_end(l) - ti->level_begin(l) >= 8 * world) { c = l; break; }
    if (cut_level >= 2 && cut_level <= L) c = cut_level;
    *cut = c;
  });
}

int smash_matrix_shard_owner(smash_matrix_t m, int64_t* owner_post) {
  return guarded([&] {
    SMASH_CHECK(m && m->impl && owner_post, SMASH_ERR_INVALID, "null argument");
    const smash::MatrixImpl* mi = m->impl;
    SMASH_CHECK(!mi->shard_owner.empty(), SMASH_ERR_INVALID, "matrix was not built sharded");
    const smash::TreeImpl* ti = mi->tree;
    std::vector<int> post(ti->n_nodes);
    smash::d2h(post.data(), ti->post.p, ti->n_nodes, ti->stream);
    smash::sync(ti->stream);
    for (int v = 0; v < ti->n_nodes; ++v) owner_post[post[v]] = mi->shard_owner[v];
  });
}

int smash_matvec_coeff_layout(smash_matrix_t m, int64_t* row_off_post, int64_t* up_pos,
                              int64_t* half_rows, void* stream) {
  return guarded([&] {
    SMASH_CHECK(m && m->impl && row_off_post && half_rows, SMASH_ERR_INVALID, "null argument");
    smash::matvec_coeff_layout(m->impl, row_off_post, up_pos, half_rows, st(stream));
  });
}

int smash_matrix_exchange_buffers(smash_matrix_t m, int64_t capacity, int64_t* n, void** ptrs,
                                  int64_t* counts, int32_t* dtypes) {
  return guarded([&] {
    SMASH_CHECK(m && m->impl && n, SMASH_ERR_INVALID, "null argument");
    std::vector<smash::ExchangeBuf> b;
    smash::matrix_exchange_buffers(m->impl, b);
    *n = (int64_t)b.size();
    SMASH_CHECK(capacity >= (int64_t)b.size(), SMASH_ERR_INVALID, "exchange list capacity too small");
    for (size_t i = 0; i < b.size(); ++i) {
      ptrs[i] = b[i].ptr;
      counts[i] = b[i].count;
      dtypes[i] = b[i].dtype;
    }
  });
}

int smash_matrix_build_finish(smash_matrix_t m, void* stream) {
  return guarded([&] {
    SMASH_CHECK(m && m->impl, SMASH_ERR_INVALID, "null matrix");
    smash::matrix_build_finish(m->impl, st(stream));
  });
}

int smash_matrix_sizes(smash_matrix_t m, int32_t side, int64_t* has_total, int64_t* ibar_total,
                       int64_t* skel_total, int64_t* g_total) {
  return guarded([&] {
    SMASH_CHECK(m && m->impl, SMASH_ERR_INVALID, "null matrix");
    SMASH_CHECK(side == 0 || side == 1, SMASH_ERR_INVALID, "side must be 0 or 1");
    const smash::SideFactors& F = side == 0 ? m->impl->rowf : *m->impl->colf;
    if (has_total) *has_total = m->impl->tree->n_nodes - 1;
    if (ibar_total) {  // exact sum of |ibar| (the device layout may hold capacity gaps)
      int n = m->impl->tree->n_nodes;
      std::vector<int> nib(n);
      smash::d2h(nib.data(), F.nib.p, n, 0);
      smash::sync(0);
      int64_t t = 0;
      for (int v = 1; v < n; ++v) t += nib[v];
      *ibar_total = t;
    }
    if (skel_total) *skel_total = F.skel_total;
    if (g_total) {
      // exact G count = sum (nib - k) * k ; computed at export; report capacity-free value
      int n = m->impl->tree->n_nodes;
      std::vector<int> nib(n), rk(n);
      smash::d2h(nib.data(), F.nib.p, n, 0);
      smash::d2h(rk.data(), F.rank.p, n, 0);
      smash::sync(0);
      int64_t g = 0;
      for (int v = 1; v < n; ++v) g += (int64_t)(nib[v] - rk[v]) * rk[v];
      *g_total = g;
    }
  });
}

int smash_matrix_export(smash_matrix_t m, int32_t side, int64_t* has, int64_t* rank,
                        int64_t* perm_ptr, int64_t* perm, int64_t* skel_ptr, int64_t* skel,
                        int64_t* g_ptr, double* G, void* stream) {
  return guarded([&] {
    SMASH_CHECK(m && m->impl, SMASH_ERR_INVALID, "null matrix");
    SMASH_CHECK(side == 0 || side == 1, SMASH_ERR_INVALID, "side must be 0 or 1");
    smash::matrix_export(m->impl, side, has, rank, perm_ptr, perm, skel_ptr, skel, g_ptr, G,
                         st(stream));
  });
}

int smash_matrix_stats(smash_matrix_t m, int64_t* swaps_row, int64_t* swaps_col) {
  return guarded([&] {
    SMASH_CHECK(m && m->impl, SMASH_ERR_INVALID, "null matrix");
    if (swaps_row) *swaps_row = m->impl->rowf.swaps;
    if (swaps_col) *swaps_col = m->impl->colf->swaps;
  });
}

int smash_ulv_factor(smash_matrix_t m, void* stream, smash_ulv_t* out) {
  return guarded([&] {
    SMASH_CHECK(m && m->impl && out, SMASH_ERR_INVALID, "null argument");
    smash::UlvImpl* f = smash::ulv_factor(m->impl, st(stream));
    *out = new smash_ulv_s{f};
  });
}

int smash_ulv_solve(smash_ulv_t f, const double* b, double* x, int64_t nrhs, void* stream) {
  return guarded([&] {
    SMASH_CHECK(f && f->impl, SMASH_ERR_INVALID, "null factorization");
    SMASH_CHECK(b && x, SMASH_ERR_INVALID, "null vector");
    smash::ulv_solve(f->impl, b, x, nrhs, st(stream));
  });
}

int smash_ulv_free(smash_ulv_t f) {
  return guarded([&] {
    if (f) {
      smash::ulv_free(f->impl);
      delete f;
    }
  });
}

int smash_matvec(smash_matrix_t m, const double* q, double* z, int64_t nrhs, void* stream) {
  return guarded([&] {
    SMASH_CHECK(m && m->impl, SMASH_ERR_INVALID, "null matrix");
    SMASH_CHECK(q && z, SMASH_ERR_INVALID, "null vector");
    smash::matvec(m->impl, q, z, nrhs, st(stream));
  });
}

int smash_matvec_levelwise(smash_matrix_t m, const double* q, double* z, int64_t nrhs,
                           void* stream) {
  return guarded([&] {
    SMASH_CHECK(m && m->impl, SMASH_ERR_INVALID, "null matrix");
    SMASH_CHECK(q && z, SMASH_ERR_INVALID, "null vector");
    smash::matvec_levelwise(m->impl, q, z, nrhs, st(stream));
  });
}

int smash_sum_matvec(int32_t n_terms, const smash_matrix_t* bases, const double* dl,
                     const double* dr, const double* q, double* z, int64_t nrhs,
                     int32_t levelwise, void* stream) {
  return guarded([&] {
    SMASH_CHECK(n_terms >= 1 && bases, SMASH_ERR_INVALID, "no terms");
    SMASH_CHECK(dl && dr && q && z, SMASH_ERR_INVALID, "null vector");
    std::vector<smash::MatrixImpl*> b(n_terms);
    for (int t = 0; t < n_terms; ++t) {
      SMASH_CHECK(bases[t] && bases[t]->impl, SMASH_ERR_INVALID, "null matrix");
      b[t] = bases[t]->impl;
    }
    smash::sum_matvec(n_terms, b.data(), dl, dr, q, z, nrhs, levelwise, st(stream));
  });
}

int smash_matvec_set_partition(smash_matrix_t m, const int64_t* own_nodes, int64_t n_own,
                               const int64_t* top_nodes, int64_t n_top, void* stream) {
  return guarded([&] {
    SMASH_CHECK(m && m->impl, SMASH_ERR_INVALID, "null matrix");
    smash::matvec_set_partition(m->impl, own_nodes, n_own, top_nodes, n_top, st(stream));
  });
}

int smash_matvec_stage(smash_matrix_t m, int32_t stage, const double* q, double* z, int64_t nrhs,
                       void* stream) {
  return guarded([&] {
    SMASH_CHECK(m && m->impl, SMASH_ERR_INVALID, "null matrix");
    smash::matvec_stage(m->impl, stage, q, z, nrhs, st(stream));
  });
}

int smash_matvec_coeffs(smash_matrix_t m, double** qhat, int64_t* rows) {
  return guarded([&] {
    SMASH_CHECK(m && m->impl && qhat && rows, SMASH_ERR_INVALID, "null argument");
    smash::matvec_coeffs(m->impl, qhat, rows);
  });
}

int smash_matvec_profile(smash_matrix_t m, int32_t enable, double* phase_ms, int64_t* launches) {
  return guarded([&] {
    SMASH_CHECK(m && m->impl, SMASH_ERR_INVALID, "null matrix");
    smash::matvec_profile(m->impl, enable, phase_ms, launches);
  });
}

int smash_matrix_free(smash_matrix_t m) {
  return guarded([&] {
    if (!m) return;
    smash::matvec_release_plan(m->impl);
    delete m->impl;
    delete m;
  });
}

int smash_kernel_block(int32_t kernel, double dx, int32_t dim, const double* X, int64_t nx,
                       const double* Y, int64_t ny, double* out, void* stream) {
  return guarded([&] {
    smash::kernel_block(kernel, dx, dim, X, nx, Y, ny, out, st(stream));
    smash::sync(st(stream));
  });
}

int smash_dense_matvec(int32_t kernel, double dx, int32_t dim, const double* X, int64_t nx,
                       const double* Y, int64_t ny, const double* q, int64_t nrhs, double* z,
                       void* stream) {
  return guarded([&] {
    SMASH_CHECK(dim >= 1 && dim <= 3, SMASH_ERR_INVALID, "dim must be 1, 2 or 3");
    smash::dense_matvec(kernel, dx, dim, X, nx, Y, ny, q, nrhs, z, st(stream));
  });
}

int smash_interp_basis(int32_t dim, const double* lo, const double* hi, const double* pts,
                       int64_t n, int32_t r, double* out, void* stream) {
  return guarded([&] {
    SMASH_CHECK(lo && hi, SMASH_ERR_INVALID, "null box");
    smash::interp_basis_single(dim, lo, hi, pts, n, r, out, st(stream));
  });
}

int smash_compr(const double* C, int64_t nrows, int64_t ncols, double s, double rtol,
                int64_t* perm, double* G, int64_t* rank, int64_t* swaps, void* stream) {
  return guarded([&] {
    SMASH_CHECK(rank && swaps, SMASH_ERR_INVALID, "null output");
    smash::compr_single(C, nrows, ncols, s, rtol, perm, G, rank, swaps, st(stream));
  });
}

}  // extern "C"
