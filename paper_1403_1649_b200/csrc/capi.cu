// capi.cu — the extern "C" boundary (include/aggmg_b200.h).  Host arrays are
// converted at the boundary (int64 <-> int32 on the device), every computation runs
// in the sm_100a kernels of this library, errors become status codes + message.
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include <thread>
#include <type_traits>

#include "../../include/aggmg_b200.h"
#include "chunked.cuh"
#include "dist_solve.cuh"
#include "mm.cuh"
#include "krylov.cuh"
#include "vecops.cuh"

#include "generators_host.hpp"

namespace aggmg_b200 {
void init_device(int device);
}  // namespace aggmg_b200

using namespace aggmg_b200;

struct aggmg_hierarchy {
  std::unique_ptr<DevHierarchy> h;
};
struct aggmg_galerkin_cache {
  GalerkinDev g;
  AggDev agg;
};
struct aggmg_dmatrix {
  DevCsrPtr A;
};
struct aggmg_comm {
  std::unique_ptr<Comm> comm;
};
struct aggmg_dist_matrix {
  Comm* comm = nullptr;
  DistCsrPtr A;
};
struct aggmg_dist_hierarchy {
  Comm* comm = nullptr;
  DistCsrPtr A0;
  std::unique_ptr<DistHierarchy> h;
};

namespace {

thread_local std::string g_last_error;

template <class F>
int guarded(F&& f) {
  try {
    f();
    g_last_error.clear();
    return AGGMG_OK;
  } catch (const Error& e) {
    g_last_error = e.what();
    return AGGMG_ERR;
  } catch (const CudaError& e) {
    g_last_error = e.what();
    return AGGMG_ERR_CUDA;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return AGGMG_ERR;
  }
}

DevCsrPtr up(const aggmg_csr* m, bool validate = false) {
  require(m != nullptr, "null matrix");
  return upload_csr(m->n_rows, m->n_cols, m->row_offsets, m->col_indices, m->values, validate);
}

// pattern-only upload (values default to 1)
DevCsrPtr up_pattern(const aggmg_csr* m) {
  std::vector<double> ones;
  const double* vals = m->values;
  if (!vals) {
    ones.assign(static_cast<size_t>(m->row_offsets[m->n_rows]), 1.0);
    vals = ones.data();
  }
  auto A = upload_csr(m->n_rows, m->n_cols, m->row_offsets, m->col_indices, vals, false);
  sync();
  return A;
}

void alloc_csr(aggmg_csr* out, int64_t rows, int64_t cols, int64_t nnz) {
  out->n_rows = rows;
  out->n_cols = cols;
  out->nnz = nnz;
  out->row_offsets = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (rows + 1)));
  out->col_indices = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (nnz > 0 ? nnz : 1)));
  out->values = static_cast<double*>(std::malloc(sizeof(double) * (nnz > 0 ? nnz : 1)));
}

void down(const DevCsr& A, aggmg_csr* out, bool unit_values = false) {
  alloc_csr(out, A.n_rows, A.n_cols, A.nnz);
  download_csr(A, out->row_offsets, out->col_indices, unit_values ? nullptr : out->values);
  if (unit_values)
    for (int64_t k = 0; k < A.nnz; ++k) out->values[k] = 1.0;
}

template <class T>
DevBuf<T> up_vec(const T* h, int64_t n) {
  DevBuf<T> d(n);
  if constexpr (std::is_same_v<T, double>) {
    if (n > 0) host_to_device_values(d.get(), h, static_cast<size_t>(n));
  } else {
    d.upload(h, n);
  }
  return d;
}

DevBuf<idx> up_index(const int64_t* h, int64_t n) {
  std::vector<idx> v(h, h + n);
  DevBuf<idx> d(n);
  d.upload(v.data(), n);
  sync();
  return d;
}

void down_index(const DevBuf<idx>& d, int64_t n, int64_t* out) {
  std::vector<idx> v(n);
  d.download(v.data(), n);
  sync();
  for (int64_t i = 0; i < n; ++i) out[i] = v[i];
}

AggDev agg_from_host(int64_t n, int64_t nc, const int64_t* assignment) {
  AggDev agg;
  agg.n_fine = n;
  agg.n_agg = nc;
  for (int64_t i = 0; i < n; ++i)
    require(assignment[i] >= 0 && assignment[i] < nc, "aggregation: assignment out of range");
  agg.assignment = up_index(assignment, n);
  build_groups(agg);
  return agg;
}

// P as CSR from (assignment, pval): one entry per row with b_i != 0 (transfer.cpp:35-46)
void p_to_host(int64_t n, int64_t nc, const DevBuf<idx>& assignment, const DevBuf<double>& pval,
               aggmg_csr* P) {
  std::vector<idx> a(n);
  std::vector<double> pv(n);
  assignment.download(a.data(), n);
  pval.download(pv.data(), n);
  sync();
  int64_t nnz = 0;
  for (int64_t i = 0; i < n; ++i) nnz += (pv[i] != 0.0) ? 1 : 0;
  alloc_csr(P, n, nc, nnz);
  P->row_offsets[0] = 0;
  int64_t p = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (pv[i] != 0.0) {
      P->col_indices[p] = a[i];
      P->values[p] = pv[i];
      ++p;
    }
    P->row_offsets[i + 1] = p;
  }
}

SetupCfg to_cfg(const aggmg_setup_config* c) {
  SetupCfg s;
  if (!c) return s;
  s.alpha = c->alpha;
  s.coarse_size_max = c->coarse_size_max;
  s.max_levels = c->max_levels;
  s.smoother = c->smoother;
  s.arnoldi_m = c->arnoldi_m;
  s.reuse_caches = c->reuse_caches;
  s.seed = c->seed;
  return s;
}
CycleCfg to_cfg(const aggmg_cycle_config* c) {
  CycleCfg s;
  if (!c) return s;
  s.kind = c->kind;
  s.k_levels = c->k_levels;
  s.t = c->t;
  s.inner = c->inner;
  return s;
}
SolverCfg to_cfg(const aggmg_solver_config* c) {
  SolverCfg s;
  if (!c) return s;
  s.method = c->method;
  s.tol = c->tol;
  s.max_iters = c->max_iters;
  s.restart = c->restart;
  return s;
}

void fill_report(const SolveOut& o, aggmg_solve_report* r) {
  if (!r) return;
  r->converged = o.converged ? 1 : 0;
  r->iterations = o.iterations;
  r->history_length = static_cast<int64_t>(o.history.size());
  if (r->history) {
    const int64_t m = std::min<int64_t>(r->history_capacity, r->history_length);
    for (int64_t i = 0; i < m; ++i) r->history[i] = o.history[i];
  }
  r->solve_seconds = o.solve_seconds;
  std::snprintf(r->note, sizeof(r->note), "%s", o.note.c_str());
}

SolveOut run_solver(const DevCsr& A, const double* b, double* x, DevHierarchy* h,
                    const aggmg_cycle_config* cycle, const aggmg_solver_config* cfg) {
  Precond M;
  M.h = h;
  M.cfg = to_cfg(cycle);
  const SolverCfg s = to_cfg(cfg);
  return s.method == AGGMG_SOLVER_PCG ? pcg(A, b, x, M, s) : fgmres(A, b, x, M, s);
}

const DevLevel& level(const aggmg_hierarchy* h, int64_t k) {
  require(h && h->h, "null hierarchy");
  require(k >= 0 && k < h->h->n_levels(), "hierarchy: level index out of range");
  return h->h->levels[k];
}

}  // namespace

namespace {
aggmg_dist_matrix* wrap_rows(aggmg_comm* c, int64_t n_global, int64_t row0, DevCsrPtr rows) {
  Comm& comm = *c->comm;
  const std::vector<int64_t> counts = comm.allgather_host({rows->n_rows});
  const std::vector<int64_t> starts = comm.allgather_host({row0});
  const Partition part = Partition::from_counts(counts);
  for (int r = 0; r < comm.size(); ++r)
    require(starts[r] == part.begin(r), "dist matrix: rank row ranges must be contiguous, in rank order");
  require(part.n() == n_global, "dist matrix: the ranks' rows do not cover the matrix");
  auto m = std::make_unique<aggmg_dist_matrix>();
  m->comm = &comm;
  m->A = make_dist(comm, part, part, *rows);
  return m.release();
}
int64_t dist_rows_begin(int64_t n, const Comm& comm) {
  return Partition::even(n, comm.size()).begin(comm.rank());
}
int64_t dist_rows_count(int64_t n, const Comm& comm) {
  return Partition::even(n, comm.size()).count(comm.rank());
}
// generic gather of `count` POD values per rank onto rank 0 (rank order)
template <class T>
void gather_pod(Comm& comm, const T* local, int64_t count, DevBuf<T>& all) {
  const std::vector<int64_t> cnt = comm.allgather_host({count});
  std::vector<CommMsg> s, r;
  s.push_back({0, const_cast<T*>(local), sizeof(T) * count});
  if (comm.rank() == 0) {
    int64_t tot = 0;
    for (int64_t v : cnt) tot += v;
    all.resize(tot);
    int64_t off = 0;
    for (int q = 0; q < comm.size(); ++q) {
      r.push_back({q, all.get() + off, sizeof(T) * cnt[q]});
      off += cnt[q];
    }
  }
  comm.exchange(s, r);
}
DistHierarchy& dh(aggmg_dist_hierarchy* h) {
  require(h && h->h, "null distributed hierarchy");
  return *h->h;
}
}  // namespace

extern "C" {

const char* aggmg_version(void) { return "0.1.0"; }
const char* aggmg_last_error(void) { return g_last_error.c_str(); }
int aggmg_init(int device) { return guarded([&] { init_device(device); }); }
int aggmg_synchronize(void) { return guarded([&] { sync(); }); }
void aggmg_set_num_threads(int) {}
void aggmg_set_exact_reductions(int on) { set_exact_reductions(on != 0); }
int aggmg_exact_reductions(void) { return exact_reductions() ? 1 : 0; }
void aggmg_set_value_dictionary(int on) { value_dictionary_switch().store(on ? 1 : 0); }
void aggmg_set_row_patterns(int on) { row_pattern_switch().store(on ? 1 : 0); }
int aggmg_num_threads(void) {
  int n = 0;
  guarded([&] { n = sm_count(); });
  return n;
}
int64_t aggmg_kernel_launches(void) { return launch_count(); }

void aggmg_setup_config_default(aggmg_setup_config* c) {
  c->alpha = 0.25;
  c->coarse_size_max = 600;
  c->max_levels = 25;
  c->smoother = AGGMG_SMOOTHER_DAMPED_JACOBI;
  c->arnoldi_m = 5;
  c->reuse_caches = 0;
  c->seed = 42;
}
void aggmg_cycle_config_default(aggmg_cycle_config* c) {
  c->kind = AGGMG_CYCLE_HYBRID;
  c->k_levels = 2;
  c->t = 0.25;
  c->inner = AGGMG_INNER_GMRES;
}
void aggmg_solver_config_default(aggmg_solver_config* c) {
  c->method = AGGMG_SOLVER_FGMRES;
  c->tol = 1e-6;
  c->max_iters = 200;
  c->restart = 30;
}
void aggmg_csr_free(aggmg_csr* m) {
  if (!m) return;
  std::free(m->row_offsets);
  std::free(m->col_indices);
  std::free(m->values);
  m->row_offsets = nullptr;
  m->col_indices = nullptr;
  m->values = nullptr;
}

// ---- L1 -----------------------------------------------------------------------

int aggmg_spmv(const aggmg_csr* A, const double* x, double* y) {
  return guarded([&] {
    auto dA = up(A);
    auto dx = up_vec(x, A->n_cols);
    DevBuf<double> dy(A->n_rows);
    spmv(*dA, dx.get(), dy.get());
    dy.download(y, A->n_rows);
    sync();
  });
}

int aggmg_transpose(const aggmg_csr* A, aggmg_csr* T) {
  return guarded([&] {
    auto dA = up(A);
    auto dT = transpose(*dA);
    down(*dT, T);
  });
}

int aggmg_dot(int64_t n, const double* a, const double* b, double* out) {
  return guarded([&] {
    auto da = up_vec(a, n), db = up_vec(b, n);
    *out = dot_host(da.get(), db.get(), n, 1);
  });
}
int aggmg_norm2(int64_t n, const double* a, double* out) {
  return guarded([&] {
    auto da = up_vec(a, n);
    *out = std::sqrt(dot_host(da.get(), da.get(), n, 1));
  });
}
int aggmg_axpy(int64_t n, double a, const double* x, double* y) {
  return guarded([&] {
    auto dx = up_vec(x, n), dy = up_vec(y, n);
    vec_axpy(n, a, dx.get(), dy.get());
    dy.download(y, n);
    sync();
  });
}
int aggmg_scale(int64_t n, double a, double* x) {
  return guarded([&] {
    auto dx = up_vec(x, n);
    vec_scale(n, a, dx.get());
    dx.download(x, n);
    sync();
  });
}

// ---- L2 --------------------------------------------------------------------------

int aggmg_classic_strength(const aggmg_csr* A, double alpha, int policy, aggmg_csr* C) {
  return guarded([&] {
    auto dA = up(A);
    auto dC = classic_strength(*dA, alpha, policy);
    down(*dC, C, true);
  });
}

int aggmg_influence_counts(const aggmg_csr* C, int64_t* counts) {
  return guarded([&] {
    auto dC = up_pattern(C);
    DevBuf<idx> infl;
    DevCsrPtr S;
    influence_and_symmetrize(*dC, infl, S);
    down_index(infl, C->n_cols, counts);
  });
}

int aggmg_symmetrize_pattern(const aggmg_csr* C, aggmg_csr* S) {
  return guarded([&] {
    auto dC = up_pattern(C);
    DevBuf<idx> infl;
    DevCsrPtr dS;
    influence_and_symmetrize(*dC, infl, dS);
    down(*dS, S, true);
  });
}

int aggmg_mis2(const aggmg_csr* S, const int64_t* influence, uint64_t seed, int8_t* state,
               int64_t* n_roots, int32_t* sweeps) {
  return guarded([&] {
    auto dS = up_pattern(S);
    auto infl = up_index(influence, S->n_rows);
    Mis2Dev m = mis2(*dS, infl.get(), seed);
    m.state.download(state, S->n_rows);
    sync();
    int64_t roots = 0;
    for (int64_t i = 0; i < S->n_rows; ++i) roots += state[i] == 1 ? 1 : 0;
    if (n_roots) *n_roots = roots;
    if (sweeps) *sweeps = m.sweeps;
  });
}

int aggmg_aggregate(const aggmg_csr* S, const aggmg_csr* A, const int8_t* state,
                    int64_t* assignment, int64_t* representatives, int64_t* n_aggregates) {
  return guarded([&] {
    auto dS = up_pattern(S);
    auto dA = up(A);
    auto st = up_vec(state, S->n_rows);
    AggDev agg = aggregate(*dS, *dA, st.get());
    down_index(agg.assignment, agg.n_fine, assignment);
    if (representatives) down_index(agg.representatives, agg.n_agg, representatives);
    *n_aggregates = agg.n_agg;
  });
}

int aggmg_build_transfer(int64_t n, int64_t nc, const int64_t* assignment, const double* fine_b,
                         aggmg_csr* P, aggmg_csr* R, double* coarse_b) {
  return guarded([&] {
    AggDev agg = agg_from_host(n, nc, assignment);
    auto db = up_vec(fine_b, n);
    TransferDev t = build_transfer(agg, db.get());
    if (P) p_to_host(n, nc, agg.assignment, t.pval, P);
    if (R) down(*t.R, R);
    if (coarse_b) {
      t.coarse_b.download(coarse_b, nc);
      sync();
    }
  });
}

int aggmg_galerkin_direct(const aggmg_csr* R, const aggmg_csr* A, const aggmg_csr* P,
                          aggmg_csr* Ac) {
  return guarded([&] {
    require(R->n_cols == A->n_rows && A->n_cols == P->n_rows && R->n_rows == P->n_cols,
            "galerkin_direct: operand shapes disagree");
    require(A->n_rows == A->n_cols, "galerkin: matrix must be square");
    // The device product is specialised to the AMG shape: P one entry per row, R = P^T.
    const int64_t n = P->n_rows, nc = P->n_cols;
    std::vector<int64_t> a(n, 0);
    std::vector<double> pv(n, 0.0);
    std::vector<int64_t> rcount(nc + 1, 0);
    for (int64_t i = 0; i < n; ++i) {
      const int64_t w = P->row_offsets[i + 1] - P->row_offsets[i];
      require(w <= 1, "galerkin_direct: the device path needs one entry per row of P");
      if (w == 1) {
        a[i] = P->col_indices[P->row_offsets[i]];
        pv[i] = P->values[P->row_offsets[i]];
        ++rcount[a[i] + 1];
      }
    }
    for (int64_t J = 0; J < nc; ++J) rcount[J + 1] += rcount[J];
    bool is_transpose = R->row_offsets[nc] == rcount[nc];
    for (int64_t J = 0; J <= nc && is_transpose; ++J) is_transpose = R->row_offsets[J] == rcount[J];
    std::vector<int64_t> cur(rcount.begin(), rcount.end() - 1);
    for (int64_t i = 0; i < n && is_transpose; ++i) {
      if (P->row_offsets[i + 1] == P->row_offsets[i]) continue;
      const int64_t k = cur[a[i]]++;
      is_transpose = R->col_indices[k] == i && R->values[k] == pv[i];
    }
    require(is_transpose, "galerkin_direct: the device path needs R = transpose(P)");
    auto dA = up(A);
    AggDev agg = agg_from_host(n, nc, a.data());
    auto dpv = up_vec(pv.data(), n);
    auto dAc = galerkin_direct(*dA, agg, dpv.get());
    down(*dAc, Ac);
  });
}

int aggmg_build_galerkin_cache(const aggmg_csr* A, int64_t nc, const int64_t* assignment,
                               aggmg_galerkin_cache** out) {
  return guarded([&] {
    require(A->n_rows == A->n_cols, "galerkin: matrix must be square");
    auto dA = up(A);
    auto c = std::make_unique<aggmg_galerkin_cache>();
    c->agg = agg_from_host(A->n_rows, nc, assignment);
    c->g = build_galerkin_cache(*dA, c->agg);
    *out = c.release();
  });
}

int aggmg_galerkin_cache_info(const aggmg_galerkin_cache* c, int64_t* n_fine, int64_t* n_coarse,
                              int64_t* nnz_fine, int64_t* nnz_coarse) {
  return guarded([&] {
    if (n_fine) *n_fine = c->g.n_fine;
    if (n_coarse) *n_coarse = c->g.n_coarse;
    if (nnz_fine) *nnz_fine = c->g.nnz_fine;
    if (nnz_coarse) *nnz_coarse = c->g.nnz_coarse;
  });
}

int aggmg_galerkin_cache_export(const aggmg_galerkin_cache* c, int64_t* coarse_row_offsets,
                                int64_t* coarse_col_indices, int64_t* entry, int64_t* entry_row,
                                int64_t* segment_offsets, int64_t* slot_of_csr,
                                int64_t* rows_by_coarse, int64_t* agg_row_offsets) {
  return guarded([&] {
    const GalerkinDev& g = c->g;
    if (coarse_row_offsets) down_index(g.coarse_rowptr, g.n_coarse + 1, coarse_row_offsets);
    if (coarse_col_indices) down_index(g.coarse_col, g.nnz_coarse, coarse_col_indices);
    if (entry) down_index(g.entry, g.nnz_fine, entry);
    if (entry_row) down_index(g.entry_row, g.nnz_fine, entry_row);
    if (segment_offsets) down_index(g.segment_offsets, g.nnz_coarse + 1, segment_offsets);
    if (slot_of_csr) down_index(g.slot_of_csr, g.nnz_fine, slot_of_csr);
    if (rows_by_coarse) down_index(c->agg.rows_by_coarse, g.n_fine, rows_by_coarse);
    if (agg_row_offsets) down_index(c->agg.agg_row_offsets, g.n_coarse + 1, agg_row_offsets);
  });
}

int aggmg_apply_galerkin_cache(const aggmg_galerkin_cache* c, const aggmg_csr* A,
                               const aggmg_csr* P, aggmg_csr* Ac) {
  return guarded([&] {
    const GalerkinDev& g = c->g;
    require(P->n_rows == g.n_fine && P->n_cols == g.n_coarse,
            "galerkin cache: prolongator shape changed; rebuild the cache");
    require(A->n_rows == g.n_fine && A->row_offsets[A->n_rows] == g.nnz_fine,
            "galerkin cache: fine matrix pattern changed; rebuild the cache");
    auto dA = up(A);
    require(pattern_fingerprint(*dA, c->agg.assignment.get()) == g.pattern_hash,
            "galerkin cache: fine matrix pattern changed; rebuild the cache");
    // per-fine-node prolongator weight (galerkin.cpp:105-118)
    std::vector<idx> a(g.n_fine);
    c->agg.assignment.download(a.data(), g.n_fine);
    sync();
    std::vector<double> pv(g.n_fine, 0.0);
    for (int64_t i = 0; i < g.n_fine; ++i) {
      const int64_t width = P->row_offsets[i + 1] - P->row_offsets[i];
      if (width > 1)
        throw Error("galerkin cache: prolongator row " + std::to_string(i) +
                    " has more than one entry");
      if (width == 1) {
        if (P->col_indices[P->row_offsets[i]] != a[i])
          throw Error("galerkin cache: prolongator disagrees with the cached aggregation");
        pv[i] = P->values[P->row_offsets[i]];
      }
    }
    auto dpv = up_vec(pv.data(), g.n_fine);
    auto dAc = apply_galerkin_cache(g, *dA, dpv.get());
    down(*dAc, Ac);
  });
}

void aggmg_galerkin_cache_free(aggmg_galerkin_cache* c) { delete c; }

int aggmg_setup_smoother(const aggmg_csr* A, int kind, int arnoldi_m, uint64_t seed,
                         double* inv_diag, double* omega, double* rho_est) {
  return guarded([&] {
    auto dA = up(A);
    SmootherDev s;
    setup_smoother(*dA, kind, arnoldi_m, seed, s);
    if (inv_diag) {
      s.inv_diag.download(inv_diag, A->n_rows);
      sync();
    }
    if (omega) *omega = s.omega;
    if (rho_est) *rho_est = s.rho_est;
  });
}

int aggmg_smooth(int kind, const double* inv_diag, double omega, const aggmg_csr* A,
                 const double* b, double* x) {
  return guarded([&] {
    const int64_t n = A->n_rows;
    auto dA = up(A);
    SmootherDev s;
    s.kind = kind;
    s.omega = omega;
    s.inv_diag = up_vec(inv_diag, n);
    s.wdiag.resize(n);
    vec_scale_into(n, kind == AGGMG_SMOOTHER_JACOBI ? 1.0 : omega, s.inv_diag.get(), s.wdiag.get());
    auto db = up_vec(b, n), dx = up_vec(x, n);
    if (kind == AGGMG_SMOOTHER_SGS) {
      build_sgs_schedule(*dA, s);
      smooth_sgs(s, *dA, db.get(), dx.get());
      dx.download(x, n);
    } else {
      DevBuf<double> xo(n);
      smooth_sweep(s, *dA, db.get(), dx.get(), xo.get());
      xo.download(x, n);
    }
    sync();
  });
}

int aggmg_hessenberg_eigenvalues(int64_t n, const double* H, double* re, double* im) {
  return guarded([&] {
    std::vector<double> h(H, H + n * n);
    auto ev = hessenberg_eigenvalues(h, static_cast<int>(n));
    for (int64_t i = 0; i < n; ++i) {
      re[i] = ev[i].real();
      im[i] = ev[i].imag();
    }
  });
}

// ---- L3 ---------------------------------------------------------------------------

int aggmg_setup_hierarchy(const aggmg_csr* A0, const double* B0, const aggmg_setup_config* cfg,
                          aggmg_hierarchy** out) {
  return guarded([&] {
    auto dA = up(A0, true);
    std::unique_ptr<DevBuf<double>> dB;
    if (B0) dB = std::make_unique<DevBuf<double>>(up_vec(B0, A0->n_rows));
    auto h = std::make_unique<aggmg_hierarchy>();
    h->h = setup_hierarchy(dA, dB ? dB->get() : nullptr, to_cfg(cfg));
    *out = h.release();
  });
}

int aggmg_refresh_values(aggmg_hierarchy* h, const double* values, int64_t count) {
  return guarded([&] {
    require(h->h->cfg.reuse_caches, "refresh: hierarchy was built without caches");
    require(count == h->h->levels[0].A->nnz,
            "refresh: value count does not match the level-0 pattern");
    auto dv = up_vec(values, count);
    refresh_values(*h->h, dv.get());
  });
}

int aggmg_hierarchy_clone(const aggmg_hierarchy* h, aggmg_hierarchy** out) {
  return guarded([&] {
    require(h && h->h, "hierarchy: null handle");
    auto c = std::make_unique<aggmg_hierarchy>();
    c->h = clone_hierarchy(*h->h);
    *out = c.release();
  });
}

void aggmg_hierarchy_free(aggmg_hierarchy* h) { delete h; }

int64_t aggmg_hierarchy_n_levels(const aggmg_hierarchy* h) { return h && h->h ? h->h->n_levels() : 0; }

int aggmg_hierarchy_level_size(const aggmg_hierarchy* h, int64_t k, int64_t* n, int64_t* nnz) {
  return guarded([&] {
    const DevLevel& L = level(h, k);
    if (n) *n = L.A->n_rows;
    if (nnz) *nnz = L.A->nnz;
  });
}

int aggmg_hierarchy_level_A(const aggmg_hierarchy* h, int64_t k, aggmg_csr* A) {
  return guarded([&] { down(*level(h, k).A, A); });
}

int aggmg_hierarchy_level_P(const aggmg_hierarchy* h, int64_t k, aggmg_csr* P) {
  return guarded([&] {
    const DevLevel& L = level(h, k);
    if (!L.has_next) {
      alloc_csr(P, 0, 0, 0);
      P->row_offsets[0] = 0;
      return;
    }
    p_to_host(L.agg.n_fine, L.agg.n_agg, L.agg.assignment, L.tr.pval, P);
  });
}

int aggmg_hierarchy_level_R(const aggmg_hierarchy* h, int64_t k, aggmg_csr* R) {
  return guarded([&] {
    const DevLevel& L = level(h, k);
    if (!L.has_next) {
      alloc_csr(R, 0, 0, 0);
      R->row_offsets[0] = 0;
      return;
    }
    down(*L.tr.R, R);
  });
}

int aggmg_hierarchy_level_B(const aggmg_hierarchy* h, int64_t k, double* B) {
  return guarded([&] {
    const DevLevel& L = level(h, k);
    L.B.download(B, L.A->n_rows);
    sync();
  });
}

int aggmg_hierarchy_level_aggregation(const aggmg_hierarchy* h, int64_t k, int64_t* assignment,
                                      int64_t* n_aggregates, int32_t* mis_sweeps) {
  return guarded([&] {
    const DevLevel& L = level(h, k);
    require(L.has_next, "hierarchy: the coarsest level has no aggregation");
    if (assignment) down_index(L.agg.assignment, L.agg.n_fine, assignment);
    if (n_aggregates) *n_aggregates = L.agg.n_agg;
    if (mis_sweeps) *mis_sweeps = L.mis_sweeps;
  });
}

int aggmg_hierarchy_level_smoother(const aggmg_hierarchy* h, int64_t k, double* omega,
                                   double* rho_est, double* inv_diag) {
  return guarded([&] {
    const DevLevel& L = level(h, k);
    if (omega) *omega = L.has_smoother ? L.smoother.omega : 1.0;
    if (rho_est) *rho_est = L.has_smoother ? L.smoother.rho_est : 1.0;
    if (inv_diag && L.has_smoother) {
      L.smoother.inv_diag.download(inv_diag, L.A->n_rows);
      sync();
    }
  });
}

int64_t aggmg_hierarchy_n_warnings(const aggmg_hierarchy* h) {
  return h && h->h ? static_cast<int64_t>(h->h->warnings.size()) : 0;
}
const char* aggmg_hierarchy_warning(const aggmg_hierarchy* h, int64_t i) {
  if (!h || !h->h || i < 0 || i >= static_cast<int64_t>(h->h->warnings.size())) return "";
  return h->h->warnings[i].c_str();
}

int aggmg_hierarchy_report(const aggmg_hierarchy* h, double* gc, double* oc) {
  return guarded([&] {  // hierarchy.cpp:106-121
    double sn = 0.0, snnz = 0.0;
    for (const auto& L : h->h->levels) {
      sn += static_cast<double>(L.A->n_rows);
      snnz += static_cast<double>(L.A->nnz);
    }
    if (gc) *gc = sn / static_cast<double>(h->h->levels[0].A->n_rows);
    if (oc) *oc = snnz / static_cast<double>(h->h->levels[0].A->nnz);
  });
}

int aggmg_hierarchy_setup_ms(const aggmg_hierarchy* h, double* ms) {
  return guarded([&] { *ms = h->h->setup_ms; });
}

// ---- L4 cycles -------------------------------------------------------------------------

static int run_cycle(const aggmg_hierarchy* h, const aggmg_cycle_config* cfg, int64_t k, bool kc,
                     const double* b, double* x) {
  return guarded([&] {
    const DevLevel& L = level(h, k);
    const int64_t n = L.A->n_rows;
    auto db = up_vec(b, n), dx = up_vec(x, n);
    DevBuf<double> xo(n);
    CycleCfg c = to_cfg(cfg);
    cycle(*h->h, c, k, kc, db.get(), dx.get(), xo.get(), nullptr);
    xo.download(x, n);
    flush_cycle_warnings();
  });
}

int aggmg_vcycle(const aggmg_hierarchy* h, int64_t k, const double* b, double* x) {
  return run_cycle(h, nullptr, k, false, b, x);
}
int aggmg_kcycle(const aggmg_hierarchy* h, const aggmg_cycle_config* cfg, int64_t k,
                 const double* b, double* x) {
  return run_cycle(h, cfg, k, true, b, x);
}

int aggmg_apply_preconditioner(const aggmg_hierarchy* h, const aggmg_cycle_config* cfg,
                               const double* r, double* z) {
  return guarded([&] {
    const int64_t n = level(h, 0).A->n_rows;
    auto dr = up_vec(r, n);
    DevBuf<double> dz(n);
    apply_preconditioner(*h->h, to_cfg(cfg), dr.get(), dz.get());
    dz.download(z, n);
    flush_cycle_warnings();
  });
}

// ---- L4 Krylov ---------------------------------------------------------------------------

static int run_krylov(const aggmg_csr* A, const double* b, const double* x0,
                      const aggmg_hierarchy* M, const aggmg_cycle_config* cycle,
                      const aggmg_solver_config* cfg, double* x, aggmg_solve_report* rep,
                      int method) {
  return guarded([&] {
    const int64_t n = A->n_rows;
    const char* who = method == AGGMG_SOLVER_PCG ? "pcg" : "fgmres";
    require(A->n_rows == A->n_cols, std::string(who) + ": matrix must be square");
    auto dA = up(A);
    auto db = up_vec(b, n), dx = up_vec(x0, n);
    aggmg_solver_config s = *cfg;
    s.method = method;
    SolveOut o = run_solver(*dA, db.get(), dx.get(), M ? M->h.get() : nullptr, cycle, &s);
    dx.download(x, n);
    sync();
    fill_report(o, rep);
  });
}

static int run_krylov_cb(const aggmg_csr* A, const double* b, const double* x0,
                         aggmg_precond_fn fn, void* user, const aggmg_solver_config* cfg,
                         double* x, aggmg_solve_report* rep, int method) {
  return guarded([&] {
    const int64_t n = A->n_rows;
    const char* who = method == AGGMG_SOLVER_PCG ? "pcg" : "fgmres";
    require(A->n_rows == A->n_cols, std::string(who) + ": matrix must be square");
    auto dA = up(A);
    auto db = up_vec(b, n), dx = up_vec(x0, n);
    Precond M;
    M.host_fn = fn;
    M.host_user = user;
    SolverCfg s = to_cfg(cfg);
    s.method = method;
    SolveOut o = method == AGGMG_SOLVER_PCG ? pcg(*dA, db.get(), dx.get(), M, s)
                                           : fgmres(*dA, db.get(), dx.get(), M, s);
    dx.download(x, n);
    sync();
    fill_report(o, rep);
  });
}

int aggmg_pcg_cb(const aggmg_csr* A, const double* b, const double* x0, aggmg_precond_fn M,
                 void* user, const aggmg_solver_config* cfg, double* x, aggmg_solve_report* report) {
  return run_krylov_cb(A, b, x0, M, user, cfg, x, report, AGGMG_SOLVER_PCG);
}
int aggmg_fgmres_cb(const aggmg_csr* A, const double* b, const double* x0, aggmg_precond_fn M,
                    void* user, const aggmg_solver_config* cfg, double* x,
                    aggmg_solve_report* report) {
  return run_krylov_cb(A, b, x0, M, user, cfg, x, report, AGGMG_SOLVER_FGMRES);
}

int aggmg_pcg(const aggmg_csr* A, const double* b, const double* x0, const aggmg_hierarchy* M,
              const aggmg_cycle_config* cycle, const aggmg_solver_config* cfg, double* x,
              aggmg_solve_report* report) {
  return run_krylov(A, b, x0, M, cycle, cfg, x, report, AGGMG_SOLVER_PCG);
}
int aggmg_fgmres(const aggmg_csr* A, const double* b, const double* x0, const aggmg_hierarchy* M,
                 const aggmg_cycle_config* cycle, const aggmg_solver_config* cfg, double* x,
                 aggmg_solve_report* report) {
  return run_krylov(A, b, x0, M, cycle, cfg, x, report, AGGMG_SOLVER_FGMRES);
}

int aggmg_setup_and_solve(const aggmg_csr* A, const double* b, const double* B0, const double* x0,
                          const aggmg_setup_config* setup, const aggmg_cycle_config* cycle,
                          const aggmg_solver_config* solver, double* x,
                          aggmg_solve_report* report) {
  return guarded([&] {
    using Clock = std::chrono::steady_clock;
    const auto t0 = Clock::now();
    const int64_t n = A->n_rows;
    auto dA = up(A, true);
    std::unique_ptr<DevBuf<double>> dB;
    if (B0) dB = std::make_unique<DevBuf<double>>(up_vec(B0, n));
    auto h = setup_hierarchy(dA, dB ? dB->get() : nullptr, to_cfg(setup));
    const double setup_s = std::chrono::duration<double>(Clock::now() - t0).count();
    auto db = up_vec(b, n);
    DevBuf<double> dx(n);
    if (x0)
      dx.upload(x0, n);
    else
      dx.zero();
    SolveOut o = run_solver(*dA, db.get(), dx.get(), h.get(), cycle, solver);
    dx.download(x, n);
    sync();
    fill_report(o, report);
    if (report) report->setup_seconds = setup_s;
  });
}

// ---- inputs --------------------------------------------------------------------------------

static void host_to_out(const HostCsr& H, aggmg_csr* A) {
  const int64_t nnz = static_cast<int64_t>(H.col.size());
  alloc_csr(A, H.n, H.ncols, nnz);
  std::memcpy(A->row_offsets, H.rp.data(), sizeof(int64_t) * (H.n + 1));
  std::memcpy(A->col_indices, H.col.data(), sizeof(int64_t) * nnz);
  std::memcpy(A->values, H.val.data(), sizeof(double) * nnz);
}

// ---- Matrix Market (matrix_market.hpp:23-35) ------------------------------------------------

int aggmg_read_matrix_market_file(const char* path, int allow_pattern, aggmg_csr* A) {
  return guarded([&] { host_to_out(read_matrix_market_file(path, allow_pattern != 0), A); });
}

int aggmg_read_matrix_market(const char* text, int64_t size, int allow_pattern, aggmg_csr* A) {
  return guarded([&] {
    host_to_out(read_matrix_market_text(text, static_cast<size_t>(size), allow_pattern != 0), A);
  });
}

int aggmg_write_matrix_market_file(const char* path, const aggmg_csr* A) {
  return guarded([&] {
    require(A != nullptr, "null matrix");
    write_matrix_market_file(path, A->n_rows, A->n_cols, A->row_offsets, A->col_indices, A->values);
  });
}

int aggmg_read_vector_market_file(const char* path, double* x, int64_t capacity, int64_t* n) {
  return guarded([&] {
    const std::vector<double> v = read_vector_market_file(path);
    *n = static_cast<int64_t>(v.size());
    if (x) {
      require(capacity >= *n, "vector market: output buffer too small");
      std::memcpy(x, v.data(), sizeof(double) * v.size());
    }
  });
}

int aggmg_write_vector_market_file(const char* path, const double* x, int64_t n) {
  return guarded([&] { write_vector_market_file(path, x, n); });
}

int aggmg_generate_poisson_rows(int dims, int64_t nx, int64_t ny, int64_t nz, double eps,
                                int weak_axis, int64_t row0, int64_t nrows, aggmg_csr* A) {
  return guarded([&] {
    host_to_out(generate_poisson_host(dims, nx, ny, nz, eps, weak_axis, row0, nrows), A);
  });
}

int aggmg_generate_jump27_rows(int64_t nx, int64_t ny, int64_t nz, double jump, int64_t block,
                               int64_t row0, int64_t nrows, aggmg_csr* A) {
  return guarded([&] { host_to_out(generate_jump27_host(nx, ny, nz, jump, block, row0, nrows), A); });
}

namespace {
// x_i = uniform_sym(seed, i) (poisson.cpp:81-87, rng.hpp:32-34)
__global__ void k_random_vector(int64_t n, uint64_t seed, double* x) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) x[i] = uniform_sym(seed, static_cast<uint64_t>(i));
}
}  // namespace

int aggmg_random_vector(int64_t n, uint64_t seed, double* x) {
  return guarded([&] {
    require(n >= 0, "random_vector: negative length");
    if (n == 0) return;
    DevBuf<double> d(n);
    AGG_LAUNCH(k_random_vector, grid_for(n, 256), 256, 0, n, seed, d.get());
    d.download(x, n);
    sync();
  });
}

int aggmg_generate_poisson(int dims, int64_t nx, int64_t ny, int64_t nz, double eps, int weak_axis,
                           aggmg_csr* A) {
  return guarded([&] { host_to_out(generate_poisson_host(dims, nx, ny, nz, eps, weak_axis), A); });
}
int aggmg_generate_jump27(int64_t nx, int64_t ny, int64_t nz, double jump, int64_t block,
                          aggmg_csr* A) {
  return guarded([&] { host_to_out(generate_jump27_host(nx, ny, nz, jump, block), A); });
}

// ---- device-resident path ------------------------------------------------------------------

int aggmg_dmatrix_from_host(const aggmg_csr* A, aggmg_dmatrix** out) {
  return guarded([&] {
    auto m = std::make_unique<aggmg_dmatrix>();
    m->A = up(A, true);
    *out = m.release();
  });
}
int aggmg_dmatrix_poisson(int dims, int64_t nx, int64_t ny, int64_t nz, double eps, int weak_axis,
                          aggmg_dmatrix** out) {
  return guarded([&] {
    auto m = std::make_unique<aggmg_dmatrix>();
    m->A = generate_poisson_device(dims, nx, ny, nz, eps, weak_axis);
    *out = m.release();
  });
}
int aggmg_dmatrix_jump27(int64_t nx, int64_t ny, int64_t nz, double jump, int64_t block,
                         aggmg_dmatrix** out) {
  return guarded([&] {
    auto m = std::make_unique<aggmg_dmatrix>();
    m->A = generate_jump27_device(nx, ny, nz, jump, block);
    *out = m.release();
  });
}
int aggmg_dmatrix_format(const aggmg_dmatrix* A, int* sell) {
  return guarded([&] { *sell = A->A->pat ? 3 : A->A->sell ? (A->A->sell_vi ? 2 : 1) : 0; });
}

int aggmg_dmatrix_size(const aggmg_dmatrix* A, int64_t* n, int64_t* nnz) {
  return guarded([&] {
    if (n) *n = A->A->n_rows;
    if (nnz) *nnz = A->A->nnz;
  });
}
int aggmg_dmatrix_to_host(const aggmg_dmatrix* A, aggmg_csr* out) {
  return guarded([&] { down(*A->A, out); });
}
void aggmg_dmatrix_free(aggmg_dmatrix* A) { delete A; }

int aggmg_setup_hierarchy_device(const aggmg_dmatrix* A0, const aggmg_setup_config* cfg,
                                 aggmg_hierarchy** out) {
  return guarded([&] {
    auto h = std::make_unique<aggmg_hierarchy>();
    // level 0's kernel layout (SELL-32 copy, value dictionary) is part of setup: rebuilt here,
    // not inherited from the matrix's creation, so a timed setup pays for it
    A0->A->plan();
    h->h = setup_hierarchy(A0->A, nullptr, to_cfg(cfg));
    *out = h.release();
  });
}

int aggmg_hierarchy_level_dmatrix(const aggmg_hierarchy* h, int64_t k, int which,
                                  aggmg_dmatrix** out) {
  return guarded([&] {
    const DevLevel& L = level(h, k);
    require(which == 0 || L.has_next, "hierarchy: the coarsest level has no restriction");
    auto m = std::make_unique<aggmg_dmatrix>();
    m->A = which == 0 ? L.A : L.tr.R;
    *out = m.release();
  });
}

int aggmg_solve_device(const aggmg_hierarchy* h, const aggmg_cycle_config* cycle,
                       const aggmg_solver_config* cfg, double* x, aggmg_solve_report* report) {
  return guarded([&] {
    const DevCsr& A = *h->h->levels[0].A;
    const int64_t n = A.n_rows;
    DevBuf<double> db(n), dx(n);
    fill_double(db.get(), n, 1.0);
    dx.zero();
    SolveOut o = run_solver(A, db.get(), dx.get(), h->h.get(), cycle, cfg);
    if (x) {
      dx.download(x, n);
      sync();
    }
    fill_report(o, report);
  });
}

// ---- measurement ----------------------------------------------------------------------------

int aggmg_profile_enable(int mask) { return guarded([&] { profile_enable(mask); }); }
int aggmg_timer_start(void) { return guarded([&] { timer_start(); }); }
int aggmg_timer_stop(double* ms) { return guarded([&] { *ms = timer_stop(); }); }
int aggmg_profile_read(int family, double* total_ms, int64_t* launches, double* bytes) {
  return guarded([&] { profile_read(family, total_ms, launches, bytes); });
}

int aggmg_bench_dot(int64_t n, int np, int exact, int reps, double* avg_ms) {
  return guarded([&] {
    require(np >= 1 && np <= 3, "bench_dot: np must be 1..3");
    DevBuf<double> a(n), b(n), out(4);
    fill_double(a.get(), n, 0.5);
    fill_double(b.get(), n, 0.25);
    DotArgs d{};
    for (int k = 0; k < np; ++k) {
      d.a[k] = a.get();
      d.b[k] = b.get();
    }
    d.np = np;
    dot_device(d, n, out.get(), nullptr, exact);
    cudaEvent_t e0, e1;
    AGG_CUDA(cudaEventCreate(&e0));
    AGG_CUDA(cudaEventCreate(&e1));
    AGG_CUDA(cudaEventRecord(e0, stream()));
    for (int r = 0; r < reps; ++r) dot_device(d, n, out.get(), nullptr, exact);
    AGG_CUDA(cudaEventRecord(e1, stream()));
    AGG_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    AGG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *avg_ms = ms / reps;
  });
}

int aggmg_bench_spmv(const aggmg_dmatrix* A, int reps, double* avg_ms, double* bytes) {
  return aggmg_bench_kernel(A, 0, reps, avg_ms, bytes);
}

int aggmg_bench_kernel(const aggmg_dmatrix* A, int kind, int reps, double* avg_ms, double* bytes) {
  return guarded([&] {
    const DevCsr& M = *A->A;
    require(kind >= 0 && kind <= 7, "bench_kernel: kind must be 0..7");
    if (kind == 7) {  // one symmetric Gauss-Seidel smooth (both directions, level-scheduled)
      SmootherDev s;
      s.kind = AGGMG_SMOOTHER_SGS;
      s.inv_diag.resize(M.n_rows);
      fill_double(s.inv_diag.get(), M.n_rows, 0.25);
      build_sgs_schedule(M, s);
      DevBuf<double> b(M.n_rows), x(M.n_rows);
      fill_double(b.get(), M.n_rows, 1.0);
      fill_double(x.get(), M.n_rows, 0.0);
      smooth_sgs(s, M, b.get(), x.get());
      cudaEvent_t e0, e1;
      AGG_CUDA(cudaEventCreate(&e0));
      AGG_CUDA(cudaEventCreate(&e1));
      AGG_CUDA(cudaEventRecord(e0, stream()));
      for (int r = 0; r < reps; ++r) smooth_sgs(s, M, b.get(), x.get());
      AGG_CUDA(cudaEventRecord(e1, stream()));
      AGG_CUDA(cudaEventSynchronize(e1));
      float ms = 0.f;
      AGG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      *avg_ms = ms / reps;
      *bytes = 2.0 * (12.0 * M.nnz + 40.0 * M.n_rows);  // per direction: A + b, inv, x in/out
      return;
    }
    const Epi epis[7] = {Epi::kSpmv, Epi::kResidual, Epi::kResidualZero, Epi::kJacobi,
                         Epi::kSpmvDot1, Epi::kScaleDiag, Epi::kJacobiDot2};
    const Epi epi = epis[kind];
    DevBuf<double> x(M.n_cols), y(M.n_rows), b(M.n_rows), d(M.n_rows), xo(M.n_rows), dots(4),
        cv(M.n_rows);
    fill_double(x.get(), M.n_cols, 1.0);
    fill_double(b.get(), M.n_rows, 1.0);
    fill_double(cv.get(), M.n_rows, 0.5);
    fill_double(d.get(), M.n_rows, 0.1);
    SpmvArgs a;
    a.x = x.get();
    a.y = y.get();
    a.b = b.get();
    a.d = d.get();
    a.u = x.get();
    a.c = cv.get();
    a.x_out = xo.get();
    a.dots_out = dots.get();
    spmv_run(M, epi, a);
    cudaEvent_t e0, e1;
    AGG_CUDA(cudaEventCreate(&e0));
    AGG_CUDA(cudaEventCreate(&e1));
    AGG_CUDA(cudaEventRecord(e0, stream()));
    for (int r = 0; r < reps; ++r) spmv_run(M, epi, a);
    AGG_CUDA(cudaEventRecord(e1, stream()));
    AGG_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    AGG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *avg_ms = ms / reps;
    *bytes = spmv_bytes(M, epi);
  });
}


// ---- row-partitioned multi-GPU path -------------------------------------------------------

int aggmg_comm_nccl_unique_id(char id[128]) {
  return guarded([&] { nccl_unique_id(id); });
}

int aggmg_comm_init_nccl(int rank, int nranks, const char id[128], aggmg_comm** out) {
  return guarded([&] {
    require(nranks >= 1 && rank >= 0 && rank < nranks, "comm: rank out of range");
    auto c = std::make_unique<aggmg_comm>();
    c->comm = make_nccl_comm(rank, nranks, id);
    *out = c.release();
  });
}

int aggmg_comm_run_threads(int nranks, const int* devices, aggmg_rank_fn fn, void* user) {
  return guarded([&] {
    require(nranks >= 1 && nranks <= 64, "comm: 1..64 ranks");
    require(fn != nullptr, "comm: null rank function");
    auto group = ThreadComm::make_group(nranks);
    std::vector<int> rc(nranks, 0);
    std::vector<std::string> msg(nranks);
    std::vector<std::thread> th;
    for (int r = 0; r < nranks; ++r)
      th.emplace_back([&, r] {
        try {
          init_device(devices ? devices[r] : 0);
          aggmg_comm c;
          c.comm = std::make_unique<ThreadComm>(group, r, nranks);
          rc[r] = fn(&c, r, user);
          if (rc[r] != 0) {
            msg[r] = aggmg_last_error();
            thread_group_abort(*group);
          }
          cudaStreamSynchronize(stream());
        } catch (const std::exception& e) {
          rc[r] = AGGMG_ERR;
          msg[r] = e.what();
          thread_group_abort(*group);
        }
      });
    for (auto& t : th) t.join();
    for (int r = 0; r < nranks; ++r)
      if (rc[r] != 0)
        throw Error("rank " + std::to_string(r) + ": " + (msg[r].empty() ? "failed" : msg[r]));
  });
}

int aggmg_comm_barrier(aggmg_comm* c) {
  return guarded([&] {
    require(c != nullptr, "null comm");
    c->comm->barrier();
    sync();
  });
}

int aggmg_comm_rank(const aggmg_comm* c) { return c ? c->comm->rank() : -1; }
int aggmg_comm_size(const aggmg_comm* c) { return c ? c->comm->size() : 0; }
const char* aggmg_comm_kind(const aggmg_comm* c) { return c ? c->comm->kind() : ""; }
void aggmg_comm_free(aggmg_comm* c) { delete c; }


int aggmg_dist_matrix_from_host(aggmg_comm* c, int64_t n_global, int64_t row0, const aggmg_csr* rows,
                                aggmg_dist_matrix** out) {
  return guarded([&] {
    require(c && rows, "dist matrix: null argument");
    require(rows->n_cols == n_global, "dist matrix: rows must use global column ids");
    DevCsrPtr R = upload_csr(rows->n_rows, rows->n_cols, rows->row_offsets, rows->col_indices,
                             rows->values, true);
    *out = wrap_rows(c, n_global, row0, R);
  });
}

int aggmg_dist_matrix_poisson(aggmg_comm* c, int dims, int64_t nx, int64_t ny, int64_t nz,
                              double epsilon, int weak_axis, aggmg_dist_matrix** out) {
  return guarded([&] {
    const int64_t n = nx * ny * (dims == 2 ? 1 : nz);
    DevCsrPtr R = generate_poisson_rows(dims, nx, ny, nz, epsilon, weak_axis,
                                        dist_rows_begin(n, *c->comm), dist_rows_count(n, *c->comm));
    *out = wrap_rows(c, n, dist_rows_begin(n, *c->comm), R);
  });
}

int aggmg_dist_matrix_jump27(aggmg_comm* c, int64_t nx, int64_t ny, int64_t nz, double jump,
                             int64_t block, aggmg_dist_matrix** out) {
  return guarded([&] {
    const int64_t n = nx * ny * nz;
    DevCsrPtr R = generate_jump27_rows(nx, ny, nz, jump, block, dist_rows_begin(n, *c->comm),
                                       dist_rows_count(n, *c->comm));
    *out = wrap_rows(c, n, dist_rows_begin(n, *c->comm), R);
  });
}

int aggmg_dist_matrix_info(const aggmg_dist_matrix* A, int64_t* n_global, int64_t* row0,
                           int64_t* n_local, int64_t* nnz_local) {
  return guarded([&] {
    require(A && A->A, "null dist matrix");
    const int me = A->comm->rank();
    if (n_global) *n_global = A->A->rows.n();
    if (row0) *row0 = A->A->rows.begin(me);
    if (n_local) *n_local = A->A->A.n_rows;
    if (nnz_local) *nnz_local = A->A->A.nnz;
  });
}

int aggmg_dist_matrix_format(const aggmg_dist_matrix* A, int* sell) {
  return guarded([&] {
    require(A && A->A, "null dist matrix");
    const DevCsr& M = A->A->A;
    *sell = M.pat ? 3 : M.sell ? (M.sell_vi ? 2 : 1) : 0;
  });
}

void aggmg_dist_matrix_free(aggmg_dist_matrix* A) { delete A; }

int aggmg_dist_setup(aggmg_comm* c, const aggmg_dist_matrix* A0, const double* B0_local,
                     const aggmg_setup_config* cfg, int64_t agglomerate_rows,
                     aggmg_dist_hierarchy** out) {
  return guarded([&] {
    require(c && A0 && A0->A, "dist setup: null argument");
    Comm& comm = *c->comm;
    DevBuf<double> B;
    if (B0_local) B = up_vec(B0_local, A0->A->A.n_rows);
    const SetupCfg s = to_cfg(cfg);
    if (agglomerate_rows <= 0) agglomerate_rows = std::max<int64_t>(s.coarse_size_max, int64_t{1} << 22);
    auto h = std::make_unique<aggmg_dist_hierarchy>();
    h->comm = &comm;
    h->A0 = A0->A;
    h->h = dist_setup_hierarchy(comm, A0->A, B0_local ? B.get() : nullptr, s, agglomerate_rows);
    *out = h.release();
  });
}

int aggmg_dist_solve(aggmg_dist_hierarchy* h, const aggmg_cycle_config* cycle,
                     const aggmg_solver_config* cfg, const double* b_local, double* x_local,
                     aggmg_solve_report* report) {
  return guarded([&] {
    DistHierarchy& H = dh(h);
    const int64_t n = h->A0->A.n_rows;
    DevBuf<double> db(n), dx(n);
    if (b_local)
      db.upload(b_local, n);
    else
      fill_double(db.get(), n, 1.0);
    dx.zero();
    SolveOut o = dist_solve(H, *h->A0, to_cfg(cycle), to_cfg(cfg), db.get(), dx.get());
    if (x_local) {
      dx.download(x_local, n);
      sync();
    }
    fill_report(o, report);
  });
}

int aggmg_dist_refresh_values(aggmg_dist_hierarchy* h, const double* new_values_local, int64_t count) {
  return guarded([&] {
    DistHierarchy& H = dh(h);
    require(count == h->A0->A.nnz, "refresh_values: value count does not match this rank's rows");
    DevBuf<double> v(count);
    v.upload(new_values_local, count);
    dist_refresh_values(H, v.get());
  });
}

int aggmg_dist_apply_preconditioner(aggmg_dist_hierarchy* h, const aggmg_cycle_config* cycle,
                                    const double* r_local, double* z_local) {
  return guarded([&] {
    DistHierarchy& H = dh(h);
    H.ensure_workspace();
    const int64_t n = h->A0->A.n_rows;
    const int64_t cap = H.kd() ? H.levels[0].halo_cap : 0;
    DevBuf<double> dr(n), dz(n + cap);
    dr.upload(r_local, n);
    dist_apply_preconditioner(H, to_cfg(cycle), dr.get(), dz.get());
    dz.download(z_local, n);
    sync();
  });
}

int aggmg_dist_hierarchy_info(const aggmg_dist_hierarchy* h, int64_t* n_levels, int64_t* n_distributed,
                              double* setup_ms) {
  return guarded([&] {
    require(h && h->h, "null distributed hierarchy");
    if (n_levels) *n_levels = h->h->n_levels_total;
    if (n_distributed) *n_distributed = h->h->kd();
    if (setup_ms) *setup_ms = h->h->setup_ms;
  });
}

int aggmg_dist_hierarchy_level_size(const aggmg_dist_hierarchy* h, int64_t k, int64_t* n, int64_t* nnz) {
  return guarded([&] {
    require(h && h->h, "null distributed hierarchy");
    require(k >= 0 && k < h->h->n_levels_total, "hierarchy: level index out of range");
    if (n) *n = h->h->level_rows[k];
    if (nnz) *nnz = h->h->level_nnz[k];
  });
}

int aggmg_dist_hierarchy_level_A(aggmg_dist_hierarchy* h, int64_t k, aggmg_csr* A) {
  return guarded([&] {
    DistHierarchy& H = dh(h);
    require(k >= 0 && k < H.n_levels_total, "hierarchy: level index out of range");
    Comm& comm = *H.comm;
    A->n_rows = A->n_cols = A->nnz = 0;
    A->row_offsets = nullptr;
    A->col_indices = nullptr;
    A->values = nullptr;
    if (k < H.kd()) {
      DevCsrPtr G = gather_to_root(comm, *H.levels[k].A, 0);
      if (comm.rank() == 0) down(*G, A);
    } else if (comm.rank() == 0) {
      down(*H.tail->levels[k - H.kd()].A, A);
    }
  });
}

int aggmg_dist_hierarchy_level_transfer(aggmg_dist_hierarchy* h, int64_t k, int64_t* assignment,
                                        double* pval, int32_t* mis_sweeps) {
  return guarded([&] {
    DistHierarchy& H = dh(h);
    require(k >= 0 && k + 1 < H.n_levels_total, "hierarchy: level has no transfer");
    Comm& comm = *H.comm;
    if (k < H.kd()) {
      const DistLevel& L = H.levels[k];
      const int64_t n = L.A->A.n_rows;
      DevBuf<idx> a_all;
      DevBuf<double> p_all;
      gather_pod<idx>(comm, L.agg_global.get(), n, a_all);
      gather_pod<double>(comm, L.pval.get(), n, p_all);
      if (comm.rank() == 0) {
        if (assignment) down_index(a_all, a_all.size(), assignment);
        if (pval) {
          p_all.download(pval, p_all.size());
          sync();
        }
        if (mis_sweeps) *mis_sweeps = L.mis_sweeps;
      }
    } else if (comm.rank() == 0) {
      const DevLevel& L = H.tail->levels[k - H.kd()];
      if (assignment) down_index(L.agg.assignment, L.agg.n_fine, assignment);
      if (pval) {
        L.tr.pval.download(pval, L.agg.n_fine);
        sync();
      }
      if (mis_sweeps) *mis_sweeps = L.mis_sweeps;
    }
  });
}

int aggmg_dist_hierarchy_level_B(aggmg_dist_hierarchy* h, int64_t k, double* B) {
  return guarded([&] {
    DistHierarchy& H = dh(h);
    require(k >= 0 && k < H.n_levels_total, "hierarchy: level index out of range");
    Comm& comm = *H.comm;
    if (k < H.kd()) {
      DevBuf<double> all;
      gather_pod<double>(comm, H.levels[k].B.get(), H.levels[k].A->A.n_rows, all);
      if (comm.rank() == 0) {
        all.download(B, all.size());
        sync();
      }
    } else if (comm.rank() == 0) {
      const DevLevel& L = H.tail->levels[k - H.kd()];
      L.B.download(B, L.A->n_rows);
      sync();
    }
  });
}

int aggmg_dist_hierarchy_level_omega(aggmg_dist_hierarchy* h, int64_t k, double* omega) {
  return guarded([&] {
    DistHierarchy& H = dh(h);
    require(k >= 0 && k < H.n_levels_total, "hierarchy: level index out of range");
    if (k < H.kd())
      *omega = H.levels[k].smoother.omega;
    else if (H.comm->rank() == 0)
      *omega = H.tail->levels[k - H.kd()].smoother.omega;
  });
}

int64_t aggmg_dist_hierarchy_n_warnings(const aggmg_dist_hierarchy* h) {
  return (h && h->h) ? static_cast<int64_t>(h->h->warnings.size()) : 0;
}
const char* aggmg_dist_hierarchy_warning(const aggmg_dist_hierarchy* h, int64_t i) {
  if (!h || !h->h || i < 0 || i >= static_cast<int64_t>(h->h->warnings.size())) return "";
  return h->h->warnings[i].c_str();
}

void aggmg_dist_hierarchy_free(aggmg_dist_hierarchy* h) { delete h; }

}  // extern "C"
