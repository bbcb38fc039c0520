// ref_shim.cpp — TEST INFRASTRUCTURE ONLY.  A thin C shim over the UNMODIFIED reference
// library (/root/reference/proj/core, compiled from its own sources by oracle/Makefile
// into oracle/_ref/).  It exposes the reference's public C++ API with the same plain-C
// signatures as include/aggmg_b200.h, prefixed aggmg_ref_, so the parity tests and the
// bench's CPU arm can call the reference and the B200 library side by side.  Nothing in
// the product links or loads this file.
#include <sstream>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "aggmg/matrix_market.hpp"
#include "aggmg/aggregation.hpp"
#include "aggmg/cycles.hpp"
#include "aggmg/dense.hpp"
#include "aggmg/galerkin.hpp"
#include "aggmg/hierarchy.hpp"
#include "aggmg/krylov.hpp"
#include "aggmg/parallel.hpp"
#include "aggmg/poisson.hpp"
#include "aggmg/smoother.hpp"
#include "aggmg/sparse.hpp"
#include "aggmg/strength.hpp"
#include "aggmg/transfer.hpp"
#include "aggmg/vector_ops.hpp"
#include "../include/aggmg_b200.h"

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    g_err.clear();
    return AGGMG_OK;
  } catch (const std::exception& e) {
    g_err = e.what();
    return AGGMG_ERR;
  }
}

aggmg::SparseMatrix to_ref(const aggmg_csr* m) {
  aggmg::SparseMatrix A(m->n_rows, m->n_cols);
  const int64_t nnz = m->row_offsets[m->n_rows];
  A.row_offsets.assign(m->row_offsets, m->row_offsets + m->n_rows + 1);
  A.col_indices.assign(m->col_indices, m->col_indices + nnz);
  if (m->values)
    A.values.assign(m->values, m->values + nnz);
  else
    A.values.assign(nnz, 1.0);
  return A;
}

void from_ref(const aggmg::SparseMatrix& A, aggmg_csr* out) {
  out->n_rows = A.n_rows;
  out->n_cols = A.n_cols;
  out->nnz = A.nnz();
  out->row_offsets = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (A.n_rows + 1)));
  out->col_indices = static_cast<int64_t*>(std::malloc(sizeof(int64_t) * (A.nnz() + 1)));
  out->values = static_cast<double*>(std::malloc(sizeof(double) * (A.nnz() + 1)));
  std::memcpy(out->row_offsets, A.row_offsets.data(), sizeof(int64_t) * (A.n_rows + 1));
  if (A.nnz()) {
    std::memcpy(out->col_indices, A.col_indices.data(), sizeof(int64_t) * A.nnz());
    std::memcpy(out->values, A.values.data(), sizeof(double) * A.nnz());
  }
}

aggmg::SetupConfig to_ref(const aggmg_setup_config* c) {
  aggmg::SetupConfig s;
  if (!c) return s;
  s.alpha = c->alpha;
  s.coarse_size_max = c->coarse_size_max;
  s.max_levels = c->max_levels;
  s.smoother = static_cast<aggmg::SmootherKind>(c->smoother);
  s.arnoldi_m = c->arnoldi_m;
  s.seed = c->seed;
  s.reuse_caches = c->reuse_caches != 0;
  return s;
}
aggmg::CycleConfig to_ref(const aggmg_cycle_config* c) {
  aggmg::CycleConfig s;
  if (!c) return s;
  s.kind = c->kind == AGGMG_CYCLE_V ? aggmg::CycleKind::v
           : c->kind == AGGMG_CYCLE_K ? aggmg::CycleKind::k
                                      : aggmg::CycleKind::hybrid;
  s.k_levels = c->k_levels;
  s.t = c->t;
  s.inner = c->inner == AGGMG_INNER_CG ? aggmg::InnerKind::cg : aggmg::InnerKind::gmres;
  return s;
}
aggmg::SolverConfig to_ref(const aggmg_solver_config* c) {
  aggmg::SolverConfig s;
  if (!c) return s;
  s.method = c->method == AGGMG_SOLVER_PCG ? aggmg::SolverMethod::pcg : aggmg::SolverMethod::fgmres;
  s.tol = c->tol;
  s.max_iters = c->max_iters;
  s.restart = c->restart;
  return s;
}

void fill_report(const aggmg::SolveReport& r, aggmg_solve_report* out) {
  if (!out) return;
  out->converged = r.converged ? 1 : 0;
  out->iterations = r.iterations;
  out->history_length = static_cast<int64_t>(r.residual_history.size());
  if (out->history)
    for (int64_t i = 0; i < std::min<int64_t>(out->history_capacity, out->history_length); ++i)
      out->history[i] = r.residual_history[i];
  out->solve_seconds = r.solve_seconds;
  std::snprintf(out->note, sizeof(out->note), "%s", r.note.c_str());
}

struct RefHierarchy {
  aggmg::Hierarchy h;
};

aggmg::Vector vec(const double* p, int64_t n) { return aggmg::Vector(p, p + n); }

}  // namespace

extern "C" {

const char* aggmg_ref_last_error(void) { return g_err.c_str(); }
void aggmg_ref_set_num_threads(int n) { aggmg::set_num_threads(n); }
int aggmg_ref_num_threads(void) { return aggmg::num_threads(); }
void aggmg_ref_csr_free(aggmg_csr* m) {
  std::free(m->row_offsets);
  std::free(m->col_indices);
  std::free(m->values);
}

int aggmg_ref_generate_poisson(int dims, int64_t nx, int64_t ny, int64_t nz, double eps, int weak,
                               aggmg_csr* A) {
  return guarded([&] {
    aggmg::PoissonSpec ps;
    ps.dims = dims;
    ps.nx = nx;
    ps.ny = ny;
    ps.nz = nz;
    ps.epsilon = eps;
    ps.weak_axis = weak;
    from_ref(aggmg::generate_poisson(ps), A);
  });
}

// Matrix Market I/O of the unmodified reference (matrix_market.hpp:23-35)
int aggmg_ref_read_matrix_market_file(const char* path, int allow_pattern, aggmg_csr* A) {
  return guarded([&] {
    aggmg::MmOptions o;
    o.allow_pattern = allow_pattern != 0;
    from_ref(aggmg::read_matrix_market_file(path, o), A);
  });
}
int aggmg_ref_read_matrix_market(const char* text, int64_t size, int allow_pattern, aggmg_csr* A) {
  return guarded([&] {
    aggmg::MmOptions o;
    o.allow_pattern = allow_pattern != 0;
    std::istringstream in(std::string(text, static_cast<size_t>(size)));
    from_ref(aggmg::read_matrix_market(in, o), A);
  });
}
int aggmg_ref_write_matrix_market_file(const char* path, const aggmg_csr* A) {
  return guarded([&] { aggmg::write_matrix_market_file(path, to_ref(A)); });
}
int aggmg_ref_read_vector_market_file(const char* path, double* x, int64_t capacity, int64_t* n) {
  return guarded([&] {
    const aggmg::Vector v = aggmg::read_vector_market_file(path);
    *n = static_cast<int64_t>(v.size());
    if (x) {
      if (capacity < *n) throw aggmg::Error("vector market: output buffer too small");
      std::copy(v.begin(), v.end(), x);
    }
  });
}
int aggmg_ref_write_vector_market_file(const char* path, const double* x, int64_t n) {
  return guarded([&] { aggmg::write_vector_market_file(path, aggmg::Vector(x, x + n)); });
}

int aggmg_ref_spmv(const aggmg_csr* A, const double* x, double* y) {
  return guarded([&] {
    auto r = aggmg::spmv(to_ref(A), vec(x, A->n_cols));
    std::memcpy(y, r.data(), sizeof(double) * r.size());
  });
}
int aggmg_ref_transpose(const aggmg_csr* A, aggmg_csr* T) {
  return guarded([&] { from_ref(aggmg::transpose(to_ref(A)), T); });
}
int aggmg_ref_dot(int64_t n, const double* a, const double* b, double* out) {
  return guarded([&] { *out = aggmg::dot(std::span<const double>(a, n), std::span<const double>(b, n)); });
}
int aggmg_ref_norm2(int64_t n, const double* a, double* out) {
  return guarded([&] { *out = aggmg::norm2(std::span<const double>(a, n)); });
}
int aggmg_ref_axpy(int64_t n, double a, const double* x, double* y) {
  return guarded([&] { aggmg::axpy(a, std::span<const double>(x, n), std::span<double>(y, n)); });
}
int aggmg_ref_scale(int64_t n, double a, double* x) {
  return guarded([&] { aggmg::scale(a, std::span<double>(x, n)); });
}

int aggmg_ref_classic_strength(const aggmg_csr* A, double alpha, int policy, aggmg_csr* C) {
  return guarded([&] {
    from_ref(aggmg::classic_strength(to_ref(A), alpha,
                                     policy ? aggmg::ZeroDiagPolicy::fail : aggmg::ZeroDiagPolicy::positive),
             C);
  });
}
int aggmg_ref_influence_counts(const aggmg_csr* C, int64_t* counts) {
  return guarded([&] {
    auto v = aggmg::influence_counts(to_ref(C));
    std::memcpy(counts, v.data(), sizeof(int64_t) * v.size());
  });
}
int aggmg_ref_symmetrize_pattern(const aggmg_csr* C, aggmg_csr* S) {
  return guarded([&] { from_ref(aggmg::symmetrize_pattern(to_ref(C)), S); });
}
int aggmg_ref_mis2(const aggmg_csr* S, const int64_t* influence, uint64_t seed, int8_t* state,
                   int64_t* n_roots, int32_t* sweeps) {
  return guarded([&] {
    std::vector<aggmg::index_t> infl(influence, influence + S->n_rows);
    auto m = aggmg::mis2(to_ref(S), infl, seed);
    std::memcpy(state, m.state.data(), m.state.size());
    if (n_roots) *n_roots = static_cast<int64_t>(m.roots.size());
    if (sweeps) *sweeps = m.sweeps;
  });
}
int aggmg_ref_aggregate(const aggmg_csr* S, const aggmg_csr* A, const int8_t* state,
                        int64_t* assignment, int64_t* representatives, int64_t* n_aggregates) {
  return guarded([&] {
    aggmg::Mis2Result m;
    m.state.assign(state, state + S->n_rows);
    for (int64_t i = 0; i < S->n_rows; ++i)
      if (state[i] == 1) m.roots.push_back(i);
    auto agg = aggmg::aggregate(to_ref(S), to_ref(A), m);
    std::memcpy(assignment, agg.assignment.data(), sizeof(int64_t) * agg.n_fine);
    if (representatives)
      std::memcpy(representatives, agg.representatives.data(), sizeof(int64_t) * agg.n_aggregates);
    *n_aggregates = agg.n_aggregates;
  });
}

static aggmg::Aggregation make_agg(int64_t n, int64_t nc, const int64_t* assignment) {
  aggmg::Aggregation agg;
  agg.n_fine = n;
  agg.n_aggregates = nc;
  agg.assignment.assign(assignment, assignment + n);
  agg.representatives.assign(nc, -1);
  for (int64_t i = 0; i < n; ++i)
    if (agg.representatives[assignment[i]] < 0) agg.representatives[assignment[i]] = i;
  return agg;
}

int aggmg_ref_build_transfer(int64_t n, int64_t nc, const int64_t* assignment, const double* b,
                             aggmg_csr* P, aggmg_csr* R, double* coarse_b) {
  return guarded([&] {
    auto t = aggmg::build_transfer(make_agg(n, nc, assignment), vec(b, n));
    if (P) from_ref(t.P, P);
    if (R) from_ref(t.R, R);
    if (coarse_b) std::memcpy(coarse_b, t.coarse_b.data(), sizeof(double) * nc);
  });
}
int aggmg_ref_galerkin_direct(const aggmg_csr* R, const aggmg_csr* A, const aggmg_csr* P,
                              aggmg_csr* Ac) {
  return guarded([&] { from_ref(aggmg::galerkin_direct(to_ref(R), to_ref(A), to_ref(P)), Ac); });
}

struct RefCache {
  aggmg::GalerkinCache c;
};
int aggmg_ref_build_galerkin_cache(const aggmg_csr* A, int64_t nc, const int64_t* assignment,
                                   void** out) {
  return guarded([&] {
    auto c = std::make_unique<RefCache>();
    c->c = aggmg::build_galerkin_cache(to_ref(A), make_agg(A->n_rows, nc, assignment));
    *out = c.release();
  });
}
int aggmg_ref_galerkin_cache_info(const void* cp, int64_t* n_fine, int64_t* n_coarse,
                                  int64_t* nnz_fine, int64_t* nnz_coarse) {
  const auto& c = static_cast<const RefCache*>(cp)->c;
  if (n_fine) *n_fine = c.n_fine;
  if (n_coarse) *n_coarse = c.n_coarse;
  if (nnz_fine) *nnz_fine = static_cast<int64_t>(c.entry.size());
  if (nnz_coarse) *nnz_coarse = static_cast<int64_t>(c.coarse_col_indices.size());
  return AGGMG_OK;
}
int aggmg_ref_galerkin_cache_export(const void* cp, int64_t* cro, int64_t* cci, int64_t* entry,
                                    int64_t* entry_row, int64_t* seg, int64_t* slot, int64_t* rbc,
                                    int64_t* aro) {
  const auto& c = static_cast<const RefCache*>(cp)->c;
  auto cp64 = [](int64_t* dst, const std::vector<aggmg::index_t>& v) {
    if (dst && !v.empty()) std::memcpy(dst, v.data(), sizeof(int64_t) * v.size());
  };
  cp64(cro, c.coarse_row_offsets);
  cp64(cci, c.coarse_col_indices);
  cp64(entry, c.entry);
  cp64(entry_row, c.entry_row);
  cp64(seg, c.segment_offsets);
  cp64(slot, c.slot_of_csr);
  cp64(rbc, c.rows_by_coarse);
  cp64(aro, c.agg_row_offsets);
  return AGGMG_OK;
}
int aggmg_ref_apply_galerkin_cache(const void* cp, const aggmg_csr* A, const aggmg_csr* P,
                                   aggmg_csr* Ac) {
  return guarded([&] {
    from_ref(aggmg::apply_galerkin_cache(static_cast<const RefCache*>(cp)->c, to_ref(A), to_ref(P)), Ac);
  });
}
void aggmg_ref_galerkin_cache_free(void* cp) { delete static_cast<RefCache*>(cp); }

int aggmg_ref_setup_smoother(const aggmg_csr* A, int kind, int m, uint64_t seed, double* inv_diag,
                             double* omega, double* rho) {
  return guarded([&] {
    auto s = aggmg::setup_smoother(to_ref(A), static_cast<aggmg::SmootherKind>(kind), m, seed);
    if (inv_diag) std::memcpy(inv_diag, s.inv_diag.data(), sizeof(double) * s.inv_diag.size());
    if (omega) *omega = s.omega;
    if (rho) *rho = s.rho_est;
  });
}
int aggmg_ref_smooth(int kind, const double* inv_diag, double omega, const aggmg_csr* A,
                     const double* b, double* x) {
  return guarded([&] {
    aggmg::SmootherState s;
    s.kind = static_cast<aggmg::SmootherKind>(kind);
    s.inv_diag = vec(inv_diag, A->n_rows);
    s.omega = omega;
    aggmg::Vector xv = vec(x, A->n_rows);
    aggmg::smooth(s, to_ref(A), vec(b, A->n_rows), xv);
    std::memcpy(x, xv.data(), sizeof(double) * xv.size());
  });
}
int aggmg_ref_hessenberg_eigenvalues(int64_t n, const double* H, double* re, double* im) {
  return guarded([&] {
    aggmg::DenseMatrix D(n, n);
    std::memcpy(D.data.data(), H, sizeof(double) * n * n);
    auto ev = aggmg::hessenberg_eigenvalues(D);
    for (int64_t i = 0; i < n; ++i) {
      re[i] = ev[i].real();
      im[i] = ev[i].imag();
    }
  });
}

int aggmg_ref_setup_hierarchy(const aggmg_csr* A0, const double* B0, const aggmg_setup_config* cfg,
                              void** out) {
  return guarded([&] {
    auto h = std::make_unique<RefHierarchy>();
    aggmg::Vector b = B0 ? vec(B0, A0->n_rows) : aggmg::ones_vector(A0->n_rows);
    h->h = aggmg::setup_hierarchy(to_ref(A0), std::move(b), to_ref(cfg));
    *out = h.release();
  });
}
int aggmg_ref_refresh_values(void* hp, const double* values, int64_t count) {
  return guarded([&] {
    auto* h = static_cast<RefHierarchy*>(hp);
    h->h = aggmg::refresh_values(std::move(h->h), std::vector<double>(values, values + count));
  });
}
void aggmg_ref_hierarchy_free(void* h) { delete static_cast<RefHierarchy*>(h); }
int64_t aggmg_ref_hierarchy_n_levels(const void* h) {
  return static_cast<const RefHierarchy*>(h)->h.n_levels();
}
int aggmg_ref_hierarchy_level_size(const void* hp, int64_t k, int64_t* n, int64_t* nnz) {
  const auto& L = static_cast<const RefHierarchy*>(hp)->h.levels[k];
  if (n) *n = L.A.n_rows;
  if (nnz) *nnz = L.A.nnz();
  return AGGMG_OK;
}
int aggmg_ref_hierarchy_level_A(const void* hp, int64_t k, aggmg_csr* A) {
  from_ref(static_cast<const RefHierarchy*>(hp)->h.levels[k].A, A);
  return AGGMG_OK;
}
int aggmg_ref_hierarchy_level_P(const void* hp, int64_t k, aggmg_csr* P) {
  from_ref(static_cast<const RefHierarchy*>(hp)->h.levels[k].P, P);
  return AGGMG_OK;
}
int aggmg_ref_hierarchy_level_R(const void* hp, int64_t k, aggmg_csr* R) {
  from_ref(static_cast<const RefHierarchy*>(hp)->h.levels[k].R, R);
  return AGGMG_OK;
}
int aggmg_ref_hierarchy_level_B(const void* hp, int64_t k, double* B) {
  const auto& L = static_cast<const RefHierarchy*>(hp)->h.levels[k];
  std::memcpy(B, L.B.data(), sizeof(double) * L.B.size());
  return AGGMG_OK;
}
int aggmg_ref_hierarchy_level_smoother(const void* hp, int64_t k, double* omega, double* rho,
                                       double* inv_diag) {
  const auto& L = static_cast<const RefHierarchy*>(hp)->h.levels[k];
  if (omega) *omega = L.smoother.omega;
  if (rho) *rho = L.smoother.rho_est;
  if (inv_diag && !L.smoother.inv_diag.empty())
    std::memcpy(inv_diag, L.smoother.inv_diag.data(), sizeof(double) * L.smoother.inv_diag.size());
  return AGGMG_OK;
}
int64_t aggmg_ref_hierarchy_n_warnings(const void* hp) {
  return static_cast<int64_t>(static_cast<const RefHierarchy*>(hp)->h.warnings.size());
}
const char* aggmg_ref_hierarchy_warning(const void* hp, int64_t i) {
  return static_cast<const RefHierarchy*>(hp)->h.warnings[i].c_str();
}

int aggmg_ref_vcycle(const void* hp, int64_t k, const double* b, double* x) {
  return guarded([&] {
    const auto& h = static_cast<const RefHierarchy*>(hp)->h;
    const int64_t n = h.levels[k].A.n_rows;
    aggmg::Vector xv = vec(x, n);
    aggmg::vcycle(h, k, vec(b, n), xv);
    std::memcpy(x, xv.data(), sizeof(double) * n);
  });
}
int aggmg_ref_kcycle(const void* hp, const aggmg_cycle_config* cfg, int64_t k, const double* b,
                     double* x) {
  return guarded([&] {
    const auto& h = static_cast<const RefHierarchy*>(hp)->h;
    const int64_t n = h.levels[k].A.n_rows;
    aggmg::Vector xv = vec(x, n);
    aggmg::kcycle(h, to_ref(cfg), k, vec(b, n), xv);
    std::memcpy(x, xv.data(), sizeof(double) * n);
  });
}
int aggmg_ref_apply_preconditioner(const void* hp, const aggmg_cycle_config* cfg, const double* r,
                                   double* z) {
  return guarded([&] {
    const auto& h = static_cast<const RefHierarchy*>(hp)->h;
    const int64_t n = h.levels[0].A.n_rows;
    auto out = aggmg::apply_preconditioner(h, to_ref(cfg), vec(r, n));
    std::memcpy(z, out.data(), sizeof(double) * n);
  });
}

static int run(const aggmg_csr* A, const double* b, const double* x0, const void* hp,
               const aggmg_cycle_config* cycle, const aggmg_solver_config* cfg, double* x,
               aggmg_solve_report* rep, bool use_pcg) {
  return guarded([&] {
    const aggmg::SparseMatrix M = to_ref(A);
    const int64_t n = A->n_rows;
    aggmg::Preconditioner P;
    const aggmg::CycleConfig cc = to_ref(cycle);
    if (hp) {
      const auto* h = static_cast<const RefHierarchy*>(hp);
      P = [h, cc](const aggmg::Vector& r) { return aggmg::apply_preconditioner(h->h, cc, r); };
    }
    const aggmg::SolverConfig sc = to_ref(cfg);
    auto res = use_pcg ? aggmg::pcg(M, vec(b, n), vec(x0, n), P, sc)
                       : aggmg::fgmres(M, vec(b, n), vec(x0, n), P, sc);
    std::memcpy(x, res.x.data(), sizeof(double) * n);
    fill_report(res.report, rep);
  });
}
int aggmg_ref_pcg(const aggmg_csr* A, const double* b, const double* x0, const void* h,
                  const aggmg_cycle_config* c, const aggmg_solver_config* s, double* x,
                  aggmg_solve_report* r) {
  return run(A, b, x0, h, c, s, x, r, true);
}
int aggmg_ref_fgmres(const aggmg_csr* A, const double* b, const double* x0, const void* h,
                     const aggmg_cycle_config* c, const aggmg_solver_config* s, double* x,
                     aggmg_solve_report* r) {
  return run(A, b, x0, h, c, s, x, r, false);
}

// the reference's Krylov solvers with a host callback preconditioner (any std::function)
static int run_cb(const aggmg_csr* A, const double* b, const double* x0, aggmg_precond_fn fn,
                  void* user, const aggmg_solver_config* cfg, double* x, aggmg_solve_report* rep,
                  bool use_pcg) {
  return guarded([&] {
    const aggmg::SparseMatrix M = to_ref(A);
    const int64_t n = A->n_rows;
    aggmg::Preconditioner P;
    if (fn)
      P = [fn, user](const aggmg::Vector& r) {
        aggmg::Vector z(r.size());
        if (fn(r.data(), z.data(), static_cast<int64_t>(r.size()), user) != 0)
          throw aggmg::Error("krylov: the preconditioner callback failed");
        return z;
      };
    const aggmg::SolverConfig sc = to_ref(cfg);
    auto res = use_pcg ? aggmg::pcg(M, vec(b, n), vec(x0, n), P, sc)
                       : aggmg::fgmres(M, vec(b, n), vec(x0, n), P, sc);
    std::memcpy(x, res.x.data(), sizeof(double) * n);
    fill_report(res.report, rep);
  });
}
int aggmg_ref_pcg_cb(const aggmg_csr* A, const double* b, const double* x0, aggmg_precond_fn fn,
                     void* user, const aggmg_solver_config* s, double* x, aggmg_solve_report* r) {
  return run_cb(A, b, x0, fn, user, s, x, r, true);
}
int aggmg_ref_fgmres_cb(const aggmg_csr* A, const double* b, const double* x0, aggmg_precond_fn fn,
                        void* user, const aggmg_solver_config* s, double* x, aggmg_solve_report* r) {
  return run_cb(A, b, x0, fn, user, s, x, r, false);
}

// Reference CLI pipeline (aggmg_main.cpp:163-210): setup then solve, timed separately.
int aggmg_ref_setup_and_solve(const aggmg_csr* A, const double* b, const double* B0,
                              const double* x0, const aggmg_setup_config* setup,
                              const aggmg_cycle_config* cycle, const aggmg_solver_config* solver,
                              double* x, aggmg_solve_report* rep) {
  return guarded([&] {
    const int64_t n = A->n_rows;
    const auto t0 = std::chrono::steady_clock::now();
    aggmg::SparseMatrix M = to_ref(A);
    aggmg::Hierarchy h = aggmg::setup_hierarchy(M, B0 ? vec(B0, n) : aggmg::ones_vector(n), to_ref(setup));
    const double setup_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    const aggmg::CycleConfig cc = to_ref(cycle);
    aggmg::Preconditioner P = [&h, cc](const aggmg::Vector& r) { return aggmg::apply_preconditioner(h, cc, r); };
    const aggmg::SolverConfig sc = to_ref(solver);
    aggmg::Vector xv = x0 ? vec(x0, n) : aggmg::Vector(n, 0.0);
    auto res = sc.method == aggmg::SolverMethod::pcg ? aggmg::pcg(M, vec(b, n), xv, P, sc)
                                                     : aggmg::fgmres(M, vec(b, n), xv, P, sc);
    std::memcpy(x, res.x.data(), sizeof(double) * n);
    fill_report(res.report, rep);
    if (rep) rep->setup_seconds = setup_s;
  });
}

}  // extern "C"
