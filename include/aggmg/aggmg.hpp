// aggmg/aggmg.hpp — header-only C++ drop-in for the reference `aggmg` setup/solve API
// (/root/reference/proj/core/include/aggmg/*.hpp), implemented over the C-ABI in
// aggmg_b200.h (link with paper_1403_1649_b200/lib/libaggmg_b200.so).
//
// Names, value types, defaults and error behaviour follow the reference so existing
// callers compile unchanged:
//   types.hpp:12-16      index_t, Vector                    error.hpp:14-27  Error, require
//   sparse.hpp:18-82     SparseMatrix, spmv, transpose      vector_ops.hpp   dot/norm2/axpy/scale
//   strength.hpp:15-31   classic_strength, influence_counts, symmetrize_pattern
//   aggregation.hpp      Mis2Result, mis2, Aggregation, aggregate
//   transfer.hpp         TransferOperators, build_transfer
//   galerkin.hpp         galerkin_direct, GalerkinCache, build/apply_galerkin_cache
//   smoother.hpp         SmootherKind, SmootherState, setup_smoother, smooth
//   hierarchy.hpp        SetupConfig, Level, Hierarchy, setup_hierarchy, refresh_values,
//                        hierarchy_report, format_table, format_records
//   cycles.hpp           CycleKind, InnerKind, CycleConfig, vcycle, kcycle, apply_preconditioner
//   krylov.hpp           SolverConfig, SolveReport, SolveResult, Preconditioner, fgmres, pcg
//   poisson.hpp          PoissonSpec, generate_poisson, ones_vector, random_vector
//   matrix_market.hpp    MmOptions, read/write_matrix_market_file, read/write_vector_market_file
// Differences, by design: the hierarchy lives in HBM (Hierarchy::device); the host copies of
// its levels (Hierarchy::levels) are materialised on first access.  pcg/fgmres take any
// Preconditioner: the AMG preconditioner returned by amg_preconditioner() runs inside the
// device Krylov loop; any other callable (a lambda around apply_preconditioner, a Jacobi
// scaling, ...) is called on the host once per application, with r and z copied across.
#ifndef AGGMG_B200_AGGMG_HPP
#define AGGMG_B200_AGGMG_HPP

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <functional>
#include <iomanip>
#include <exception>
#include <memory>
#include <mutex>
#include <span>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "../aggmg_b200.h"

namespace aggmg {

using index_t = std::int64_t;
using Vector = std::vector<double>;
inline constexpr const char* version() { return "0.1.0"; }

class Error : public std::runtime_error {
 public:
  explicit Error(const std::string& what) : std::runtime_error(what) {}
};
inline void require(bool cond, const std::string& msg) {
  if (!cond) throw Error(msg);
}

namespace detail {
inline void check(int rc) {
  if (rc != AGGMG_OK) throw Error(aggmg_last_error());
}
}  // namespace detail

inline void set_num_threads(int n) { aggmg_set_num_threads(n); }
// B200 extension: bit-identical solves (see aggmg_set_exact_reductions in aggmg_b200.h)
inline void set_exact_reductions(bool on) { aggmg_set_exact_reductions(on ? 1 : 0); }
inline int num_threads() { return aggmg_num_threads(); }

// ---- sparse.hpp ------------------------------------------------------------------------

struct SparseMatrix {
  index_t n_rows = 0;
  index_t n_cols = 0;
  std::vector<index_t> row_offsets;
  std::vector<index_t> col_indices;
  std::vector<double> values;

  SparseMatrix() : row_offsets(1, 0) {}
  SparseMatrix(index_t rows, index_t cols)
      : n_rows(rows), n_cols(cols), row_offsets(static_cast<size_t>(rows) + 1, 0) {}
  index_t nnz() const { return static_cast<index_t>(col_indices.size()); }
  double at(index_t i, index_t j) const {
    for (index_t k = row_offsets[i]; k < row_offsets[i + 1]; ++k)
      if (col_indices[k] == j) return values[k];
    return 0.0;
  }
  aggmg_csr c() const {
    return aggmg_csr{n_rows, n_cols, nnz(), const_cast<index_t*>(row_offsets.data()),
                     const_cast<index_t*>(col_indices.data()), const_cast<double*>(values.data())};
  }
  static SparseMatrix adopt(aggmg_csr& m) {  // take a library-allocated result
    SparseMatrix A(m.n_rows, m.n_cols);
    A.row_offsets.assign(m.row_offsets, m.row_offsets + m.n_rows + 1);
    A.col_indices.assign(m.col_indices, m.col_indices + m.nnz);
    A.values.assign(m.values, m.values + m.nnz);
    aggmg_csr_free(&m);
    return A;
  }
};

inline Vector spmv(const SparseMatrix& A, const Vector& x) {
  require(static_cast<index_t>(x.size()) == A.n_cols,
          "spmv: matrix has " + std::to_string(A.n_cols) + " columns but vector has " +
              std::to_string(x.size()) + " entries");
  Vector y(A.n_rows);
  const aggmg_csr c = A.c();
  detail::check(aggmg_spmv(&c, x.data(), y.data()));
  return y;
}
inline SparseMatrix transpose(const SparseMatrix& A) {
  const aggmg_csr c = A.c();
  aggmg_csr out{};
  detail::check(aggmg_transpose(&c, &out));
  return SparseMatrix::adopt(out);
}

// ---- vector_ops.hpp (reference 8192-chunk order) ------------------------------------------

inline double dot(std::span<const double> a, std::span<const double> b) {
  require(a.size() == b.size(), "dot: length mismatch");
  double out = 0.0;
  detail::check(aggmg_dot(static_cast<int64_t>(a.size()), a.data(), b.data(), &out));
  return out;
}
inline double norm2(std::span<const double> a) {
  double out = 0.0;
  detail::check(aggmg_norm2(static_cast<int64_t>(a.size()), a.data(), &out));
  return out;
}
inline void axpy(double a, std::span<const double> x, std::span<double> y) {
  require(x.size() == y.size(), "axpy: length mismatch");
  detail::check(aggmg_axpy(static_cast<int64_t>(x.size()), a, x.data(), y.data()));
}
inline void scale(double a, std::span<double> x) {
  detail::check(aggmg_scale(static_cast<int64_t>(x.size()), a, x.data()));
}

// ---- strength / aggregation / transfer / galerkin ------------------------------------------

enum class ZeroDiagPolicy { positive, fail };
inline SparseMatrix classic_strength(const SparseMatrix& A, double alpha,
                                     ZeroDiagPolicy p = ZeroDiagPolicy::positive) {
  const aggmg_csr c = A.c();
  aggmg_csr out{};
  detail::check(aggmg_classic_strength(&c, alpha, p == ZeroDiagPolicy::fail, &out));
  return SparseMatrix::adopt(out);
}
inline std::vector<index_t> influence_counts(const SparseMatrix& C) {
  std::vector<index_t> v(C.n_cols);
  const aggmg_csr c = C.c();
  detail::check(aggmg_influence_counts(&c, v.data()));
  return v;
}
inline SparseMatrix symmetrize_pattern(const SparseMatrix& C) {
  const aggmg_csr c = C.c();
  aggmg_csr out{};
  detail::check(aggmg_symmetrize_pattern(&c, &out));
  return SparseMatrix::adopt(out);
}

struct Mis2Result {
  std::vector<std::int8_t> state;
  std::vector<index_t> roots;
  int sweeps = 0;
};
inline Mis2Result mis2(const SparseMatrix& S, const std::vector<index_t>& influence,
                       std::uint64_t seed) {
  require(static_cast<index_t>(influence.size()) == S.n_rows, "mis2: influence length mismatch");
  Mis2Result r;
  r.state.resize(S.n_rows);
  int64_t nr = 0;
  int32_t sw = 0;
  const aggmg_csr c = S.c();
  detail::check(aggmg_mis2(&c, influence.data(), seed, r.state.data(), &nr, &sw));
  r.sweeps = sw;
  for (index_t i = 0; i < S.n_rows; ++i)
    if (r.state[i] == 1) r.roots.push_back(i);
  return r;
}

struct Aggregation {
  index_t n_fine = 0;
  index_t n_aggregates = 0;
  std::vector<index_t> assignment;
  std::vector<index_t> representatives;
};
inline Aggregation aggregate(const SparseMatrix& S, const SparseMatrix& A, const Mis2Result& mis) {
  Aggregation g;
  g.n_fine = S.n_rows;
  g.assignment.resize(S.n_rows);
  g.representatives.resize(S.n_rows);
  const aggmg_csr cs = S.c(), ca = A.c();
  detail::check(aggmg_aggregate(&cs, &ca, mis.state.data(), g.assignment.data(),
                                g.representatives.data(), &g.n_aggregates));
  g.representatives.resize(g.n_aggregates);
  return g;
}

struct TransferOperators {
  SparseMatrix P, R;
  Vector coarse_b;
};
inline TransferOperators build_transfer(const Aggregation& agg, const Vector& fine_b) {
  require(static_cast<index_t>(fine_b.size()) == agg.n_fine,
          "transfer: near-null-space vector length mismatch");
  TransferOperators t;
  t.coarse_b.resize(agg.n_aggregates);
  aggmg_csr P{}, R{};
  detail::check(aggmg_build_transfer(agg.n_fine, agg.n_aggregates, agg.assignment.data(),
                                     fine_b.data(), &P, &R, t.coarse_b.data()));
  t.P = SparseMatrix::adopt(P);
  t.R = SparseMatrix::adopt(R);
  return t;
}

inline SparseMatrix galerkin_direct(const SparseMatrix& R, const SparseMatrix& A,
                                    const SparseMatrix& P) {
  const aggmg_csr cr = R.c(), ca = A.c(), cp = P.c();
  aggmg_csr out{};
  detail::check(aggmg_galerkin_direct(&cr, &ca, &cp, &out));
  return SparseMatrix::adopt(out);
}

struct GalerkinCache {
  index_t n_fine = 0, n_coarse = 0;
  std::vector<index_t> coarse_row_offsets, coarse_col_indices, entry, entry_row,
      segment_offsets, slot_of_csr, rows_by_coarse, agg_row_offsets;
  std::shared_ptr<aggmg_galerkin_cache> device;
};
inline GalerkinCache build_galerkin_cache(const SparseMatrix& A, const Aggregation& agg) {
  const aggmg_csr ca = A.c();
  aggmg_galerkin_cache* h = nullptr;
  detail::check(aggmg_build_galerkin_cache(&ca, agg.n_aggregates, agg.assignment.data(), &h));
  GalerkinCache c;
  c.device.reset(h, aggmg_galerkin_cache_free);
  int64_t nnzf = 0, nnzc = 0;
  detail::check(aggmg_galerkin_cache_info(h, &c.n_fine, &c.n_coarse, &nnzf, &nnzc));
  c.coarse_row_offsets.resize(c.n_coarse + 1);
  c.coarse_col_indices.resize(nnzc);
  c.entry.resize(nnzf);
  c.entry_row.resize(nnzf);
  c.segment_offsets.resize(nnzc + 1);
  c.slot_of_csr.resize(nnzf);
  c.rows_by_coarse.resize(c.n_fine);
  c.agg_row_offsets.resize(c.n_coarse + 1);
  detail::check(aggmg_galerkin_cache_export(
      h, c.coarse_row_offsets.data(), c.coarse_col_indices.data(), c.entry.data(),
      c.entry_row.data(), c.segment_offsets.data(), c.slot_of_csr.data(), c.rows_by_coarse.data(),
      c.agg_row_offsets.data()));
  return c;
}
inline SparseMatrix apply_galerkin_cache(const GalerkinCache& c, const SparseMatrix& A,
                                         const SparseMatrix& P) {
  const aggmg_csr ca = A.c(), cp = P.c();
  aggmg_csr out{};
  detail::check(aggmg_apply_galerkin_cache(c.device.get(), &ca, &cp, &out));
  return SparseMatrix::adopt(out);
}

// ---- smoother.hpp ----------------------------------------------------------------------------

enum class SmootherKind { jacobi, damped_jacobi, sgs };
struct SmootherState {
  SmootherKind kind = SmootherKind::damped_jacobi;
  Vector inv_diag;
  double omega = 1.0;
  double rho_est = 1.0;
  int arnoldi_m = 5;
};
inline SmootherState setup_smoother(const SparseMatrix& A, SmootherKind kind, int arnoldi_m = 5,
                                    std::uint64_t seed = 0) {
  SmootherState s;
  s.kind = kind;
  s.arnoldi_m = arnoldi_m;
  s.inv_diag.resize(A.n_rows);
  const aggmg_csr ca = A.c();
  detail::check(aggmg_setup_smoother(&ca, static_cast<int>(kind), arnoldi_m, seed,
                                     s.inv_diag.data(), &s.omega, &s.rho_est));
  return s;
}
inline void smooth(const SmootherState& s, const SparseMatrix& A, const Vector& b, Vector& x) {
  require(static_cast<index_t>(b.size()) == A.n_rows && static_cast<index_t>(x.size()) == A.n_rows,
          "smooth: vector length mismatch");
  const aggmg_csr ca = A.c();
  detail::check(aggmg_smooth(static_cast<int>(s.kind), s.inv_diag.data(), s.omega, &ca, b.data(),
                             x.data()));
}

// ---- hierarchy.hpp ---------------------------------------------------------------------------

struct SetupConfig {
  double alpha = 0.25;
  index_t coarse_size_max = 600;
  int max_levels = 25;
  SmootherKind smoother = SmootherKind::damped_jacobi;
  int arnoldi_m = 5;
  std::uint64_t seed = 42;
  bool reuse_caches = false;
  bool keep_host_levels = true;  // B200 addition (kept for source compatibility): levels are
                                 // always materialised lazily, on first access
  aggmg_setup_config c() const {
    return aggmg_setup_config{alpha, coarse_size_max, max_levels, static_cast<int32_t>(smoother),
                              arnoldi_m, reuse_caches ? 1 : 0, seed};
  }
};

struct Level {
  SparseMatrix A, P, R;
  Vector B;
  SmootherState smoother;
};

// Host view of the device levels (hierarchy.hpp:46 `std::vector<Level> levels`): the reads a
// reference caller makes (size, [k], at, front, back, iteration) materialise every level's
// A / P / R / B / smoother from HBM on first use, once, shared by copies of the Hierarchy.
class LevelList {
 public:
  LevelList() = default;
  LevelList(std::shared_ptr<aggmg_hierarchy> dev, SmootherKind kind)
      : state_(std::make_shared<State>()) {
    state_->dev = std::move(dev);
    state_->kind = kind;
  }
  size_t size() const {
    const auto dev = state_ ? state_->dev.lock() : nullptr;
    return dev ? static_cast<size_t>(aggmg_hierarchy_n_levels(dev.get())) : 0;
  }
  bool empty() const { return size() == 0; }
  const Level& operator[](size_t k) const { return all()[k]; }
  const Level& at(size_t k) const { return all().at(k); }
  const Level& front() const { return all().front(); }
  const Level& back() const { return all().back(); }
  std::vector<Level>::const_iterator begin() const { return all().begin(); }
  std::vector<Level>::const_iterator end() const { return all().end(); }

 private:
  struct State {
    std::weak_ptr<aggmg_hierarchy> dev;  // not an owner: Hierarchy::device's use count stays
                                         // the number of Hierarchy values holding it
    SmootherKind kind = SmootherKind::damped_jacobi;
    std::once_flag once;
    std::vector<Level> levels;
  };
  static void check(int rc) {
    if (rc != AGGMG_OK) throw Error(aggmg_last_error());
  }
  const std::vector<Level>& all() const {
    static const std::vector<Level> none;
    if (!state_) return none;
    std::call_once(state_->once, [s = state_.get()] {
      const auto dev = s->dev.lock();
      require(dev != nullptr, "hierarchy: levels read after the hierarchy was destroyed");
      const int64_t L = aggmg_hierarchy_n_levels(dev.get());
      for (int64_t k = 0; k < L; ++k) {
        Level lvl;
        aggmg_csr m{};
        check(aggmg_hierarchy_level_A(dev.get(), k, &m));
        lvl.A = SparseMatrix::adopt(m);
        check(aggmg_hierarchy_level_P(dev.get(), k, &m));
        lvl.P = SparseMatrix::adopt(m);
        check(aggmg_hierarchy_level_R(dev.get(), k, &m));
        lvl.R = SparseMatrix::adopt(m);
        lvl.B.resize(lvl.A.n_rows);
        check(aggmg_hierarchy_level_B(dev.get(), k, lvl.B.data()));
        lvl.smoother.kind = s->kind;
        lvl.smoother.inv_diag.resize(lvl.A.n_rows);
        check(aggmg_hierarchy_level_smoother(dev.get(), k, &lvl.smoother.omega,
                                             &lvl.smoother.rho_est, lvl.smoother.inv_diag.data()));
        s->levels.push_back(std::move(lvl));
      }
    });
    return state_->levels;
  }
  std::shared_ptr<State> state_;
};

struct Hierarchy {
  LevelList levels;  // host view, materialised on first access
  SetupConfig config;
  std::vector<std::string> warnings;
  std::shared_ptr<aggmg_hierarchy> device;
  index_t n_levels() const { return device ? aggmg_hierarchy_n_levels(device.get()) : 0; }
  index_t coarsest() const { return n_levels() - 1; }
};

namespace detail {
inline void mirror(Hierarchy& h) {
  h.warnings.clear();
  for (int64_t i = 0; i < aggmg_hierarchy_n_warnings(h.device.get()); ++i)
    h.warnings.emplace_back(aggmg_hierarchy_warning(h.device.get(), i));
  h.levels = LevelList(h.device, h.config.smoother);
}
}  // namespace detail

inline Hierarchy setup_hierarchy(SparseMatrix A0, Vector B0, const SetupConfig& config) {
  require(static_cast<index_t>(B0.size()) == A0.n_rows,
          "setup: near-null-space vector length mismatch");
  const aggmg_csr ca = A0.c();
  const aggmg_setup_config cfg = config.c();
  aggmg_hierarchy* raw = nullptr;
  detail::check(aggmg_setup_hierarchy(&ca, B0.data(), &cfg, &raw));
  Hierarchy h;
  h.config = config;
  h.device.reset(raw, aggmg_hierarchy_free);
  detail::mirror(h);
  return h;
}

// hierarchy.cpp:90-104.  Value semantics as in the reference: when the caller still holds the
// hierarchy (auto h2 = refresh_values(h, v)), the refresh runs on a device copy and h keeps
// solving the old system; refresh_values(std::move(h), v) refreshes in place.
inline Hierarchy refresh_values(Hierarchy h, const std::vector<double>& new_values) {
  if (h.device.use_count() > 1) {
    aggmg_hierarchy* copy = nullptr;
    detail::check(aggmg_hierarchy_clone(h.device.get(), &copy));
    h.device.reset(copy, aggmg_hierarchy_free);
  }
  detail::check(aggmg_refresh_values(h.device.get(), new_values.data(),
                                     static_cast<int64_t>(new_values.size())));
  detail::mirror(h);
  return h;
}

struct LevelStats {
  index_t n = 0;
  index_t nnz = 0;
  double nnz_per_row = 0.0;
};
struct HierarchyReport {
  std::vector<LevelStats> levels;
  double grid_complexity = 0.0;
  double operator_complexity = 0.0;
};
inline HierarchyReport hierarchy_report(const Hierarchy& h) {  // hierarchy.cpp:106-121
  HierarchyReport r;
  double sn = 0.0, snnz = 0.0;
  for (index_t k = 0; k < h.n_levels(); ++k) {
    LevelStats s;
    detail::check(aggmg_hierarchy_level_size(h.device.get(), k, &s.n, &s.nnz));
    s.nnz_per_row = s.n > 0 ? static_cast<double>(s.nnz) / static_cast<double>(s.n) : 0.0;
    sn += static_cast<double>(s.n);
    snnz += static_cast<double>(s.nnz);
    r.levels.push_back(s);
  }
  r.grid_complexity = sn / static_cast<double>(r.levels.front().n);
  r.operator_complexity = snnz / static_cast<double>(r.levels.front().nnz);
  return r;
}
inline std::string format_table(const HierarchyReport& r) {
  std::ostringstream out;
  out << "level       unknowns            nnz   nnz/row\n";
  for (size_t k = 0; k < r.levels.size(); ++k)
    out << std::setw(5) << k << std::setw(15) << r.levels[k].n << std::setw(15) << r.levels[k].nnz
        << std::setw(10) << std::fixed << std::setprecision(2) << r.levels[k].nnz_per_row << "\n";
  out << "grid complexity     " << std::setprecision(4) << r.grid_complexity << "\n";
  out << "operator complexity " << std::setprecision(4) << r.operator_complexity << "\n";
  return out.str();
}
inline std::string format_records(const HierarchyReport& r) {
  std::ostringstream out;
  for (size_t k = 0; k < r.levels.size(); ++k)
    out << "level " << k << " " << r.levels[k].n << " " << r.levels[k].nnz << " "
        << std::setprecision(17) << r.levels[k].nnz_per_row << "\n";
  out << "grid_complexity " << std::setprecision(17) << r.grid_complexity << "\n";
  out << "operator_complexity " << std::setprecision(17) << r.operator_complexity << "\n";
  return out.str();
}

// ---- cycles.hpp ----------------------------------------------------------------------------

enum class CycleKind { v, k, hybrid };
enum class InnerKind { cg, gmres };
struct CycleConfig {
  CycleKind kind = CycleKind::hybrid;
  int k_levels = 2;
  double t = 0.25;
  InnerKind inner = InnerKind::gmres;
  aggmg_cycle_config c() const {
    return aggmg_cycle_config{kind == CycleKind::v ? AGGMG_CYCLE_V
                              : kind == CycleKind::k ? AGGMG_CYCLE_K
                                                     : AGGMG_CYCLE_HYBRID,
                              k_levels, t, inner == InnerKind::cg ? AGGMG_INNER_CG : AGGMG_INNER_GMRES};
  }
};

inline void vcycle(const Hierarchy& h, index_t k, const Vector& b, Vector& x) {
  detail::check(aggmg_vcycle(h.device.get(), k, b.data(), x.data()));
}
inline void kcycle(const Hierarchy& h, const CycleConfig& cfg, index_t k, const Vector& b,
                   Vector& x) {
  const aggmg_cycle_config c = cfg.c();
  detail::check(aggmg_kcycle(h.device.get(), &c, k, b.data(), x.data()));
}
inline Vector apply_preconditioner(const Hierarchy& h, const CycleConfig& cfg, const Vector& r) {
  Vector z(r.size());
  const aggmg_cycle_config c = cfg.c();
  detail::check(aggmg_apply_preconditioner(h.device.get(), &c, r.data(), z.data()));
  return z;
}

// ---- krylov.hpp ----------------------------------------------------------------------------

enum class SolverMethod { fgmres, pcg };
struct SolverConfig {
  SolverMethod method = SolverMethod::fgmres;
  double tol = 1e-6;
  int max_iters = 200;
  int restart = 30;
  aggmg_solver_config c() const {
    return aggmg_solver_config{method == SolverMethod::pcg ? AGGMG_SOLVER_PCG : AGGMG_SOLVER_FGMRES,
                               tol, max_iters, restart};
  }
};
struct SolveReport {
  bool converged = false;
  int iterations = 0;
  std::vector<double> residual_history;
  double setup_seconds = 0.0;
  double solve_seconds = 0.0;
  std::string note;
};
struct SolveResult {
  Vector x;
  SolveReport report;
};
using Preconditioner = std::function<Vector(const Vector&)>;

// The AMG preconditioner r -> apply_preconditioner(h, cfg, r) in a form the device
// Krylov solvers recognise (the call operator also works as a plain host callback).
struct AmgPreconditioner {
  std::shared_ptr<aggmg_hierarchy> device;
  CycleConfig cfg;
  Vector operator()(const Vector& r) const {
    Vector z(r.size());
    const aggmg_cycle_config c = cfg.c();
    detail::check(aggmg_apply_preconditioner(device.get(), &c, r.data(), z.data()));
    return z;
  }
};
inline Preconditioner amg_preconditioner(const Hierarchy& h, const CycleConfig& cfg) {
  return AmgPreconditioner{h.device, cfg};
}

namespace detail {
// C trampoline for an arbitrary host Preconditioner (aggmg_precond_fn); exceptions thrown by
// the callable are carried across the C boundary and rethrown by krylov()
struct HostPrecond {
  const Preconditioner* M = nullptr;
  std::exception_ptr error;
  static int call(const double* r, double* z, int64_t n, void* user) {
    auto* self = static_cast<HostPrecond*>(user);
    try {
      const Vector zv = (*self->M)(Vector(r, r + n));
      require(static_cast<int64_t>(zv.size()) == n, "krylov: preconditioner output length mismatch");
      std::copy(zv.begin(), zv.end(), z);
      return 0;
    } catch (...) {
      self->error = std::current_exception();
      return 1;
    }
  }
};

inline SolveResult krylov(bool use_pcg, const SparseMatrix& A, const Vector& b, const Vector& x0,
                          const Preconditioner& M, const SolverConfig& cfg) {
  const aggmg_hierarchy* h = nullptr;
  aggmg_cycle_config cc;
  aggmg_cycle_config_default(&cc);
  const AmgPreconditioner* amg = M ? M.target<AmgPreconditioner>() : nullptr;
  if (amg) {  // the device cycle, inside the device Krylov loop
    h = amg->device.get();
    cc = amg->cfg.c();
  }
  SolveResult out;
  out.x.resize(A.n_rows);
  out.report.residual_history.resize(static_cast<size_t>(cfg.max_iters) + 2);
  aggmg_solve_report rep{};
  rep.history = out.report.residual_history.data();
  rep.history_capacity = static_cast<int64_t>(out.report.residual_history.size());
  const aggmg_csr ca = A.c();
  const aggmg_solver_config sc = cfg.c();
  if (M && !amg) {  // any other callable: a host callback per application
    HostPrecond hp;
    hp.M = &M;
    const int rc = use_pcg ? aggmg_pcg_cb(&ca, b.data(), x0.data(), &HostPrecond::call, &hp, &sc,
                                          out.x.data(), &rep)
                           : aggmg_fgmres_cb(&ca, b.data(), x0.data(), &HostPrecond::call, &hp,
                                             &sc, out.x.data(), &rep);
    if (hp.error) std::rethrow_exception(hp.error);
    check(rc);
  } else {
    check(use_pcg ? aggmg_pcg(&ca, b.data(), x0.data(), h, &cc, &sc, out.x.data(), &rep)
                  : aggmg_fgmres(&ca, b.data(), x0.data(), h, &cc, &sc, out.x.data(), &rep));
  }
  out.report.converged = rep.converged != 0;
  out.report.iterations = rep.iterations;
  out.report.residual_history.resize(static_cast<size_t>(rep.history_length));
  out.report.solve_seconds = rep.solve_seconds;
  out.report.note = rep.note;
  return out;
}
}  // namespace detail

inline SolveResult fgmres(const SparseMatrix& A, const Vector& b, const Vector& x0,
                          const Preconditioner& M, const SolverConfig& cfg) {
  return detail::krylov(false, A, b, x0, M, cfg);
}
inline SolveResult pcg(const SparseMatrix& A, const Vector& b, const Vector& x0,
                       const Preconditioner& M, const SolverConfig& cfg) {
  return detail::krylov(true, A, b, x0, M, cfg);
}

// ---- poisson.hpp -----------------------------------------------------------------------------

struct PoissonSpec {
  int dims = 2;
  index_t nx = 0, ny = 0, nz = 1;
  double epsilon = 1.0;
  int weak_axis = -1;
};
inline SparseMatrix generate_poisson(const PoissonSpec& s) {
  aggmg_csr out{};
  detail::check(aggmg_generate_poisson(s.dims, s.nx, s.ny, s.nz, s.epsilon, s.weak_axis, &out));
  return SparseMatrix::adopt(out);
}
inline Vector ones_vector(index_t n) { return Vector(static_cast<size_t>(n), 1.0); }
inline Vector random_vector(index_t n, std::uint64_t seed) {  // poisson.hpp:30
  Vector x(static_cast<size_t>(n));
  detail::check(aggmg_random_vector(n, seed, x.data()));
  return x;
}

// ---- matrix_market.hpp ---------------------------------------------------------------------

struct MmOptions {
  bool allow_pattern = false;
};
inline SparseMatrix read_matrix_market_file(const std::string& path, const MmOptions& opts = {}) {
  aggmg_csr out{};
  detail::check(aggmg_read_matrix_market_file(path.c_str(), opts.allow_pattern ? 1 : 0, &out));
  return SparseMatrix::adopt(out);
}
inline void write_matrix_market_file(const std::string& path, const SparseMatrix& A) {
  const aggmg_csr c = A.c();
  detail::check(aggmg_write_matrix_market_file(path.c_str(), &c));
}
inline Vector read_vector_market_file(const std::string& path) {
  int64_t n = 0;
  detail::check(aggmg_read_vector_market_file(path.c_str(), nullptr, 0, &n));
  Vector x(static_cast<size_t>(n));
  detail::check(aggmg_read_vector_market_file(path.c_str(), x.data(), n, &n));
  return x;
}
inline void write_vector_market_file(const std::string& path, const Vector& x) {
  detail::check(aggmg_write_vector_market_file(path.c_str(), x.data(), static_cast<int64_t>(x.size())));
}

}  // namespace aggmg

#endif  // AGGMG_B200_AGGMG_HPP
