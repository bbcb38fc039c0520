// cpp_dropin_demo.cpp — a reference-style C++ caller compiled against the drop-in
// header (include/aggmg/aggmg.hpp) and linked with the B200 library.  It re-runs the
// reference's acceptance criteria that exercise the public setup/solve API
// (acceptance_main.cpp:68-139, :356-417) and prints one PASS/FAIL line per criterion.
//
//   built by `make` (see the Makefile rule for build/cpp_dropin_demo)
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <random>
#include <string>
#include <tuple>
#include <vector>

#include "aggmg/aggmg.hpp"

using namespace aggmg;

namespace {

SparseMatrix poisson2d(index_t nx, index_t ny, double eps = 1.0) {
  PoissonSpec ps;
  ps.nx = nx;
  ps.ny = ny;
  ps.epsilon = eps;
  return generate_poisson(ps);
}

int failures = 0;
void report(const char* name, bool ok, const std::string& detail) {
  std::printf("%s %s: %s\n", ok ? "PASS" : "FAIL", name, detail.c_str());
  if (!ok) ++failures;
}

// acceptance_main.cpp:68-96 — hierarchy sparsity bounds on the 1000^2 anisotropic problem
void criterion_sparsity() {
  const SparseMatrix A = poisson2d(1000, 1000, 0.01);
  SetupConfig cfg;
  cfg.keep_host_levels = false;
  const Hierarchy h = setup_hierarchy(A, ones_vector(A.n_rows), cfg);
  const HierarchyReport rep = hierarchy_report(h);
  double worst = 0.0;
  for (size_t k = 1; k < rep.levels.size(); ++k) worst = std::max(worst, rep.levels[k].nnz_per_row);
  const bool ok = A.n_rows == 1000000 && A.nnz() == 4996000 && worst <= 8.0 &&
                  rep.operator_complexity <= 1.7;
  report("sparsity", ok,
         std::to_string(rep.levels.size()) + " levels, max coarse nnz/row " + std::to_string(worst) +
             ", operator complexity " + std::to_string(rep.operator_complexity));
  std::printf("%s", format_table(rep).c_str());
}

int iterations(const SparseMatrix& A, CycleKind kind) {
  SetupConfig scfg;
  scfg.keep_host_levels = false;
  const Hierarchy h = setup_hierarchy(A, ones_vector(A.n_rows), scfg);
  CycleConfig c;
  c.kind = kind;
  SolverConfig k;
  k.tol = 1e-6;
  k.max_iters = 500;
  const SolveResult r = fgmres(A, ones_vector(A.n_rows), Vector(A.n_rows, 0.0),
                               amg_preconditioner(h, c), k);
  return r.report.converged ? r.report.iterations : k.max_iters;
}

// acceptance_main.cpp:100-139 — grid-independent convergence of the hybrid cycle
void criterion_grid_independence() {
  std::vector<int> hyb, vee;
  for (index_t s : {index_t{64}, index_t{128}, index_t{256}}) {
    const SparseMatrix A = poisson2d(s, s);
    hyb.push_back(iterations(A, CycleKind::hybrid));
    vee.push_back(iterations(A, CycleKind::v));
  }
  auto ratio = [](const std::vector<int>& v) {
    return double(*std::max_element(v.begin(), v.end())) / *std::min_element(v.begin(), v.end());
  };
  const bool ok = *std::max_element(hyb.begin(), hyb.end()) <= 30 && ratio(hyb) <= 1.5 &&
                  ratio(vee) > ratio(hyb);
  report("grid_independence", ok,
         "hybrid {" + std::to_string(hyb[0]) + ", " + std::to_string(hyb[1]) + ", " +
             std::to_string(hyb[2]) + "}, V {" + std::to_string(vee[0]) + ", " +
             std::to_string(vee[1]) + ", " + std::to_string(vee[2]) + "}");
}

// acceptance_main.cpp:356-388 — refresh reuses the symbolic setup and is faster
void criterion_refresh() {
  using Clock = std::chrono::steady_clock;
  const SparseMatrix A = poisson2d(512, 512);
  SetupConfig cfg;
  cfg.reuse_caches = true;
  cfg.keep_host_levels = false;
  Hierarchy h = setup_hierarchy(A, ones_vector(A.n_rows), cfg);
  std::vector<double> v(A.values);
  for (double& x : v) x *= 2.0;
  auto t0 = Clock::now();
  h = refresh_values(std::move(h), v);
  const double t_refresh = std::chrono::duration<double>(Clock::now() - t0).count();
  SparseMatrix A2 = A;
  A2.values = v;
  t0 = Clock::now();
  const Hierarchy fresh = setup_hierarchy(A2, ones_vector(A.n_rows), cfg);
  const double t_setup = std::chrono::duration<double>(Clock::now() - t0).count();
  report("refresh", fresh.n_levels() == h.n_levels(),
         "refresh " + std::to_string(t_refresh * 1e3) + " ms vs fresh setup " +
             std::to_string(t_setup * 1e3) + " ms");
}

// acceptance_main.cpp:392-417 — histories are reproducible run to run
void criterion_determinism() {
  const SparseMatrix A = poisson2d(128, 128);
  std::vector<double> first;
  bool same = true;
  int its = 0;
  for (int run = 0; run < 3; ++run) {
    SetupConfig cfg;
    cfg.keep_host_levels = false;
    const Hierarchy h = setup_hierarchy(A, ones_vector(A.n_rows), cfg);
    SolverConfig k;
    k.tol = 1e-6;
    const SolveResult r = fgmres(A, ones_vector(A.n_rows), Vector(A.n_rows, 0.0),
                                 amg_preconditioner(h, CycleConfig{}), k);
    its = r.report.iterations;
    if (run == 0)
      first = r.report.residual_history;
    else
      same = same && r.report.residual_history == first;
  }
  report("determinism", same, std::to_string(its) + " iterations, histories bit-identical over 3 runs");
}

// ---- reference caller code, unchanged in form ----------------------------------------

// aggmg_main.cpp:163-210 (run_pipeline): the CLI wires the preconditioner as a LAMBDA around
// apply_preconditioner, not through amg_preconditioner(); the drop-in must accept it.
struct Outcome {
  SolveReport report;
  HierarchyReport hierarchy;
};
Outcome run_pipeline(const SparseMatrix& A, const Vector& b, SolverMethod method) {
  SetupConfig scfg;
  scfg.reuse_caches = true;
  const Hierarchy h = setup_hierarchy(A, ones_vector(A.n_rows), scfg);
  CycleConfig ccfg;
  SolverConfig kcfg;
  kcfg.method = method;
  kcfg.tol = 1e-8;
  kcfg.max_iters = 500;
  const Preconditioner M = [&](const Vector& r) { return apply_preconditioner(h, ccfg, r); };
  const Vector x0(A.n_rows, 0.0);
  SolveResult res = (kcfg.method == SolverMethod::pcg) ? pcg(A, b, x0, M, kcfg)
                                                       : fgmres(A, b, x0, M, kcfg);
  return {std::move(res.report), hierarchy_report(h)};
}

void criterion_cli_lambda() {
  const SparseMatrix A = poisson2d(256, 256);
  const Vector b = ones_vector(A.n_rows);
  for (SolverMethod m : {SolverMethod::pcg, SolverMethod::fgmres}) {
    const Outcome lam = run_pipeline(A, b, m);
    // the same solve with the device-resident preconditioner
    SetupConfig scfg;
    scfg.reuse_caches = true;
    const Hierarchy h = setup_hierarchy(A, ones_vector(A.n_rows), scfg);
    SolverConfig k;
    k.method = m;
    k.tol = 1e-8;
    k.max_iters = 500;
    const SolveResult dev = m == SolverMethod::pcg
                                ? pcg(A, b, Vector(A.n_rows, 0.0), amg_preconditioner(h, {}), k)
                                : fgmres(A, b, Vector(A.n_rows, 0.0), amg_preconditioner(h, {}), k);
    double worst = 0.0;
    const auto& hl = lam.report.residual_history;
    const auto& hd = dev.report.residual_history;
    for (size_t i = 0; i < std::min(hl.size(), hd.size()); ++i)
      worst = std::max(worst, std::abs(hl[i] - hd[i]) / hd[0]);
    const bool ok = lam.report.converged && lam.report.iterations == dev.report.iterations &&
                    hl.size() == hd.size() && worst <= 1e-10;
    report(m == SolverMethod::pcg ? "cli_lambda_pcg" : "cli_lambda_fgmres", ok,
           std::to_string(lam.report.iterations) + " iterations (lambda) vs " +
               std::to_string(dev.report.iterations) + " (device cycle), max |dh|/h0 " +
               std::to_string(worst));
  }
}

// tests/support/test_helpers.hpp:34-77 generators (std::mt19937_64 + uniform_real_distribution,
// the same libstdc++ sequences), assembled as triplets_to_csr does (rows, then ascending columns)
SparseMatrix random_spd(index_t n, double density, std::uint64_t seed) {
  std::mt19937_64 g(seed);
  std::uniform_real_distribution<double> val(-1.0, 1.0);
  std::uniform_real_distribution<double> coin(0.0, 1.0);
  std::vector<std::tuple<index_t, index_t, double>> t;
  std::vector<double> rowsum(n, 0.0);
  for (index_t i = 0; i < n; ++i)
    for (index_t j = i + 1; j < n; ++j)
      if (coin(g) < density) {
        const double v = val(g);
        t.emplace_back(i, j, v);
        t.emplace_back(j, i, v);
        rowsum[i] += std::abs(v);
        rowsum[j] += std::abs(v);
      }
  for (index_t i = 0; i < n; ++i) t.emplace_back(i, i, rowsum[i] + 1.0);
  std::sort(t.begin(), t.end(), [](const auto& a, const auto& b) {
    return std::tie(std::get<0>(a), std::get<1>(a)) < std::tie(std::get<0>(b), std::get<1>(b));
  });
  SparseMatrix A(n, n);
  for (const auto& [i, j, v] : t) {
    A.col_indices.push_back(j);
    A.values.push_back(v);
    ++A.row_offsets[i + 1];
  }
  for (index_t i = 0; i < n; ++i) A.row_offsets[i + 1] += A.row_offsets[i];
  return A;
}
Vector random_dense_vector(index_t n, std::uint64_t seed) {
  std::mt19937_64 g(seed);
  std::uniform_real_distribution<double> d(-1.0, 1.0);
  Vector v(n);
  for (auto& x : v) x = d(g);
  return v;
}
// test_helpers.hpp:335-370: textbook PCG on dense matrices
std::vector<double> reference_pcg(const SparseMatrix& A, const Vector& b, const Vector& dinv,
                                  int max_iters, double tol) {
  const index_t n = A.n_rows;
  auto mul = [&](const Vector& v) {
    Vector y(n, 0.0);
    for (index_t i = 0; i < n; ++i)
      for (index_t j = 0; j < n; ++j) y[i] += A.at(i, j) * v[j];
    return y;
  };
  auto norm = [](const Vector& v) {
    double s = 0.0;
    for (double y : v) s += y * y;
    return std::sqrt(s);
  };
  auto vdot = [](const Vector& a, const Vector& c) {
    double s = 0.0;
    for (size_t i = 0; i < a.size(); ++i) s += a[i] * c[i];
    return s;
  };
  Vector x(n, 0.0), r = b;
  std::vector<double> history{norm(r)};
  const double target = tol * norm(b);
  Vector z(n);
  for (index_t i = 0; i < n; ++i) z[i] = dinv[i] * r[i];
  Vector p = z;
  double rz = vdot(r, z);
  for (int it = 0; it < max_iters && norm(r) > target; ++it) {
    const Vector Ap = mul(p);
    const double alpha = rz / vdot(p, Ap);
    for (index_t i = 0; i < n; ++i) x[i] += alpha * p[i];
    for (index_t i = 0; i < n; ++i) r[i] -= alpha * Ap[i];
    history.push_back(norm(r));
    for (index_t i = 0; i < n; ++i) z[i] = dinv[i] * r[i];
    const double rz_new = vdot(r, z);
    const double beta = rz_new / rz;
    for (index_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
    rz = rz_new;
  }
  return history;
}

// test_krylov.cpp:129-156 "jacobi-preconditioned cg matches the dense reference history",
// the test body unchanged: the preconditioner is a plain host lambda
void criterion_jacobi_pcg() {
  const SparseMatrix A = random_spd(20, 0.3, 4010);
  const Vector b = random_dense_vector(20, 4011);
  SolverConfig cfg;
  cfg.tol = 1e-10;
  cfg.max_iters = 100;
  const Preconditioner jacobi = [&](const Vector& r) {
    Vector z(r.size());
    for (index_t i = 0; i < A.n_rows; ++i) z[i] = r[i] / A.at(i, i);
    return z;
  };
  Vector dinv(20);
  for (index_t i = 0; i < 20; ++i) dinv[i] = 1.0 / A.at(i, i);
  const SolveResult s = pcg(A, b, Vector(20, 0.0), jacobi, cfg);
  const std::vector<double> ref = reference_pcg(A, b, dinv, cfg.max_iters, cfg.tol);
  bool ok = s.report.converged && s.report.residual_history.size() == ref.size();
  for (size_t k = 0; ok && k < ref.size(); ++k) {
    const double tol = std::max(2e-2 * ref[k], 1e-12 * ref[0]);
    ok = std::abs(s.report.residual_history[k] - ref[k]) <= tol;
  }
  report("jacobi_pcg", ok,
         std::to_string(s.report.iterations) + " iterations, history of " +
             std::to_string(s.report.residual_history.size()) + " vs dense reference " +
             std::to_string(ref.size()));
}

// hierarchy.cpp:90: refresh_values takes the hierarchy by value — the caller's copy must keep
// solving the OLD system after `auto h2 = refresh_values(h, v)`
void criterion_refresh_value_semantics() {
  const SparseMatrix A = poisson2d(200, 200);
  SetupConfig cfg;
  cfg.reuse_caches = true;
  const Hierarchy h = setup_hierarchy(A, ones_vector(A.n_rows), cfg);
  SolverConfig k;
  k.method = SolverMethod::pcg;
  k.tol = 1e-8;
  const Vector b = ones_vector(A.n_rows), x0(A.n_rows, 0.0);
  const SolveResult before = pcg(A, b, x0, amg_preconditioner(h, {}), k);
  std::vector<double> v(A.values);
  for (index_t i = 0; i < A.n_rows; ++i)
    for (index_t e = A.row_offsets[i]; e < A.row_offsets[i + 1]; ++e)
      if (A.col_indices[e] == i) v[e] *= 1.5;  // a different operator on the same pattern
  const Hierarchy h2 = refresh_values(h, v);
  SparseMatrix A2 = A;
  A2.values = v;
  const SolveResult after_old = pcg(A, b, x0, amg_preconditioner(h, {}), k);
  const SolveResult fresh = pcg(A2, b, x0, amg_preconditioner(setup_hierarchy(A2, ones_vector(A.n_rows), cfg), {}), k);
  const SolveResult after_new = pcg(A2, b, x0, amg_preconditioner(h2, {}), k);
  const bool ok = after_old.report.residual_history == before.report.residual_history &&
                  after_new.report.iterations == fresh.report.iterations &&
                  h.levels[1].A.values != h2.levels[1].A.values;
  report("refresh_value_semantics", ok,
         "old hierarchy " + std::to_string(after_old.report.iterations) + " its (unchanged), refreshed " +
             std::to_string(after_new.report.iterations) + " its vs fresh setup " +
             std::to_string(fresh.report.iterations));
}

}  // namespace

int main() {
  try {
    criterion_sparsity();
    criterion_grid_independence();
    criterion_refresh();
    criterion_determinism();
    criterion_cli_lambda();
    criterion_jacobi_pcg();
    criterion_refresh_value_semantics();
  } catch (const Error& e) {
    std::printf("FAIL exception: %s\n", e.what());
    return 1;
  }
  return failures;
}
