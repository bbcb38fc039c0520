// cpp_dropin_demo.cpp — a reference-style C++ caller compiled against the drop-in
// header (include/aggmg/aggmg.hpp) and linked with the B200 library.  It re-runs the
// reference's acceptance criteria that exercise the public setup/solve API
// (acceptance_main.cpp:68-139, :356-417) and prints one PASS/FAIL line per criterion.
//
//   built by `make` (see the Makefile rule for build/cpp_dropin_demo)
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <string>
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

}  // namespace

int main() {
  try {
    criterion_sparsity();
    criterion_grid_independence();
    criterion_refresh();
    criterion_determinism();
  } catch (const Error& e) {
    std::printf("FAIL exception: %s\n", e.what());
    return 1;
  }
  return failures;
}
