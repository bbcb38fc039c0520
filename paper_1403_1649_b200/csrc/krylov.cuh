// krylov.cuh — flexible PCG and restarted FGMRES (reference krylov.cpp:36-201) with all
// vectors in HBM.  The host keeps only the scalar recurrences it must branch on.
#pragma once

#include <string>
#include <vector>

#include "cycles.cuh"

namespace aggmg_b200 {

struct SolverCfg {
  int method = 0;  // 0 fgmres, 1 pcg
  double tol = 1e-6;
  int max_iters = 200;
  int restart = 30;
};

struct SolveOut {
  bool converged = false;
  int iterations = 0;
  std::vector<double> history;
  double solve_seconds = 0.0;
  std::string note;
};

// Preconditioner: nullptr hierarchy = identity (krylov.cpp:23-25).
struct Precond {
  DevHierarchy* h = nullptr;
  CycleCfg cfg;
};

// x (device, n) holds x0 on entry and the solution on exit.
SolveOut pcg(const DevCsr& A, const double* b, double* x, const Precond& M, const SolverCfg& cfg);
SolveOut fgmres(const DevCsr& A, const double* b, double* x, const Precond& M,
                const SolverCfg& cfg);

}  // namespace aggmg_b200
