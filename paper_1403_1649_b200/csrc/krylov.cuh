// krylov.cuh — flexible PCG and restarted FGMRES (reference krylov.cpp:36-201) with all
// vectors in HBM.  The host keeps only the scalar recurrences it must branch on.
#pragma once

#include <functional>
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

// Host preconditioner z = M(r) over host arrays of n entries (the reference's std::function
// Preconditioner, krylov.hpp:38); nonzero return = failure.
using HostPrecondFn = int (*)(const double* r, double* z, int64_t n, void* user);

// Preconditioner: the device AMG cycle of h, or a host callback, or (neither) the identity
// (krylov.cpp:23-25).
struct Precond {
  DevHierarchy* h = nullptr;
  CycleCfg cfg;
  HostPrecondFn host_fn = nullptr;
  void* host_user = nullptr;
  mutable std::vector<double> host_r, host_z;  // staging of the callback's arguments
};

// Hooks for a row-partitioned operator (dist_solve.cu): A is this rank's rows with local
// column ids, vectors that feed an SpMV carry n_alloc >= n entries (owned + halo), every
// dot product written to device memory is summed over ranks in rank order, and the
// preconditioner is the partitioned cycle.  nullptr = the one-GPU path.
struct KrylovDist {
  int64_t n_alloc = 0;
  std::function<void(Epi, const SpmvArgs&, int)> spmv;  // halo exchange + SpMV on the rows
  std::function<void(double*, int)> allreduce;       // device scalars, in place
  std::function<void(const double*, double*)> precond;
  // precond + (rr . z, rold . z) summed over ranks into q; false = dots not produced
  std::function<bool(const double*, const double*, double*, double*)> precond_dots;
  std::function<void()> flush_warnings;
};

// x (device, n; n_alloc with dist) holds x0 on entry and the solution on exit.
SolveOut pcg(const DevCsr& A, const double* b, double* x, const Precond& M, const SolverCfg& cfg,
             const KrylovDist* dist = nullptr);
SolveOut fgmres(const DevCsr& A, const double* b, double* x, const Precond& M,
                const SolverCfg& cfg, const KrylovDist* dist = nullptr);

}  // namespace aggmg_b200
