// smoother.cuh — smoother setup (a12) and sweeps (a15).
#pragma once

#include <functional>

#include "sparse.cuh"

namespace aggmg_b200 {

struct SmootherDev {
  int kind = 1;  // AGGMG_SMOOTHER_*
  DevBuf<double> inv_diag;
  DevBuf<double> wdiag;  // omega * inv_diag, the damped-Jacobi scaling
  double omega = 1.0;
  double rho_est = 1.0;
  int arnoldi_m = 5;
};

// Hooks that run the Arnoldi estimate on a row-partitioned operator: the Krylov vectors
// carry a halo (n_alloc entries), the start vector uses global indices, dots are summed
// over ranks.  nullptr = the one-GPU path.
struct ArnoldiOps {
  int64_t n_alloc = 0, n_global = 0, row0 = 0;
  std::function<void(double*)> start;
  std::function<void(double*)> before_spmv;
  std::function<double(const double*, const double*)> dot;
  std::function<void(double*, int)> allreduce_dev;  // device scalars summed over ranks
};

// smoother.cpp:86-99 (inverse diagonal with "zero diagonal at row i"; Arnoldi rho for
// damped Jacobi with start vector uniform_sym(seed, i)).
void setup_smoother(const DevCsr& A, int kind, int arnoldi_m, uint64_t seed, SmootherDev& s,
                    const ArnoldiOps* ops = nullptr);

// One sweep on device vectors (smoother.cpp:101-124): jacobi/damped Jacobi out of place
// into x_out (x_out may not alias x); sgs in place on x.
void smooth_sweep(const SmootherDev& s, const DevCsr& A, const double* b, const double* x,
                  double* x_out, const int* pred = nullptr, int prof = 0);
void smooth_sgs(const SmootherDev& s, const DevCsr& A, const double* b, double* x);

}  // namespace aggmg_b200
