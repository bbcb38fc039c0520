// smoother.cuh — smoother setup (a12) and sweeps (a15).
#pragma once

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

// smoother.cpp:86-99 (inverse diagonal with "zero diagonal at row i"; Arnoldi rho for
// damped Jacobi with start vector uniform_sym(seed, i)).
void setup_smoother(const DevCsr& A, int kind, int arnoldi_m, uint64_t seed, SmootherDev& s);

// One sweep on device vectors (smoother.cpp:101-124): jacobi/damped Jacobi out of place
// into x_out (x_out may not alias x); sgs in place on x.
void smooth_sweep(const SmootherDev& s, const DevCsr& A, const double* b, const double* x,
                  double* x_out, const int* pred = nullptr, int prof = 0);
void smooth_sgs(const SmootherDev& s, const DevCsr& A, const double* b, double* x);

}  // namespace aggmg_b200
