// cycles.cuh — V-/K-/hybrid cycles on the device (reference cycles.cpp:16-146).
//
// The whole cycle is a fixed kernel sequence: the K-cycle's scalar branches
// (rho1 == 0, ||rt|| <= t ||rc||, rho2 == 0; cycles.cpp:96-127) are evaluated on the
// device and steer later kernels through device predicates, so an application of the
// preconditioner needs no host synchronisation.
#pragma once

#include "hierarchy.cuh"

namespace aggmg_b200 {

struct CycleCfg {
  int kind = 2;  // AGGMG_CYCLE_HYBRID
  int k_levels = 2;
  double t = 0.25;
  int inner = 1;  // AGGMG_INNER_GMRES
};

// x_out = cycle(k) applied to b from the initial guess x_in (nullptr = zero guess,
// the case every internal call uses).  x_out must not alias b or x_in.
void cycle(DevHierarchy& h, const CycleCfg& cfg, int64_t k, bool accelerated_top,
           const double* b, const double* x_in, double* x_out, const int* pred);

// z = M r (apply_preconditioner, cycles.cpp:140-146)
void apply_preconditioner(DevHierarchy& h, const CycleCfg& cfg, const double* r, double* z);

// Host-visible warnings raised by device-side branch fallbacks (cycles.cpp:97,124).
void flush_cycle_warnings();

// dense coarse solve x = A_L^{-1} b
void coarse_solve(DevHierarchy& h, const double* b, double* x, const int* pred);

}  // namespace aggmg_b200
