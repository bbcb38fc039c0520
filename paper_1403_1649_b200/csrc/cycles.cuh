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
// The level-0 damped-Jacobi zero-guess sweep z = 0 + wd .* r every cycle of h starts with
// (nullptr when it does not: one level, or SGS).  A caller that produces r elementwise can
// write that z alongside and mark it done for the next apply_preconditioner(h, cfg, r, z).
const double* top_zero_sweep_diag(const DevHierarchy& h);
void mark_top_zero_sweep(DevHierarchy& h, const double* r, double* z);

// Host-visible warnings raised by device-side branch fallbacks (cycles.cpp:97,124).
void flush_cycle_warnings();

// Workspace of one coarse correction (vectors of the coarse level).
struct CoarseWork {
  double *c, *v, *rt, *d, *w;
  KScalars* ks;
};
// Coarse half of a cycle visit (cycles.cpp:56-132): level kc of h receives rc, returns xc.
void coarse_correction(DevHierarchy& h, const CycleCfg& cfg, bool kparent, int64_t kc,
                       const double* rc, double* xc, const CoarseWork& w, const int* pred);

// Building blocks of the row-partitioned cycle (dist_solve.cu).
void launch_jacobi_zero(int64_t n, const double* wd, const double* b, double* x, const int* pred);
void launch_prolong(int64_t n, const double* x, const idx* agg, const double* pval, const double* xc,
                    double* t, const int* pred);
// rt = rc - s1 v and this rank's ||rt||^2, ||rc||^2 into ks->nrt/nrc
void launch_kstep1(int64_t n, const double* rc, const double* v, double* rt, KScalars* ks, double t,
                   const int* pred, int level);
// second-step flag from the (summed) norms
void launch_kflag(KScalars* ks, double t, const int* pred);
void launch_kcombine(int64_t n, const double* c, const double* d, double* xc, const KScalars* ks,
                     const int* pred, int level);
bool cycle_accelerated(const CycleCfg& cfg, int64_t k);  // cycles.cpp:16-20
bool cycle_graphs_enabled();  // AGGMG_GRAPHS != 0

// dense coarse solve x = A_L^{-1} b
void coarse_solve(DevHierarchy& h, const double* b, double* x, const int* pred);

}  // namespace aggmg_b200
