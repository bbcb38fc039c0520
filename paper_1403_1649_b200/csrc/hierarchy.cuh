// hierarchy.cuh — device-resident AMG hierarchy (reference hierarchy.hpp:21-48) and the
// setup loop (hierarchy.cpp:34-104).
#pragma once

#include <string>
#include <vector>

#include "dense_host.hpp"
#include "setup.cuh"
#include "smoother.cuh"

namespace aggmg_b200 {

struct SetupCfg {
  double alpha = 0.25;
  int64_t coarse_size_max = 600;
  int max_levels = 25;
  int smoother = 1;
  int arnoldi_m = 5;
  int reuse_caches = 0;
  uint64_t seed = 42;
  // Global index of this hierarchy's level 0 (> 0 for the agglomerated tail of a
  // row-partitioned hierarchy): seeds, K-cycle level policy and messages use k + offset.
  int64_t level_offset = 0;
};

// K-cycle scalars of one level, resident in device memory (cycles.cpp:88-132).
struct KScalars {
  double rho1, alpha1;       // written by the fused SpMV+dot of c
  double nrt, nrc;           // ||rt||^2, ||rc||^2
  double gamma, beta, alpha2;  // written by the fused SpMV+dot of d
  int flag2;                 // run the second inner cycle
  int pad;
};

struct DevLevel {
  DevCsrPtr A;
  DevBuf<double> B;  // near-null-space vector on this level
  SmootherDev smoother;
  bool has_smoother = false;
  // transfer to the next level (empty on the coarsest level)
  bool has_next = false;
  AggDev agg;
  TransferDev tr;
  GalerkinDev gal;
  int mis_sweeps = 0;
  // cycle workspace on this level (size n_k)
  DevBuf<double> r, t;
  // coarse-side vectors owned by this level's cycle (size n_{k+1})
  DevBuf<double> rc, xc, c, v, rt, d, w;
  DevBuf<KScalars> ks;
  // set while capturing / issuing a cycle: the restriction into this level already wrote the
  // zero-guess damped-Jacobi sweep of right-hand side zs_b into zs_x (Epi::kSpmvZero)
  const double* zs_b = nullptr;
  double* zs_x = nullptr;
};

// Captured CUDA graph of one coarse sub-cycle launch (levels >= 1 are launch-latency
// bound: ~100 small kernels per preconditioner application).
struct SubcycleGraph {
  cudaGraphExec_t exec = nullptr;
  int64_t kernels = 0;
};

struct DevHierarchy {
  ~DevHierarchy();
  std::vector<DevLevel> levels;
  std::vector<std::pair<std::string, SubcycleGraph>> graphs;  // key -> graph
  int graph_uses = 0;
  SetupCfg cfg;
  std::vector<std::string> warnings;
  DevBuf<double> coarse_inv;  // explicit inverse of the coarsest operator (row-major)
  // exact-reduction mode (aggmg_set_exact_reductions(1) before setup): the reference's LU
  // factors (dense.cpp:16-79, host restatement) for a bit-identical substitution
  DevBuf<double> coarse_lu;
  DevBuf<double> coarse_lu_t;  // the same, column-major (the forward substitution's order)
  DevBuf<int> coarse_perm;
  bool coarse_lu_ready = false;
  double setup_ms = 0.0;
  bool workspace_ready = false;
  // PCG hook: the finest level's last damped-Jacobi sweep of a preconditioner application
  // also produces (r . z, top_dot_c . z) into top_dot_out (set by pcg, cleared after use);
  // top_dot_done reports whether the fused path ran.
  const double* top_dot_c = nullptr;
  double* top_dot_out = nullptr;
  bool top_dot_done = false;


  int64_t n_levels() const { return static_cast<int64_t>(levels.size()); }
  int64_t coarsest() const { return n_levels() - 1; }
  void ensure_workspace();
};

// B0 == nullptr means ones (aggmg_main.cpp:177).
std::unique_ptr<DevHierarchy> setup_hierarchy(DevCsrPtr A0, const double* B0_dev,
                                              const SetupCfg& cfg);
void refresh_values(DevHierarchy& h, const double* new_values_dev);
// Deep copy (every level's operator, transfer, cache and smoother; no captured graphs): the
// reference's refresh_values takes the hierarchy BY VALUE (hierarchy.cpp:90), so a refresh of
// a hierarchy someone else still holds works on a copy.
std::unique_ptr<DevHierarchy> clone_hierarchy(const DevHierarchy& h);
DevCsrPtr clone_csr(const DevCsr& A);
void factor_coarsest(DevHierarchy& h);
// Explicit inverse of the coarsest operator (row-major) by device Gauss-Jordan (coarse.cu).
void invert_coarsest(const DevCsr& A, DevBuf<double>& inv);

}  // namespace aggmg_b200
