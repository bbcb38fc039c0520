// smoother.cuh — smoother setup (a12) and sweeps (a15).
#pragma once

#include <functional>
#include <memory>
#include <vector>

#include "sparse.cuh"

namespace aggmg_b200 {

// Level schedule of one symmetric Gauss-Seidel direction (sgs.cu; built on the host at
// setup).  Row i's level is 1 + the highest level of the rows it reads new values from (j < i
// going forward, j > i going backward); rows of one level are independent.  Slot t = the
// t-th row in level order; A is stored per slot with the diagonal dropped, the first `ell`
// entries in an ELL block whose codes say where each x value comes from (sgs.cu).
struct SgsDirection {
  int ell = 4, cta = 512;           // ELL width and single-CTA run size
  DevBuf<int> rows;                 // slot t -> row id
  DevBuf<int4> rec;                 // slot t: {row, off-diagonal count, 1/A_ii}
  DevBuf<int> offsets;              // level l = slots [offsets[l], offsets[l+1])
  std::vector<int64_t> h_offsets;   // host copy
  DevBuf<uint32_t> code;            // ELL block: codes in uint4 chunks, values in double2
  DevBuf<double> val;               //   chunks; entries past `ell` continue in
                                    //   ocol[optr[t], optr[t+1])
  DevBuf<idx> optr, ocol;
  DevBuf<double> oval;
  struct Run { int64_t l0, l1; bool narrow; };
  std::vector<Run> runs;            // consecutive narrow levels share one single-CTA launch
};

struct SmootherDev {
  int kind = 1;  // AGGMG_SMOOTHER_*
  DevBuf<double> inv_diag;
  DevBuf<double> wdiag;  // omega * inv_diag, the damped-Jacobi scaling
  double omega = 1.0;
  double rho_est = 1.0;
  int arnoldi_m = 5;
  SgsDirection sgs_fw, sgs_bw;           // kind == sgs only
  DevBuf<double> sgs_tmp, sgs_bp, sgs_xp;  // forward output; b and x in slot order (n each)
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

// Smoother setup for every level of a one-GPU hierarchy with the damped-Jacobi Arnoldi
// estimates overlapped with the rest of setup.  add() computes the inverse diagonal at once
// (zero diagonals fail there, in level order) and issues the level's Arnoldi process
// (smoother.cpp:43-84) entirely on the device on the side stream — breakdown handled by a
// device flag, no host reads — so the latency-bound dot chains run under the next levels'
// coarsening.  finish() joins, reads each Hessenberg matrix once, and sets rho/omega exactly
// as setup_smoother does (same kernels, same operation order: omega is bit-identical).
class SmootherBatch {
 public:
  SmootherBatch();
  ~SmootherBatch();  // joins the side stream if finish() was not reached (error paths)
  // `s` must stay at a stable address only during add(); finish() resolves each job's state
  // again through level(key) (hierarchy levels live in a growing vector)
  void add(const DevCsr& A, int kind, int arnoldi_m, uint64_t seed, SmootherDev& s, int key);
  void finish(const std::function<SmootherDev&(int)>& level);

 private:
  struct Job;
  std::vector<std::unique_ptr<Job>> jobs_;
};

// One sweep on device vectors (smoother.cpp:101-124): jacobi/damped Jacobi out of place
// into x_out (x_out may not alias x); sgs in place on x.
void smooth_sweep(const SmootherDev& s, const DevCsr& A, const double* b, const double* x,
                  double* x_out, const int* pred = nullptr, int prof = 0);
// Symmetric Gauss-Seidel in place on x; the level schedule comes from setup_smoother (or
// build_sgs_schedule for a caller-supplied state).  pred = device flag gating the sweep.
void smooth_sgs(const SmootherDev& s, const DevCsr& A, const double* b, double* x,
                const int* pred = nullptr);
void build_sgs_schedule(const DevCsr& A, SmootherDev& s);

}  // namespace aggmg_b200
