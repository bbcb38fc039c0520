// smoother.cu — inverse diagonal, Arnoldi spectral-radius estimate, sweeps.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "chunked.cuh"
#include "dense_host.hpp"
#include "smoother.cuh"
#include "vecops.cuh"

namespace aggmg_b200 {

namespace {

__global__ void k_inv_diag(const idx* rp, const idx* col, const double* val, int64_t n,
                           double* inv, int* bad_row) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double d = 0.0;
  for (idx k = rp[i]; k < rp[i + 1]; ++k)
    if (col[k] == i) d = val[k];
  if (d == 0.0) {
    atomicMin(bad_row, static_cast<int>(i));
    inv[i] = 0.0;
    return;
  }
  inv[i] = __ddiv_rn(1.0, d);
}

// One fused MGS step of the Arnoldi column on the device, in the reference's chunked dot
// order: w = w + (-h) V_i (skipped for the column's first step), then (V_next . w,
// V_next . V_next) — or (w . w, 0) after the last basis vector.  The host path this replaces
// ran dot2 (sync) + axpy per coefficient; the fused form makes one pass per coefficient and
// one host read per column, with bit-identical coefficients (same operations, same order).
struct ArnoldiStepOp {
  const double* hsrc;  // device coefficient h to subtract with (nullptr: first step)
  const double* vi;
  double* w;
  const double* vn;  // next basis vector (nullptr: last step, out = w . w)
  double mh;
  __device__ bool active() const { return true; }
  __device__ void inactive() const {}
  __device__ void init() { mh = hsrc ? -*hsrc : 0.0; }
  __device__ void operator()(int64_t t, double* p) const {
    double wt = w[t];
    if (hsrc) {
      wt = __dadd_rn(wt, __dmul_rn(mh, vi[t]));  // vec_axpy(-h, V_i, w)
      w[t] = wt;
    }
    if (vn) {
      const double v = vn[t];
      p[0] = __dmul_rn(v, wt);
      p[1] = __dmul_rn(v, v);
    } else {
      p[0] = __dmul_rn(wt, wt);
      p[1] = 0.0;
    }
  }
  __device__ void finalize(double*) const {}
};

__global__ void k_hdiv(const double* s, double* h) { *h = s[0] / s[1]; }

double estimate_rho(const DevCsr& A, const double* inv_diag, int m, uint64_t seed,
                    const ArnoldiOps* ops) {
  const int64_t n = A.n_rows;
  const int64_t n_alloc = ops ? ops->n_alloc : n;
  m = static_cast<int>(std::min<int64_t>(m, ops ? ops->n_global : n));
  auto dot = [&](const double* a, const double* b) {
    return ops ? ops->dot(a, b) : dot_host(a, b, n, 1);
  };
  std::vector<DevBuf<double>> V;
  V.emplace_back(n_alloc);
  if (ops)
    ops->start(V[0].get());
  else
    vec_uniform_sym(n, seed, V[0].get());
  const double qn = std::sqrt(dot(V[0].get(), V[0].get()));
  require(qn > 0.0, "smoother: degenerate start vector");
  vec_scale(n, 1.0 / qn, V[0].get());

  std::vector<double> H(static_cast<size_t>(m + 1) * m, 0.0);  // row-major (m+1) x m
  auto h = [&](int i, int j) -> double& { return H[static_cast<size_t>(i) * m + j]; };
  int m_eff = m;
  // device copies: column j's coefficients Hc[i] (i <= j), step slots, the final ||w||^2
  DevBuf<double> w(n), Hc(m + 1), slots(2);
  double* pin = pinned_scratch(m + 2);
  for (int j = 0; j < m; ++j) {
    if (ops) ops->before_spmv(V[j].get());  // halo of the Krylov vector
    SpmvArgs a;
    a.x = V[j].get();
    a.y = w.get();
    a.d = inv_diag;
    spmv_run(A, Epi::kScaleDiag, a);
    for (int i = -1; i <= j; ++i) {  // i = -1: the first dots, no axpy
      ArnoldiStepOp op;
      op.hsrc = i >= 0 ? Hc.get() + i : nullptr;
      op.vi = i >= 0 ? V[i].get() : nullptr;
      op.w = w.get();
      op.vn = i < j ? V[i + 1].get() : nullptr;
      if (n > 0)
        launch_chunked<2>(op, n, slots.get());
      else
        slots.zero();
      if (ops) ops->allreduce_dev(slots.get(), 2);
      if (i < j)
        AGG_LAUNCH(k_hdiv, 1, 1, 0, slots.get(), Hc.get() + i + 1);  // h(i+1, j)
    }
    // one read per column: h(0..j, j) and ||w||^2
    AGG_CUDA(cudaMemcpyAsync(pin, Hc.get(), sizeof(double) * (j + 1), cudaMemcpyDeviceToHost, stream()));
    AGG_CUDA(cudaMemcpyAsync(pin + j + 1, slots.get(), sizeof(double), cudaMemcpyDeviceToHost, stream()));
    sync();
    double h_scale = 0.0;
    for (int i = 0; i <= j; ++i) {
      h(i, j) = pin[i];
      h_scale = std::max(h_scale, std::abs(pin[i]));
    }
    const double hj = std::sqrt(pin[j + 1]);
    if (hj <= 1e-12 * std::max(h_scale, 1.0)) {
      m_eff = j + 1;
      break;
    }
    h(j + 1, j) = hj;
    if (j + 1 < m) {
      V.emplace_back(n_alloc);
      vec_scale_into(n, 1.0 / hj, w.get(), V.back().get());
    }
  }
  std::vector<double> Hm(static_cast<size_t>(m_eff) * m_eff);
  for (int i = 0; i < m_eff; ++i)
    for (int j = 0; j < m_eff; ++j) Hm[static_cast<size_t>(i) * m_eff + j] = h(i, j);
  double rho = 0.0;
  for (const auto& ev : hessenberg_eigenvalues(Hm, m_eff)) rho = std::max(rho, std::abs(ev));
  require(rho > 0.0, "smoother: spectral radius estimate collapsed to zero");
  return rho;
}

__global__ void k_scale_diag(const double* inv, double omega, int64_t n, double* wd) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) wd[i] = __dmul_rn(omega, inv[i]);
}

}  // namespace

void setup_smoother(const DevCsr& A, int kind, int arnoldi_m, uint64_t seed, SmootherDev& s,
                    const ArnoldiOps* ops) {
  require(ops || A.n_rows == A.n_cols, "smoother: matrix must be square");
  require(arnoldi_m >= 1 && arnoldi_m <= 5, "smoother: arnoldi_m must be in [1, 5]");
  const int64_t n = A.n_rows;
  s.kind = kind;
  s.arnoldi_m = arnoldi_m;
  s.inv_diag.resize(n);
  DevBuf<int> bad(1);
  fill_int(bad.get(), 1, INT32_MAX);
  if (n > 0)
    AGG_LAUNCH(k_inv_diag, grid_for(n, 256), 256, 0, A.rowptr.get(), A.col.get(), A.val.get(), n,
               s.inv_diag.get(), bad.get());
  const int b = read_scalar(bad.get());
  if (b != INT32_MAX)
    throw Error("smoother: zero diagonal at row " + std::to_string(b + (ops ? ops->row0 : 0)));
  s.omega = 1.0;
  s.rho_est = 1.0;
  if (kind == 1) {  // damped Jacobi
    s.rho_est = estimate_rho(A, s.inv_diag.get(), arnoldi_m, seed, ops);
    s.omega = (4.0 / 3.0) / s.rho_est;
  }
  if (kind == 2) build_sgs_schedule(A, s);
  const double w = (kind == 0) ? 1.0 : s.omega;  // smoother.cpp:120
  s.wdiag.resize(n);
  if (n > 0)
    AGG_LAUNCH(k_scale_diag, grid_for(n, 256), 256, 0, s.inv_diag.get(), w, n, s.wdiag.get());
}

void smooth_sweep(const SmootherDev& s, const DevCsr& A, const double* b, const double* x,
                  double* x_out, const int* pred, int prof) {
  SpmvArgs a;
  a.x = x;
  a.y = x_out;
  a.b = b;
  a.d = s.wdiag.get();
  a.pred = pred;
  spmv_run(A, Epi::kJacobi, a, prof);
}

}  // namespace aggmg_b200
