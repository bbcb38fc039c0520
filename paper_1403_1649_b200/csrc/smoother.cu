// smoother.cu — inverse diagonal, Arnoldi spectral-radius estimate, sweeps.
#include <algorithm>
#include <cmath>
#include <vector>

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

// Sequential symmetric Gauss-Seidel (smoother.cpp:105-119): strictly ordered by
// definition, so one thread walks the rows.
__global__ void k_sgs(const idx* rp, const idx* col, const double* val, int64_t n,
                      const double* inv, const double* b, double* x) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  for (int64_t i = 0; i < n; ++i) {
    double s = b[i];
    for (idx k = rp[i]; k < rp[i + 1]; ++k)
      if (col[k] != i) s = __dsub_rn(s, __dmul_rn(val[k], x[col[k]]));
    x[i] = __dmul_rn(s, inv[i]);
  }
  for (int64_t i = n - 1; i >= 0; --i) {
    double s = b[i];
    for (idx k = rp[i]; k < rp[i + 1]; ++k)
      if (col[k] != i) s = __dsub_rn(s, __dmul_rn(val[k], x[col[k]]));
    x[i] = __dmul_rn(s, inv[i]);
  }
}

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
  DevBuf<double> w(n), dots(2);
  for (int j = 0; j < m; ++j) {
    if (ops) ops->before_spmv(V[j].get());  // halo of the Krylov vector
    SpmvArgs a;
    a.x = V[j].get();
    a.y = w.get();
    a.d = inv_diag;
    spmv_run(A, Epi::kScaleDiag, a);
    double h_scale = 0.0;
    for (int i = 0; i <= j; ++i) {
      double hv[2];
      if (ops) {
        ops->dot2(V[i].get(), w.get(), V[i].get(), V[i].get(), hv);
      } else {
        DotArgs d{};
        d.a[0] = V[i].get();
        d.b[0] = w.get();
        d.a[1] = V[i].get();
        d.b[1] = V[i].get();
        d.np = 2;
        dot_device(d, n, dots.get(), nullptr, 1);
        dots.download(hv, 2);
        sync();
      }
      const double hij = hv[0] / hv[1];
      h(i, j) = hij;
      vec_axpy(n, -hij, V[i].get(), w.get());
      h_scale = std::max(h_scale, std::abs(hij));
    }
    const double hj = std::sqrt(dot(w.get(), w.get()));
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

void smooth_sgs(const SmootherDev& s, const DevCsr& A, const double* b, double* x) {
  AGG_LAUNCH(k_sgs, 1, 32, 0, A.rowptr.get(), A.col.get(), A.val.get(), A.n_rows,
             s.inv_diag.get(), b, x);
}

}  // namespace aggmg_b200
