// dense_host.cpp — host LU for the coarsest level and the Hessenberg eigenvalue solver
// used by the Arnoldi spectral-radius estimate.
#include "dense_host.hpp"

#include <algorithm>
#include <cmath>
#include <string>

#include "common.cuh"

namespace aggmg_b200 {

void HostLu::factor(std::vector<double> a, int64_t dim) {
  n = dim;
  lu = std::move(a);
  perm.resize(n);
  for (int64_t i = 0; i < n; ++i) perm[i] = i;
  auto at = [&](int64_t i, int64_t j) -> double& { return lu[i * n + j]; };
  for (int64_t k = 0; k < n; ++k) {
    int64_t piv = k;
    double best = std::fabs(at(k, k));
    for (int64_t i = k + 1; i < n; ++i)
      if (std::fabs(at(i, k)) > best) {
        best = std::fabs(at(i, k));
        piv = i;
      }
    if (best == 0.0) throw Error("lu_factor: zero pivot at index " + std::to_string(k));
    if (piv != k) {
      std::swap_ranges(lu.begin() + k * n, lu.begin() + (k + 1) * n, lu.begin() + piv * n);
      std::swap(perm[k], perm[piv]);
    }
    const double inv = 1.0 / at(k, k);
    for (int64_t i = k + 1; i < n; ++i) {
      const double m = at(i, k) * inv;
      at(i, k) = m;
      double* ri = &lu[i * n];
      const double* rk = &lu[k * n];
      for (int64_t j = k + 1; j < n; ++j) ri[j] = ri[j] - m * rk[j];
    }
  }
}

void HostLu::solve(const double* b, double* x) const {
  for (int64_t i = 0; i < n; ++i) {
    double s = b[perm[i]];
    const double* ri = &lu[i * n];
    for (int64_t j = 0; j < i; ++j) s = s - ri[j] * x[j];
    x[i] = s;
  }
  for (int64_t i = n - 1; i >= 0; --i) {
    double s = x[i];
    const double* ri = &lu[i * n];
    for (int64_t j = i + 1; j < n; ++j) s = s - ri[j] * x[j];
    x[i] = s / ri[i];
  }
}

std::vector<double> HostLu::inverse() const {
  std::vector<double> inv(static_cast<size_t>(n) * n), e(n, 0.0), col(n);
  for (int64_t j = 0; j < n; ++j) {
    e[j] = 1.0;
    solve(e.data(), col.data());
    e[j] = 0.0;
    for (int64_t i = 0; i < n; ++i) inv[i * n + j] = col[i];
  }
  return inv;
}

// Complex single-shift QR with Wilkinson shifts and Givens rotations on the active
// window; deflation on negligible subdiagonals.  Converges for the <= 5x5 Hessenberg
// matrices produced by the Arnoldi estimate; complex pairs come out naturally.
std::vector<std::complex<double>> hessenberg_eigenvalues(const std::vector<double>& h, int n) {
  using cd = std::complex<double>;
  std::vector<std::complex<double>> eig;
  if (n <= 0) return eig;
  std::vector<cd> H(static_cast<size_t>(n) * n);
  for (int i = 0; i < n * n; ++i) H[i] = cd(h[i], 0.0);
  auto at = [&](int i, int j) -> cd& { return H[static_cast<size_t>(i) * n + j]; };
  int hi = n - 1;
  int iters = 0;
  const int max_iters = 60 * n + 100;
  while (hi >= 0) {
    if (hi == 0) {
      eig.push_back(at(0, 0));
      break;
    }
    // find the active window [lo, hi]
    int lo = hi;
    while (lo > 0) {
      const double off = std::abs(at(lo, lo - 1));
      const double sc = std::abs(at(lo - 1, lo - 1)) + std::abs(at(lo, lo));
      if (off <= 1e-15 * (sc > 0.0 ? sc : 1.0)) {
        at(lo, lo - 1) = 0.0;
        break;
      }
      --lo;
    }
    if (lo == hi) {
      eig.push_back(at(hi, hi));
      --hi;
      continue;
    }
    if (++iters > max_iters) throw Error("hessenberg_eigenvalues: QR iteration did not converge");
    // Wilkinson shift: eigenvalue of the trailing 2x2 closest to H(hi,hi)
    const cd a = at(hi - 1, hi - 1), b = at(hi - 1, hi), c = at(hi, hi - 1), d = at(hi, hi);
    const cd tr = a + d, det = a * d - b * c;
    const cd disc = std::sqrt(tr * tr * 0.25 - det);
    const cd l1 = tr * 0.5 + disc, l2 = tr * 0.5 - disc;
    cd mu = (std::abs(l1 - d) < std::abs(l2 - d)) ? l1 : l2;
    if (iters % 11 == 0) mu += cd(std::abs(c), 0.0);  // exceptional shift
    for (int i = lo; i <= hi; ++i) at(i, i) -= mu;
    // QR by Givens on the window, then RQ
    std::vector<cd> cs(hi - lo), sn(hi - lo);
    for (int k = lo; k < hi; ++k) {
      const cd x = at(k, k), y = at(k + 1, k);
      const double r = std::sqrt(std::norm(x) + std::norm(y));
      cd cc = 1.0, ss = 0.0;
      if (r > 0.0) {
        cc = x / r;
        ss = y / r;
      }
      cs[k - lo] = cc;
      sn[k - lo] = ss;
      for (int j = k; j < n; ++j) {
        const cd t1 = at(k, j), t2 = at(k + 1, j);
        at(k, j) = std::conj(cc) * t1 + std::conj(ss) * t2;
        at(k + 1, j) = -ss * t1 + cc * t2;
      }
    }
    for (int k = lo; k < hi; ++k) {
      const cd cc = cs[k - lo], ss = sn[k - lo];
      for (int i = 0; i <= std::min(k + 1, hi); ++i) {
        const cd t1 = at(i, k), t2 = at(i, k + 1);
        at(i, k) = t1 * cc + t2 * ss;
        at(i, k + 1) = -t1 * std::conj(ss) + t2 * std::conj(cc);
      }
    }
    for (int i = lo; i <= hi; ++i) at(i, i) += mu;
  }
  return eig;
}

}  // namespace aggmg_b200
