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

// Francis double-shift QR on an upper-Hessenberg matrix, eigenvalues only.  The
// floating-point operation sequence is the reference's (dense.cpp:81-212) so that the
// Arnoldi spectral-radius estimate, and therefore omega, is bit-identical to the CPU
// oracle: deflation test 1e-14, closed-form 1x1 / 2x2 blocks, Householder bulge chase
// with the 3-vector (x, y, z), a closing Givens rotation, exceptional shift every 20.
namespace {

class FrancisQR {
 public:
  FrancisQR(std::vector<double> h, int n) : h_(std::move(h)), n_(n) {}

  std::vector<std::complex<double>> run() {
    int hi = n_ - 1, since = 0, steps = 0;
    while (hi >= 0) {
      if (!(steps++ < 30 * n_ + 100)) throw Error("hessenberg_eigenvalues: QR iteration did not converge");
      const int lo = active_start(hi);
      if (lo == hi) {
        out_.emplace_back(a(hi, hi), 0.0);
        hi -= 1;
        since = 0;
      } else if (lo + 1 == hi) {
        block2(a(lo, lo), a(lo, hi), a(hi, lo), a(hi, hi));
        hi -= 2;
        since = 0;
      } else {
        sweep(lo, hi, ++since % 20 == 0);
      }
    }
    return out_;
  }

 private:
  double& a(int i, int j) { return h_[static_cast<size_t>(i) * n_ + j]; }

  int active_start(int hi) {  // walk up until a negligible subdiagonal entry
    int lo = hi;
    while (lo > 0) {
      const double scale = std::fabs(a(lo - 1, lo - 1)) + std::fabs(a(lo, lo));
      if (std::fabs(a(lo, lo - 1)) <= 1e-14 * (scale > 0.0 ? scale : 1.0)) {
        a(lo, lo - 1) = 0.0;
        return lo;
      }
      --lo;
    }
    return 0;
  }

  void block2(double p, double q, double r, double s) {
    const double tr = p + s;
    const double det = p * s - q * r;
    const double disc = tr * tr / 4.0 - det;
    if (disc >= 0.0) {
      const double w = std::sqrt(disc);
      out_.emplace_back(tr / 2.0 + w, 0.0);
      out_.emplace_back(tr / 2.0 - w, 0.0);
    } else {
      const double w = std::sqrt(-disc);
      out_.emplace_back(tr / 2.0, w);
      out_.emplace_back(tr / 2.0, -w);
    }
  }

  // one implicit double-shift step on the window [lo, hi]
  void sweep(int lo, int hi, bool exceptional) {
    double s = a(hi - 1, hi - 1) + a(hi, hi);
    double t = a(hi - 1, hi - 1) * a(hi, hi) - a(hi - 1, hi) * a(hi, hi - 1);
    if (exceptional) {
      const double w = std::fabs(a(hi, hi - 1)) + std::fabs(a(hi - 1, hi - 2));
      s = 1.5 * w;
      t = w * w;
    }
    double x = a(lo, lo) * a(lo, lo) + a(lo, lo + 1) * a(lo + 1, lo) - s * a(lo, lo) + t;
    double y = a(lo + 1, lo) * (a(lo, lo) + a(lo + 1, lo + 1) - s);
    double z = a(lo + 2, lo + 1) * a(lo + 1, lo);
    for (int k = lo; k <= hi - 2; ++k) {
      double nrm = std::sqrt(x * x + y * y + z * z);
      if (nrm != 0.0) {
        if (x > 0.0) nrm = -nrm;
        const double u0 = x - nrm;
        const double beta = 2.0 / (u0 * u0 + y * y + z * z);
        reflect_rows(k, (k > lo) ? k - 1 : lo, hi, u0, y, z, beta);
        reflect_cols(k, lo, std::min(k + 3, hi), u0, y, z, beta);
      }
      x = a(k + 1, k);
      y = a(k + 2, k);
      z = (k + 3 <= hi) ? a(k + 3, k) : 0.0;
    }
    const int k = hi - 1;
    const double r = std::hypot(x, y);
    if (r > 0.0) {
      const double c = x / r, sn = y / r;
      for (int j = k - 1; j <= hi; ++j) {
        const double t1 = a(k, j), t2 = a(k + 1, j);
        a(k, j) = c * t1 + sn * t2;
        a(k + 1, j) = -sn * t1 + c * t2;
      }
      for (int i = lo; i <= hi; ++i) {
        const double t1 = a(i, k), t2 = a(i, k + 1);
        a(i, k) = c * t1 + sn * t2;
        a(i, k + 1) = -sn * t1 + c * t2;
      }
    }
  }

  void reflect_rows(int k, int j0, int j1, double u0, double u1, double u2, double beta) {
    for (int j = j0; j <= j1; ++j) {
      double d = u0 * a(k, j) + u1 * a(k + 1, j) + u2 * a(k + 2, j);
      d *= beta;
      a(k, j) -= d * u0;
      a(k + 1, j) -= d * u1;
      a(k + 2, j) -= d * u2;
    }
  }
  void reflect_cols(int k, int i0, int i1, double u0, double u1, double u2, double beta) {
    for (int i = i0; i <= i1; ++i) {
      double d = u0 * a(i, k) + u1 * a(i, k + 1) + u2 * a(i, k + 2);
      d *= beta;
      a(i, k) -= d * u0;
      a(i, k + 1) -= d * u1;
      a(i, k + 2) -= d * u2;
    }
  }

  std::vector<double> h_;
  int n_;
  std::vector<std::complex<double>> out_;
};

}  // namespace

std::vector<std::complex<double>> hessenberg_eigenvalues(const std::vector<double>& h, int n) {
  if (n <= 0) return {};
  return FrancisQR(h, n).run();
}

}  // namespace aggmg_b200
