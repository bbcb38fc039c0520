// dense_host.hpp — small dense kernels that stay on the host (coarsest level, <= 5000
// unknowns; Arnoldi Hessenberg <= 5x5).
#pragma once

#include <complex>
#include <cstdint>
#include <vector>

namespace aggmg_b200 {

// Partial-pivot LU of a row-major n x n matrix (reference dense.cpp:24-57 semantics:
// first maximal |pivot| wins, "lu_factor: zero pivot at index k" on failure).
struct HostLu {
  int64_t n = 0;
  std::vector<double> lu;
  std::vector<int64_t> perm;
  void factor(std::vector<double> a, int64_t n);
  void solve(const double* b, double* x) const;  // dense.cpp:59-73 substitution order
  std::vector<double> inverse() const;           // row-major A^-1 from n unit solves
};

// Eigenvalues of a small upper-Hessenberg matrix (shifted QR; dense.hpp:45 contract).
std::vector<std::complex<double>> hessenberg_eigenvalues(const std::vector<double>& h, int n);

}  // namespace aggmg_b200
