// generators_host.cpp — host problem generators (harness inputs).
// Poisson follows poisson.cpp:15-77 (lexicographic rows, ascending columns, Dirichlet
// rows eliminated); the 27-point jump operator is defined in DESIGN.md §7 and is
// bit-identical to the device generator in sparse.cu.
#include <string>
#include <vector>

#include "common.cuh"
#include "generators_host.hpp"

namespace aggmg_b200 {

HostCsr generate_poisson_host(int dims, int64_t nx, int64_t ny, int64_t nz, double eps,
                              int weak_axis, int64_t row0, int64_t nrows) {
  require(dims == 2 || dims == 3, "poisson: dims must be 2 or 3");
  if (dims == 2) nz = 1;
  require(nx >= 1 && ny >= 1 && nz >= 1, "poisson: grid extents must be positive");
  require(eps > 0.0, "poisson: epsilon must be positive");
  const int weak = weak_axis < 0 ? (dims == 2 ? 1 : 2) : weak_axis;
  require(weak < dims, "poisson: weak axis " + std::to_string(weak) + " out of range for " +
                           std::to_string(dims) + "D");
  const double cx = weak == 0 ? -eps : -1.0, cy = weak == 1 ? -eps : -1.0,
               cz = weak == 2 ? -eps : -1.0;
  const double diag = -2.0 * (cx + cy + (dims == 3 ? cz : 0.0));
  HostCsr A;
  A.ncols = nx * ny * nz;
  if (nrows < 0) nrows = A.ncols - row0;
  require(row0 >= 0 && row0 + nrows <= A.ncols, "poisson: row range outside the grid");
  A.n = nrows;
  A.rp.assign(A.n + 1, 0);
  A.col.reserve(static_cast<size_t>(A.n) * (dims == 3 ? 7 : 5));
  A.val.reserve(A.col.capacity());
  for (int64_t r = row0; r < row0 + A.n; ++r) {
    const int64_t i = r % nx, j = (r / nx) % ny, k = r / (nx * ny);
    auto put = [&](int64_t c, double v) {
      A.col.push_back(c);
      A.val.push_back(v);
    };
    if (k > 0) put(r - nx * ny, cz);
    if (j > 0) put(r - nx, cy);
    if (i > 0) put(r - 1, cx);
    put(r, diag);
    if (i + 1 < nx) put(r + 1, cx);
    if (j + 1 < ny) put(r + nx, cy);
    if (k + 1 < nz) put(r + nx * ny, cz);
    A.rp[r - row0 + 1] = static_cast<int64_t>(A.col.size());
  }
  return A;
}

HostCsr generate_jump27_host(int64_t nx, int64_t ny, int64_t nz, double jump, int64_t block,
                             int64_t row0, int64_t nrows) {
  require(nx >= 1 && ny >= 1 && nz >= 1 && block >= 1, "jump27: extents must be positive");
  require(jump > 0.0, "jump27: jump must be positive");
  auto kappa = [&](int64_t x, int64_t y, int64_t z) {
    return (((x / block) + (y / block) + (z / block)) & 1) ? jump : 1.0;
  };
  HostCsr A;
  A.ncols = nx * ny * nz;
  if (nrows < 0) nrows = A.ncols - row0;
  require(row0 >= 0 && row0 + nrows <= A.ncols, "jump27: row range outside the grid");
  A.n = nrows;
  A.rp.assign(A.n + 1, 0);
  for (int64_t r = row0; r < row0 + A.n; ++r) {
    const int64_t i = r % nx, j = (r / nx) % ny, k = r / (nx * ny);
    const double ki = kappa(i, j, k);
    double diag = 0.0;
    size_t pdiag = 0;
    for (int dz = -1; dz <= 1; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          const int64_t x = i + dx, y = j + dy, z = k + dz;
          const bool inside = x >= 0 && x < nx && y >= 0 && y < ny && z >= 0 && z < nz;
          if (dx == 0 && dy == 0 && dz == 0) {
            pdiag = A.col.size();
            A.col.push_back(r);
            A.val.push_back(0.0);
            continue;
          }
          if (!inside) {
            diag = diag + ki;
            continue;
          }
          const double kj = kappa(x, y, z);
          const double kij = ((2.0 * ki) * kj) / (ki + kj);
          diag = diag + kij;
          A.col.push_back((z * ny + y) * nx + x);
          A.val.push_back(-kij);
        }
    A.val[pdiag] = diag;
    A.rp[r - row0 + 1] = static_cast<int64_t>(A.col.size());
  }
  return A;
}

}  // namespace aggmg_b200
