// generators_host.hpp — host problem generators (poisson.hpp:17-26 analogue).
#pragma once

#include <cstdint>
#include <vector>

namespace aggmg_b200 {

struct HostCsr {
  int64_t n = 0;      // rows held (a slab of the grid operator, or all of it)
  int64_t ncols = 0;  // global column count
  std::vector<int64_t> rp, col;
  std::vector<double> val;
};

// rows [row0, row0 + nrows) (nrows < 0: all) with global column ids
HostCsr generate_poisson_host(int dims, int64_t nx, int64_t ny, int64_t nz, double eps,
                              int weak_axis, int64_t row0 = 0, int64_t nrows = -1);
HostCsr generate_jump27_host(int64_t nx, int64_t ny, int64_t nz, double jump, int64_t block,
                             int64_t row0 = 0, int64_t nrows = -1);

}  // namespace aggmg_b200
