// generators_host.hpp — host problem generators (poisson.hpp:17-26 analogue).
#pragma once

#include <cstdint>
#include <vector>

namespace aggmg_b200 {

struct HostCsr {
  int64_t n = 0;
  std::vector<int64_t> rp, col;
  std::vector<double> val;
};

HostCsr generate_poisson_host(int dims, int64_t nx, int64_t ny, int64_t nz, double eps,
                              int weak_axis);
HostCsr generate_jump27_host(int64_t nx, int64_t ny, int64_t nz, double jump, int64_t block);

}  // namespace aggmg_b200
