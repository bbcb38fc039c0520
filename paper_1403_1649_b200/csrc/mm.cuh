// mm.cuh — Matrix Market reader / writer (reference matrix_market.hpp:23-35).
#pragma once

#include <string>
#include <vector>

#include "generators_host.hpp"
#include "runtime.cuh"

namespace aggmg_b200 {

// read_matrix_market (matrix_market.cpp:93-145): host parse on all cores, CSR assembly on the
// device (stable (row, col) sort + in-order duplicate sums, sparse.cpp:153-181).
HostCsr read_matrix_market_text(const char* data, size_t size, bool allow_pattern);
HostCsr read_matrix_market_file(const std::string& path, bool allow_pattern);
std::vector<double> read_vector_market_file(const std::string& path);
// 17-significant-digit writers (matrix_market.cpp:176-220), byte-identical to the reference's.
void write_matrix_market_file(const std::string& path, int64_t n_rows, int64_t n_cols,
                              const int64_t* rp, const int64_t* col, const double* val);
void write_vector_market_file(const std::string& path, const double* x, int64_t n);
// triplets -> canonical CSR on the device (TripletList order decides duplicate sums)
HostCsr triplets_to_csr_device(int64_t n_rows, int64_t n_cols, const std::vector<int64_t>& ti,
                               const std::vector<int64_t>& tj, const std::vector<double>& tv);

}  // namespace aggmg_b200
