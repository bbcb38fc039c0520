// vecops.cuh — elementwise vector kernels with the reference's exact rounding
// sequence (vector_ops.hpp:44-52): axpy is y + (a*x), scale is x*a.
#pragma once

#include "runtime.cuh"

namespace aggmg_b200 {

void vec_axpy(int64_t n, double a, const double* x, double* y);        // y = y + a*x
void vec_scale(int64_t n, double a, double* x);                        // x = x*a
void vec_scale_into(int64_t n, double a, const double* x, double* y);  // y = x*a
void vec_sub(int64_t n, const double* b, const double* ax, double* r); // r = b - ax
void vec_uniform_sym(int64_t n, uint64_t seed, double* x);             // rng.hpp:32-34

}  // namespace aggmg_b200
