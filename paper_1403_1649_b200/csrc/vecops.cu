// vecops.cu — elementwise kernels (grid-stride, 2 doubles per thread-step).
#include "vecops.cuh"

namespace aggmg_b200 {

namespace {
constexpr int kB = 256;
unsigned vgrid(int64_t n) { return grid_for(n, kB, 16 * static_cast<int64_t>(sm_count())); }

__global__ void k_axpy(int64_t n, double a, const double* __restrict__ x, double* __restrict__ y) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    y[i] = __dadd_rn(y[i], __dmul_rn(a, x[i]));
}
__global__ void k_scale_into(int64_t n, double a, const double* x, double* y) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    y[i] = __dmul_rn(x[i], a);
}
__global__ void k_sub(int64_t n, const double* b, const double* ax, double* r) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    r[i] = __dsub_rn(b[i], ax[i]);
}
__global__ void k_uniform_sym(int64_t n, uint64_t seed, double* x) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    x[i] = uniform_sym(seed, static_cast<uint64_t>(i));
}
}  // namespace

void vec_axpy(int64_t n, double a, const double* x, double* y) {
  if (n > 0) AGG_LAUNCH(k_axpy, vgrid(n), kB, 0, n, a, x, y);
}
void vec_scale(int64_t n, double a, double* x) {
  if (n > 0) AGG_LAUNCH(k_scale_into, vgrid(n), kB, 0, n, a, x, x);
}
void vec_scale_into(int64_t n, double a, const double* x, double* y) {
  if (n > 0) AGG_LAUNCH(k_scale_into, vgrid(n), kB, 0, n, a, x, y);
}
void vec_sub(int64_t n, const double* b, const double* ax, double* r) {
  if (n > 0) AGG_LAUNCH(k_sub, vgrid(n), kB, 0, n, b, ax, r);
}
void vec_uniform_sym(int64_t n, uint64_t seed, double* x) {
  if (n > 0) AGG_LAUNCH(k_uniform_sym, vgrid(n), kB, 0, n, seed, x);
}

}  // namespace aggmg_b200
