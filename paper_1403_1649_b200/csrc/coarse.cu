// coarse.cu — the coarsest-level direct solve (dense.cpp:16-79, hierarchy.cpp:83-86) on the
// device: the explicit inverse of the dense coarsest operator by Gauss-Jordan elimination with
// the reference's partial pivoting (first maximal |pivot| in the column wins; an exactly zero
// pivot fails with "lu_factor: zero pivot at index k"), used by the cycle as one GEMV.  The
// solve tolerance is <= 1e-10, so an inverse is admissible; the pivot
// sequence is the reference LU's (the rows below the pivot receive the same updates).
//
// One cooperative kernel does all n steps.  The augmented matrix [A | I] is column-major;
// step k reads column k (never written again: columns <= k of the A half are finished) and
// every warp updates one column j > k of the 2n, so a step needs exactly one grid barrier.
#include <cooperative_groups.h>

#include <string>

#include "hierarchy.cuh"

namespace cg = cooperative_groups;

namespace aggmg_b200 {
namespace {

constexpr int kGjThreads = 256;

__global__ void k_dense_aug(const idx* rp, const idx* col, const double* val, int64_t n,
                            double* aug) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (idx k = rp[i]; k < rp[i + 1]; ++k) aug[static_cast<int64_t>(col[k]) * n + i] = val[k];
  aug[(n + i) * n + i] = 1.0;
}

__global__ void __launch_bounds__(kGjThreads) k_gauss_jordan(double* aug, int n, int* bad) {
  cg::grid_group grid = cg::this_grid();
  __shared__ double s_best[kGjThreads / 32];
  __shared__ int s_idx[kGjThreads / 32];
  __shared__ int s_piv;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t nn = n;
  const int warps = gridDim.x * (kGjThreads / 32);
  const int gw = blockIdx.x * (kGjThreads / 32) + wid;
  for (int k = 0; k < n; ++k) {
    const double* ck = aug + k * nn;
    // pivot: first maximal |a_ik|, i >= k (every CTA computes the same answer)
    double best = -1.0;
    int bi = n;
    for (int i = k + threadIdx.x; i < n; i += kGjThreads) {
      const double v = fabs(ck[i]);
      if (v > best) best = v, bi = i;  // ascending i per thread: first max kept
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_down_sync(0xffffffffu, best, o);
      const int oi = __shfl_down_sync(0xffffffffu, bi, o);
      if (ob > best || (ob == best && oi < bi)) best = ob, bi = oi;
    }
    if (lane == 0) s_best[wid] = best, s_idx[wid] = bi;
    __syncthreads();
    if (threadIdx.x == 0) {
      double b = s_best[0];
      int p = s_idx[0];
      for (int w = 1; w < kGjThreads / 32; ++w)
        if (s_best[w] > b || (s_best[w] == b && s_idx[w] < p)) b = s_best[w], p = s_idx[w];
      s_piv = b == 0.0 ? -1 : p;
    }
    __syncthreads();
    const int p = s_piv;
    if (p < 0) {  // all CTAs see it: leave together
      if (blockIdx.x == 0 && threadIdx.x == 0) *bad = k;
      return;
    }
    const double inv = 1.0 / ck[p];
    const double mk = ck[k];  // multiplier of the old row k, which moves to row p
    for (int64_t j = k + 1 + gw; j < 2 * nn; j += warps) {
      double* cj = aug + j * nn;
      const double u = cj[p] * inv;  // the new row k: pivot row scaled
      const double akj = cj[k];
      __syncwarp();
      for (int i = lane; i < n; i += 32) {
        double v;
        if (i == k)
          v = u;
        else if (i == p)
          v = akj - mk * u;
        else
          v = cj[i] - ck[i] * u;
        cj[i] = v;
      }
    }
    grid.sync();
  }
}

// right half of the column-major augmented matrix -> row-major inverse
__global__ void k_take_inverse(const double* aug, int64_t n, double* inv) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n * n) return;
  const int64_t i = t / n, j = t % n;
  inv[t] = aug[(n + j) * n + i];
}

}  // namespace

void invert_coarsest(const DevCsr& A, DevBuf<double>& inv) {
  const int64_t n = A.n_rows;
  require(n < (int64_t{1} << 31) / 2, "setup: coarsest level too large for a dense solve");
  inv.resize(n * n);
  if (n == 0) return;
  DevBuf<double> aug(2 * n * n);
  aug.zero();
  AGG_LAUNCH(k_dense_aug, grid_for(n, 256), 256, 0, A.rowptr.get(), A.col.get(), A.val.get(), n,
             aug.get());
  DevBuf<int> bad(1);
  fill_int(bad.get(), 1, -1);
  int per_sm = 0, sms = 0, dev = current_device();
  AGG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_gauss_jordan, kGjThreads, 0));
  AGG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  const int64_t want = (2 * n + kGjThreads / 32 - 1) / (kGjThreads / 32);
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(want, int64_t{per_sm} * sms)));
  double* a = aug.get();
  int ni = static_cast<int>(n);
  int* b = bad.get();
  void* args[] = {&a, &ni, &b};
  AGG_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_gauss_jordan), grid, kGjThreads,
                                       args, 0, stream()));
  const int k = read_scalar(bad.get());
  if (k >= 0) throw Error("lu_factor: zero pivot at index " + std::to_string(k));
  AGG_LAUNCH(k_take_inverse, grid_for(n * n, 256), 256, 0, aug.get(), n, inv.get());
}

}  // namespace aggmg_b200
