// primitives.cuh — device building blocks: exclusive scans, deterministic reductions,
// segmented rank sort.  All results are independent of launch timing: reductions use a
// fixed grid and a fixed combination order (the GPU analogue of the reference's fixed
// 8192-chunk reductions, vector_ops.hpp:16-40).
#pragma once

#include "runtime.cuh"

namespace aggmg_b200 {

// offsets[0..n] = exclusive scan of counts[0..n-1]; returns offsets[n] (synchronises).
int64_t scan_to_offsets(const idx* counts, idx* offsets, int64_t n);
// Same without reading the total back to the host.
void scan_to_offsets_async(const idx* counts, idx* offsets, int64_t n);

// ---- deterministic dot products ------------------------------------------------
// Up to three products reduced in one pass: out[k] = sum_i a_k[i] * b_k[i].
struct DotArgs {
  const double* a[3];
  const double* b[3];
  int np;
};
// Writes the results to device memory out[0..np-1].
void dot_device(const DotArgs& args, int64_t n, double* out, const int* pred = nullptr,
                int exact = -1);  // exact: 1 reference chunk order, 0 tree, -1 library mode
// Convenience host-returning dot (synchronises).
double dot_host(const double* a, const double* b, int64_t n, int exact = -1);

// Reduction scratch: the grid size used by every reduction over n elements.
unsigned reduce_grid(int64_t n);
// Global scratch (partials + completion ticket) shared by all reductions on the stream.
double* reduce_partials();
unsigned* reduce_ticket();

// Block-level reduction of NP doubles; result valid in thread 0.  Fixed tree order.
template <int NP>
__device__ inline void block_reduce(double (&v)[NP], double* smem /* >= 32*NP */) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NP; ++k)
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v[k] = __dadd_rn(v[k], __shfl_down_sync(0xffffffffu, v[k], o));
  if (lane == 0)
#pragma unroll
    for (int k = 0; k < NP; ++k) smem[warp * NP + k] = v[k];
  __syncthreads();
  const int nw = (blockDim.x + 31) >> 5;
  if (warp == 0) {
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      v[k] = lane < nw ? smem[lane * NP + k] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v[k] = __dadd_rn(v[k], __shfl_down_sync(0xffffffffu, v[k], o));
    }
  }
  __syncthreads();
}

// Called by every block after writing its partials: the last block to arrive sums
// partials[0..nblocks) (stride NP) in a fixed order and writes out[k].  Returns true
// in the block that finished the reduction.
template <int NP>
__device__ inline bool finish_reduction(double* partials, unsigned* ticket, double* out,
                                        double* smem) {
  __shared__ bool last;
  __threadfence();
  if (threadIdx.x == 0) last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return false;
  __threadfence();
  double v[NP];
#pragma unroll
  for (int k = 0; k < NP; ++k) v[k] = 0.0;
  for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x)
#pragma unroll
    for (int k = 0; k < NP; ++k) v[k] = __dadd_rn(v[k], ((volatile double*)partials)[b * NP + k]);
  block_reduce<NP>(v, smem);
  if (threadIdx.x == 0) {
#pragma unroll
    for (int k = 0; k < NP; ++k) out[k] = v[k];
    *ticket = 0u;
  }
  return true;
}

// ---- segmented sort ---------------------------------------------------------------
// Sorts keys inside each segment [offsets[s], offsets[s+1]) ascending; keys must be
// unique within a segment.  Optional payload moves with its key.  Out of place.
void segmented_sort(const idx* offsets, int64_t nseg, const idx* keys_in, idx* keys_out,
                    const double* vals_in = nullptr, double* vals_out = nullptr);

// ---- small helpers ---------------------------------------------------------------
void fill_int(idx* p, int64_t n, idx v);
void fill_double(double* p, int64_t n, double v);
void copy_double(double* dst, const double* src, int64_t n);

}  // namespace aggmg_b200
