// chunked.cuh — reductions in the reference's exact summation order.
//
// The reference sums dot products over fixed 8192-element chunks, sequentially inside
// a chunk, then the chunk partials sequentially in chunk order (vector_ops.hpp:16-40).
// k_chunked reproduces that order bit for bit: one CTA per chunk; every tile of 1024
// elements is computed by all threads (the elementwise part of a fused operation and
// its products) into a double-buffered shared-memory tile, and one lane per product
// chain accumulates the tile sequentially while the rest of the CTA computes the next
// tile.  The last CTA to finish sums the chunk partials in order.
#pragma once

#include "primitives.cuh"

namespace aggmg_b200 {

constexpr int kChunk = 8192;       // vector_ops.hpp:18
constexpr int kChunkThreads = 256;
// elements per pipeline stage (two stages of NP tiles must fit in 48 KB static smem)
template <int NP>
struct ChunkTile {
  static constexpr int value = NP >= 3 ? 512 : 1024;
};

// Process-wide switch for the solve-phase reductions: exact (reference order) or tree
// (default).  The smoother setup and the public dot/norm2 always use the exact order.
bool exact_reductions();
void set_exact_reductions(bool on);

template <int NP, class Op>
__global__ void __launch_bounds__(kChunkThreads)
    k_chunked(int64_t n, Op op, double* partials, unsigned* ticket, double* out) {
  constexpr int kChunkTile = ChunkTile<NP>::value;
  __shared__ double tile[2][NP][kChunkTile];
  __shared__ bool last;
  if (!op.active()) {
    if (blockIdx.x == 0 && threadIdx.x == 0) op.inactive();
    return;
  }
  op.init();
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * kChunk;
  const int len = static_cast<int>(min(static_cast<int64_t>(kChunk), n - c0));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool summer = lane == 0 && warp < NP;
  double acc = 0.0;
  for (int tb = 0, t = 0; tb < len; tb += kChunkTile, ++t) {
    double(*buf)[kChunkTile] = tile[t & 1];
#pragma unroll
    for (int j = 0; j < kChunkTile / kChunkThreads; ++j) {
      const int pos = tb + j * kChunkThreads + threadIdx.x;
      if (pos < len) {
        double p[NP];
        op(c0 + pos, p);
#pragma unroll
        for (int k = 0; k < NP; ++k) buf[k][pos - tb] = p[k];
      }
    }
    __syncthreads();
    if (summer) {
      const int m = min(kChunkTile, len - tb);
      const double* src = buf[warp];
      int q = 0;
      for (; q + 8 <= m; q += 8) {
        const double2 a = *reinterpret_cast<const double2*>(src + q);
        const double2 b = *reinterpret_cast<const double2*>(src + q + 2);
        const double2 c = *reinterpret_cast<const double2*>(src + q + 4);
        const double2 d = *reinterpret_cast<const double2*>(src + q + 6);
        acc = __dadd_rn(acc, a.x);
        acc = __dadd_rn(acc, a.y);
        acc = __dadd_rn(acc, b.x);
        acc = __dadd_rn(acc, b.y);
        acc = __dadd_rn(acc, c.x);
        acc = __dadd_rn(acc, c.y);
        acc = __dadd_rn(acc, d.x);
        acc = __dadd_rn(acc, d.y);
      }
      for (; q < m; ++q) acc = __dadd_rn(acc, src[q]);
    }
  }
  if (summer) partials[blockIdx.x * NP + warp] = acc;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x < NP) {
    const volatile double* vp = partials;
    double s;
    if (gridDim.x == 1) {
      s = vp[threadIdx.x];  // single chunk: the reference returns the chunk sum itself
    } else {
      s = 0.0;
      for (unsigned c = 0; c < gridDim.x; ++c) s = __dadd_rn(s, vp[c * NP + threadIdx.x]);
    }
    out[threadIdx.x] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *ticket = 0u;
    op.finalize(out);
  }
}

inline unsigned chunk_grid(int64_t n) {
  return static_cast<unsigned>(std::max<int64_t>(1, (n + kChunk - 1) / kChunk));
}

// Launch k_chunked for a fused elementwise op over n elements; out[0..NP) receives the
// reference-ordered sums.  n == 0 still runs the op's inactive/finalize semantics via a
// single empty chunk.
template <int NP, class Op>
void launch_chunked(const Op& op, int64_t n, double* out) {
  auto kern = k_chunked<NP, Op>;
  AGG_LAUNCH(kern, chunk_grid(n), kChunkThreads, 0, n, op, reduce_partials(), reduce_ticket(), out);
}

// ---- elementwise ops ---------------------------------------------------------------

// plain multi-dot: p_k = a_k[i] * b_k[i]   (vector_ops.hpp:20-40)
template <int NP>
struct DotOp {
  const double* a[NP];
  const double* b[NP];
  const int* pred;
  __device__ bool active() const { return !pred || *pred; }
  __device__ void inactive() const {}
  __device__ void init() {}
  __device__ void operator()(int64_t i, double* p) const {
#pragma unroll
    for (int k = 0; k < NP; ++k) p[k] = __dmul_rn(a[k][i], b[k][i]);
  }
  __device__ void finalize(double*) const {}
};

template <int NP>
void launch_dot_exact(const DotOp<NP>& op, int64_t n, double* out) {
  if (n <= 0) {
    AGG_CUDA(cudaMemsetAsync(out, 0, sizeof(double) * NP, stream()));
    return;
  }
  launch_chunked<NP>(op, n, out);
}

}  // namespace aggmg_b200
