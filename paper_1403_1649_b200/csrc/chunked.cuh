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

constexpr int kChunk = 8192;  // vector_ops.hpp:18
// CTA layout: warp 0 is the consumer (lanes 0..NP-1 each run one sequential chain),
// warps 1..3 produce tiles (elementwise op + products) into a double buffer.
constexpr int kChunkThreads = 128;
constexpr int kChunkProducers = kChunkThreads - 32;
constexpr int kChunkTile = 4 * kChunkProducers;  // 384 elements per stage: 12 KB, 16 CTAs per SM

// Process-wide switch for the solve-phase reductions: exact (reference order) or tree
// (default).  The smoother setup and the public dot/norm2 always use the exact order.
bool exact_reductions();
void set_exact_reductions(bool on);

// Shared-memory mbarriers for the producer/consumer hand-off.  (Named barriers did the same
// job but a CTA holding four of them caps residency at four CTAs per SM — 3.5 waves of chunk
// chains for a 16.7 M vector; mbarriers carry no such limit.)
__device__ inline unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ inline void mbar_init(unsigned long long* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ inline void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ inline void mbar_wait(unsigned long long* bar, unsigned parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "MBAR_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra MBAR_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// One CTA per 8192-element chunk.  Producers fill stage b = t & 1 and arrive on FULL[b];
// the consumer waits on FULL[b], adds the stage sequentially, arrives on EMPTY[b]; the
// producers wait on EMPTY[b] before refilling it two tiles later.  The chain latency
// (8192 dependent adds) overlaps the memory traffic, and 16 CTAs per SM put every chunk
// of a 16.7 M vector in flight at once.
template <int NP, class Op>
__global__ void __launch_bounds__(kChunkThreads)
    k_chunked(int64_t n, Op op, double* partials, unsigned* ticket, double* out) {
  __shared__ __align__(16) double tile[2][NP][kChunkTile];
  __shared__ bool last;
  __shared__ unsigned long long full[2], empty[2];
  if (!op.active()) {
    if (blockIdx.x == 0 && threadIdx.x == 0) op.inactive();
    return;
  }
  if (threadIdx.x == 0) {
    mbar_init(&full[0], kChunkProducers);
    mbar_init(&full[1], kChunkProducers);
    mbar_init(&empty[0], 1);
    mbar_init(&empty[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  op.init();
  const int64_t c0 = static_cast<int64_t>(blockIdx.x) * kChunk;
  const int len = static_cast<int>(min(static_cast<int64_t>(kChunk), n - c0));
  const int ntiles = (len + kChunkTile - 1) / kChunkTile;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double acc = 0.0;
  if (warp > 0) {  // producers
    const int pt = threadIdx.x - 32;
    for (int t = 0; t < ntiles; ++t) {
      const int b = t & 1;
      if (t >= 2) mbar_wait(&empty[b], ((t >> 1) - 1) & 1);  // consumer freed use t-2
      const int tb = t * kChunkTile;
#pragma unroll
      for (int j = 0; j < kChunkTile / kChunkProducers; ++j) {
        const int pos = tb + j * kChunkProducers + pt;
        if (pos < len) {
          double p[NP];
          op(c0 + pos, p);
#pragma unroll
          for (int k = 0; k < NP; ++k) tile[b][k][pos - tb] = p[k];
        }
      }
      mbar_arrive(&full[b]);
    }
  } else {  // consumer warp
    for (int t = 0; t < ntiles; ++t) {
      const int b = t & 1;
      mbar_wait(&full[b], (t >> 1) & 1);
      if (lane < NP) {
        const int m = min(kChunkTile, len - t * kChunkTile);
        const double* src = tile[b][lane];
        // (the chain is bound by the fp64 add latency, ~10 cycles: 8192 adds ~ 45 us per
        // chunk; software-pipelining the smem loads measured no faster)
        int q = 0;
        for (; q + 8 <= m; q += 8) {
          const double2 a = *reinterpret_cast<const double2*>(src + q);
          const double2 c = *reinterpret_cast<const double2*>(src + q + 2);
          const double2 d = *reinterpret_cast<const double2*>(src + q + 4);
          const double2 e = *reinterpret_cast<const double2*>(src + q + 6);
          acc = __dadd_rn(acc, a.x);
          acc = __dadd_rn(acc, a.y);
          acc = __dadd_rn(acc, c.x);
          acc = __dadd_rn(acc, c.y);
          acc = __dadd_rn(acc, d.x);
          acc = __dadd_rn(acc, d.y);
          acc = __dadd_rn(acc, e.x);
          acc = __dadd_rn(acc, e.y);
        }
        for (; q < m; ++q) acc = __dadd_rn(acc, src[q]);
      }
      __syncwarp();
      if (lane == 0 && t + 2 < ntiles) mbar_arrive(&empty[b]);
    }
    if (lane < NP) partials[blockIdx.x * NP + lane] = acc;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  // Chunk partials in chunk order.  All threads stage tiles of partials into shared memory
  // (coalesced, in flight together); lanes 0..NP-1 walk each tile sequentially, so the
  // dependent chain pays the add latency, not a global-load latency per chunk.
  double s = 0.0;
  const unsigned nc = gridDim.x;
  double* stage = &tile[0][0][0];  // reuse: 2 * NP * kChunkTile >= NP * kFinalTile
  constexpr int kFinalTile = kChunkTile;
  for (unsigned base = 0; base < nc; base += kFinalTile) {
    const int cnt = static_cast<int>(min(static_cast<unsigned>(kFinalTile), nc - base));
    __syncthreads();
    for (int q = threadIdx.x; q < cnt * NP; q += kChunkThreads) {
      const int c = q / NP, k = q - c * NP;
      stage[k * kFinalTile + c] = __ldcg(partials + (base + c) * NP + k);
    }
    __syncthreads();
    if (threadIdx.x < NP) {
      const double* src = stage + threadIdx.x * kFinalTile;
      if (nc == 1) {
        s = src[0];  // single chunk: the reference returns the chunk sum itself
      } else {
        for (int c = 0; c < cnt; ++c) s = __dadd_rn(s, src[c]);
      }
    }
  }
  if (threadIdx.x < NP) out[threadIdx.x] = s;
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
