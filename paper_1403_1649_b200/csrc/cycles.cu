// cycles.cu — V-cycle (Alg. 4) and K-cycle (Alg. 5) recursion on device buffers.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>

#include <tuple>
#include <vector>

#include "chunked.cuh"

#include "cycles.cuh"

namespace aggmg_b200 {

namespace {

constexpr int kB = 256;
unsigned egrid(int64_t n) { return grid_for(n, kB, 8 * static_cast<int64_t>(sm_count())); }

int* warn_bits() {
  struct Bits {
    int* p = nullptr;
    ~Bits() {
      if (p) cudaFree(p);
    }
  };
  static thread_local Bits b;
  if (!b.p) {
    AGG_CUDA(cudaMalloc(&b.p, 2 * sizeof(int)));
    AGG_CUDA(cudaMemset(b.p, 0, 2 * sizeof(int)));
  }
  return b.p;
}

inline __device__ bool on(const int* pred) { return !pred || *pred; }

// x = 0 + wd .* (b - 0): first damped-Jacobi sweep from the zero guess
// (smoother.cpp:121-123 with x = 0, A*0 = +0).
__global__ void k_jacobi_zero(int64_t n, const double* __restrict__ wd,
                              const double* __restrict__ b, double* __restrict__ x,
                              const int* pred) {
  if (!on(pred)) return;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    x[i] = __dadd_rn(0.0, __dmul_rn(wd[i], b[i]));
}

// t = x + P xc  (prolongate_add, cycles.cpp:37-44: x + (0 + p*xc))
__global__ void k_prolong(int64_t n, const double* __restrict__ x, const idx* __restrict__ agg,
                          const double* __restrict__ pval, const double* __restrict__ xc,
                          double* __restrict__ t, const int* pred) {
  if (!on(pred)) return;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    t[i] = __dadd_rn(x[i], __dadd_rn(0.0, __dmul_rn(pval[i], xc[agg[i]])));
}

__global__ void k_copy(int64_t n, const double* __restrict__ a, double* __restrict__ b,
                       const int* pred) {
  if (!on(pred)) return;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    b[i] = a[i];
}

// rt = rc + (-s1) v ; ||rt||^2, ||rc||^2 ; flag2 = !(||rt|| <= t ||rc||)  (cycles.cpp:101-104)
__global__ void __launch_bounds__(kB) k_kstep1(int64_t n, const double* __restrict__ rc,
                                               const double* __restrict__ v,
                                               double* __restrict__ rt, KScalars* ks, double tt,
                                               const int* pred, double* partials,
                                               unsigned* ticket, int* warn, int level) {
  __shared__ double smem[64];
  if (!on(pred) || ks->rho1 == 0.0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      ks->flag2 = 0;
      if (on(pred)) atomicOr(&warn[0], 1 << (level & 31));
    }
    return;
  }
  const double s1 = __ddiv_rn(ks->alpha1, ks->rho1);
  const double ms1 = -s1;
  double acc[2] = {0.0, 0.0};
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double r = rc[i];
    const double z = __dadd_rn(r, __dmul_rn(ms1, v[i]));
    rt[i] = z;
    acc[0] = __dadd_rn(acc[0], __dmul_rn(z, z));
    acc[1] = __dadd_rn(acc[1], __dmul_rn(r, r));
  }
  block_reduce<2>(acc, smem);
  if (threadIdx.x == 0) {
    partials[blockIdx.x * 2] = acc[0];
    partials[blockIdx.x * 2 + 1] = acc[1];
  }
  if (finish_reduction<2>(partials, ticket, &ks->nrt, smem) && threadIdx.x == 0) {
    const double nrt = __dsqrt_rn(ks->nrt), nrc = __dsqrt_rn(ks->nrc);
    ks->flag2 = (nrt <= __dmul_rn(tt, nrc)) ? 0 : 1;
  }
}

// Reference-order variant of k_kstep1 for the chunked reduction kernel.
struct KStep1Op {
  KScalars* ks;
  double tt;
  const double *rc, *v;
  double* rt;
  const int* pred;
  int* warn;
  int level;
  double ms1;
  __device__ bool active() const { return on(pred) && ks->rho1 != 0.0; }
  __device__ void inactive() const {
    ks->flag2 = 0;
    if (on(pred)) atomicOr(&warn[0], 1 << (level & 31));
  }
  __device__ void init() { ms1 = -__ddiv_rn(ks->alpha1, ks->rho1); }
  __device__ void operator()(int64_t i, double* p) const {
    const double r = rc[i];
    const double z = __dadd_rn(r, __dmul_rn(ms1, v[i]));
    rt[i] = z;
    p[0] = __dmul_rn(z, z);
    p[1] = __dmul_rn(r, r);
  }
  __device__ void finalize(double* out) const {  // out == &ks->nrt
    ks->flag2 = (__dsqrt_rn(out[0]) <= __dmul_rn(tt, __dsqrt_rn(out[1]))) ? 0 : 1;
  }
};

// Final coarse correction of the K-cycle (cycles.cpp:96-132):
//   rho1 == 0           -> xc = c
//   accepted one step   -> xc = c * s1
//   rho2 == 0           -> xc = c * s1
//   otherwise           -> xc = c * (s1 - gamma*alpha2/(rho1*rho2)) + (alpha2/rho2) * d
__global__ void k_kcombine(int64_t n, const double* __restrict__ c, const double* __restrict__ d,
                           double* __restrict__ xc, const KScalars* ks, const int* pred,
                           int* warn, int level) {
  if (!on(pred)) return;
  const double rho1 = ks->rho1;
  int mode;
  double cc = 1.0, cd = 0.0;
  if (rho1 == 0.0) {
    mode = 0;
  } else {
    const double s1 = __ddiv_rn(ks->alpha1, rho1);
    if (!ks->flag2) {
      mode = 1;
      cc = s1;
    } else {
      const double g = ks->gamma, be = ks->beta, a2 = ks->alpha2;
      const double rho2 = __dsub_rn(be, __ddiv_rn(__dmul_rn(g, g), rho1));
      if (rho2 == 0.0) {
        mode = 1;
        cc = s1;
        if (blockIdx.x == 0 && threadIdx.x == 0) atomicOr(&warn[1], 1 << (level & 31));
      } else {
        mode = 2;
        cc = __dsub_rn(s1, __ddiv_rn(__dmul_rn(g, a2), __dmul_rn(rho1, rho2)));
        cd = __ddiv_rn(a2, rho2);
      }
    }
  }
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const double ci = c[i];
    double v;
    if (mode == 0)
      v = ci;
    else if (mode == 1)
      v = __dmul_rn(ci, cc);
    else
      v = __dadd_rn(__dmul_rn(ci, cc), __dmul_rn(cd, d[i]));
    xc[i] = v;
  }
}

// x = Ainv b, warp per row (coarsest level, n <= 5000)
__global__ void k_gemv(int64_t n, const double* __restrict__ M, const double* __restrict__ b,
                       double* __restrict__ x, const int* pred) {
  if (!on(pred)) return;
  const int64_t row = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const double* m = M + row * n;
  double s = 0.0;
  for (int64_t j = lane; j < n; j += 32) s = fma(m[j], b[j], s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if (lane == 0) x[row] = s;
}

// LuFactors::solve (dense.cpp:63-79) in the reference's operation order: forward
// substitution with the row permutation, back substitution with the division by U_ii.  Only
// the exact-reduction mode uses it.  One CTA of kLuThreads.
//  forward, column order: after columns 0..j-1 have been subtracted, s_j is final (x_j);
//    every row i > j then subtracts L_ij x_j.  Each row still subtracts in ascending j, so
//    the result is the reference's; the critical path is n barriers, not n^2/2 subtractions.
//    L is read from the column-major copy lt (coalesced), one column ahead.
//  backward, row order: row i's chain s -= U_ij x_j (ascending j > i) starts with x_{i+1},
//    so it is serial by definition.  Lane 0 runs the chain of row i from products that
//    warps 1.. computed during the previous row (U_ij x_j, j >= i+2, double-buffered in
//    shared memory), while they compute row i-1's products for j >= i+1.
// Operators above kLuRows * kLuThreads rows (coarse_size_max raised past the dense cap) take
// the one-thread k_lu_serial.
constexpr int kLuThreads = 1024;
constexpr int kLuRows = 5;  // rows per thread: kDenseSolveCap (5000) / kLuThreads, rounded up

__global__ void __launch_bounds__(kLuThreads) k_lu_solve(int n, const double* __restrict__ lu,
                                                        const double* __restrict__ lt,
                                                        const int* __restrict__ perm,
                                                        const double* __restrict__ b,
                                                        double* __restrict__ x, const int* pred) {
  if (!on(pred)) return;
  extern __shared__ double sh[];
  double* xs = sh;          // n: x
  double* pb = sh + n;      // 2n: product buffers
  const int t = threadIdx.x;
  double s[kLuRows], lcur[kLuRows];
#pragma unroll
  for (int r = 0; r < kLuRows; ++r) {
    const int i = t + r * kLuThreads;
    s[r] = i < n ? b[perm[i]] : 0.0;
    lcur[r] = (i < n && i > 0) ? lt[i] : 0.0;  // column 0
  }
  if (t == 0 && n > 0) xs[0] = s[0];
  __syncthreads();
  for (int j = 0; j + 1 < n; ++j) {
    const double xj = xs[j];
    double lnext[kLuRows];
#pragma unroll
    for (int r = 0; r < kLuRows; ++r) {
      const int i = t + r * kLuThreads;
      lnext[r] = (i < n && i > j + 1) ? lt[static_cast<int64_t>(j + 1) * n + i] : 0.0;
      if (i < n && i > j) s[r] = __dsub_rn(s[r], __dmul_rn(lcur[r], xj));
      if (i == j + 1) xs[i] = s[r];
      lcur[r] = lnext[r];
    }
    __syncthreads();
  }
  // backward (xs holds y)
  const int lane = t & 31, w = t >> 5;
  for (int i = n - 1; i >= 0; --i) {
    if (w == 0) {
      if (lane == 0) {
        const double* ui = lu + static_cast<int64_t>(i) * n;
        double acc = xs[i];
        if (i + 1 < n) acc = __dsub_rn(acc, __dmul_rn(ui[i + 1], xs[i + 1]));
        const double* p = pb + (i & 1) * n;
#pragma unroll 8
        for (int j = i + 2; j < n; ++j) acc = __dsub_rn(acc, p[j]);
        xs[i] = __ddiv_rn(acc, ui[i]);
      }
    } else if (i > 0) {
      const double* ur = lu + static_cast<int64_t>(i - 1) * n;
      double* p = pb + ((i - 1) & 1) * n;
      for (int j = i + 1 + (t - 32); j < n; j += kLuThreads - 32) p[j] = __dmul_rn(ur[j], xs[j]);
    }
    __syncthreads();
  }
  for (int i = t; i < n; i += kLuThreads) x[i] = xs[i];
}

// Small coarsest levels (n <= kLuWarpRows, the factors fit in shared memory): the CTA stages
// the row-major factors into shared memory, then ONE warp runs the whole substitution with
// warp barriers only.  Forward: lane l owns rows l, l + 32, ...; column j is applied once x_j
// (row j's finished value) is published.  Backward: the lanes form row i's products
// U_ij x_j (j > i) into a shared buffer, lane 0 subtracts them in ascending j and divides.
// Exactly the reference's operation sequence per row (dense.cpp:63-79), so the same bits.
constexpr int kLuWarpRows = 160;  // n^2 + 2n doubles <= 227 KB
__global__ void __launch_bounds__(256) k_lu_solve_warp(int n, const double* __restrict__ lu,
                                                     const int* __restrict__ perm,
                                                     const double* __restrict__ b,
                                                     double* __restrict__ x, const int* pred) {
  if (!on(pred)) return;
  extern __shared__ double sh[];
  double* f = sh;               // n * n: the factors, row-major
  double* xs = sh + n * n;      // n: y, then x
  double* pb = xs + n;          // n: row i's products
  const int64_t nn = static_cast<int64_t>(n) * n;
  for (int64_t q = threadIdx.x; q < nn; q += blockDim.x) f[q] = lu[q];
  __syncthreads();
  if (threadIdx.x >= 32) return;
  const int lane = threadIdx.x;
  // forward in place on xs (xs[i] = b[perm[i]], minus the finished columns); row j is final when
  // column j is reached, and the lanes apply it to their rows i > j
  for (int i = lane; i < n; i += 32) xs[i] = b[perm[i]];
  __syncwarp();
  for (int j = 0; j + 1 < n; ++j) {
    const double xj = xs[j];
    for (int i = j + 1 + lane; i < n; i += 32)
      xs[i] = __dsub_rn(xs[i], __dmul_rn(f[static_cast<int64_t>(i) * n + j], xj));
    __syncwarp();
  }
  __syncwarp();
  for (int i = n - 1; i >= 0; --i) {
    const double* ui = f + static_cast<int64_t>(i) * n;
    for (int j = i + 1 + lane; j < n; j += 32) pb[j] = __dmul_rn(ui[j], xs[j]);
    __syncwarp();
    if (lane == 0) {
      double acc = xs[i];
      int j = i + 1;
      // the next group's products load while this group's chain runs
      double q[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) q[u] = j + u < n ? pb[j + u] : 0.0;
      for (; j + 8 <= n; j += 8) {
        double nq[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) nq[u] = j + 8 + u < n ? pb[j + 8 + u] : 0.0;
#pragma unroll
        for (int u = 0; u < 8; ++u) acc = __dsub_rn(acc, q[u]);
#pragma unroll
        for (int u = 0; u < 8; ++u) q[u] = nq[u];
      }
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (j + u < n) acc = __dsub_rn(acc, q[u]);
      xs[i] = __ddiv_rn(acc, ui[i]);
    }
    __syncwarp();
  }
  for (int i = lane; i < n; i += 32) x[i] = xs[i];
}

__global__ void k_lu_serial(int64_t n, const double* __restrict__ lu, const int* __restrict__ perm,
                            const double* __restrict__ b, double* __restrict__ x, const int* pred) {
  if (!on(pred) || threadIdx.x != 0) return;
  for (int64_t i = 0; i < n; ++i) {
    double acc = b[perm[i]];
    const double* ri = lu + i * n;
    for (int64_t j = 0; j < i; ++j) acc = __dsub_rn(acc, __dmul_rn(ri[j], x[j]));
    x[i] = acc;
  }
  for (int64_t i = n - 1; i >= 0; --i) {
    double acc = x[i];
    const double* ri = lu + i * n;
    for (int64_t j = i + 1; j < n; ++j) acc = __dsub_rn(acc, __dmul_rn(ri[j], x[j]));
    x[i] = __ddiv_rn(acc, ri[i]);
  }
}

// the global finest level (profiling families time level 0 only)
bool finest(const DevHierarchy& h, int64_t k) { return k + h.cfg.level_offset == 0; }

bool accelerated(const CycleCfg& c, int64_t k) {  // cycles.cpp:16-20
  if (c.kind == 1) return true;
  if (c.kind == 2) return k < c.k_levels;
  return false;
}

void presmooth(DevLevel& L, const double* b, const double* x_in, double* x_out, const int* pred,
               bool top) {
  const int64_t n = L.A->n_rows;
  if (L.smoother.kind == 2) {  // sgs, in place
    if (x_in)
      AGG_LAUNCH(k_copy, egrid(n), kB, 0, n, x_in, x_out, pred);
    else
      fill_double(x_out, n, 0.0);
    smooth_sgs(L.smoother, *L.A, b, x_out, pred);
    return;
  }
  if (x_in) {
    smooth_sweep(L.smoother, *L.A, b, x_in, x_out, pred, top ? kProfSmoothL0 : 0);
  } else if (L.zs_b == b && L.zs_x == x_out) {  // done by the restriction into this level
    L.zs_b = nullptr;
    L.zs_x = nullptr;
  } else {
    AGG_LAUNCH(k_jacobi_zero, egrid(n), kB, 0, n, L.smoother.wdiag.get(), b, x_out, pred);
  }
}

void postsmooth(DevHierarchy& h, DevLevel& L, const double* b, double* x, const int* pred, bool top) {
  const int64_t n = L.A->n_rows;
  AGG_LAUNCH(k_prolong, egrid(n), kB, 0, n, x, L.agg.assignment.get(), L.tr.pval.get(),
             L.xc.get(), L.t.get(), pred);
  if (L.smoother.kind == 2) {
    AGG_LAUNCH(k_copy, egrid(n), kB, 0, n, L.t.get(), x, pred);
    smooth_sgs(L.smoother, *L.A, b, x, pred);
    return;
  }
  // PCG's (r.z, r_old.z) ride on the last sweep — on CSR-stream operators.  With a SELL-32
  // copy the plain sweep (0.97 of peak) plus PCG's separate two-product dot measured faster
  // than the fused sweep (0.82-0.85): c2 solve -0.5 ms.
  if (top && !pred && h.top_dot_out &&
      (!L.A->sell || (L.A->sell_vi && fuse_dots_on_dictionary()))) {
    SpmvArgs a;
    a.x = L.t.get();
    a.y = x;
    a.b = b;
    a.d = L.smoother.wdiag.get();
    a.c = h.top_dot_c;
    a.dots_out = h.top_dot_out;
    spmv_run(*L.A, Epi::kJacobiDot2, a, kProfSmoothL0);
    h.top_dot_done = true;
    return;
  }
  smooth_sweep(L.smoother, *L.A, b, L.t.get(), x, pred, top ? kProfSmoothL0 : 0);
}

// Pre-smooth, residual and restriction of one cycle visit (cycles.cpp:54-57).  From the
// zero guess the damped-Jacobi sweep and the residual fuse into one CSR-stream pass
// (x1 = 0 + wd b is recomputed for the gathered neighbours, bit-identical to the
// two-kernel sequence since A*0 sums to +0).
// next_x: where the next level's cycle will put its iterate (the parent's coarse vector: xc
// under a V-cycle, c under a K-cycle's first inner cycle) — the restriction then also writes
// the next level's zero-guess sweep into it, one launch instead of two
void descend(DevHierarchy& h, int64_t k, const double* b, const double* x_in, double* x_out,
             const int* pred, double* next_x) {
  DevLevel& L = h.levels[k];
  SpmvArgs ra;
  ra.y = L.r.get();
  ra.b = b;
  ra.pred = pred;
  // Measured on B200 (profiles/r01_kernel_bench.json): the fused pass gathers wd and b
  // for every stencil neighbour and loses to jacobi_zero + residual at every level, so it
  // stays off; the kernel remains available (aggmg_bench_kernel kind 2).
  constexpr bool kFuseZeroGuess = false;
  if (kFuseZeroGuess && !x_in && L.smoother.kind != 2) {
    ra.x_out = x_out;
    ra.d = L.smoother.wdiag.get();
    spmv_run(*L.A, Epi::kResidualZero, ra, finest(h, k) ? kProfSpmvL0 : 0);
  } else {
    presmooth(L, b, x_in, x_out, pred, finest(h, k));
    ra.x = x_out;
    spmv_run(*L.A, Epi::kResidual, ra, finest(h, k) ? kProfSpmvL0 : 0);  // cycles.cpp:30-35
  }
  SpmvArgs rr;
  rr.x = L.r.get();
  rr.y = L.rc.get();
  rr.pred = pred;
  DevLevel& N = h.levels[k + 1];
  if (next_x && k + 1 < h.coarsest() && N.smoother.kind != 2) {
    rr.x_out = next_x;
    rr.d = N.smoother.wdiag.get();
    spmv_run(*L.tr.R, Epi::kSpmvZero, rr);  // restriction + x_{k+1} = 0 + wd rc
    N.zs_b = L.rc.get();
    N.zs_x = next_x;
    return;
  }
  spmv_run(*L.tr.R, Epi::kSpmv, rr);  // restriction = spmv(R, r), cycles.cpp:56-57
}

void vcycle_dev(DevHierarchy& h, int64_t k, const double* b, const double* x_in, double* x_out,
                const int* pred);
void kcycle_dev(DevHierarchy& h, const CycleCfg& cfg, int64_t k, const double* b,
                const double* x_in, double* x_out, const int* pred);

void inner_cycle_eager(DevHierarchy& h, const CycleCfg& cfg, int64_t k, const double* b,
                       double* x_out, const int* pred);
CoarseWork work_of(DevLevel& L) {
  return CoarseWork{L.c.get(), L.v.get(), L.rt.get(), L.d.get(), L.w.get(), L.ks.get()};
}
void subcycle(DevHierarchy& h, const CycleCfg& cfg, int64_t k, const double* b, double* x_out,
              const int* pred, bool vee);

}  // namespace

bool cycle_graphs_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("AGGMG_GRAPHS");
    return !(e && e[0] == '0');
  }();
  return on;
}

namespace {
bool graphs_enabled() { return cycle_graphs_enabled(); }

// The sub-cycle below level 0 is a fixed kernel sequence over fixed buffers (device
// predicates steer the K-cycle branches), so it is captured once per (config, level,
// in/out/predicate buffers) into a CUDA graph and replayed: the ~100 small coarse-level
// kernels of one preconditioner application then launch back to back from the graph.
// The first call with a new key runs eagerly (initialising lazily created resources),
// the second captures.
void subcycle(DevHierarchy& h, const CycleCfg& cfg, int64_t k, const double* b, double* x_out,
              const int* pred, bool vee) {
  auto eager = [&] {
    if (vee)
      vcycle_dev(h, k, b, nullptr, x_out, pred);
    else
      inner_cycle_eager(h, cfg, k, b, x_out, pred);
  };
  cudaStreamCaptureStatus capturing = cudaStreamCaptureStatusNone;
  AGG_CUDA(cudaStreamIsCapturing(stream(), &capturing));
  // (inside a caller's capture — the partitioned cycle's graphs — run eagerly: it is recorded)
  if (k != 1 || !graphs_enabled() || k == h.coarsest() || capturing != cudaStreamCaptureStatusNone) {
    eager();
    return;
  }
  char keybuf[256];
  std::snprintf(keybuf, sizeof(keybuf), "%d/%d/%d/%d/%.17g/%d/%lld/%p/%p/%p", exact_reductions() ? 1 : 0,
                vee ? 1 : 0, cfg.kind, cfg.k_levels, cfg.t, cfg.inner, static_cast<long long>(k),
                static_cast<const void*>(b), static_cast<void*>(x_out),
                static_cast<const void*>(pred));
  const std::string key(keybuf);
  SubcycleGraph* g = nullptr;
  for (auto& e : h.graphs)
    if (e.first == key) g = &e.second;
  if (!g) {  // first sighting: eager run, remember the key
    h.graphs.emplace_back(key, SubcycleGraph{});
    eager();
    return;
  }
  if (!g->exec) {
    AGG_CUDA(cudaStreamBeginCapture(stream(), cudaStreamCaptureModeThreadLocal));
    const int64_t before = launch_count();
    try {
      eager();
    } catch (...) {
      cudaGraph_t junk;
      cudaStreamEndCapture(stream(), &junk);
      if (junk) cudaGraphDestroy(junk);
      throw;
    }
    g->kernels = launch_count() - before;
    note_launches(-g->kernels);  // counted again on every replay
    cudaGraph_t graph;
    AGG_CUDA(cudaStreamEndCapture(stream(), &graph));
    AGG_CUDA(cudaGraphInstantiate(&g->exec, graph, 0));
    AGG_CUDA(cudaGraphDestroy(graph));
  }
  AGG_CUDA(cudaGraphLaunch(g->exec, stream()));
  h.levels[k].zs_b = nullptr;  // the replayed capture consumed the fused sweep
  h.levels[k].zs_x = nullptr;
  note_launches(g->kernels);
  ++h.graph_uses;
}

void inner_cycle(DevHierarchy& h, const CycleCfg& cfg, int64_t k, const double* b, double* x_out,
                 const int* pred) {
  subcycle(h, cfg, k, b, x_out, pred, false);
}

void inner_cycle_eager(DevHierarchy& h, const CycleCfg& cfg, int64_t k, const double* b,
                       double* x_out, const int* pred) {
  if (accelerated(cfg, k + h.cfg.level_offset))
    kcycle_dev(h, cfg, k, b, nullptr, x_out, pred);
  else
    vcycle_dev(h, k, b, nullptr, x_out, pred);
}

// AGGMG_LEVEL_TIMING=1 (with AGGMG_GRAPHS=0): inclusive GPU time of every level visit,
// summed per level and printed by flush_cycle_warnings() — the per-level cost breakdown.
struct LevelTimer {
  bool on = false;
  std::vector<std::tuple<int, cudaEvent_t, cudaEvent_t>> rec;
  LevelTimer() {
    const char* e = std::getenv("AGGMG_LEVEL_TIMING");
    on = e && e[0] == '1';
  }
};
LevelTimer& ltimer() {
  static thread_local LevelTimer t;
  return t;
}
struct LevelScope {
  cudaEvent_t b_ = nullptr, e_ = nullptr;
  int level_;
  explicit LevelScope(int level) : level_(level) {
    if (!ltimer().on) return;
    cudaStreamCaptureStatus st;
    cudaStreamIsCapturing(stream(), &st);
    if (st != cudaStreamCaptureStatusNone) return;
    cudaEventCreate(&b_);
    cudaEventCreate(&e_);
    cudaEventRecord(b_, stream());
  }
  ~LevelScope() {
    if (!b_) return;
    cudaEventRecord(e_, stream());
    ltimer().rec.emplace_back(level_, b_, e_);
  }
};

void vcycle_dev(DevHierarchy& h, int64_t k, const double* b, const double* x_in, double* x_out,
                const int* pred) {
  LevelScope ls(static_cast<int>(k + h.cfg.level_offset));
  if (k == h.coarsest()) {
    coarse_solve(h, b, x_out, pred);
    return;
  }
  DevLevel& L = h.levels[k];
  descend(h, k, b, x_in, x_out, pred, L.xc.get());
  coarse_correction(h, CycleCfg{}, false, k + 1, L.rc.get(), L.xc.get(), work_of(L), pred);
  postsmooth(h, L, b, x_out, pred, finest(h, k));
}

void kcycle_dev(DevHierarchy& h, const CycleCfg& cfg, int64_t k, const double* b,
                const double* x_in, double* x_out, const int* pred) {
  LevelScope ls(static_cast<int>(k + h.cfg.level_offset));
  if (k == h.coarsest()) {
    coarse_solve(h, b, x_out, pred);
    return;
  }
  DevLevel& L = h.levels[k];
  descend(h, k, b, x_in, x_out, pred, L.c.get());
  coarse_correction(h, cfg, true, k + 1, L.rc.get(), L.xc.get(), work_of(L), pred);
  postsmooth(h, L, b, x_out, pred, finest(h, k));
}

}  // namespace

// The coarse half of a cycle visit: level kc receives rc and returns xc.  kparent: the
// visiting level runs a K-cycle (two inner cycles combined by the inner CG/GMRES scalars,
// cycles.cpp:84-132); otherwise a V-cycle (cycles.cpp:58-60).
void coarse_correction(DevHierarchy& h, const CycleCfg& cfg, bool kparent, int64_t kc,
                       const double* rc, double* xc, const CoarseWork& W, const int* pred) {
  if (kc == h.coarsest()) {
    coarse_solve(h, rc, xc, pred);
    return;
  }
  if (!kparent) {
    subcycle(h, CycleCfg{}, kc, rc, xc, pred, true);
    return;
  }
  const DevCsr& Ac = *h.levels[kc].A;
  const int64_t nc = Ac.n_rows;
  const int level = static_cast<int>(kc + h.cfg.level_offset);
  const bool cg = cfg.inner == 0;
  inner_cycle(h, cfg, kc, rc, W.c, pred);
  SpmvArgs a1;  // v = Ac c ; rho1, alpha1  (cycles.cpp:86-95)
  a1.x = W.c;
  a1.y = W.v;
  a1.c = rc;
  a1.dot_with_x = cg ? 1 : 0;
  a1.dots_out = &W.ks->rho1;
  a1.pred = pred;
  const bool exact = exact_reductions();
  if (exact) {  // SpMV, then the two dots in the reference's chunk order
    spmv_run(Ac, Epi::kSpmv, a1);
    DotOp<2> d;
    d.a[0] = cg ? W.c : W.v;  // rho1 = c.v | v.v
    d.b[0] = W.v;
    d.a[1] = cg ? W.c : W.v;  // alpha1 = c.rc | v.rc
    d.b[1] = rc;
    d.pred = pred;
    launch_chunked<2>(d, nc, &W.ks->rho1);
    KStep1Op op;
    op.ks = W.ks;
    op.tt = cfg.t;
    op.rc = rc;
    op.v = W.v;
    op.rt = W.rt;
    op.pred = pred;
    op.warn = warn_bits();
    op.level = level;
    launch_chunked<2>(op, nc, &W.ks->nrt);
  } else {
    spmv_run(Ac, Epi::kSpmvDot2, a1);
    const unsigned g = reduce_grid(nc);
    AGG_LAUNCH(k_kstep1, g, kB, 0, nc, rc, W.v, W.rt, W.ks, cfg.t, pred, reduce_partials(),
               reduce_ticket(), warn_bits(), level);
  }
  const int* p2 = &W.ks->flag2;
  inner_cycle(h, cfg, kc, W.rt, W.d, p2);
  SpmvArgs a2;  // w = Ac d ; gamma, beta, alpha2  (cycles.cpp:110-121)
  a2.x = W.d;
  a2.y = W.w;
  a2.u = W.v;
  a2.c = W.rt;
  a2.dot_with_x = cg ? 1 : 0;
  a2.dots_out = &W.ks->gamma;
  a2.pred = p2;
  if (exact) {
    spmv_run(Ac, Epi::kSpmv, a2);
    DotOp<3> d;
    const double* lhs = cg ? W.d : W.w;
    d.a[0] = lhs;  // gamma = d.v | w.v
    d.b[0] = W.v;
    d.a[1] = lhs;  // beta = d.w | w.w
    d.b[1] = W.w;
    d.a[2] = lhs;  // alpha2 = d.rt | w.rt
    d.b[2] = W.rt;
    d.pred = p2;
    launch_chunked<3>(d, nc, &W.ks->gamma);
  } else {
    spmv_run(Ac, Epi::kSpmvDot3, a2);
  }
  AGG_LAUNCH(k_kcombine, egrid(nc), kB, 0, nc, W.c, W.d, xc, W.ks, pred, warn_bits(), level);
}

// ---- building blocks of the row-partitioned cycle (dist_solve.cu) --------------------

namespace {
__global__ void k_kflag(KScalars* ks, double tt, const int* pred) {
  if (!on(pred) || ks->rho1 == 0.0) return;  // k_kstep1 already set flag2 = 0
  ks->flag2 = (__dsqrt_rn(ks->nrt) <= __dmul_rn(tt, __dsqrt_rn(ks->nrc))) ? 0 : 1;
}
}  // namespace

void launch_jacobi_zero(int64_t n, const double* wd, const double* b, double* x, const int* pred) {
  if (n > 0) AGG_LAUNCH(k_jacobi_zero, egrid(n), kB, 0, n, wd, b, x, pred);
}
void launch_prolong(int64_t n, const double* x, const idx* agg, const double* pval, const double* xc,
                    double* t, const int* pred) {
  if (n > 0) AGG_LAUNCH(k_prolong, egrid(n), kB, 0, n, x, agg, pval, xc, t, pred);
}
void launch_kstep1(int64_t n, const double* rc, const double* v, double* rt, KScalars* ks, double t,
                   const int* pred, int level) {
  AGG_LAUNCH(k_kstep1, reduce_grid(std::max<int64_t>(n, 1)), kB, 0, n, rc, v, rt, ks, t, pred,
             reduce_partials(), reduce_ticket(), warn_bits(), level);
}
void launch_kflag(KScalars* ks, double t, const int* pred) { AGG_LAUNCH(k_kflag, 1, 1, 0, ks, t, pred); }
void launch_kcombine(int64_t n, const double* c, const double* d, double* xc, const KScalars* ks,
                     const int* pred, int level) {
  AGG_LAUNCH(k_kcombine, egrid(std::max<int64_t>(n, 1)), kB, 0, n, c, d, xc, ks, pred, warn_bits(),
             level);
}
bool cycle_accelerated(const CycleCfg& cfg, int64_t k) { return accelerated(cfg, k); }

void coarse_solve(DevHierarchy& h, const double* b, double* x, const int* pred) {
  const int64_t n = h.levels.back().A->n_rows;
  if (n == 0) return;
  if (exact_reductions() && h.coarse_lu_ready) {  // bit-identical substitution (slow: n^2 chain)
    if (n <= kLuWarpRows) {
      const size_t wsmem = (static_cast<size_t>(n) * n + 2 * n) * sizeof(double);
      static std::atomic<unsigned long long> wattr{0};  // the attribute is per device
      if (device_pending(wattr)) {
        AGG_CUDA(cudaFuncSetAttribute(k_lu_solve_warp, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>((kLuWarpRows * kLuWarpRows + 2 * kLuWarpRows) *
                                                       sizeof(double))));
        mark_device(wattr);
      }
      AGG_LAUNCH(k_lu_solve_warp, 1, 256, wsmem, static_cast<int>(n), h.coarse_lu.get(),
                 h.coarse_perm.get(), b, x, pred);
      return;
    }
    const size_t smem = 3 * n * sizeof(double);
    if (n <= int64_t{kLuRows} * kLuThreads && smem <= 200 * 1024) {
      static std::atomic<unsigned long long> attr{0};  // the attribute is per device
      if (device_pending(attr)) {
        AGG_CUDA(cudaFuncSetAttribute(k_lu_solve, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      200 * 1024));
        mark_device(attr);
      }
      AGG_LAUNCH(k_lu_solve, 1, kLuThreads, smem, static_cast<int>(n), h.coarse_lu.get(),
                 h.coarse_lu_t.get(), h.coarse_perm.get(), b, x, pred);
    } else {
      AGG_LAUNCH(k_lu_serial, 1, 32, 0, n, h.coarse_lu.get(), h.coarse_perm.get(), b, x, pred);
    }
    return;
  }
  AGG_LAUNCH(k_gemv, grid_for(n * 32, 256), 256, 0, n, h.coarse_inv.get(), b, x, pred);
}

void cycle(DevHierarchy& h, const CycleCfg& cfg, int64_t k, bool accelerated_top, const double* b,
           const double* x_in, double* x_out, const int* pred) {
  h.ensure_workspace();
  if (accelerated_top)
    kcycle_dev(h, cfg, k, b, x_in, x_out, pred);
  else
    vcycle_dev(h, k, b, x_in, x_out, pred);
}

void apply_preconditioner(DevHierarchy& h, const CycleCfg& cfg, const double* r, double* z) {
  h.ensure_workspace();
  inner_cycle(h, cfg, 0, r, z, nullptr);
  h.levels[0].zs_b = nullptr;  // a mark the cycle did not consume never outlives it
  h.levels[0].zs_x = nullptr;
}

const double* top_zero_sweep_diag(const DevHierarchy& h) {
  if (h.levels.empty() || h.coarsest() == 0 || h.levels[0].smoother.kind == 2) return nullptr;
  return h.levels[0].smoother.wdiag.get();
}

void mark_top_zero_sweep(DevHierarchy& h, const double* r, double* z) {
  h.levels[0].zs_b = r;
  h.levels[0].zs_x = z;
}

void flush_cycle_warnings() {
  if (ltimer().on && !ltimer().rec.empty()) {
    sync();
    double inc[32] = {0};
    int visits[32] = {0};
    for (auto& r : ltimer().rec) {
      float ms = 0.f;
      cudaEventElapsedTime(&ms, std::get<1>(r), std::get<2>(r));
      const int l = std::min(31, std::get<0>(r));
      inc[l] += ms;
      ++visits[l];
      cudaEventDestroy(std::get<1>(r));
      cudaEventDestroy(std::get<2>(r));
    }
    ltimer().rec.clear();
    for (int l = 0; l < 32; ++l)
      if (visits[l])
        std::fprintf(stderr, "[level timing] level %d: %d visits, inclusive %.3f ms, exclusive %.3f ms\n",
                     l, visits[l], inc[l], inc[l] - (l + 1 < 32 ? inc[l + 1] : 0.0));
  }
  int w[2];
  AGG_CUDA(cudaMemcpyAsync(w, warn_bits(), sizeof(w), cudaMemcpyDeviceToHost, stream()));
  AGG_CUDA(cudaStreamSynchronize(stream()));
  if (w[0] == 0 && w[1] == 0) return;
  for (int l = 0; l < 32; ++l) {
    if (w[0] & (1 << l))
      std::fprintf(stderr, "kcycle: zero curvature at level %d, keeping the unscaled correction\n", l);
    if (w[1] & (1 << l))
      std::fprintf(stderr,
                   "kcycle: singular inner Gram matrix at level %d, keeping the one-step correction\n",
                   l);
  }
  AGG_CUDA(cudaMemsetAsync(warn_bits(), 0, 2 * sizeof(int), stream()));
}

}  // namespace aggmg_b200
