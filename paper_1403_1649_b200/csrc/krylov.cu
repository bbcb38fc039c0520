// krylov.cu — device PCG / FGMRES.  Vector work is fused into few HBM passes; the
// per-iteration host readback is one small pinned copy (the residual or the Hessenberg
// column the host's Givens recurrence needs).
#include <chrono>
#include <algorithm>
#include <cmath>

#include "chunked.cuh"
#include "krylov.cuh"
#include "vecops.cuh"

namespace aggmg_b200 {

namespace {

using Clock = std::chrono::steady_clock;
constexpr int kB = 256;

struct PcgSlots {
  double pAp;
  double res2;
  double q[2][2];  // q[par] = {r.z, r_old.z} of the iteration that produced it
  double pad[2];
};

// alpha = rz/pAp; rn = r + (-alpha) Ap; res2 = ||rn||^2  (krylov.cpp:181-186).  x += alpha p
// is deferred to k_pcg_p (which reads p anyway) or, after the last iteration, to k_pcg_x.
// wd: also the preconditioner's first operation, z = 0 + wd .* rn (the level-0 zero-guess
// damped-Jacobi sweep, k_jacobi_zero's arithmetic), while rn is in registers
__global__ void __launch_bounds__(kB) k_pcg_update(int64_t n, PcgSlots* s, int par,
                                                   const double* __restrict__ p,
                                                   const double* __restrict__ Ap,
                                                   const double* __restrict__ r, double* __restrict__ x,
                                                   double* __restrict__ rn, double* partials,
                                                   unsigned* ticket, const double* __restrict__ wd,
                                                   double* __restrict__ z) {
  __shared__ double smem[32];
  const double alpha = __ddiv_rn(s->q[par][0], s->pAp);
  const double malpha = -alpha;
  double acc[1] = {0.0};
  // 128-bit loads/stores: pairs (2i, 2i+1); the odd tail element goes to the last pair slot
  const int64_t npair = n >> 1;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < npair; q += stride) {
    const double2 aq = reinterpret_cast<const double2*>(Ap)[q];
    const double2 rq = reinterpret_cast<const double2*>(r)[q];
    const double v0 = __dadd_rn(rq.x, __dmul_rn(malpha, aq.x));
    const double v1 = __dadd_rn(rq.y, __dmul_rn(malpha, aq.y));
    reinterpret_cast<double2*>(rn)[q] = make_double2(v0, v1);
    if (wd) {
      const double2 w = reinterpret_cast<const double2*>(wd)[q];
      reinterpret_cast<double2*>(z)[q] =
          make_double2(__dadd_rn(0.0, __dmul_rn(w.x, v0)), __dadd_rn(0.0, __dmul_rn(w.y, v1)));
    }
    acc[0] = __dadd_rn(acc[0], __dmul_rn(v0, v0));
    acc[0] = __dadd_rn(acc[0], __dmul_rn(v1, v1));
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t i = n - 1;
    const double v = __dadd_rn(r[i], __dmul_rn(malpha, Ap[i]));
    rn[i] = v;
    if (wd) z[i] = __dadd_rn(0.0, __dmul_rn(wd[i], v));
    acc[0] = __dadd_rn(acc[0], __dmul_rn(v, v));
  }
  block_reduce<1>(acc, smem);
  if (threadIdx.x == 0) partials[blockIdx.x] = acc[0];
  finish_reduction<1>(partials, ticket, &s->res2, smem);
}

// x += alpha p (this iteration's alpha = rz / pAp, krylov.cpp:182), then
// beta = (rz_new - r_old.z) / rz ; p = z + beta p  (krylov.cpp:191-195)
__global__ void k_pcg_p(int64_t n, const PcgSlots* s, int cur, const double* __restrict__ z,
                        double* __restrict__ p, double* __restrict__ x) {
  const double alpha = __ddiv_rn(s->q[cur ^ 1][0], s->pAp);
  const double beta = __ddiv_rn(__dsub_rn(s->q[cur][0], s->q[cur][1]), s->q[cur ^ 1][0]);
  const int64_t np = n >> 1, stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < np; q += stride) {
    const double2 pq = reinterpret_cast<const double2*>(p)[q];
    const double2 zq = reinterpret_cast<const double2*>(z)[q];
    if (x) {
      double2 xq = reinterpret_cast<double2*>(x)[q];
      xq.x = __dadd_rn(xq.x, __dmul_rn(alpha, pq.x));
      xq.y = __dadd_rn(xq.y, __dmul_rn(alpha, pq.y));
      reinterpret_cast<double2*>(x)[q] = xq;
    }
    reinterpret_cast<double2*>(p)[q] =
        make_double2(__dadd_rn(zq.x, __dmul_rn(beta, pq.x)), __dadd_rn(zq.y, __dmul_rn(beta, pq.y)));
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t i = n - 1;
    const double pi = p[i];
    if (x) x[i] = __dadd_rn(x[i], __dmul_rn(alpha, pi));
    p[i] = __dadd_rn(z[i], __dmul_rn(beta, pi));
  }
}
// the last iteration's x += alpha p (no p update follows)
__global__ void k_pcg_x(int64_t n, const PcgSlots* s, int par, const double* __restrict__ p,
                        double* __restrict__ x) {
  const double alpha = __ddiv_rn(s->q[par][0], s->pAp);
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
}

// MGS step i of column j (krylov.cpp:85-89): w = w + (-h_i) V_i, then the next
// coefficient dot(V_{i+1}, w) or, after the last basis vector, ||w||^2.
__global__ void __launch_bounds__(kB) k_mgs_step(int64_t n, const double* hcol, int i,
                                                 const double* __restrict__ Vi,
                                                 const double* __restrict__ Vnext,
                                                 double* __restrict__ w, double* out,
                                                 double* partials, unsigned* ticket) {
  __shared__ double smem[32];
  const double mh = -hcol[i];
  double acc[1] = {0.0};
  // 16-byte accesses: three streams of a 450 MB basis vector per step need the bytes in flight
  const int64_t np = n >> 1;
  const double2* Vi2 = reinterpret_cast<const double2*>(Vi);
  const double2* Vn2 = reinterpret_cast<const double2*>(Vnext);
  double2* w2 = reinterpret_cast<double2*>(w);
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < np;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double2 v = w2[t];
    const double2 a = Vi2[t];
    v.x = __dadd_rn(v.x, __dmul_rn(mh, a.x));
    v.y = __dadd_rn(v.y, __dmul_rn(mh, a.y));
    w2[t] = v;
    const double2 o = Vnext ? Vn2[t] : v;
    acc[0] = __dadd_rn(acc[0], __dmul_rn(o.x, v.x));
    acc[0] = __dadd_rn(acc[0], __dmul_rn(o.y, v.y));
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const int64_t t = n - 1;
    const double v = __dadd_rn(w[t], __dmul_rn(mh, Vi[t]));
    w[t] = v;
    const double o = Vnext ? Vnext[t] : v;
    acc[0] = __dadd_rn(acc[0], __dmul_rn(o, v));
  }
  block_reduce<1>(acc, smem);
  if (threadIdx.x == 0) partials[blockIdx.x] = acc[0];
  finish_reduction<1>(partials, ticket, out, smem);
}
unsigned mgs_grid(int64_t n) {
  const int64_t want = (n / 2 + kB - 1) / kB;
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(want, 8 * int64_t{sm_count()})));
}

// ---- reference-order (exact) variants of the fused vector kernels ---------------------

// x += alpha p ; rn = r + (-alpha) Ap ; chain: rn_i^2   (krylov.cpp:181-186)
struct PcgUpdateOp {
  PcgSlots* s;
  int par;
  const double *p, *Ap, *r;
  double *x, *rn;
  double alpha, malpha;
  __device__ bool active() const { return true; }
  __device__ void inactive() const {}
  __device__ void init() {
    alpha = __ddiv_rn(s->q[par][0], s->pAp);
    malpha = -alpha;
  }
  __device__ void operator()(int64_t i, double* out) const {
    x[i] = __dadd_rn(x[i], __dmul_rn(alpha, p[i]));
    const double v = __dadd_rn(r[i], __dmul_rn(malpha, Ap[i]));
    rn[i] = v;
    out[0] = __dmul_rn(v, v);
  }
  __device__ void finalize(double*) const {}
};

// w = w + (-h_i) V_i ; chain: V_{i+1}.w or w.w   (krylov.cpp:85-89)
struct MgsOp {
  const double* hcol;
  int idx;
  const double *Vi, *Vnext;
  double* w;
  double mh;
  __device__ bool active() const { return true; }
  __device__ void inactive() const {}
  __device__ void init() { mh = -hcol[idx]; }
  __device__ void operator()(int64_t t, double* out) const {
    const double v = __dadd_rn(w[t], __dmul_rn(mh, Vi[t]));
    w[t] = v;
    out[0] = __dmul_rn(Vnext ? Vnext[t] : v, v);
  }
  __device__ void finalize(double*) const {}
};

struct AxpyList {
  const double* z[32];
  double y[32];
  int count;
};
// x = x + y_0 Z_0, then + y_1 Z_1, ... (krylov.cpp:128), one pass over x
__global__ void k_multi_axpy(int64_t n, AxpyList L, double* __restrict__ x) {
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double v = x[t];
    for (int i = 0; i < L.count; ++i) v = __dadd_rn(v, __dmul_rn(L.y[i], L.z[i][t]));
    x[t] = v;
  }
}

unsigned egrid(int64_t n) { return grid_for(n, kB, 8 * static_cast<int64_t>(sm_count())); }

void apply_M(const Precond& M, const double* r, double* z, int64_t n, const KrylovDist* dist) {
  if (dist && dist->precond) {
    dist->precond(r, z);
  } else if (M.host_fn) {  // one device->host->device round trip per application
    M.host_r.resize(n);
    M.host_z.resize(n);
    device_to_host(M.host_r.data(), r, sizeof(double) * n);
    sync();
    require(M.host_fn(M.host_r.data(), M.host_z.data(), n, M.host_user) == 0,
            "krylov: the preconditioner callback failed");
    host_to_device(z, M.host_z.data(), sizeof(double) * n);
  } else if (M.h)
    apply_preconditioner(*M.h, M.cfg, r, z);
  else
    copy_double(z, r, n);
}

void residual(const DevCsr& A, const double* b, const double* x, double* r, const KrylovDist* dist) {
  SpmvArgs a;
  a.x = x;
  a.y = r;
  a.b = b;
  if (dist)
    dist->spmv(Epi::kResidual, a, 0);  // halo exchange overlapped with the interior rows
  else
    spmv_run(A, Epi::kResidual, a);
}

double norm_host(const double* v, int64_t n, const KrylovDist* dist = nullptr) {
  if (!dist) return std::sqrt(dot_host(v, v, n));
  DevBuf<double> d(1);
  DotArgs a{};
  a.a[0] = v;
  a.b[0] = v;
  a.np = 1;
  if (n > 0)
    dot_device(a, n, d.get(), nullptr, 0);
  else
    d.zero();
  dist->allreduce(d.get(), 1);
  return std::sqrt(read_scalar(d.get()));
}
void reduce(const KrylovDist* dist, double* v, int k) {
  if (dist) dist->allreduce(v, k);
}

double seconds_since(Clock::time_point t0) {
  return std::chrono::duration<double>(Clock::now() - t0).count();
}

}  // namespace

SolveOut pcg(const DevCsr& A, const double* b, double* x, const Precond& M, const SolverCfg& cfg,
             const KrylovDist* dist) {
  require(dist || A.n_rows == A.n_cols, "pcg: matrix must be square");
  require(cfg.tol > 0.0, "pcg: tol must be positive");
  const auto t0 = Clock::now();
  const int64_t n = A.n_rows;
  SolveOut out;
  const double norm_b = norm_host(b, n, dist);
  if (norm_b == 0.0) {
    fill_double(x, n, 0.0);
    out.converged = true;
    out.history.push_back(0.0);
    sync();
    out.solve_seconds = seconds_since(t0);
    return out;
  }
  const double target = cfg.tol * norm_b;
  const bool exact = exact_reductions() && !dist;
  const int64_t n_alloc = dist ? dist->n_alloc : n;  // SpMV inputs and cycle outputs carry a halo
  DevBuf<double> rA(n), rB(n), z(n_alloc), p(n_alloc), Ap(n);
  DevBuf<PcgSlots> slots(1);
  slots.zero();
  double* r = rA.get();
  double* rn = rB.get();
  residual(A, b, x, r, dist);
  double res = norm_host(r, n, dist);
  out.history.push_back(res);
  // (r.z, r_old.z) fused into the preconditioner's last level-0 sweep when possible
  const bool fuse = !exact && (dist ? static_cast<bool>(dist->precond_dots) : M.h != nullptr);
  auto precond_dots = [&](const double* rr, const double* rold, double* q, int np) {
    bool fused = false;
    if (fuse && dist) {
      fused = dist->precond_dots(rr, rold, z.get(), q);
    } else {
      if (fuse) {
        M.h->top_dot_c = rold;
        M.h->top_dot_out = q;
        M.h->top_dot_done = false;
      }
      apply_M(M, rr, z.get(), n, dist);
      fused = fuse && M.h->top_dot_done;
      if (fuse) {
        M.h->top_dot_c = nullptr;
        M.h->top_dot_out = nullptr;
      }
    }
    if (!fused) {
      DotArgs d{};
      d.a[0] = rr;
      d.b[0] = z.get();
      d.a[1] = rold;
      d.b[1] = z.get();
      d.np = np;
      dot_device(d, n, q);
      reduce(dist, q, np);
    }
  };
  precond_dots(r, r, &slots.get()->q[0][0], 1);
  copy_double(p.get(), z.get(), n);
  // the update pass also writes the preconditioner's level-0 zero-guess sweep into z
  const double* wd0 = (fuse && !dist && M.h && !M.host_fn) ? top_zero_sweep_diag(*M.h) : nullptr;
  double* pinned = pinned_scratch(8);
  int par = 0;  // q[par][0] holds the current r.z
  while (res > target && out.iterations < cfg.max_iters) {
    SpmvArgs a;  // Ap = A p ; pAp
    a.x = p.get();
    a.y = Ap.get();
    a.u = p.get();
    a.dots_out = &slots.get()->pAp;
    if (exact) {
      spmv_run(A, Epi::kSpmv, a, kProfSpmvL0);
      DotOp<1> d1;
      d1.a[0] = p.get();
      d1.b[0] = Ap.get();
      d1.pred = nullptr;
      launch_chunked<1>(d1, n, &slots.get()->pAp);
      PcgUpdateOp u;
      u.s = slots.get();
      u.par = par;
      u.p = p.get();
      u.Ap = Ap.get();
      u.r = r;
      u.x = x;
      u.rn = rn;
      launch_chunked<1>(u, n, &slots.get()->res2);
    } else {
      if (dist)
        dist->spmv(Epi::kSpmvDot1, a, kProfSpmvL0);
      else
        spmv_run(A, Epi::kSpmvDot1, a, kProfSpmvL0);
      reduce(dist, &slots.get()->pAp, 1);
      AGG_LAUNCH(k_pcg_update, reduce_grid(n), kB, 0, n, slots.get(), par, p.get(), Ap.get(), r, x,
                 rn, reduce_partials(), reduce_ticket(), wd0, z.get());
      reduce(dist, &slots.get()->res2, 1);
    }
    AGG_CUDA(cudaMemcpyAsync(pinned, slots.get(), 2 * sizeof(double), cudaMemcpyDeviceToHost,
                             stream()));
    sync();
    const double pAp = pinned[0];
    require(pAp > 0.0, "pcg: non-positive curvature (matrix not positive definite); use fgmres");
    ++out.iterations;
    res = std::sqrt(pinned[1]);
    out.history.push_back(res);
    std::swap(r, rn);  // r = new residual, rn = r_old
    if (res <= target) {
      if (!exact) AGG_LAUNCH(k_pcg_x, egrid(n), kB, 0, n, slots.get(), par, p.get(), x);
      break;
    }
    const int cur = par ^ 1;
    if (wd0) mark_top_zero_sweep(*M.h, r, z.get());  // z = 0 + wd .* r is in place already
    precond_dots(r, rn, &slots.get()->q[cur][0], 2);  // {r.z, r_old.z}
    if (exact) {
      AGG_LAUNCH(k_pcg_p, reduce_grid(n), kB, 0, n, slots.get(), cur, z.get(), p.get(), nullptr);
    } else {
      AGG_LAUNCH(k_pcg_p, reduce_grid(n), kB, 0, n, slots.get(), cur, z.get(), p.get(), x);
    }
    par = cur;
  }
  if (dist && dist->flush_warnings)
    dist->flush_warnings();
  else if (M.h)
    flush_cycle_warnings();
  out.converged = res <= target;
  sync();
  out.solve_seconds = seconds_since(t0);
  return out;
}

SolveOut fgmres(const DevCsr& A, const double* b, double* x, const Precond& M,
                const SolverCfg& cfg, const KrylovDist* dist) {
  require(dist || A.n_rows == A.n_cols, "fgmres: matrix must be square");
  require(cfg.tol > 0.0, "fgmres: tol must be positive");
  require(cfg.restart >= 1, "fgmres: restart must be at least 1");
  const auto t0 = Clock::now();
  const int64_t n = A.n_rows;
  const int m = cfg.restart;
  SolveOut out;
  const double norm_b = norm_host(b, n, dist);
  if (norm_b == 0.0) {
    fill_double(x, n, 0.0);
    out.converged = true;
    out.history.push_back(0.0);
    sync();
    out.solve_seconds = seconds_since(t0);
    return out;
  }
  const double target = cfg.tol * norm_b;
  const bool exact = exact_reductions() && !dist;
  const int64_t nz_alloc = dist ? dist->n_alloc : n;
  DevBuf<double> r(n), w(n), hcol(m + 2);
  std::vector<DevBuf<double>> V, Z;
  residual(A, b, x, r.get(), dist);
  double beta = norm_host(r.get(), n, dist);
  out.history.push_back(beta);
  std::vector<double> H(static_cast<size_t>(m + 1) * m, 0.0);  // column-major, ld m+1
  auto h = [&](int i, int j) -> double& { return H[static_cast<size_t>(j) * (m + 1) + i]; };
  std::vector<double> cs(m), sn(m), g(m + 1);
  double* pinned = pinned_scratch(m + 2);
  double prev_outer = beta;
  while (beta > target && out.iterations < cfg.max_iters) {
    if (V.empty()) V.emplace_back(n);
    vec_scale_into(n, 1.0 / beta, r.get(), V[0].get());
    std::fill(g.begin(), g.end(), 0.0);
    g[0] = beta;
    std::fill(H.begin(), H.end(), 0.0);
    int j = 0;
    for (; j < m && out.iterations < cfg.max_iters; ++j) {
      if (static_cast<int>(Z.size()) <= j) Z.emplace_back(nz_alloc);
      apply_M(M, V[j].get(), Z[j].get(), n, dist);
      SpmvArgs a;  // w = A Z_j ; h(0,j) = V_0 . w
      a.x = Z[j].get();
      a.y = w.get();
      a.u = V[0].get();
      a.dots_out = hcol.get();
      if (exact) {
        spmv_run(A, Epi::kSpmv, a, kProfSpmvL0);
        DotOp<1> d1;
        d1.a[0] = V[0].get();
        d1.b[0] = w.get();
        d1.pred = nullptr;
        launch_chunked<1>(d1, n, hcol.get());
      } else {
        if (dist)
          dist->spmv(Epi::kSpmvDot1, a, kProfSpmvL0);
        else
          spmv_run(A, Epi::kSpmvDot1, a, kProfSpmvL0);
        reduce(dist, hcol.get(), 1);
      }
      for (int i = 0; i <= j; ++i) {
        const double* vnext = (i < j) ? V[i + 1].get() : nullptr;
        if (exact) {
          MgsOp op;
          op.hcol = hcol.get();
          op.idx = i;
          op.Vi = V[i].get();
          op.Vnext = vnext;
          op.w = w.get();
          launch_chunked<1>(op, n, hcol.get() + i + 1);
        } else {
          AGG_LAUNCH(k_mgs_step, mgs_grid(n), kB, 0, n, hcol.get(), i, V[i].get(), vnext,
                     w.get(), hcol.get() + i + 1, reduce_partials(), reduce_ticket());
          reduce(dist, hcol.get() + i + 1, 1);
        }
      }
      AGG_CUDA(cudaMemcpyAsync(pinned, hcol.get(), sizeof(double) * (j + 2),
                               cudaMemcpyDeviceToHost, stream()));
      sync();
      for (int i = 0; i <= j; ++i) h(i, j) = pinned[i];
      h(j + 1, j) = std::sqrt(pinned[j + 1]);
      const bool breakdown = (h(j + 1, j) == 0.0);
      if (!breakdown) {
        if (static_cast<int>(V.size()) <= j + 1) V.emplace_back(n);
        vec_scale_into(n, 1.0 / h(j + 1, j), w.get(), V[j + 1].get());
      }
      for (int i = 0; i < j; ++i) {  // apply previous rotations (krylov.cpp:95-99)
        const double t = cs[i] * h(i, j) + sn[i] * h(i + 1, j);
        h(i + 1, j) = -sn[i] * h(i, j) + cs[i] * h(i + 1, j);
        h(i, j) = t;
      }
      const double denom = std::hypot(h(j, j), h(j + 1, j));
      if (denom == 0.0) {
        cs[j] = 1.0;
        sn[j] = 0.0;
      } else {
        cs[j] = h(j, j) / denom;
        sn[j] = h(j + 1, j) / denom;
      }
      h(j, j) = cs[j] * h(j, j) + sn[j] * h(j + 1, j);
      h(j + 1, j) = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      ++out.iterations;
      out.history.push_back(std::abs(g[j + 1]));
      if (std::abs(g[j + 1]) <= target || breakdown) {
        ++j;
        break;
      }
    }
    std::vector<double> y(j);  // krylov.cpp:122-127
    for (int i = j - 1; i >= 0; --i) {
      double s = g[i];
      for (int l = i + 1; l < j; ++l) s -= h(i, l) * y[l];
      y[i] = s / h(i, i);
    }
    for (int i0 = 0; i0 < j; i0 += 32) {  // same left-to-right sequence per element
      AxpyList L{};
      L.count = std::min(32, j - i0);
      for (int i = 0; i < L.count; ++i) {
        L.z[i] = Z[i0 + i].get();
        L.y[i] = y[i0 + i];
      }
      AGG_LAUNCH(k_multi_axpy, egrid(n), kB, 0, n, L, x);
    }
    residual(A, b, x, r.get(), dist);
    beta = norm_host(r.get(), n, dist);
    out.history.back() = beta;
    if (beta > target && beta >= prev_outer && j == m)
      out.note = "stagnation: no residual decrease over a full restart cycle";
    prev_outer = beta;
  }
  if (dist && dist->flush_warnings)
    dist->flush_warnings();
  else if (M.h)
    flush_cycle_warnings();
  out.converged = beta <= target;
  sync();
  out.solve_seconds = seconds_since(t0);
  return out;
}

}  // namespace aggmg_b200
