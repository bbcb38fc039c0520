// smoother.cu — inverse diagonal, Arnoldi spectral-radius estimate, sweeps.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "chunked.cuh"
#include "dense_host.hpp"
#include "smoother.cuh"
#include "vecops.cuh"

namespace aggmg_b200 {

namespace {

__global__ void k_inv_diag(const idx* rp, const idx* col, const double* val, int64_t n,
                           double* inv, int* bad_row) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double d = 0.0;
  for (idx k = rp[i]; k < rp[i + 1]; ++k)
    if (col[k] == i) d = val[k];
  if (d == 0.0) {
    atomicMin(bad_row, static_cast<int>(i));
    inv[i] = 0.0;
    return;
  }
  inv[i] = __ddiv_rn(1.0, d);
}

// One fused MGS step of the Arnoldi column on the device, in the reference's chunked dot
// order: w = w + (-h) V_i (skipped for the column's first step), then (V_next . w,
// V_next . V_next) — or (w . w, 0) after the last basis vector.  The host path this replaces
// ran dot2 (sync) + axpy per coefficient; the fused form makes one pass per coefficient and
// one host read per column, with bit-identical coefficients (same operations, same order).
struct ArnoldiStepOp {
  const double* hsrc;  // device coefficient h to subtract with (nullptr: first step)
  const double* vi;
  double* w;
  const double* vn;  // next basis vector (nullptr: last step, out = w . w)
  double mh;
  const int* go;  // device flag (batched setup): 0 after an Arnoldi breakdown
  __device__ bool active() const { return !go || *go; }
  __device__ void inactive() const {}
  __device__ void init() { mh = hsrc ? -*hsrc : 0.0; }
  __device__ void operator()(int64_t t, double* p) const {
    double wt = w[t];
    if (hsrc) {
      wt = __dadd_rn(wt, __dmul_rn(mh, vi[t]));  // vec_axpy(-h, V_i, w)
      w[t] = wt;
    }
    if (vn) {
      const double v = vn[t];
      p[0] = __dmul_rn(v, wt);
      p[1] = __dmul_rn(v, v);
    } else {
      p[0] = __dmul_rn(wt, wt);
      p[1] = 0.0;
    }
  }
  __device__ void finalize(double*) const {}
};

__global__ void k_hdiv(const double* s, double* h, const int* go = nullptr) {
  if (!go || *go) *h = s[0] / s[1];
}

double estimate_rho(const DevCsr& A, const double* inv_diag, int m, uint64_t seed,
                    const ArnoldiOps* ops) {
  const int64_t n = A.n_rows;
  const int64_t n_alloc = ops ? ops->n_alloc : n;
  m = static_cast<int>(std::min<int64_t>(m, ops ? ops->n_global : n));
  auto dot = [&](const double* a, const double* b) {
    return ops ? ops->dot(a, b) : dot_host(a, b, n, 1);
  };
  std::vector<DevBuf<double>> V;
  V.emplace_back(n_alloc);
  if (ops)
    ops->start(V[0].get());
  else
    vec_uniform_sym(n, seed, V[0].get());
  const double qn = std::sqrt(dot(V[0].get(), V[0].get()));
  require(qn > 0.0, "smoother: degenerate start vector");
  vec_scale(n, 1.0 / qn, V[0].get());

  std::vector<double> H(static_cast<size_t>(m + 1) * m, 0.0);  // row-major (m+1) x m
  auto h = [&](int i, int j) -> double& { return H[static_cast<size_t>(i) * m + j]; };
  int m_eff = m;
  // device copies: column j's coefficients Hc[i] (i <= j), step slots, the final ||w||^2
  DevBuf<double> w(n), Hc(m + 1), slots(2);
  double* pin = pinned_scratch(m + 2);
  for (int j = 0; j < m; ++j) {
    if (ops) ops->before_spmv(V[j].get());  // halo of the Krylov vector
    SpmvArgs a;
    a.x = V[j].get();
    a.y = w.get();
    a.d = inv_diag;
    spmv_run(A, Epi::kScaleDiag, a);
    for (int i = -1; i <= j; ++i) {  // i = -1: the first dots, no axpy
      ArnoldiStepOp op;
      op.go = nullptr;
      op.hsrc = i >= 0 ? Hc.get() + i : nullptr;
      op.vi = i >= 0 ? V[i].get() : nullptr;
      op.w = w.get();
      op.vn = i < j ? V[i + 1].get() : nullptr;
      if (n > 0)
        launch_chunked<2>(op, n, slots.get());
      else
        slots.zero();
      if (ops) ops->allreduce_dev(slots.get(), 2);
      if (i < j)
        AGG_LAUNCH(k_hdiv, 1, 1, 0, slots.get(), Hc.get() + i + 1);  // h(i+1, j)
    }
    // one read per column: h(0..j, j) and ||w||^2
    AGG_CUDA(cudaMemcpyAsync(pin, Hc.get(), sizeof(double) * (j + 1), cudaMemcpyDeviceToHost, stream()));
    AGG_CUDA(cudaMemcpyAsync(pin + j + 1, slots.get(), sizeof(double), cudaMemcpyDeviceToHost, stream()));
    sync();
    double h_scale = 0.0;
    for (int i = 0; i <= j; ++i) {
      h(i, j) = pin[i];
      h_scale = std::max(h_scale, std::abs(pin[i]));
    }
    const double hj = std::sqrt(pin[j + 1]);
    if (hj <= 1e-12 * std::max(h_scale, 1.0)) {
      m_eff = j + 1;
      break;
    }
    h(j + 1, j) = hj;
    if (j + 1 < m) {
      V.emplace_back(n_alloc);
      vec_scale_into(n, 1.0 / hj, w.get(), V.back().get());
    }
  }
  std::vector<double> Hm(static_cast<size_t>(m_eff) * m_eff);
  for (int i = 0; i < m_eff; ++i)
    for (int j = 0; j < m_eff; ++j) Hm[static_cast<size_t>(i) * m_eff + j] = h(i, j);
  double rho = 0.0;
  for (const auto& ev : hessenberg_eigenvalues(Hm, m_eff)) rho = std::max(rho, std::abs(ev));
  require(rho > 0.0, "smoother: spectral radius estimate collapsed to zero");
  return rho;
}

__global__ void k_scale_diag(const double* inv, double omega, int64_t n, double* wd) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) wd[i] = __dmul_rn(omega, inv[i]);
}

}  // namespace

void setup_smoother(const DevCsr& A, int kind, int arnoldi_m, uint64_t seed, SmootherDev& s,
                    const ArnoldiOps* ops) {
  require(ops || A.n_rows == A.n_cols, "smoother: matrix must be square");
  require(arnoldi_m >= 1 && arnoldi_m <= 5, "smoother: arnoldi_m must be in [1, 5]");
  const int64_t n = A.n_rows;
  s.kind = kind;
  s.arnoldi_m = arnoldi_m;
  s.inv_diag.resize(n);
  DevBuf<int> bad(1);
  fill_int(bad.get(), 1, INT32_MAX);
  if (n > 0)
    AGG_LAUNCH(k_inv_diag, grid_for(n, 256), 256, 0, A.rowptr.get(), A.col.get(), A.val.get(), n,
               s.inv_diag.get(), bad.get());
  const int b = read_scalar(bad.get());
  if (b != INT32_MAX)
    throw Error("smoother: zero diagonal at row " + std::to_string(b + (ops ? ops->row0 : 0)));
  s.omega = 1.0;
  s.rho_est = 1.0;
  if (kind == 1) {  // damped Jacobi
    s.rho_est = estimate_rho(A, s.inv_diag.get(), arnoldi_m, seed, ops);
    s.omega = (4.0 / 3.0) / s.rho_est;
  }
  if (kind == 2) build_sgs_schedule(A, s);
  const double w = (kind == 0) ? 1.0 : s.omega;  // smoother.cpp:120
  s.wdiag.resize(n);
  if (n > 0)
    AGG_LAUNCH(k_scale_diag, grid_for(n, 256), 256, 0, s.inv_diag.get(), w, n, s.wdiag.get());
}

void smooth_sweep(const SmootherDev& s, const DevCsr& A, const double* b, const double* x,
                  double* x_out, const int* pred, int prof) {
  SpmvArgs a;
  a.x = x;
  a.y = x_out;
  a.b = b;
  a.d = s.wdiag.get();
  a.pred = pred;
  spmv_run(A, Epi::kJacobi, a, prof);
}

// ---- batched (overlapped) smoother setup ---------------------------------------------------

namespace {

// qn = ||V0|| from the exact dot; V0 *= 1/qn (smoother.cpp:51-54)
__global__ void k_arn_start(const double* d2, double* inv_qn, int* go, int* status) {
  const double qn = sqrt(d2[0]);
  if (!(qn > 0.0)) {
    *status = 1;
    *go = 0;
  } else {
    *inv_qn = 1.0 / qn;
  }
}
__global__ void k_scale_by(int64_t n, const double* f, const double* x, double* y, const int* go) {
  if (!*go) return;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) y[i] = __dmul_rn(x[i], *f);
}
// end of column j (smoother.cpp:62-81): record h(0..j, j), breakdown test, h(j+1, j), 1/h
__global__ void k_arn_col(int j, int m, const double* Hc, const double* slots, double* H,
                          double* inv_h, int* meff, int* go) {
  if (!*go) return;
  double h_scale = 0.0;
  for (int i = 0; i <= j; ++i) {
    H[i * m + j] = Hc[i];
    h_scale = fmax(h_scale, fabs(Hc[i]));
  }
  const double hj = sqrt(slots[0]);
  if (hj <= 1e-12 * fmax(h_scale, 1.0)) {
    *meff = j + 1;
    *go = 0;
    return;
  }
  H[(j + 1) * m + j] = hj;
  *inv_h = 1.0 / hj;
}

}  // namespace

struct SmootherBatch::Job {
  int key = 0;
  int m = 0;
  std::vector<DevBuf<double>> V;
  DevBuf<double> w, Hc, slots, H, scal;  // scal: [0] |V0|^2, [1] 1/|V0|, [2] 1/h
  DevBuf<int> flags;                     // [0] go, [1] m_eff, [2] status
  cudaEvent_t done = nullptr;
  ~Job() {
    if (done) cudaEventDestroy(done);
  }
};

SmootherBatch::SmootherBatch() = default;

SmootherBatch::~SmootherBatch() {
  if (!jobs_.empty()) cudaStreamSynchronize(background_stream());  // buffers die after the chains
}

void SmootherBatch::add(const DevCsr& A, int kind, int arnoldi_m, uint64_t seed, SmootherDev& s,
                        int key) {
  const int64_t n = A.n_rows;
  if (kind != 1 || n == 0) {  // nothing to overlap
    setup_smoother(A, kind, arnoldi_m, seed, s);
    return;
  }
  require(A.n_rows == A.n_cols, "smoother: matrix must be square");
  require(arnoldi_m >= 1 && arnoldi_m <= 5, "smoother: arnoldi_m must be in [1, 5]");
  s.kind = kind;
  s.arnoldi_m = arnoldi_m;
  s.inv_diag.resize(n);
  DevBuf<int> bad(1);
  fill_int(bad.get(), 1, INT32_MAX);
  AGG_LAUNCH(k_inv_diag, grid_for(n, 256), 256, 0, A.rowptr.get(), A.col.get(), A.val.get(), n,
             s.inv_diag.get(), bad.get());
  const int b = read_scalar(bad.get());
  if (b != INT32_MAX) throw Error("smoother: zero diagonal at row " + std::to_string(b));

  auto job = std::make_unique<Job>();
  const int m = static_cast<int>(std::min<int64_t>(arnoldi_m, n));
  job->key = key;
  job->m = m;
  // every buffer the side stream touches is allocated here, on the main stream, and lives
  // until finish() has joined
  for (int j = 0; j < m; ++j) job->V.emplace_back(n);
  job->w.resize(n);
  job->Hc.resize(m + 1);
  job->slots.resize(2);
  job->H.resize(static_cast<int64_t>(m + 1) * m);
  job->H.zero();
  job->scal.resize(3);
  job->flags.resize(3);
  const int f0[3] = {1, m, 0};
  job->flags.upload(f0, 3);
  cudaEvent_t ready;
  AGG_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  AGG_CUDA(cudaEventRecord(ready, stream()));  // A, inv_diag and the buffers are ready
  cudaStream_t side = background_stream();
  AGG_CUDA(cudaStreamWaitEvent(side, ready, 0));
  cudaEventDestroy(ready);
  {
    StreamRedirect on_side(side);
    const int* go = job->flags.get();
    int* gom = job->flags.get();
    double* V0 = job->V[0].get();
    vec_uniform_sym(n, seed, V0);
    DotOp<1> d0;
    d0.a[0] = V0;
    d0.b[0] = V0;
    d0.pred = nullptr;
    launch_dot_exact<1>(d0, n, job->scal.get());
    AGG_LAUNCH(k_arn_start, 1, 1, 0, job->scal.get(), job->scal.get() + 1, gom,
               job->flags.get() + 2);
    AGG_LAUNCH(k_scale_by, grid_for(n, 256), 256, 0, n, job->scal.get() + 1, V0, V0, go);
    for (int j = 0; j < m; ++j) {
      SpmvArgs a;
      a.x = job->V[j].get();
      a.y = job->w.get();
      a.d = s.inv_diag.get();
      a.pred = go;
      spmv_run(A, Epi::kScaleDiag, a);
      for (int i = -1; i <= j; ++i) {
        ArnoldiStepOp op;
        op.go = go;
        op.hsrc = i >= 0 ? job->Hc.get() + i : nullptr;
        op.vi = i >= 0 ? job->V[i].get() : nullptr;
        op.w = job->w.get();
        op.vn = i < j ? job->V[i + 1].get() : nullptr;
        launch_chunked<2>(op, n, job->slots.get());
        if (i < j) AGG_LAUNCH(k_hdiv, 1, 1, 0, job->slots.get(), job->Hc.get() + i + 1, go);
      }
      AGG_LAUNCH(k_arn_col, 1, 1, 0, j, m, job->Hc.get(), job->slots.get(), job->H.get(),
                 job->scal.get() + 2, job->flags.get() + 1, gom);
      if (j + 1 < m)
        AGG_LAUNCH(k_scale_by, grid_for(n, 256), 256, 0, n, job->scal.get() + 2, job->w.get(),
                   job->V[j + 1].get(), go);
    }
    AGG_CUDA(cudaEventCreateWithFlags(&job->done, cudaEventDisableTiming));
    AGG_CUDA(cudaEventRecord(job->done, side));
  }
  jobs_.push_back(std::move(job));
}

void SmootherBatch::finish(const std::function<SmootherDev&(int)>& level) {
  if (jobs_.empty()) return;
  AGG_CUDA(cudaStreamSynchronize(background_stream()));
  auto jobs = std::move(jobs_);
  for (auto& j : jobs) {
    const int m = j->m;
    std::vector<double> H(static_cast<size_t>(m + 1) * m);
    int flags[3];
    AGG_CUDA(cudaMemcpy(H.data(), j->H.get(), sizeof(double) * H.size(), cudaMemcpyDeviceToHost));
    AGG_CUDA(cudaMemcpy(flags, j->flags.get(), sizeof(flags), cudaMemcpyDeviceToHost));
    require(flags[2] == 0, "smoother: degenerate start vector");
    const int m_eff = flags[1];
    std::vector<double> Hm(static_cast<size_t>(m_eff) * m_eff);
    for (int r = 0; r < m_eff; ++r)
      for (int c = 0; c < m_eff; ++c) Hm[static_cast<size_t>(r) * m_eff + c] = H[static_cast<size_t>(r) * m + c];
    double rho = 0.0;
    for (const auto& ev : hessenberg_eigenvalues(Hm, m_eff)) rho = std::max(rho, std::abs(ev));
    require(rho > 0.0, "smoother: spectral radius estimate collapsed to zero");
    SmootherDev& s = level(j->key);
    s.rho_est = rho;
    s.omega = (4.0 / 3.0) / rho;
    const int64_t n = s.inv_diag.size();
    s.wdiag.resize(n);
    AGG_LAUNCH(k_scale_diag, grid_for(n, 256), 256, 0, s.inv_diag.get(), s.omega, n, s.wdiag.get());
  }
}

}  // namespace aggmg_b200
