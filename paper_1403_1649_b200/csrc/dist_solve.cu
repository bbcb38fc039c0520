// dist_solve.cu — the solve stage on a row-partitioned hierarchy (SURVEY §8(e) "solve
// collectives"): halo exchange before every SpMV-family kernel, rank-ordered allreduce of
// every Krylov / K-cycle scalar, gather of the restricted residual onto rank 0 at the
// agglomeration level and scatter of the coarse correction back.
//
// The kernel sequence per level is the one-GPU sequence of cycles.cu (cycles.cpp:16-146),
// so on one rank the partitioned solve is bit-identical to the one-GPU solve, and on R
// ranks it differs only by the summation order of the dot products.
#include <algorithm>
#include <cstdio>
#include <string>

#include "dist_solve.cuh"
#include "primitives.cuh"

namespace aggmg_b200 {

void DistHierarchy::ensure_workspace() {
  if (workspace_ready) return;
  const int64_t kd_ = kd();
  // halo capacity per level: A's and R's column halos of the level, P's of the level above
  std::vector<int64_t> cap(kd_ + 1, 0), nl(kd_ + 1, 0);
  for (int64_t k = 0; k < kd_; ++k) {
    DistLevel& L = levels[k];
    nl[k] = L.A->A.n_rows;
    cap[k] = std::max(cap[k], std::max(L.A->halo.nhalo, L.R->halo.nhalo));
    cap[k + 1] = std::max(cap[k + 1], L.P_halo.nhalo);
  }
  nl[kd_] = tail_rows.count(comm->rank());
  for (int64_t k = 0; k < kd_; ++k) {
    DistLevel& L = levels[k];
    L.halo_cap = cap[k];
    L.r.resize(nl[k] + cap[k]);
    L.t.resize(nl[k] + cap[k]);
    const int64_t nc = nl[k + 1] + cap[k + 1];
    L.rc.resize(nc);
    L.xc.resize(nc);
    L.c.resize(nc);
    L.v.resize(nc);
    L.rt.resize(nc);
    L.d.resize(nc);
    L.w.resize(nc);
    L.ks.resize(1);
    L.ks.zero();
  }
  if (tail) {
    tail->ensure_workspace();
    const int64_t n = tail->levels[0].A->n_rows;
    tail_b.resize(n);
    tail_x.resize(n);
    tail_work_c.resize(n);
    tail_work_v.resize(n);
    tail_work_rt.resize(n);
    tail_work_d.resize(n);
    tail_work_w.resize(n);
    tail_ks.resize(1);
    tail_ks.zero();
  }
  workspace_ready = true;
}

namespace {

void dist_cycle(DistHierarchy& h, const CycleCfg& cfg, int64_t k, bool kc, const double* b,
                double* x, const int* pred);
void dist_subcycle(DistHierarchy& h, const CycleCfg& cfg, int64_t k, bool kc, const double* b,
                   double* x, const int* pred);

// A sub-cycle of a distributed level, captured into a CUDA graph on its second use and replayed
// afterwards (first use eager), keyed by level, cycle kind and buffers.  Only when no exchange
// needs the host: one rank, or NCCL (its send/recv/allgather capture as graph nodes);
// in-process rank threads rendezvous on the host and stay eager.
void dist_subcycle(DistHierarchy& h, const CycleCfg& cfg, int64_t k, bool kc, const double* b,
                   double* x, const int* pred) {
  Comm& comm = *h.comm;
  const bool capturable = cycle_graphs_enabled() && (comm.size() == 1 || std::string(comm.kind()) == "nccl");
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  AGG_CUDA(cudaStreamIsCapturing(stream(), &cap));
  if (!capturable || cap != cudaStreamCaptureStatusNone) {
    dist_cycle(h, cfg, k, kc, b, x, pred);
    return;
  }
  char keybuf[256];
  std::snprintf(keybuf, sizeof(keybuf), "%d/%d/%d/%.17g/%d/%lld/%p/%p/%p", kc ? 1 : 0, cfg.kind,
                cfg.k_levels, cfg.t, cfg.inner, static_cast<long long>(k), static_cast<const void*>(b),
                static_cast<void*>(x), static_cast<const void*>(pred));
  const std::string key(keybuf);
  for (auto& g : h.graphs)
    if (g.first == key) {
      if (!g.second) {  // second use: capture
        AGG_CUDA(cudaStreamBeginCapture(stream(), cudaStreamCaptureModeThreadLocal));
        const int64_t before = launch_count();
        try {
          dist_cycle(h, cfg, k, kc, b, x, pred);
        } catch (...) {
          cudaGraph_t junk = nullptr;
          cudaStreamEndCapture(stream(), &junk);
          if (junk) cudaGraphDestroy(junk);
          throw;
        }
        const int64_t kernels = launch_count() - before;
        cudaGraph_t graph;
        AGG_CUDA(cudaStreamEndCapture(stream(), &graph));
        AGG_CUDA(cudaGraphInstantiate(&g.second, graph, 0));
        AGG_CUDA(cudaGraphDestroy(graph));
        note_launches(-kernels);  // counted again on every replay below
        h.graph_kernels[key] = kernels;
      }
      AGG_CUDA(cudaGraphLaunch(g.second, stream()));
      note_launches(h.graph_kernels[key]);
      return;
    }
  h.graphs.emplace_back(key, nullptr);  // first use: eager
  dist_cycle(h, cfg, k, kc, b, x, pred);
}

// coarse half of a visit of distributed level k (cycles.cpp:56-132)
void dist_coarse(DistHierarchy& h, const CycleCfg& cfg, int64_t k, bool kparent, const int* pred) {
  Comm& comm = *h.comm;
  DistLevel& L = h.levels[k];
  if (k + 1 == h.kd()) {  // the agglomerated tail, replicated on every rank
    allgather_vector(comm, h.tail_rows, L.rc.get(), h.tail_b.get());
    CoarseWork W{h.tail_work_c.get(), h.tail_work_v.get(), h.tail_work_rt.get(),
                 h.tail_work_d.get(), h.tail_work_w.get(), h.tail_ks.get()};
    coarse_correction(*h.tail, cfg, kparent, 0, h.tail_b.get(), h.tail_x.get(), W, pred);
    // every rank computed the same correction: keep this rank's rows, no scatter
    const int me = comm.rank();
    copy_double(L.xc.get(), h.tail_x.get() + h.tail_rows.begin(me), h.tail_rows.count(me));
    return;
  }
  DistLevel& C = h.levels[k + 1];
  if (!kparent) {  // V-cycle below a V-cycle
    dist_subcycle(h, cfg, k + 1, false, L.rc.get(), L.xc.get(), pred);
    return;
  }
  const int64_t nc = C.A->A.n_rows;
  const bool cg = cfg.inner == 0;
  const bool inner_k = cycle_accelerated(cfg, k + 1);
  const int level = static_cast<int>(k + 1);
  dist_subcycle(h, cfg, k + 1, inner_k, L.rc.get(), L.c.get(), pred);
  SpmvArgs a1;  // v = Ac c ; rho1, alpha1
  a1.x = L.c.get();
  a1.y = L.v.get();
  a1.c = L.rc.get();
  a1.dot_with_x = cg ? 1 : 0;
  a1.dots_out = &L.ks.get()->rho1;
  a1.pred = pred;
  dist_spmv(comm, *C.A, Epi::kSpmvDot2, a1);
  comm.allreduce_sum(&L.ks.get()->rho1, 2);
  launch_kstep1(nc, L.rc.get(), L.v.get(), L.rt.get(), L.ks.get(), cfg.t, pred, level);
  comm.allreduce_sum(&L.ks.get()->nrt, 2);
  launch_kflag(L.ks.get(), cfg.t, pred);
  const int* p2 = &L.ks.get()->flag2;
  dist_subcycle(h, cfg, k + 1, inner_k, L.rt.get(), L.d.get(), p2);
  SpmvArgs a2;  // w = Ac d ; gamma, beta, alpha2
  a2.x = L.d.get();
  a2.y = L.w.get();
  a2.u = L.v.get();
  a2.c = L.rt.get();
  a2.dot_with_x = cg ? 1 : 0;
  a2.dots_out = &L.ks.get()->gamma;
  a2.pred = p2;
  dist_spmv(comm, *C.A, Epi::kSpmvDot3, a2);
  comm.allreduce_sum(&L.ks.get()->gamma, 3);
  launch_kcombine(nc, L.c.get(), L.d.get(), L.xc.get(), L.ks.get(), pred, level);
}

// x = cycle(k) applied to b from the zero guess; kc: K-cycle (else V-cycle) at level k.
void dist_cycle(DistHierarchy& h, const CycleCfg& cfg, int64_t k, bool kc, const double* b,
                double* x, const int* pred) {
  Comm& comm = *h.comm;
  DistLevel& L = h.levels[k];
  const int64_t n = L.A->A.n_rows;
  const int prof = k == 0 ? kProfSmoothL0 : 0;
  // pre-smooth from zero, residual, restriction (cycles.cpp:54-57)
  launch_jacobi_zero(n, L.smoother.wdiag.get(), b, x, pred);
  SpmvArgs ra;
  ra.x = x;
  ra.y = L.r.get();
  ra.b = b;
  ra.pred = pred;
  dist_spmv(comm, *L.A, Epi::kResidual, ra, k == 0 ? kProfSpmvL0 : 0);
  SpmvArgs rr;
  rr.x = L.r.get();
  rr.y = L.rc.get();
  rr.pred = pred;
  dist_spmv(comm, *L.R, Epi::kSpmv, rr);
  dist_coarse(h, cfg, k, kc, pred);
  // prolongation + post-smooth (cycles.cpp:37-44, 59-60)
  halo_update<double>(comm, L.P_halo, L.xc.get());
  launch_prolong(n, x, L.agg_local.get(), L.pval.get(), L.xc.get(), L.t.get(), pred);
  SpmvArgs ja;
  ja.x = L.t.get();
  ja.y = x;
  ja.b = b;
  ja.d = L.smoother.wdiag.get();
  ja.pred = pred;
  // PCG's (r.z, r_old.z) ride on the last sweep on CSR-stream and value-dictionary operators
  // (plain SELL-32: plain sweep + PCG's separate dot), as on one GPU
  if (k == 0 && !pred && h.top_dot_out &&
      (!L.A->A.sell || (L.A->A.sell_vi && fuse_dots_on_dictionary()))) {
    ja.c = h.top_dot_c;
    ja.dots_out = h.top_dot_out;
    dist_spmv(comm, *L.A, Epi::kJacobiDot2, ja, prof);
    comm.allreduce_sum(h.top_dot_out, 2);
    h.top_dot_done = true;
    return;
  }
  dist_spmv(comm, *L.A, Epi::kJacobi, ja, prof);
}

}  // namespace

void dist_apply_preconditioner(DistHierarchy& h, const CycleCfg& cfg, const double* r, double* z) {
  h.ensure_workspace();
  if (h.kd() == 0) {  // everything agglomerated: the one-GPU cycle, replicated on every rank
    Comm& comm = *h.comm;
    allgather_vector(comm, h.tail_rows, r, h.tail_b.get());
    apply_preconditioner(*h.tail, cfg, h.tail_b.get(), h.tail_x.get());
    copy_double(z, h.tail_x.get() + h.tail_rows.begin(comm.rank()), h.tail_rows.count(comm.rank()));
    return;
  }
  dist_cycle(h, cfg, 0, cycle_accelerated(cfg, 0), r, z, nullptr);
}

SolveOut dist_solve(DistHierarchy& h, const DistCsr& A, const CycleCfg& cyc, const SolverCfg& cfg,
                    const double* b, double* x) {
  h.ensure_workspace();
  Comm& comm = *h.comm;
  KrylovDist d;
  d.n_alloc = A.A.n_rows + std::max<int64_t>(A.halo.nhalo, h.kd() ? h.levels[0].halo_cap : 0);
  d.spmv = [&](Epi epi, const SpmvArgs& a, int prof) { dist_spmv(comm, A, epi, a, prof); };
  d.allreduce = [&](double* v, int k) { comm.allreduce_sum(v, k); };
  d.precond = [&](const double* r, double* z) { dist_apply_preconditioner(h, cyc, r, z); };
  d.precond_dots = [&](const double* r, const double* rold, double* z, double* q) {
    h.top_dot_c = rold;
    h.top_dot_out = q;
    h.top_dot_done = false;
    dist_apply_preconditioner(h, cyc, r, z);
    h.top_dot_c = nullptr;
    h.top_dot_out = nullptr;
    return h.top_dot_done;
  };
  d.flush_warnings = [&] {
    if (comm.rank() == 0) flush_cycle_warnings();
  };
  Precond M;
  M.cfg = cyc;
  // x needs halo room for the residual SpMV: solve in a workspace copy
  DevBuf<double> xw(d.n_alloc);
  xw.zero();
  copy_double(xw.get(), x, A.A.n_rows);
  SolveOut out = cfg.method == 1 ? pcg(A.A, b, xw.get(), M, cfg, &d) : fgmres(A.A, b, xw.get(), M, cfg, &d);
  copy_double(x, xw.get(), A.A.n_rows);
  sync();
  return out;
}

}  // namespace aggmg_b200
