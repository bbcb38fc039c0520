// hierarchy.cu — Algorithm 1 setup loop on the device (hierarchy.cpp:34-104).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <sstream>

#include "hierarchy.cuh"
#include "chunked.cuh"
#include "vecops.cuh"

namespace aggmg_b200 {

constexpr int64_t kDenseSolveCap = 5000;  // hierarchy.cpp:23

namespace {
// AGGMG_SETUP_TIMING=1: per-phase GPU-synchronised wall time of setup_hierarchy (stderr);
// =2: no synchronisation — an event per phase boundary on the stream (the overlapped run's
// own critical path) beside the host's issue time of the boundary
struct SetupTimer {
  int mode = 0;
  std::chrono::steady_clock::time_point t, t0;
  std::vector<std::pair<std::string, double>> acc;
  std::vector<std::tuple<std::string, cudaEvent_t, double>> ev;
  SetupTimer() {
    const char* e = std::getenv("AGGMG_SETUP_TIMING");
    mode = e ? std::atoi(e) : 0;
    if (mode == 1) sync();
    t = t0 = std::chrono::steady_clock::now();
    if (mode == 2) push("start");
  }
  void push(const std::string& name) {
    cudaEvent_t x;
    AGG_CUDA(cudaEventCreate(&x));
    AGG_CUDA(cudaEventRecord(x, stream()));
    ev.emplace_back(name, x,
                    std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count());
  }
  void mark(const std::string& name) {
    if (mode == 2) push(name);
    if (mode != 1) return;
    sync();
    const auto now = std::chrono::steady_clock::now();
    const double ms = std::chrono::duration<double, std::milli>(now - t).count();
    t = now;
    for (auto& a : acc)
      if (a.first == name) {
        a.second += ms;
        return;
      }
    acc.emplace_back(name, ms);
  }
  ~SetupTimer() {
    for (auto& a : acc) std::fprintf(stderr, "[setup] %-14s %8.3f ms\n", a.first.c_str(), a.second);
    if (mode != 2 || ev.empty()) return;
    sync();
    for (size_t k = 1; k < ev.size(); ++k) {
      float ms = 0.f, at = 0.f;
      cudaEventElapsedTime(&ms, std::get<1>(ev[k - 1]), std::get<1>(ev[k]));
      cudaEventElapsedTime(&at, std::get<1>(ev[0]), std::get<1>(ev[k]));
      std::fprintf(stderr, "[setup-ev] %-14s gpu %8.3f ms (ends at %8.3f)  host issued at %8.3f\n",
                   std::get<0>(ev[k]).c_str(), ms, at, std::get<2>(ev[k]));
    }
    for (auto& e : ev) cudaEventDestroy(std::get<1>(e));
  }
};
}  // namespace

void factor_coarsest(DevHierarchy& h) {
  DevLevel& L = h.levels.back();
  const int64_t nL = L.A->n_rows;
  require(nL <= std::max<int64_t>(h.cfg.coarse_size_max, kDenseSolveCap),
          "setup: coarsest level has " + std::to_string(nL) + " unknowns, too large for a dense solve");
  invert_coarsest(*L.A, h.coarse_inv);  // coarse.cu (dense.cpp:16-79 on the device)
  h.coarse_lu_ready = false;
  if (exact_reductions() && nL > 0) {
    // the reference's own factorisation order, for the bit-identical substitution kernel
    std::vector<int64_t> rp(nL + 1), col(L.A->nnz);
    std::vector<double> val(L.A->nnz);
    download_csr(*L.A, rp.data(), col.data(), val.data());
    std::vector<double> dense(static_cast<size_t>(nL) * nL, 0.0);  // dense.cpp:16-22
    for (int64_t i = 0; i < nL; ++i)
      for (int64_t k = rp[i]; k < rp[i + 1]; ++k) dense[i * nL + col[k]] = val[k];
    HostLu lu;
    lu.factor(std::move(dense), nL);
    h.coarse_lu.resize(nL * nL);
    h.coarse_lu.upload(lu.lu.data(), nL * nL);
    std::vector<double> lt(static_cast<size_t>(nL) * nL);
    for (int64_t i = 0; i < nL; ++i)
      for (int64_t j = 0; j < nL; ++j) lt[j * nL + i] = lu.lu[i * nL + j];
    h.coarse_lu_t.resize(nL * nL);
    h.coarse_lu_t.upload(lt.data(), nL * nL);
    std::vector<int> perm(lu.perm.begin(), lu.perm.end());
    h.coarse_perm.resize(nL);
    h.coarse_perm.upload(perm.data(), nL);
    h.coarse_lu_ready = true;
  }
  sync();
}

std::unique_ptr<DevHierarchy> setup_hierarchy(DevCsrPtr A0, const double* B0_dev,
                                              const SetupCfg& cfg) {
  require(A0->n_rows == A0->n_cols, "setup: matrix must be square");
  require(cfg.coarse_size_max >= 1, "setup: coarse_size_max must be at least 1");
  require(cfg.max_levels >= 1, "setup: max_levels must be at least 1");
  // working set of setup + a Krylov solve: ~16x the operator (strength graphs, Galerkin
  // scratch and caches, coarse levels, FGMRES(30) basis)
  pool_reserve(16 * static_cast<size_t>(A0->nnz * 12 + A0->n_rows * 8) + (size_t{256} << 20));
  cudaEvent_t e0, e1;
  AGG_CUDA(cudaEventCreate(&e0));
  AGG_CUDA(cudaEventCreate(&e1));
  AGG_CUDA(cudaEventRecord(e0, stream()));

  auto h = std::make_unique<DevHierarchy>();
  SmootherBatch smoothers;  // after h: joins the side stream before h's buffers die
  h->cfg = cfg;
  h->levels.emplace_back();
  h->levels[0].A = A0;
  h->levels[0].B.resize(A0->n_rows);
  if (B0_dev)
    copy_double(h->levels[0].B.get(), B0_dev, A0->n_rows);
  else
    fill_double(h->levels[0].B.get(), A0->n_rows, 1.0);
  const double nb = std::sqrt(dot_host(h->levels[0].B.get(), h->levels[0].B.get(), A0->n_rows));
  require(nb > 0.0, "setup: near-null-space vector is zero");

  SetupTimer st;
  while (h->levels.back().A->n_rows > cfg.coarse_size_max &&
         static_cast<int>(h->levels.size()) < cfg.max_levels) {
    const int64_t k = h->coarsest();
    DevLevel& fine = h->levels[k];
    const DevCsr& A = *fine.A;
    const int64_t n = A.n_rows;

    const std::string lv = "L" + std::to_string(k) + " ";
    DevCsrPtr C = classic_strength(A, cfg.alpha, 0);
    st.mark(lv + "strength");
    DevBuf<idx> influence;
    DevCsrPtr S;
    influence_and_symmetrize(*C, influence, S);
    C.reset();
    st.mark(lv + "symmetrize");
    Mis2Dev mis = mis2(*S, influence.get(), level_seed(cfg.seed, k + cfg.level_offset, kMisTag));
    st.mark(lv + "mis2");
    AggDev agg = aggregate(*S, A, mis.state.get());
    S.reset();
    st.mark(lv + "aggregate");

    if (static_cast<double>(agg.n_agg) >= 0.95 * static_cast<double>(n)) {
      std::ostringstream msg;
      msg << "coarsening stalled at level " << k + cfg.level_offset << " (" << n << " -> " << agg.n_agg
          << " aggregates); solving this level directly";
      h->warnings.push_back(msg.str());
      break;
    }
    fine.mis_sweeps = mis.sweeps;
    fine.tr = build_transfer(agg, fine.B.get());
    st.mark(lv + "transfer");
    DevCsrPtr Ac;
    if (cfg.reuse_caches) {  // hierarchy.cpp:69-71: cached sort / segmented reduce
      DevBuf<double> vals;
      fine.gal = build_galerkin_cache(A, agg, false, false, true, fine.tr.pval.get(), &vals);
      Ac = fine.gal.lean ? coarse_from_cache(fine.gal, std::move(vals))
                         : apply_galerkin_cache(fine.gal, A, fine.tr.pval.get());
    } else {  // hierarchy.cpp:73: galerkin_direct, the reference default
      Ac = galerkin_direct(A, agg, fine.tr.pval.get());
    }
    st.mark(lv + "galerkin");
    smoothers.add(A, cfg.smoother, cfg.arnoldi_m,
                  level_seed(cfg.seed, k + cfg.level_offset, kSmootherTag), fine.smoother,
                  static_cast<int>(k));
    st.mark(lv + "smoother");
    fine.has_smoother = true;
    fine.agg = std::move(agg);
    fine.has_next = true;
    DevLevel next;
    next.A = Ac;
    next.B = std::move(fine.tr.coarse_b);
    h->levels.push_back(std::move(next));
  }
  factor_coarsest(*h);
  st.mark("coarsest LU");
  // the Arnoldi estimates ran on the side stream under the coarsening
  smoothers.finish([&](int k) -> SmootherDev& { return h->levels[k].smoother; });
  st.mark("smoother join");
  AGG_CUDA(cudaEventRecord(e1, stream()));
  AGG_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  AGG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  h->setup_ms = ms;
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return h;
}

// hierarchy.cpp:90-104: numeric half only; aggregates, P and R are untouched.
void refresh_values(DevHierarchy& h, const double* new_values_dev) {
  // the smoother arrays are reallocated below: captured sub-cycle graphs become stale
  for (auto& g : h.graphs)
    if (g.second.exec) cudaGraphExecDestroy(g.second.exec);
  h.graphs.clear();
  DevLevel& L0 = h.levels[0];
  // level 0 may share its storage with the caller's device matrix (setup_hierarchy_device):
  // the refresh must not rewrite the caller's values
  if (L0.A.use_count() > 1) L0.A = clone_csr(*L0.A);
  copy_double(L0.A->val.get(), new_values_dev, L0.A->nnz);
  L0.A->refresh_sell();
  SmootherBatch smoothers;
  for (int64_t k = 0; k + 1 < h.n_levels(); ++k) {
    DevLevel& fine = h.levels[k];
    DevCsrPtr Ac = apply_galerkin_cache(fine.gal, *fine.A, fine.tr.pval.get());
    copy_double(h.levels[k + 1].A->val.get(), Ac->val.get(), Ac->nnz);
    h.levels[k + 1].A->refresh_sell();
    smoothers.add(*fine.A, h.cfg.smoother, h.cfg.arnoldi_m,
                  level_seed(h.cfg.seed, k + h.cfg.level_offset, kSmootherTag), fine.smoother,
                  static_cast<int>(k));
  }
  factor_coarsest(h);
  smoothers.finish([&](int k) -> SmootherDev& { return h.levels[k].smoother; });
}

DevCsrPtr clone_csr(const DevCsr& A) {
  auto C = std::make_shared<DevCsr>();
  C->n_rows = A.n_rows;
  C->n_cols = A.n_cols;
  C->nnz = A.nnz;
  C->rowptr.copy_from(A.rowptr);
  C->col.copy_from(A.col);
  C->val.copy_from(A.val);
  C->max_row = A.max_row;
  C->rows_per_block = A.rows_per_block;
  C->smem_entries = A.smem_entries;
  C->sell = A.sell;
  C->sell_short = A.sell_short;
  C->sell_ptr.copy_from(A.sell_ptr);
  C->sell_col.copy_from(A.sell_col);
  C->sell_val.copy_from(A.sell_val);
  C->sell_perm.copy_from(A.sell_perm);
  C->sell_sigma_ok = A.sell_sigma_ok;
  C->sell_vi = A.sell_vi;
  C->sell_pad4 = A.sell_pad4;
  C->sell_code.copy_from(A.sell_code);
  C->sell_tab.copy_from(A.sell_tab);
  C->sell_pcol.copy_from(A.sell_pcol);
  C->sell_len.copy_from(A.sell_len);
  C->sell_d16 = A.sell_d16;
  C->sell_col16.copy_from(A.sell_col16);
  C->sell_slots = A.sell_slots;
  C->pat = A.pat;
  C->pat_w = A.pat_w;
  C->pat_id.copy_from(A.pat_id);
  C->pat_len.copy_from(A.pat_len);
  C->pat_delta.copy_from(A.pat_delta);
  C->pat_val.copy_from(A.pat_val);
  return C;
}

namespace {
void clone_sgs(SgsDirection& d, const SgsDirection& s) {
  d.ell = s.ell;
  d.cta = s.cta;
  d.rows.copy_from(s.rows);
  d.rec.copy_from(s.rec);
  d.offsets.copy_from(s.offsets);
  d.h_offsets = s.h_offsets;
  d.code.copy_from(s.code);
  d.val.copy_from(s.val);
  d.optr.copy_from(s.optr);
  d.ocol.copy_from(s.ocol);
  d.oval.copy_from(s.oval);
  d.runs = s.runs;
}
}  // namespace

std::unique_ptr<DevHierarchy> clone_hierarchy(const DevHierarchy& h) {
  auto c = std::make_unique<DevHierarchy>();
  c->cfg = h.cfg;
  c->warnings = h.warnings;
  c->setup_ms = h.setup_ms;
  c->coarse_inv.copy_from(h.coarse_inv);
  c->coarse_lu.copy_from(h.coarse_lu);
  c->coarse_lu_t.copy_from(h.coarse_lu_t);
  c->coarse_perm.copy_from(h.coarse_perm);
  c->coarse_lu_ready = h.coarse_lu_ready;
  c->levels.resize(h.levels.size());
  for (size_t k = 0; k < h.levels.size(); ++k) {
    const DevLevel& s = h.levels[k];
    DevLevel& d = c->levels[k];
    d.A = clone_csr(*s.A);
    d.B.copy_from(s.B);
    d.has_smoother = s.has_smoother;
    d.smoother.kind = s.smoother.kind;
    d.smoother.inv_diag.copy_from(s.smoother.inv_diag);
    d.smoother.wdiag.copy_from(s.smoother.wdiag);
    d.smoother.omega = s.smoother.omega;
    d.smoother.rho_est = s.smoother.rho_est;
    d.smoother.arnoldi_m = s.smoother.arnoldi_m;
    clone_sgs(d.smoother.sgs_fw, s.smoother.sgs_fw);
    clone_sgs(d.smoother.sgs_bw, s.smoother.sgs_bw);
    d.smoother.sgs_tmp.copy_from(s.smoother.sgs_tmp);
    d.smoother.sgs_bp.copy_from(s.smoother.sgs_bp);
    d.smoother.sgs_xp.copy_from(s.smoother.sgs_xp);
    d.has_next = s.has_next;
    d.mis_sweeps = s.mis_sweeps;
    d.agg.n_fine = s.agg.n_fine;
    d.agg.n_agg = s.agg.n_agg;
    d.agg.assignment.copy_from(s.agg.assignment);
    d.agg.representatives.copy_from(s.agg.representatives);
    d.agg.agg_row_offsets.copy_from(s.agg.agg_row_offsets);
    d.agg.rows_by_coarse.copy_from(s.agg.rows_by_coarse);
    d.tr.pval.copy_from(s.tr.pval);
    d.tr.coarse_b.copy_from(s.tr.coarse_b);
    d.tr.R = s.tr.R;  // never written after setup (refresh keeps P and R)
    d.tr.p_nnz = s.tr.p_nnz;
    d.gal.n_fine = s.gal.n_fine;
    d.gal.n_coarse = s.gal.n_coarse;
    d.gal.nnz_fine = s.gal.nnz_fine;
    d.gal.nnz_coarse = s.gal.nnz_coarse;
    d.gal.coarse_rowptr.copy_from(s.gal.coarse_rowptr);
    d.gal.coarse_col.copy_from(s.gal.coarse_col);
    d.gal.entry.copy_from(s.gal.entry);
    d.gal.entry_row.copy_from(s.gal.entry_row);
    d.gal.segment_offsets.copy_from(s.gal.segment_offsets);
    d.gal.slot_of_csr.copy_from(s.gal.slot_of_csr);
    d.gal.group_offsets.copy_from(s.gal.group_offsets);
    d.gal.group_rows.copy_from(s.gal.group_rows);
    d.gal.max_coarse_row = s.gal.max_coarse_row;
    d.gal.pattern_hash = s.gal.pattern_hash;
    d.gal.lean = s.gal.lean;
  }
  sync();
  return c;
}

DevHierarchy::~DevHierarchy() {
  for (auto& g : graphs)
    if (g.second.exec) cudaGraphExecDestroy(g.second.exec);
}

void DevHierarchy::ensure_workspace() {
  if (workspace_ready) return;
  for (int64_t k = 0; k < n_levels(); ++k) {
    DevLevel& L = levels[k];
    const int64_t n = L.A->n_rows;
    L.r.resize(n);
    L.t.resize(n);
    if (k + 1 < n_levels()) {
      const int64_t nc = levels[k + 1].A->n_rows;
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
  }
  workspace_ready = true;
}

}  // namespace aggmg_b200
