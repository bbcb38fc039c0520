// dist_hierarchy.cuh — the row-partitioned AMG hierarchy.
//
// Levels 0..kd-1 are split into contiguous row slabs across the ranks of a Comm; every
// setup artefact (strength, MIS(2) states, aggregates, P, R, B, coarse operators) equals the
// one-GPU hierarchy bit for bit.  Level kd — the first level at or below the agglomeration
// threshold (or the coarsest / stalled level) — is gathered onto rank 0 and continued there
// as an ordinary DevHierarchy whose level 0 is global level kd (SetupCfg::level_offset).
#pragma once

#include <map>
#include <memory>
#include <string>
#include <vector>

#include "dist.cuh"
#include "hierarchy.cuh"

namespace aggmg_b200 {

// What refresh_values needs to redo this level's Galerkin product with new values: the cached
// sort over the extended row set, its column weights, and which local entries travel where.
struct DistGalerkin {
  GalerkinDev gal;
  DevCsrPtr Aext;
  DevBuf<double> pvc;
  DevBuf<idx> exrow, exoff;  // exported rows (destination order) and their entry offsets
  int64_t nexp = 0, nie = 0;
  std::vector<int64_t> ent_cnt;  // exported entries per destination rank
};

struct DistLevel {
  DistCsrPtr A;       // this level's operator (rows = cols partition)
  DevBuf<double> B;   // near-null-space vector, owned rows
  SmootherDev smoother;
  int mis_sweeps = 0;
  // transfer to level k+1 (always present: the last distributed level feeds the tail)
  DistCsrPtr R;          // rows = owned coarse rows, cols = this level's rows (members)
  HaloPlan P_halo;       // plan over the coarse space for prolongation
  DevBuf<idx> agg_local; // coarse id of every owned row in P_halo's local numbering
  DevBuf<idx> agg_global;
  DevBuf<double> pval;
  // cycle workspace: fine vectors carry a halo (max of A's and R's), coarse ones P's
  int64_t halo_cap = 0;
  DevBuf<double> r, t;
  DevBuf<double> rc, xc, c, v, rt, d, w;  // level k+1 vectors (owned + halo)
  DevBuf<KScalars> ks;
  std::unique_ptr<DistGalerkin> galc;  // kept when SetupConfig::reuse_caches
};

struct DistHierarchy {
  ~DistHierarchy();
  Comm* comm = nullptr;
  SetupCfg cfg;
  int64_t agglomerate_rows = 0;
  std::vector<DistLevel> levels;       // distributed levels 0..kd-1
  Partition tail_rows;                 // row partition of level kd before the gather
  DistCsrPtr tail_A;                   // level kd's rows on this rank (refresh_values)
  int64_t tail_halo_cap = 0;           // halo slots the level-kd vectors need (P of level kd-1)
  std::unique_ptr<DevHierarchy> tail;  // global levels kd.., replicated on every rank
  int64_t n_levels_total = 0;          // global level count (same on every rank)
  std::vector<int64_t> level_rows, level_nnz;  // global sizes per level
  std::vector<std::string> warnings;
  double setup_ms = 0.0;
  bool workspace_ready = false;
  // tail-side buffers (the allgathered rc, the replicated correction) and tail workspace
  DevBuf<double> tail_b, tail_x;
  DevBuf<double> tail_work_c, tail_work_v, tail_work_rt, tail_work_d, tail_work_w;
  DevBuf<KScalars> tail_ks;
  // captured sub-cycles of the distributed levels (NCCL or one rank: no host rendezvous)
  std::vector<std::pair<std::string, cudaGraphExec_t>> graphs;
  std::map<std::string, int64_t> graph_kernels;
  // PCG hook (see DevHierarchy::top_dot_*): fused (r.z, r_old.z) on the last level-0 sweep
  const double* top_dot_c = nullptr;
  double* top_dot_out = nullptr;
  bool top_dot_done = false;

  int64_t kd() const { return static_cast<int64_t>(levels.size()); }
  void ensure_workspace();
  void drop_graphs();
};

// Collective over comm: every rank passes its own rows [A0.rows.begin(me), ...).
// B0_local == nullptr means ones.
// refresh_values (hierarchy.cpp:90-104) on the ranks: new values of level 0's local rows, the
// cached Galerkin products and smoothers redone level by level (needs reuse_caches).
void dist_refresh_values(DistHierarchy& h, const double* new_values_local);

std::unique_ptr<DistHierarchy> dist_setup_hierarchy(Comm& comm, DistCsrPtr A0,
                                                    const double* B0_local, const SetupCfg& cfg,
                                                    int64_t agglomerate_rows);

}  // namespace aggmg_b200
