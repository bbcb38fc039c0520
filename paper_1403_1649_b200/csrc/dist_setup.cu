// dist_setup.cu — setup of the row-partitioned levels (SURVEY §8(e) "setup collectives").
//
// Each step restates the one-GPU kernel of setup.cu (and through it the reference lines it
// cites) for a slab of rows, plus the exchange the step needs:
//   strength            row-local                                   (strength.cpp:28-72)
//   influence           column counts + reverse halo add            (strength.cpp:74-78)
//   S = C u C^T         transpose pairs shipped to the row owner    (strength.cpp:80-111)
//   MIS(2)              two tuple halos + one count allreduce/sweep (aggregation.cpp:45-86)
//   aggregation         state/representative halos, A_ji requests,
//                       global renumbering by representative node   (aggregation.cpp:88-159)
//   transfer            members shipped to the aggregate owner,
//                       summed in ascending global order            (transfer.cpp:15-49)
//   Galerkin            (I, J, (p_i a_ij) p_j) records shipped to the owner of I in global
//                       (row, entry) order, stable sort by (I, J), ordered segment sums —
//                       the reference cache order                   (galerkin.cpp:38-137)
//   smoother            inverse diagonal + Arnoldi with halo SpMVs  (smoother.cpp:21-99)
// Integer / index results and coarse values are bit-identical to the one-GPU hierarchy;
// omega differs only by the order of the Arnoldi dot products (<= 1e-12 relative).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cub/cub.cuh>
#include <cstdio>
#include <cstdlib>
#include <sstream>

#include "dist_hierarchy.cuh"
#include "primitives.cuh"
#include "vecops.cuh"

namespace aggmg_b200 {

namespace {

template <class F>
void cub_call(F&& f) {
  size_t bytes = 0;
  AGG_CUDA(f(nullptr, bytes));
  DevBuf<char> tmp(static_cast<int64_t>(std::max<size_t>(bytes, 1)));
  AGG_CUDA(f(tmp.get(), bytes));
}

constexpr int kMaxRanks = 64;
struct PartDev {
  int64_t off[kMaxRanks + 1];
  int nranks;
};
PartDev part_dev(const Partition& p) {
  require(p.off.size() <= kMaxRanks + 1, "distributed path supports at most 64 ranks");
  PartDev d{};
  d.nranks = static_cast<int>(p.off.size()) - 1;
  for (size_t r = 0; r < p.off.size(); ++r) d.off[r] = p.off[r];
  return d;
}
__device__ inline int dev_owner(const PartDev& p, int64_t g) {
  int lo = 0, hi = p.nranks - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (p.off[mid] <= g)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

__device__ inline double dmax_ref(double a, double b) { return (a < b) ? b : a; }

// global id of local column c
__device__ inline idx gcol_of(idx c, int64_t nloc, int64_t c0, const idx* halo) {
  return c < nloc ? static_cast<idx>(c + c0) : halo[c - nloc];
}

// value of A(i, gj) for local row i by binary search over the row's global column ids
__device__ inline double row_at(const idx* rp, const idx* gcol, const double* val, idx i, idx gj) {
  idx lo = rp[i], hi = rp[i + 1];
  while (lo < hi) {
    const idx mid = lo + ((hi - lo) >> 1);
    if (gcol[mid] < gj)
      lo = mid + 1;
    else
      hi = mid;
  }
  return (lo < rp[i + 1] && gcol[lo] == gj) ? val[lo] : 0.0;
}

// ---- influence / symmetrize -----------------------------------------------------------
__global__ void k_count_cols(const idx* col, int64_t nnz, idx* cnt) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < nnz) atomicAdd(&cnt[col[k]], 1);
}
// transpose pairs (row = global column of C, col = global row), destination = owner of row
// sorted merge of C row i and C^T row i (strength.cpp:86-103), global ids.  mode 0 counts.
__global__ void k_merge_rows_g(const idx* crp, const idx* ccol, const idx* trp, const idx* tcol,
                               int64_t n, int mode, const idx* srp, idx* out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  idx a = crp[i], ae = crp[i + 1], b = trp[i], be = trp[i + 1];
  idx cnt = 0;
  idx* o = mode ? out + srp[i] : nullptr;
  while (a < ae || b < be) {
    idx j;
    if (b >= be || (a < ae && ccol[a] <= tcol[b])) {
      j = ccol[a];
      if (b < be && tcol[b] == j) ++b;
      ++a;
    } else {
      j = tcol[b++];
    }
    if (o) o[cnt] = j;
    ++cnt;
  }
  if (!mode) out[i] = cnt;
}

// ---- MIS(2) ---------------------------------------------------------------------------
struct __align__(16) Tuple {
  double v;
  int i;  // global node id
  int s;
};
__device__ inline bool tuple_less(const Tuple& a, const Tuple& b) {
  if (a.s != b.s) return a.s < b.s;
  if (a.v != b.v) return a.v < b.v;
  return a.i < b.i;
}
struct DMisCtl {
  long long undecided;  // global
  long long dec;        // decided this sweep (local, then summed)
  int active;
  int sweeps;
};
__global__ void k_dmis_init(const idx* infl, int64_t n, int64_t row0, uint64_t seed, Tuple* cur,
                            int8_t* state) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  Tuple t;
  t.v = __dadd_rn(static_cast<double>(infl[i]),
                  uniform_open01(seed, static_cast<uint64_t>(row0 + i)));
  t.i = static_cast<int>(row0 + i);
  t.s = 0;
  cur[i] = t;
  state[i] = 0;
}
__global__ void k_dmis_pass1(const idx* rp, const idx* col, int64_t n, const Tuple* cur, Tuple* mid,
                             DMisCtl* ctl) {
  const long long und = ctl->undecided;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ctl->active = und > 0 ? 1 : 0;
    if (und > 0) ctl->sweeps += 1;
  }
  if (und == 0) return;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  Tuple best = cur[i];
  for (idx k = rp[i]; k < rp[i + 1]; ++k) {
    const Tuple t = cur[col[k]];
    if (tuple_less(best, t)) best = t;
  }
  mid[i] = best;
}
__global__ void k_dmis_pass2(const idx* rp, const idx* col, int64_t n, int64_t row0, const Tuple* mid,
                             Tuple* cur, int8_t* state, DMisCtl* ctl) {
  if (!ctl->active) return;
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  int decided = 0;
  if (i < n && state[i] == 0) {
    Tuple far = mid[i];
    for (idx k = rp[i]; k < rp[i + 1]; ++k) {
      const Tuple t = mid[col[k]];
      if (tuple_less(far, t)) far = t;
    }
    int8_t st = 0;
    if (far.i == static_cast<int>(row0 + i))
      st = 1;
    else if (far.s == 1)
      st = -1;
    if (st != 0) {
      state[i] = st;
      cur[i].s = st;
      decided = 1;
    }
  }
  const unsigned ballot = __ballot_sync(0xffffffffu, decided);
  if ((threadIdx.x & 31) == 0 && ballot) atomicAdd(reinterpret_cast<unsigned long long*>(&ctl->dec),
                                                   static_cast<unsigned long long>(__popc(ballot)));
}
__global__ void k_dmis_update(DMisCtl* ctl) {
  if (ctl->active) ctl->undecided -= ctl->dec;
  ctl->dec = 0;
}

// ---- aggregation ------------------------------------------------------------------------
// pass 1: representative (global root id) and the local column of that root (via1)
__global__ void k_dagg_pass1(const idx* rp, const idx* col, int64_t n, int64_t row0, int64_t nloc,
                             const idx* halo, const int8_t* state, idx* rep, idx* via) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  idx r = -1, v = -1;
  if (state[i] == 1) {
    r = static_cast<idx>(row0 + i);
  } else {
    for (idx k = rp[i]; k < rp[i + 1]; ++k) {
      const idx c = col[k];
      if (state[c] == 1) {
        r = gcol_of(c, nloc, row0, halo);
        v = c;
        break;
      }
    }
  }
  rep[i] = r;
  via[i] = v;
}
// S cross entries that pass 2 needs A(j, i) for: rows still unassigned after pass 1
__global__ void k_dagg_req_count(const idx* srp, const idx* scol, int64_t n, int64_t nloc,
                                 const idx* rep, idx* cnt) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  idx c = 0;
  if (rep[i] == -1)
    for (idx k = srp[i]; k < srp[i + 1]; ++k) c += (scol[k] >= nloc && rep[scol[k]] != -1) ? 1 : 0;
  cnt[i] = c;
}
__global__ void k_dagg_req_fill(const idx* srp, const idx* scol, int64_t n, int64_t row0, int64_t nloc,
                                const idx* halo, const idx* rep, const idx* off, int2* req, idx* slot) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  idx p = off[i];
  for (idx k = srp[i]; k < srp[i + 1]; ++k) {
    slot[k] = -1;
    if (rep[i] != -1) continue;
    const idx c = scol[k];
    if (c >= nloc && rep[c] != -1) {
      req[p] = make_int2(halo[c - nloc], static_cast<int>(row0 + i));  // A(j, i)
      slot[k] = p;
      ++p;
    }
  }
}
// pass 2 against the pass-1 snapshot (aggregation.cpp:118-136), leftovers singletons
__global__ void k_dagg_pass2(const idx* srp, const idx* scol, const idx* arp, const idx* agcol,
                             const double* aval, int64_t n, int64_t row0, int64_t nloc,
                             const idx* halo, const idx* rep, const idx* slot, const double* tval,
                             idx* rep2, idx* via2, idx* isrep) {
  const int64_t ii = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (ii >= n) return;
  const idx i = static_cast<idx>(ii);
  const idx gi = static_cast<idx>(row0 + i);
  idx r = rep[i], v = -1;
  if (r == -1) {
    idx best = -1;
    double best_w = -1.0;
    for (idx k = srp[i]; k < srp[i + 1]; ++k) {
      const idx c = scol[k];
      const idx ja = rep[c];
      if (ja == -1) continue;
      const idx gj = gcol_of(c, nloc, row0, halo);
      const double aij = row_at(arp, agcol, aval, i, gj);
      const double aji = c < nloc ? row_at(arp, agcol, aval, c, gi) : tval[slot[k]];
      const double w = dmax_ref(fabs(aij), fabs(aji));
      if (w > best_w || (w == best_w && ja < best)) {
        best_w = w;
        best = ja;
        v = c;
      }
    }
    r = best == -1 ? gi : best;
    if (best == -1) v = -1;
  }
  rep2[i] = r;
  via2[i] = v;
  isrep[i] = (r == gi) ? 1 : 0;
}
__global__ void k_dagg_fid_reps(const idx* isrep, const idx* rank, int64_t n, int64_t cbase, idx* fid) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) fid[i] = isrep[i] ? static_cast<idx>(cbase + rank[i]) : -1;
}
// phase 1: pass-1 members copy their root's id; phase 2: pass-2 members copy their neighbour's
__global__ void k_dagg_fid_copy(const idx* via, const idx* rep_or_null, const idx* isrep, int64_t n,
                                int phase, idx* fid) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n || isrep[i]) return;
  const bool pass1_member = rep_or_null[i] != -1;
  if ((phase == 1) == pass1_member) fid[i] = fid[via[i]];
}

// ---- pair requests: A(row_g, col_g) from the owner of row_g ------------------------------
__global__ void k_req_owner(const int2* req, int64_t m, PartDev p, unsigned* own, idx* perm) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= m) return;
  own[k] = static_cast<unsigned>(dev_owner(p, req[k].x));
  perm[k] = static_cast<idx>(k);
}
__global__ void k_req_gather(const int2* req, const idx* perm, int64_t m, int2* out) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < m) out[k] = req[perm[k]];
}
__global__ void k_req_answer(const int2* req, int64_t m, int64_t row0, const idx* arp, const idx* agcol,
                             const double* aval, double* out) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < m) out[k] = row_at(arp, agcol, aval, static_cast<idx>(req[k].x - row0), req[k].y);
}
__global__ void k_scatter_back(const double* in, const idx* perm, int64_t m, double* out) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < m) out[perm[k]] = in[k];
}
__global__ void k_count_u(const unsigned* own, int64_t m, long long* cnt) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < m) atomicAdd(reinterpret_cast<unsigned long long*>(&cnt[own[k]]), 1ull);
}

// ---- transfer: an exported member row (global aggregate id, global row id, b_i) ----------
struct __align__(16) MemberRec {
  int J;
  int gid;
  double b;
};

__global__ void k_uniform_sym_off(int64_t n, int64_t row0, uint64_t seed, double* x) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) x[i] = uniform_sym(seed, static_cast<uint64_t>(row0 + i));
}

double dist_dot(Comm& comm, const double* a, const double* b, int64_t n) {
  DevBuf<double> d(1);
  DotArgs args{};
  args.a[0] = a;
  args.b[0] = b;
  args.np = 1;
  if (n > 0)
    dot_device(args, n, d.get(), nullptr, 1);
  else
    d.zero();
  comm.allreduce_sum(d.get(), 1);
  return read_scalar(d.get());
}

}  // namespace


namespace {



// ---- C^T pieces ------------------------------------------------------------------------------
__global__ void k_cross_count(const idx* rp, const idx* col, const idx* gcol, int64_t n, int64_t nloc,
                              PartDev p, unsigned long long* cnt) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (idx k = rp[i]; k < rp[i + 1]; ++k)
    if (col[k] >= nloc) atomicAdd(&cnt[dev_owner(p, gcol[k])], 1ull);
}
__global__ void k_cross_fill(const idx* rp, const idx* col, const idx* gcol, int64_t n, int64_t nloc,
                             int64_t row0, PartDev p, const int64_t* off, unsigned long long* cursor,
                             int2* out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (idx k = rp[i]; k < rp[i + 1]; ++k) {
    if (col[k] < nloc) continue;
    const int q = dev_owner(p, gcol[k]);
    const unsigned long long slot = atomicAdd(&cursor[q], 1ull);
    out[off[q] + slot] = make_int2(gcol[k], static_cast<int>(row0 + i));
  }
}
__global__ void k_tcount_local(const idx* rp, const idx* col, int64_t n, int64_t nloc, idx* cnt) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (idx k = rp[i]; k < rp[i + 1]; ++k)
    if (col[k] < nloc) atomicAdd(&cnt[col[k]], 1);
}
__global__ void k_tcount_remote(const int2* pr, int64_t m, int64_t row0, idx* cnt) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < m) atomicAdd(&cnt[pr[k].x - row0], 1);
}
__global__ void k_tfill_local(const idx* rp, const idx* col, int64_t n, int64_t nloc, int64_t row0,
                              const idx* trp, idx* cur, idx* out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (idx k = rp[i]; k < rp[i + 1]; ++k) {
    const idx c = col[k];
    if (c < nloc) out[trp[c] + atomicAdd(&cur[c], 1)] = static_cast<idx>(row0 + i);
  }
}
__global__ void k_tfill_remote(const int2* pr, int64_t m, int64_t row0, const idx* trp, idx* cur, idx* out) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const int64_t r = pr[k].x - row0;
  out[trp[r] + atomicAdd(&cur[r], 1)] = pr[k].y;
}

// ---- extended row set (transfer / Galerkin across ranks) ------------------------------------
struct __align__(16) EntRec {
  double a;    // entry value
  double pvc;  // P weight of the entry's column
};
static_assert(sizeof(EntRec) == 16, "EntRec travels as a 16-byte unit");
__global__ void k_agg_owner(const idx* fid, int64_t n, PartDev cp, int me, unsigned* dest, idx* ex) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int o = dev_owner(cp, fid[i]);
  dest[i] = static_cast<unsigned>(o);
  ex[i] = (o != me) ? 1 : 0;
}
__global__ void k_export_list(const idx* ex, const idx* pos, const unsigned* dest, int64_t n, idx* rows,
                              unsigned* d) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n || !ex[i]) return;
  rows[pos[i]] = static_cast<idx>(i);
  d[pos[i]] = dest[i];
}
__global__ void k_export_members(const idx* rows, int64_t m, const idx* fid, const double* b, int64_t row0,
                                 MemberRec* out) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const idx i = rows[k];
  MemberRec r;
  r.J = fid[i];
  r.gid = static_cast<int>(row0 + i);
  r.b = b[i];
  out[k] = r;
}
__global__ void k_ext_rows(const double* b, int64_t nloc, int64_t ntot, int64_t row0, const MemberRec* imp,
                           int64_t m, double* b_ext, idx* gid_ext) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < nloc) {
    b_ext[i] = b[i];
    gid_ext[i] = static_cast<idx>(row0 + i);
  } else if (i < ntot) {
    gid_ext[i] = -1;
  } else if (i < ntot + m) {
    const MemberRec r = imp[i - ntot];
    b_ext[i] = r.b;
    gid_ext[i] = r.gid;
  }
}
__global__ void k_group_count(const idx* fid, const idx* ex, int64_t nloc, const MemberRec* imp, int64_t m,
                              int64_t cbase, idx* cnt) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < nloc) {
    if (!ex[t]) atomicAdd(&cnt[fid[t] - cbase], 1);
  } else if (t < nloc + m) {
    atomicAdd(&cnt[imp[t - nloc].J - cbase], 1);
  }
}
// keys = global row id (unique), payload = extended row index (exact as a double)
__global__ void k_group_fill(const idx* fid, const idx* ex, int64_t nloc, int64_t ntot, int64_t row0,
                             const MemberRec* imp, int64_t m, int64_t cbase, const idx* off, idx* cur,
                             idx* keys, double* pay) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  int64_t Jl, gid, ext;
  if (t < nloc) {
    if (ex[t]) return;
    Jl = fid[t] - cbase;
    gid = row0 + t;
    ext = t;
  } else if (t < nloc + m) {
    Jl = imp[t - nloc].J - cbase;
    gid = imp[t - nloc].gid;
    ext = ntot + (t - nloc);
  } else {
    return;
  }
  const idx p = off[Jl] + atomicAdd(&cur[Jl], 1);
  keys[p] = static_cast<idx>(gid);
  pay[p] = static_cast<double>(ext);
}
__global__ void k_payload_to_idx(const double* pay, int64_t n, idx* out) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t < n) out[t] = static_cast<idx>(pay[t]);
}
__global__ void k_export_J(const idx* rows, int64_t m, const idx* fid, idx* q) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < m) q[k] = fid[rows[k]];
}
// p_i = b_i / ||b_J|| (transfer.cpp:42-45) for local rows of owned aggregates and imports
__global__ void k_ext_pval(const double* b_ext, const idx* fid, const idx* ex, int64_t nloc, int64_t ntot,
                           const MemberRec* imp, int64_t m, int64_t cbase, const double* cb, double* pv) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < nloc) {
    if (ex[i]) return;
    const double bi = b_ext[i];
    pv[i] = (bi != 0.0) ? __ddiv_rn(bi, cb[fid[i] - cbase]) : 0.0;
  } else if (i >= ntot && i < ntot + m) {
    const double bi = b_ext[i];
    pv[i] = (bi != 0.0) ? __ddiv_rn(bi, cb[imp[i - ntot].J - cbase]) : 0.0;
  }
}
__global__ void k_export_pval(const idx* rows, const double* cb, const double* b, int64_t m, double* pv) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const idx i = rows[k];
  const double bi = b[i];
  pv[i] = (bi != 0.0) ? __ddiv_rn(bi, cb[k]) : 0.0;
}
__global__ void k_map_idx(idx* x, int64_t n, const idx* map) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < n) x[k] = map[x[k]];
}
__global__ void k_export_len(const idx* rows, int64_t m, const idx* rp, idx* len) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < m) len[k] = rp[rows[k] + 1] - rp[rows[k]];
}
__global__ void k_export_entries(const idx* rows, int64_t m, const idx* off, const idx* rp, const idx* col,
                                 const double* val, const idx* fid, const double* pv, EntRec* out,
                                 idx* jc) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const idx i = rows[k];
  idx p = off[k];
  for (idx e = rp[i]; e < rp[i + 1]; ++e, ++p) {
    EntRec r;
    r.a = val[e];
    r.pvc = pv[col[e]];
    out[p] = r;
    jc[p] = fid[col[e]];
  }
}
__global__ void k_ext_entries(const EntRec* ent, const idx* jc, int64_t nie, int64_t base, int64_t next,
                              idx* col, double* val, idx* asg, double* pvc) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nie) return;
  col[base + t] = static_cast<idx>(next + t);
  val[base + t] = ent[t].a;
  asg[next + t] = jc[t];
  pvc[next + t] = ent[t].pvc;
}
__global__ void k_pack_row_values(const idx* rows, int64_t m, const idx* off, const idx* rp,
                                  const double* val, double* out) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const idx i = rows[k];
  idx p = off[k];
  for (idx e = rp[i]; e < rp[i + 1]; ++e) out[p++] = val[e];
}
__global__ void k_ext_len(const idx* rp, int64_t nloc, int64_t ntot, const idx* ilen, int64_t m, idx* len) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < nloc)
    len[i] = rp[i + 1] - rp[i];
  else if (i < ntot)
    len[i] = 0;
  else if (i < ntot + m)
    len[i] = ilen[i - ntot];
}

// AGGMG_DIST_TIMING=1: per-phase wall time of the distributed setup on rank 0 (stderr).
struct PhaseTimer {
  bool on = false;
  int rank = 0;
  std::chrono::steady_clock::time_point t;
  std::vector<std::pair<std::string, double>> acc;
  PhaseTimer() {
    const char* e = std::getenv("AGGMG_DIST_TIMING");
    on = e && e[0] == '1';
    t = std::chrono::steady_clock::now();
  }
  void mark(const char* name) {
    if (!on) return;
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
  void report() {
    if (!on || rank != 0) return;
    for (auto& a : acc) std::fprintf(stderr, "[dist setup] %-12s %8.2f ms\n", a.first.c_str(), a.second);
  }
};
thread_local PhaseTimer* g_phase = nullptr;
void phase(const char* name) {
  if (g_phase) g_phase->mark(name);
}

struct Coarsened {
  bool stalled = false;
  int64_t n_agg_global = 0;
  DistCsrPtr Ac;
  DevBuf<double> Bc;
};

Coarsened coarsen_level(Comm& comm, DistLevel& L, const SetupCfg& cfg, int64_t k) {
  const int me = comm.rank(), P = comm.size();
  const DistCsr& A = *L.A;
  const int64_t nloc = A.A.n_rows, nh = A.halo.nhalo, row0 = A.rows.begin(me);
  const int64_t ntot = nloc + nh;
  const int64_t n_glob = A.rows.n();
  const PartDev rp_dev = part_dev(A.rows);
  const unsigned g = grid_for(std::max<int64_t>(nloc, 1), 256);
  Coarsened out;

  // ---- a3 strength, a4 influence ----
  DevCsrPtr C = strength_rows(A.A, cfg.alpha, 0);
  DevBuf<idx> infl(ntot);
  infl.zero();
  if (C->nnz) AGG_LAUNCH(k_count_cols, grid_for(C->nnz, 256), 256, 0, C->col.get(), C->nnz, infl.get());
  halo_reverse_add(comm, A.halo, infl.get());
  phase("strength");

  // ---- a5 S = C u C^T (global ids), then local ids over A's halo ----
  DevBuf<idx> Cg(C->nnz);
  globalize_cols(A.halo, C->col.get(), C->nnz, Cg.get());
  // C^T: entries with an owned column are transposed locally; the cross entries travel to
  // the owner of their column as (row, col) pairs (global ids)
  DevBuf<unsigned long long> tcnt(P), tcur(P);
  tcnt.zero();
  tcur.zero();
  if (nloc)
    AGG_LAUNCH(k_cross_count, g, 256, 0, C->rowptr.get(), C->col.get(), Cg.get(), nloc, nloc, rp_dev,
               tcnt.get());
  std::vector<unsigned long long> tc(P);
  tcnt.download(tc.data(), P);
  sync();
  std::vector<int64_t> tsend(P), toff(P + 1, 0);
  for (int q = 0; q < P; ++q) {
    tsend[q] = static_cast<int64_t>(tc[q]);
    toff[q + 1] = toff[q] + tsend[q];
  }
  DevBuf<int64_t> toff_d(P + 1);
  toff_d.upload(toff.data(), P + 1);
  DevBuf<int2> tpairs(toff[P]);
  if (nloc && toff[P])
    AGG_LAUNCH(k_cross_fill, g, 256, 0, C->rowptr.get(), C->col.get(), Cg.get(), nloc, nloc, row0, rp_dev,
               toff_d.get(), tcur.get(), tpairs.get());
  DevBuf<int2> mine = alltoallv<int2>(comm, tpairs.get(), tsend);
  tpairs.reset();
  const int64_t mt = mine.size();
  DevBuf<idx> trp(nloc + 1), trow_cnt(nloc), tcur2(nloc), ttmp(C->nnz + mt), tcol(C->nnz + mt);
  trow_cnt.zero();
  tcur2.zero();
  if (nloc)
    AGG_LAUNCH(k_tcount_local, g, 256, 0, C->rowptr.get(), C->col.get(), nloc, nloc, trow_cnt.get());
  if (mt) AGG_LAUNCH(k_tcount_remote, grid_for(mt, 256), 256, 0, mine.get(), mt, row0, trow_cnt.get());
  scan_to_offsets_async(trow_cnt.get(), trp.get(), nloc);
  if (nloc)
    AGG_LAUNCH(k_tfill_local, g, 256, 0, C->rowptr.get(), C->col.get(), nloc, nloc, row0, trp.get(),
               tcur2.get(), ttmp.get());
  if (mt)
    AGG_LAUNCH(k_tfill_remote, grid_for(mt, 256), 256, 0, mine.get(), mt, row0, trp.get(), tcur2.get(),
               ttmp.get());
  segmented_sort(trp.get(), nloc, ttmp.get(), tcol.get());
  ttmp.reset();
  DevBuf<idx> scnt(nloc), srp(nloc + 1);
  if (nloc)
    AGG_LAUNCH(k_merge_rows_g, g, 256, 0, C->rowptr.get(), Cg.get(), trp.get(), tcol.get(), nloc, 0,
               nullptr, scnt.get());
  const int64_t snnz = scan_to_offsets(scnt.get(), srp.get(), nloc);
  DevBuf<idx> sg(snnz), scol(snnz);
  if (nloc && snnz)
    AGG_LAUNCH(k_merge_rows_g, g, 256, 0, C->rowptr.get(), Cg.get(), trp.get(), tcol.get(), nloc, 1,
               srp.get(), sg.get());
  localize_cols(A.halo, sg.get(), snnz, scol.get(),
                "distributed setup requires a structurally symmetric matrix (strength graph "
                "reaches a column outside the operator's halo)");
  C.reset();
  Cg.reset();
  sg.reset();
  mine.reset();
  phase("symmetrize");

  // ---- a6 MIS(2) ----
  DevBuf<Tuple> cur(ntot), mid(ntot);
  DevBuf<int8_t> state(ntot);
  DevBuf<DMisCtl> ctl(1);
  DMisCtl h0{static_cast<long long>(n_glob), 0, 0, 0};
  ctl.upload(&h0, 1);
  const uint64_t seed = level_seed(cfg.seed, k, kMisTag);
  if (nloc) AGG_LAUNCH(k_dmis_init, g, 256, 0, infl.get(), nloc, row0, seed, cur.get(), state.get());
  int batch = 8;
  while (true) {
    for (int b = 0; b < batch; ++b) {
      halo_update<double2>(comm, A.halo, reinterpret_cast<double2*>(cur.get()));
      AGG_LAUNCH(k_dmis_pass1, g, 256, 0, srp.get(), scol.get(), nloc, cur.get(), mid.get(), ctl.get());
      halo_update<double2>(comm, A.halo, reinterpret_cast<double2*>(mid.get()));
      AGG_LAUNCH(k_dmis_pass2, g, 256, 0, srp.get(), scol.get(), nloc, row0, mid.get(), cur.get(),
                 state.get(), ctl.get());
      comm.allreduce_sum(reinterpret_cast<int64_t*>(&ctl.get()->dec), 1);
      AGG_LAUNCH(k_dmis_update, 1, 1, 0, ctl.get());
    }
    const DMisCtl h = read_scalar(ctl.get());
    if (h.sweeps > n_glob) throw Error("mis2: failed to decide all nodes");
    if (h.undecided == 0) {
      L.mis_sweeps = h.sweeps;
      break;
    }
    batch = 4;
  }
  cur.reset();
  mid.reset();
  phase("mis2");

  // ---- a7 aggregation ----
  halo_update<int8_t>(comm, A.halo, state.get());
  DevBuf<idx> rep(ntot), via1(nloc), rep2(nloc), via2(nloc), isrep(nloc), rank(nloc + 1);
  if (nloc)
    AGG_LAUNCH(k_dagg_pass1, g, 256, 0, srp.get(), scol.get(), nloc, row0, nloc, A.halo.halo_gid.get(),
               state.get(), rep.get(), via1.get());
  halo_update<idx>(comm, A.halo, rep.get());
  // A(j, i) for the cross edges pass 2 looks at
  DevBuf<idx> Ag = global_cols(A);
  DevBuf<idx> rq_cnt(nloc), rq_off(nloc + 1), slot(snnz);
  if (nloc)
    AGG_LAUNCH(k_dagg_req_count, g, 256, 0, srp.get(), scol.get(), nloc, nloc, rep.get(), rq_cnt.get());
  const int64_t nreq = scan_to_offsets(rq_cnt.get(), rq_off.get(), nloc);
  DevBuf<int2> req(nreq);
  if (nloc)
    AGG_LAUNCH(k_dagg_req_fill, g, 256, 0, srp.get(), scol.get(), nloc, row0, nloc,
               A.halo.halo_gid.get(), rep.get(), rq_off.get(), req.get(), slot.get());
  DevBuf<double> tval(nreq);
  {
    DevBuf<unsigned> own(nreq);
    DevBuf<idx> perm(nreq);
    if (nreq) AGG_LAUNCH(k_req_owner, grid_for(nreq, 256), 256, 0, req.get(), nreq, rp_dev, own.get(), perm.get());
    // requests grouped (stably) by owner; the permutation routes the answers back
    DevBuf<unsigned> own_s(nreq);
    DevBuf<idx> perm_s(nreq);
    DevBuf<long long> cnt_d(P);
    cnt_d.zero();
    DevBuf<int2> grouped(nreq);
    if (nreq) {
      AGG_LAUNCH(k_count_u, grid_for(nreq, 256), 256, 0, own.get(), nreq, cnt_d.get());
      const int nbits = std::max(1, 32 - __builtin_clz(static_cast<unsigned>(P)));
      cub_call([&](void* t, size_t& b) {
        return cub::DeviceRadixSort::SortPairs(t, b, own.get(), own_s.get(), perm.get(), perm_s.get(),
                                               static_cast<int>(nreq), 0, nbits, stream());
      });
      AGG_LAUNCH(k_req_gather, grid_for(nreq, 256), 256, 0, req.get(), perm_s.get(), nreq, grouped.get());
    }
    std::vector<long long> c(P);
    cnt_d.download(c.data(), P);
    sync();
    std::vector<int64_t> cnt(c.begin(), c.end()), rc;
    DevBuf<int2> incoming = alltoallv<int2>(comm, grouped.get(), cnt, &rc);
    const int64_t nin = incoming.size();
    DevBuf<double> ans(nin);
    if (nin)
      AGG_LAUNCH(k_req_answer, grid_for(nin, 256), 256, 0, incoming.get(), nin, row0, A.A.rowptr.get(),
                 Ag.get(), A.A.val.get(), ans.get());
    DevBuf<double> back = alltoallv<double>(comm, ans.get(), rc);
    if (nreq) AGG_LAUNCH(k_scatter_back, grid_for(nreq, 256), 256, 0, back.get(), perm_s.get(), nreq, tval.get());
  }
  if (nloc)
    AGG_LAUNCH(k_dagg_pass2, g, 256, 0, srp.get(), scol.get(), A.A.rowptr.get(), Ag.get(),
               A.A.val.get(), nloc, row0, nloc, A.halo.halo_gid.get(), rep.get(), slot.get(),
               tval.get(), rep2.get(), via2.get(), isrep.get());
  const int64_t nrep = scan_to_offsets(isrep.get(), rank.get(), nloc);
  const std::vector<int64_t> reps_all = comm.allgather_host({nrep});
  const Partition cpart = Partition::from_counts(reps_all);
  out.n_agg_global = cpart.n();
  if (static_cast<double>(out.n_agg_global) >= 0.95 * static_cast<double>(n_glob)) {
    out.stalled = true;
    return out;
  }
  const int64_t cbase = cpart.begin(me), ncl = cpart.count(me);
  DevBuf<idx> fid(ntot);
  if (nloc) AGG_LAUNCH(k_dagg_fid_reps, g, 256, 0, isrep.get(), rank.get(), nloc, cbase, fid.get());
  halo_update<idx>(comm, A.halo, fid.get());
  if (nloc) AGG_LAUNCH(k_dagg_fid_copy, g, 256, 0, via1.get(), rep.get(), isrep.get(), nloc, 1, fid.get());
  halo_update<idx>(comm, A.halo, fid.get());
  if (nloc) AGG_LAUNCH(k_dagg_fid_copy, g, 256, 0, via2.get(), rep.get(), isrep.get(), nloc, 2, fid.get());
  halo_update<idx>(comm, A.halo, fid.get());
  srp.reset();
  scol.reset();
  phase("aggregate");

  // ---- a8 transfer / a9-a10 Galerkin over the EXTENDED row set ----
  // Rows whose aggregate lives on another rank are exported to the aggregate's owner.  The
  // owner's extended row space is [0, nloc) local rows, [nloc, ntot) halo (empty rows),
  // [ntot, ntot + m) imported rows; member groups are ordered by global row id, so the
  // one-GPU group kernels (ascending-member norms, R rows, the Galerkin sort / ordered
  // segment sums) run unchanged and reproduce the reference order across ranks.
  const PartDev cp_dev = part_dev(cpart);
  DevBuf<unsigned> odest(nloc);
  DevBuf<idx> exflag(nloc), expos(nloc + 1);
  if (nloc)
    AGG_LAUNCH(k_agg_owner, g, 256, 0, fid.get(), nloc, cp_dev, me, odest.get(), exflag.get());
  const int64_t nexp = scan_to_offsets(exflag.get(), expos.get(), nloc);
  // exported rows in row order, grouped (stably) by destination
  DevBuf<idx> exrow(nexp), exrow_s(nexp);
  DevBuf<unsigned> exdest(nexp), exdest_s(nexp);
  std::vector<int64_t> ecnt(P, 0);
  if (nexp) {
    AGG_LAUNCH(k_export_list, g, 256, 0, exflag.get(), expos.get(), odest.get(), nloc, exrow.get(),
               exdest.get());
    DevBuf<long long> cnt_d(P);
    cnt_d.zero();
    AGG_LAUNCH(k_count_u, grid_for(nexp, 256), 256, 0, exdest.get(), nexp, cnt_d.get());
    const int nbits = std::max(1, 32 - __builtin_clz(static_cast<unsigned>(P)));
    cub_call([&](void* t, size_t& bb) {
      return cub::DeviceRadixSort::SortPairs(t, bb, exdest.get(), exdest_s.get(), exrow.get(),
                                             exrow_s.get(), static_cast<int>(nexp), 0, nbits, stream());
    });
    std::vector<long long> c(P);
    cnt_d.download(c.data(), P);
    sync();
    for (int q = 0; q < P; ++q) ecnt[q] = c[q];
  }
  // round 1: (gid, J, b) of every exported row
  DevBuf<MemberRec> mrec(nexp);
  if (nexp)
    AGG_LAUNCH(k_export_members, grid_for(nexp, 256), 256, 0, exrow_s.get(), nexp, fid.get(),
               L.B.get(), row0, mrec.get());
  std::vector<int64_t> icnt;
  DevBuf<double2> imp_buf = alltoallv<double2>(comm, reinterpret_cast<const double2*>(mrec.get()), ecnt, &icnt);
  const MemberRec* imp = reinterpret_cast<const MemberRec*>(imp_buf.get());
  const int64_t m = imp_buf.size();
  const int64_t next = ntot + m;  // extended row space
  DevBuf<double> b_ext(next);
  DevBuf<idx> gid_ext(next);
  b_ext.zero();
  if (next)
    AGG_LAUNCH(k_ext_rows, grid_for(next, 256), 256, 0, L.B.get(), nloc, ntot, row0, imp, m,
               b_ext.get(), gid_ext.get());
  // member groups of the owned aggregates, ascending global row id
  DevBuf<idx> gcnt(ncl), goff(ncl + 1), gcur(ncl), gkeys(nloc + m), gsorted(nloc + m);
  DevBuf<double> gpay(nloc + m), gpay_s(nloc + m);
  gcnt.zero();
  gcur.zero();
  if (nloc + m)
    AGG_LAUNCH(k_group_count, grid_for(nloc + m, 256), 256, 0, fid.get(), exflag.get(), nloc, imp, m,
               cbase, gcnt.get());
  scan_to_offsets_async(gcnt.get(), goff.get(), ncl);
  if (nloc + m)
    AGG_LAUNCH(k_group_fill, grid_for(nloc + m, 256), 256, 0, fid.get(), exflag.get(), nloc, ntot,
               row0, imp, m, cbase, goff.get(), gcur.get(), gkeys.get(), gpay.get());
  segmented_sort(goff.get(), ncl, gkeys.get(), gsorted.get(), gpay.get(), gpay_s.get());
  DevBuf<idx> rows_ext(nloc + m);
  if (nloc + m)
    AGG_LAUNCH(k_payload_to_idx, grid_for(nloc + m, 256), 256, 0, gpay_s.get(), nloc + m, rows_ext.get());
  gkeys.reset();
  gpay.reset();
  gpay_s.reset();
  gsorted.reset();
  // coarse norms (transfer.cpp:21-29) and R rows
  out.Bc.resize(ncl);
  DevBuf<idx> rcnt(ncl);
  {
    const int64_t bad = transfer_norms_groups(goff.get(), rows_ext.get(), b_ext.get(), ncl,
                                              out.Bc.get(), rcnt.get());
    const int64_t worst = comm.allreduce_host_max(bad < 0 ? -1 : cbase + bad);
    if (worst >= 0)
      throw Error("transfer: near-null-space vector vanishes on aggregate " + std::to_string(worst));
  }
  // P values: owned aggregates here, the others from their owners' norms
  DevBuf<idx> fq(nexp);
  DevBuf<double> fcb(nexp);
  if (nexp)
    AGG_LAUNCH(k_export_J, grid_for(nexp, 256), 256, 0, exrow.get(), nexp, fid.get(), fq.get());
  fetch_remote<double>(comm, cpart, out.Bc.get(), fq.get(), nexp, fcb.get());
  DevBuf<double> pv_ext(next);
  pv_ext.zero();
  if (next)
    AGG_LAUNCH(k_ext_pval, grid_for(next, 256), 256, 0, b_ext.get(), fid.get(), exflag.get(), nloc,
               ntot, imp, m, cbase, out.Bc.get(), pv_ext.get());
  if (nexp)
    AGG_LAUNCH(k_export_pval, grid_for(nexp, 256), 256, 0, exrow.get(), fcb.get(), L.B.get(), nexp,
               pv_ext.get());
  auto Rg = std::make_shared<DevCsr>();
  Rg->n_rows = ncl;
  Rg->n_cols = n_glob;
  Rg->rowptr.resize(ncl + 1);
  Rg->nnz = scan_to_offsets(rcnt.get(), Rg->rowptr.get(), ncl);
  Rg->col.resize(Rg->nnz);
  Rg->val.resize(Rg->nnz);
  transfer_R_groups(goff.get(), rows_ext.get(), pv_ext.get(), ncl, Rg->rowptr.get(), Rg->col.get(),
                    Rg->val.get());
  if (Rg->nnz)
    AGG_LAUNCH(k_map_idx, grid_for(Rg->nnz, 256), 256, 0, Rg->col.get(), Rg->nnz, gid_ext.get());
  L.R = make_dist(comm, cpart, A.rows, *Rg, "restriction: member outside the plan");
  // P on this rank's rows: coarse id (local numbering over the P plan) and value
  L.pval.resize(ntot);
  AGG_CUDA(cudaMemcpyAsync(L.pval.get(), pv_ext.get(), sizeof(double) * ntot, cudaMemcpyDeviceToDevice,
                           stream()));
  halo_update<double>(comm, A.halo, L.pval.get());
  AGG_CUDA(cudaMemcpyAsync(pv_ext.get(), L.pval.get(), sizeof(double) * ntot, cudaMemcpyDeviceToDevice,
                           stream()));  // halo columns' weights for the Galerkin products
  build_halo_plan(comm, cpart, fid.get(), nloc, L.P_halo);
  L.agg_local.resize(nloc);
  localize_cols(L.P_halo, fid.get(), nloc, L.agg_local.get(), "prolongation: aggregate outside the plan");
  L.agg_global.resize(nloc);
  if (nloc)
    AGG_CUDA(cudaMemcpyAsync(L.agg_global.get(), fid.get(), sizeof(idx) * nloc, cudaMemcpyDeviceToDevice,
                             stream()));
  phase("transfer");

  // round 2: the exported rows' entries (coarse column, value, column weight)
  DevBuf<idx> exlen(nexp), exoff(nexp + 1);
  if (nexp)
    AGG_LAUNCH(k_export_len, grid_for(nexp, 256), 256, 0, exrow_s.get(), nexp, A.A.rowptr.get(), exlen.get());
  const int64_t nent = scan_to_offsets(exlen.get(), exoff.get(), nexp);
  DevBuf<EntRec> erec(nent);
  DevBuf<idx> ejc(nent);
  if (nexp)
    AGG_LAUNCH(k_export_entries, grid_for(nexp, 256), 256, 0, exrow_s.get(), nexp, exoff.get(),
               A.A.rowptr.get(), A.A.col.get(), A.A.val.get(), fid.get(), L.pval.get(), erec.get(),
               ejc.get());
  std::vector<int64_t> ent_cnt(P, 0);
  {
    std::vector<int64_t> rowc(P, 0), pos(P + 1, 0);
    for (int q = 0; q < P; ++q) pos[q + 1] = pos[q] + ecnt[q];
    std::vector<idx> off_h(nexp + 1);
    if (nexp) {
      exoff.download(off_h.data(), nexp + 1);
      sync();
    }
    for (int q = 0; q < P; ++q) ent_cnt[q] = nexp ? off_h[pos[q + 1]] - off_h[pos[q]] : 0;
  }
  DevBuf<idx> ilen = alltoallv<idx>(comm, exlen.get(), ecnt);
  DevBuf<double2> ient_buf = alltoallv<double2>(comm, reinterpret_cast<const double2*>(erec.get()), ent_cnt);
  DevBuf<idx> ijc = alltoallv<idx>(comm, ejc.get(), ent_cnt);
  const EntRec* ient = reinterpret_cast<const EntRec*>(ient_buf.get());
  const int64_t nie = ient_buf.size();
  // extended CSR: local rows, empty halo rows, imported rows; imported columns get private
  // slots [next, next + nie) carrying their coarse id and weight
  auto Aext = std::make_shared<DevCsr>();
  Aext->n_rows = next;
  Aext->n_cols = next + nie;
  Aext->nnz = A.A.nnz + nie;
  Aext->rowptr.resize(next + 1);
  Aext->col.resize(Aext->nnz);
  Aext->val.resize(Aext->nnz);
  {
    DevBuf<idx> len(next);
    if (next)
      AGG_LAUNCH(k_ext_len, grid_for(next, 256), 256, 0, A.A.rowptr.get(), nloc, ntot, ilen.get(), m,
                 len.get());
    scan_to_offsets(len.get(), Aext->rowptr.get(), next);
  }
  if (A.A.nnz) {
    AGG_CUDA(cudaMemcpyAsync(Aext->col.get(), A.A.col.get(), sizeof(idx) * A.A.nnz,
                             cudaMemcpyDeviceToDevice, stream()));
    AGG_CUDA(cudaMemcpyAsync(Aext->val.get(), A.A.val.get(), sizeof(double) * A.A.nnz,
                             cudaMemcpyDeviceToDevice, stream()));
  }
  DevBuf<idx> asg_ext(next + nie);
  DevBuf<double> pvc_ext(next + nie);
  AGG_CUDA(cudaMemcpyAsync(asg_ext.get(), fid.get(), sizeof(idx) * ntot, cudaMemcpyDeviceToDevice, stream()));
  AGG_CUDA(cudaMemcpyAsync(pvc_ext.get(), pv_ext.get(), sizeof(double) * next, cudaMemcpyDeviceToDevice,
                           stream()));
  if (nie)
    AGG_LAUNCH(k_ext_entries, grid_for(nie, 256), 256, 0, ient, ijc.get(), nie, A.A.nnz, next,
               Aext->col.get(), Aext->val.get(), asg_ext.get(), pvc_ext.get());
  AggDev gx;
  gx.n_fine = next;
  gx.n_agg = ncl;
  gx.assignment = std::move(asg_ext);
  gx.agg_row_offsets = std::move(goff);
  gx.rows_by_coarse = std::move(rows_ext);
  GalerkinDev gal = build_galerkin_cache(*Aext, gx, true);
  DevCsrPtr Acg = apply_galerkin_cache(gal, *Aext, pvc_ext.get());
  Acg->n_cols = cpart.n();
  if (cfg.reuse_caches) {  // keep what refresh_values needs (galerkin.cpp:98-137 reuse)
    auto gc = std::make_unique<DistGalerkin>();
    gc->gal = std::move(gal);
    gc->Aext = Aext;
    gc->pvc = std::move(pvc_ext);
    gc->exrow = std::move(exrow_s);
    gc->exoff = std::move(exoff);
    gc->nexp = nexp;
    gc->nie = nie;
    gc->ent_cnt = ent_cnt;
    L.galc = std::move(gc);
  }
  phase("galerkin");
  out.Ac = make_dist(comm, cpart, cpart, *Acg);
  phase("coarse-plan");
  return out;
}

void dist_smoother(Comm& comm, DistLevel& L, const SetupCfg& cfg, int64_t k) {
  const DistCsr& A = *L.A;
  const int me = comm.rank();
  const int64_t nloc = A.A.n_rows, row0 = A.rows.begin(me);
  const uint64_t seed = level_seed(cfg.seed, k, kSmootherTag);
  ArnoldiOps ops;
  ops.n_alloc = nloc + A.halo.nhalo;
  ops.n_global = A.rows.n();
  ops.row0 = row0;
  ops.start = [&](double* v) {
    if (nloc) AGG_LAUNCH(k_uniform_sym_off, grid_for(nloc, 256), 256, 0, nloc, row0, seed, v);
  };
  ops.before_spmv = [&](double* v) { halo_update<double>(comm, A.halo, v); };
  ops.dot = [&](const double* a, const double* b) { return dist_dot(comm, a, b, nloc); };
  ops.allreduce_dev = [&](double* v, int k) { comm.allreduce_sum(v, k); };
  // a zero diagonal on any rank must fail every rank
  std::string err;
  try {
    setup_smoother(A.A, cfg.smoother, cfg.arnoldi_m, seed, L.smoother, &ops);
  } catch (const Error& e) {
    err = e.what();
  }
  if (comm.allreduce_host_sum(err.empty() ? 0 : 1) > 0)
    throw Error(err.empty() ? "smoother: zero diagonal on another rank" : err);
}

}  // namespace

DistHierarchy::~DistHierarchy() { drop_graphs(); }

void DistHierarchy::drop_graphs() {
  for (auto& g : graphs)
    if (g.second) cudaGraphExecDestroy(g.second);
  graphs.clear();
  graph_kernels.clear();
}

std::unique_ptr<DistHierarchy> dist_setup_hierarchy(Comm& comm, DistCsrPtr A0, const double* B0_local,
                                                    const SetupCfg& cfg, int64_t agglomerate_rows) {
  require(A0->rows.n() == A0->cols.n(), "setup: matrix must be square");
  require(cfg.coarse_size_max >= 1, "setup: coarse_size_max must be at least 1");
  require(cfg.max_levels >= 1, "setup: max_levels must be at least 1");
  // sgs is one global sequential sweep (smoother.cpp:105-119): no row partition reproduces it
  require(cfg.smoother != 2,
          "setup: the sgs smoother is a global sequential sweep; a row-partitioned hierarchy "
          "supports jacobi and damped_jacobi");
  const int me = comm.rank();
  pool_reserve(16 * static_cast<size_t>(A0->A.nnz * 12 + A0->A.n_rows * 8) + (size_t{256} << 20));
  comm.barrier();
  const auto t0 = std::chrono::steady_clock::now();
  PhaseTimer timer;
  timer.rank = me;
  g_phase = timer.on ? &timer : nullptr;
  auto h = std::make_unique<DistHierarchy>();
  h->comm = &comm;
  h->cfg = cfg;
  h->agglomerate_rows = std::max<int64_t>(agglomerate_rows, cfg.coarse_size_max);

  DistCsrPtr A = A0;
  DevBuf<double> B(A->A.n_rows);
  if (B0_local)
    copy_double(B.get(), B0_local, A->A.n_rows);
  else
    fill_double(B.get(), A->A.n_rows, 1.0);
  {
    const double nb = std::sqrt(dist_dot(comm, B.get(), B.get(), A->A.n_rows));
    require(nb > 0.0, "setup: near-null-space vector is zero");
  }
  int64_t k = 0;
  while (true) {
    const int64_t n_glob = A->rows.n();
    if (n_glob <= h->agglomerate_rows || k + 1 >= cfg.max_levels) break;
    DistLevel L;
    L.A = A;
    L.B = std::move(B);
    Coarsened c = coarsen_level(comm, L, cfg, k);
    if (c.stalled) {  // the tail re-runs this level and records the reference's warning
      B = std::move(L.B);
      break;
    }
    dist_smoother(comm, L, cfg, k);
    phase("smoother");
    A = c.Ac;
    B = std::move(c.Bc);
    h->levels.push_back(std::move(L));
    ++k;
  }
  phase("levels");
  // agglomerate level kd onto EVERY rank and continue with the one-GPU setup there: the ranks
  // build (and later run) identical copies of the tail — deterministic kernels on identical
  // inputs — so no rank idles while another works and the solve needs no scatter back
  h->tail_rows = A->rows;
  h->tail_A = A;
  DevCsrPtr Ag = gather_to_all(comm, *A);
  DevBuf<double> Bg(A->rows.n());
  allgather_vector(comm, A->rows, B.get(), Bg.get());
  std::vector<int64_t> meta(3, 0);  // tail level count, warnings flag
  {
    SetupCfg tc = cfg;
    tc.level_offset = k;
    tc.max_levels = cfg.max_levels - static_cast<int>(k);
    h->tail = setup_hierarchy(Ag, Bg.get(), tc);
    meta[0] = h->tail->n_levels();
  }
  const std::vector<int64_t> m_all = comm.allgather_host(meta);
  h->n_levels_total = k + m_all[0];
  h->warnings = h->tail->warnings;
  // global sizes per level (same on every rank)
  for (auto& L : h->levels) {
    h->level_rows.push_back(L.A->rows.n());
    h->level_nnz.push_back(comm.allreduce_host_sum(L.A->A.nnz));
  }
  std::vector<int64_t> tail_sizes;
  if (me == 0)  // (every rank holds the same tail; rank 0's sizes are published)
    for (auto& L : h->tail->levels) {
      tail_sizes.push_back(L.A->n_rows);
      tail_sizes.push_back(L.A->nnz);
    }
  tail_sizes.resize(2 * m_all[0], 0);
  const std::vector<int64_t> ts_all = comm.allgather_host(tail_sizes);
  for (int64_t l = 0; l < m_all[0]; ++l) {
    h->level_rows.push_back(ts_all[2 * l]);
    h->level_nnz.push_back(ts_all[2 * l + 1]);
  }
  if (!h->levels.empty()) h->tail_halo_cap = h->levels.back().P_halo.nhalo;
  phase("tail");
  timer.report();
  g_phase = nullptr;
  comm.barrier();
  h->setup_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  return h;
}

}  // namespace aggmg_b200

namespace aggmg_b200 {

void dist_refresh_values(DistHierarchy& h, const double* new_values_local) {
  Comm& comm = *h.comm;
  require(h.cfg.reuse_caches, "refresh_values: hierarchy was built without caches; rebuild it");
  h.drop_graphs();  // the smoother arrays are rebuilt below; captured pointers would dangle
  DistCsr& A0 = h.kd() ? *h.levels[0].A : *h.tail_A;
  copy_double(A0.A.val.get(), new_values_local, A0.A.nnz);
  A0.A.refresh_sell();
  for (int64_t k = 0; k < h.kd(); ++k) {
    DistLevel& L = h.levels[k];
    DistGalerkin& g = *L.galc;
    const DevCsr& A = L.A->A;
    // the exported rows' new values travel to their aggregates' owners, as in setup
    int64_t nent = 0;
    for (int64_t c : g.ent_cnt) nent += c;
    DevBuf<double> send(std::max<int64_t>(nent, 1));
    if (g.nexp)
      AGG_LAUNCH(k_pack_row_values, grid_for(g.nexp, 256), 256, 0, g.exrow.get(), g.nexp, g.exoff.get(),
                 A.rowptr.get(), A.val.get(), send.get());
    DevBuf<double> recv = alltoallv<double>(comm, send.get(), g.ent_cnt);
    require(recv.size() == g.nie, "refresh_values: imported entry count changed");
    if (A.nnz)
      AGG_CUDA(cudaMemcpyAsync(g.Aext->val.get(), A.val.get(), sizeof(double) * A.nnz,
                               cudaMemcpyDeviceToDevice, stream()));
    if (g.nie)
      AGG_CUDA(cudaMemcpyAsync(g.Aext->val.get() + A.nnz, recv.get(), sizeof(double) * g.nie,
                               cudaMemcpyDeviceToDevice, stream()));
    DevCsrPtr Ac = apply_galerkin_cache(g.gal, *g.Aext, g.pvc.get());
    DistCsr& next = (k + 1 < h.kd()) ? *h.levels[k + 1].A : *h.tail_A;
    require(Ac->nnz == next.A.nnz, "refresh_values: coarse pattern changed");
    copy_double(next.A.val.get(), Ac->val.get(), Ac->nnz);
    next.A.refresh_sell();
    dist_smoother(comm, L, h.cfg, k);
  }
  // the agglomerated tail: level kd's new values (row order = rank order) to every rank, each
  // refreshing its copy of the tail
  const std::vector<int64_t> cnt = comm.allgather_host({h.tail_A->A.nnz});
  DevBuf<double> all;
  std::vector<CommMsg> s, r;
  int64_t tot = 0;
  for (int64_t c : cnt) tot += c;
  all.resize(tot);
  int64_t off = 0;
  for (int q = 0; q < comm.size(); ++q) {
    s.push_back({q, h.tail_A->A.val.get(), sizeof(double) * h.tail_A->A.nnz});
    r.push_back({q, all.get() + off, sizeof(double) * cnt[q]});
    off += cnt[q];
  }
  comm.exchange(s, r);
  refresh_values(*h.tail, all.get());
  comm.barrier();
}

}  // namespace aggmg_b200
