// setup.cu — strength, symmetrization, MIS(2), aggregation, transfer and the Galerkin
// sort / segmented reduce.  Every kernel reproduces the reference's arithmetic and
// tie-breaking exactly; the file is compiled with --fmad=false and
// uses explicit _rn intrinsics where a rounding sequence is part of the contract.
#include <algorithm>
#include <string>

#include "setup.cuh"

namespace aggmg_b200 {

namespace {

__device__ inline double dmax_ref(double a, double b) { return (a < b) ? b : a; }  // std::max

// ---- a3 strength ---------------------------------------------------------------------
// mode 0: count (cnt[i]); mode 1: fill columns at out_rowptr[i].
__global__ void k_strength(const idx* __restrict__ rowptr, const idx* __restrict__ col,
                           const double* __restrict__ val, int64_t n, double alpha, int fail_zero,
                           int mode, const idx* out_rowptr, idx* out, int* bad_row) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const idx lo = rowptr[i], hi = rowptr[i + 1];
  double d = 0.0;
  for (idx k = lo; k < hi; ++k)
    if (col[k] == i) d = val[k];
  double s;
  if (d == 0.0) {  // strength.cpp:18-21
    if (fail_zero) atomicMin(bad_row, static_cast<int>(i));
    s = 1.0;
  } else {
    s = d > 0.0 ? 1.0 : -1.0;
  }
  const double ns = -s;
  double m = 0.0;
  for (idx k = lo; k < hi; ++k) {
    if (col[k] == i) continue;
    m = dmax_ref(m, __dmul_rn(ns, val[k]));
  }
  const double thr = __dmul_rn(alpha, m);
  if (mode == 0) {
    idx c = 0;
    if (m > 0.0)
      for (idx k = lo; k < hi; ++k)
        if (col[k] != i && __dmul_rn(ns, val[k]) > thr) ++c;
    out[i] = c;
  } else {
    if (!(m > 0.0)) return;
    idx p = out_rowptr[i];
    for (idx k = lo; k < hi; ++k)
      if (col[k] != i && __dmul_rn(ns, val[k]) > thr) out[p++] = col[k];
  }
}

// The same row rule over CSR-stream row blocks (sparse.cuh): the block's columns and values
// are staged into shared memory with coalesced vector loads, then one thread per row applies
// k_strength's three passes from shared memory (same operations, same order).
constexpr int kStrThreads = 256;
__global__ void __launch_bounds__(kStrThreads)
    k_strength_stream(const idx* __restrict__ rowptr, const idx* __restrict__ col,
                      const double* __restrict__ val, int64_t n, int rpb, int64_t nblocks,
                      int stage, double alpha, int fail_zero, int mode, const idx* out_rowptr,
                      idx* out, int* bad_row) {
  extern __shared__ __align__(16) double sstage[];
  double* sv = sstage;
  idx* sc = reinterpret_cast<idx*>(sstage + stage);
  for (int64_t rb = blockIdx.x; rb < nblocks; rb += gridDim.x) {
    const int64_t r0 = rb * rpb, r1 = min(r0 + static_cast<int64_t>(rpb), n);
    const idx e0 = rowptr[r0], e1 = rowptr[r1];
    const idx ea = e0 & ~1;
    for (idx e = ea + 2 * static_cast<idx>(threadIdx.x); e < e1; e += 2 * kStrThreads) {
      const double2 v2 = __ldcs(reinterpret_cast<const double2*>(val + e));
      const int2 c2 = __ldcs(reinterpret_cast<const int2*>(col + e));
      *reinterpret_cast<double2*>(sv + (e - ea)) = v2;
      *reinterpret_cast<int2*>(sc + (e - ea)) = c2;
    }
    __syncthreads();
    const int64_t i = r0 + threadIdx.x;
    if (threadIdx.x < rpb && i < r1) {
      const idx lo = rowptr[i] - ea, hi = rowptr[i + 1] - ea;
      const idx ii = static_cast<idx>(i);
      double d = 0.0;
      for (idx k = lo; k < hi; ++k)
        if (sc[k] == ii) d = sv[k];
      double sg;
      if (d == 0.0) {  // strength.cpp:18-21
        if (fail_zero) atomicMin(bad_row, static_cast<int>(i));
        sg = 1.0;
      } else {
        sg = d > 0.0 ? 1.0 : -1.0;
      }
      const double ns = -sg;
      double m = 0.0;
      for (idx k = lo; k < hi; ++k) {
        if (sc[k] == ii) continue;
        m = dmax_ref(m, __dmul_rn(ns, sv[k]));
      }
      const double thr = __dmul_rn(alpha, m);
      if (mode == 0) {
        idx c = 0;
        if (m > 0.0)
          for (idx k = lo; k < hi; ++k)
            if (sc[k] != ii && __dmul_rn(ns, sv[k]) > thr) ++c;
        out[i] = c;
      } else if (m > 0.0) {
        idx p = out_rowptr[i];
        for (idx k = lo; k < hi; ++k)
          if (sc[k] != ii && __dmul_rn(ns, sv[k]) > thr) out[p++] = sc[k];
      }
    }
    __syncthreads();
  }
}

// ---- a4/a5 influence + symmetrize -------------------------------------------------------
__global__ void k_col_count(const idx* col, int64_t nnz, idx* cnt) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < nnz) atomicAdd(&cnt[col[k]], 1);
}
// S = C u C^T and the influence counts without materialising C^T (strength.cpp:74-111).
// Strength graphs are structurally symmetric almost everywhere, so each entry (r, c) is
// probed for its mirror (c, r) by binary search in the sorted row c: a mirrored entry adds
// nothing to S, an unmirrored one adds r to row c of S.  influence(c) = |{r : c in C_r}| =
// (entries of row c whose mirror exists) + (unmirrored entries pointing at c).
__device__ __forceinline__ bool row_has(const idx* ccol, idx lo, idx hi, idx v) {
  while (lo < hi) {
    const idx mid = (lo + hi) >> 1;
    const idx x = __ldg(ccol + mid);
    if (x == v) return true;
    if (x < v) lo = mid + 1;
    else hi = mid;
  }
  return false;
}
// pass 1: mirrored count per row, unmirrored entries counted per receiving row
__global__ void k_sym_probe(const idx* __restrict__ crp, const idx* __restrict__ ccol, int64_t n,
                            idx* mirrored, idx* extra_cnt, int8_t* has_extra,
                            unsigned long long* total) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  unsigned u = 0;
  if (r < n) {
    idx f = 0;
    const idx k1 = crp[r + 1];
    for (idx k = crp[r]; k < k1; ++k) {
      const idx c = ccol[k];
      if (row_has(ccol, __ldg(crp + c), __ldg(crp + c + 1), static_cast<idx>(r))) {
        ++f;
      } else {
        atomicAdd(&extra_cnt[c], 1);
        ++u;
      }
    }
    mirrored[r] = f;
    has_extra[r] = u ? 1 : 0;
  }
  for (int o = 16; o > 0; o >>= 1) u += __shfl_down_sync(0xffffffffu, u, o);
  if ((threadIdx.x & 31) == 0 && u) atomicAdd(total, static_cast<unsigned long long>(u));
}
// pass 2 (rows with unmirrored entries only): r goes into row c's extra bucket
__global__ void k_sym_extras(const idx* __restrict__ crp, const idx* __restrict__ ccol, int64_t n,
                             const int8_t* has_extra, const idx* eoff, idx* cursor, idx* ecol) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n || !has_extra[r]) return;
  for (idx k = crp[r]; k < crp[r + 1]; ++k) {
    const idx c = ccol[k];
    if (!row_has(ccol, __ldg(crp + c), __ldg(crp + c + 1), static_cast<idx>(r)))
      ecol[eoff[c] + atomicAdd(&cursor[c], 1)] = static_cast<idx>(r);
  }
}
__global__ void k_sym_counts(const idx* crp, const idx* mirrored, const idx* extra_cnt, int64_t n,
                             idx* influence, idx* scnt) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  influence[r] = mirrored[r] + extra_cnt[r];
  scnt[r] = crp[r + 1] - crp[r] + extra_cnt[r];
}
// S row = C row merged with its (sorted) extra bucket; buckets are rare and short
__global__ void k_sym_fill(const idx* __restrict__ crp, const idx* __restrict__ ccol,
                           const idx* srp, const idx* eoff, const idx* extra_cnt, idx* ecol,
                           int64_t n, idx* scol) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  idx a = crp[r];
  const idx ae = crp[r + 1];
  idx* o = scol + srp[r];
  const idx ne = extra_cnt[r];
  if (ne == 0) {
    for (; a < ae; ++a) *o++ = ccol[a];
    return;
  }
  idx* e = ecol + eoff[r];
  for (idx x = 1; x < ne; ++x) {  // insertion sort of the bucket
    const idx v = e[x];
    idx y = x;
    for (; y > 0 && e[y - 1] > v; --y) e[y] = e[y - 1];
    e[y] = v;
  }
  idx b = 0;
  while (a < ae || b < ne) {
    if (b >= ne || (a < ae && ccol[a] < e[b])) *o++ = ccol[a++];
    else *o++ = e[b++];
  }
}

// ---- a6 MIS(2) ---------------------------------------------------------------------------
struct __align__(16) Tuple {
  double v;
  int i;
  int s;
};
// lexicographic (s, v, i) — aggregation.cpp:24-28
__device__ inline bool tuple_less(const Tuple& a, const Tuple& b) {
  if (a.s != b.s) return a.s < b.s;
  if (a.v != b.v) return a.v < b.v;
  return a.i < b.i;
}
__device__ inline Tuple load_tuple(const Tuple* p) {
  const double2 raw = __ldg(reinterpret_cast<const double2*>(p));
  Tuple t;
  t.v = raw.x;
  const int2 is = *reinterpret_cast<const int2*>(&raw.y);
  t.i = is.x;
  t.s = is.y;
  return t;
}
struct MisCtl {
  int undecided;
  int active;
  int sweeps;
  int pad;
};

__global__ void k_mis_init(const idx* infl, int64_t n, uint64_t seed, Tuple* cur, int8_t* state) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  Tuple t;
  t.v = __dadd_rn(static_cast<double>(infl[i]), uniform_open01(seed, static_cast<uint64_t>(i)));
  t.i = static_cast<int>(i);
  t.s = 0;
  cur[i] = t;
  state[i] = 0;
}

// mid_i = max over {i} u N(i) of cur (aggregation.cpp:31-41).  Grid-stride over the rows (a
// persistent grid): pass 2 then reduces its decided count per CTA, one atomic per CTA.
__global__ void k_mis_pass1(const idx* __restrict__ rp, const idx* __restrict__ col, int64_t n,
                            const Tuple* cur, Tuple* mid, MisCtl* ctl) {
  const int undecided = *reinterpret_cast<volatile int*>(&ctl->undecided);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ctl->active = undecided > 0 ? 1 : 0;
    if (undecided > 0) ctl->sweeps += 1;
  }
  if (undecided == 0) return;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    Tuple best = load_tuple(cur + i);
    const idx k0 = rp[i], k1 = rp[i + 1];
#pragma unroll 8
    for (idx k = k0; k < k1; ++k) {  // unrolled: the gathers of a row issue together
      const Tuple t = load_tuple(cur + col[k]);
      if (tuple_less(best, t)) best = t;
    }
    mid[i] = best;
  }
}

// far_i = max over {i} u N(i) of mid; decide; broadcast the state (aggregation.cpp:64-79)
__global__ void __launch_bounds__(256) k_mis_pass2(const idx* __restrict__ rp, const idx* __restrict__ col,
                                                   int64_t n, const Tuple* mid, Tuple* cur,
                                                   int8_t* state, MisCtl* ctl) {
  __shared__ int s_dec[8];
  if (!ctl->active) return;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int decided = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    if (state[i] != 0) continue;
    Tuple far = load_tuple(mid + i);
    const idx k0 = rp[i], k1 = rp[i + 1];
#pragma unroll 8
    for (idx k = k0; k < k1; ++k) {
      const Tuple t = load_tuple(mid + col[k]);
      if (tuple_less(far, t)) far = t;
    }
    int8_t st = 0;
    if (far.i == static_cast<int>(i))
      st = 1;
    else if (far.s == 1)
      st = -1;
    if (st != 0) {
      state[i] = st;
      cur[i].s = st;
      ++decided;
    }
  }
  // one atomic per CTA (a same-address atomic per warp serialised 0.5 M of them per sweep)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) decided += __shfl_down_sync(0xffffffffu, decided, o);
  if ((threadIdx.x & 31) == 0) s_dec[threadIdx.x >> 5] = decided;
  __syncthreads();
  if (threadIdx.x == 0) {
    int tot = 0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) tot += s_dec[w];
    if (tot) atomicSub(&ctl->undecided, tot);
  }
}

// ---- MIS(2) late sweeps on the undecided set -----------------------------------------------
// After the first sweeps most nodes are decided, but the two full passes still visit every
// row.  far_i = max over j in {i} u N(i) of max over l in {j} u N(j) of T_l, so an undecided
// node can read its two-hop neighbourhood directly; once fewer than a quarter of the nodes are
// undecided the sweeps run over a compact list of them: decide (reading the sweep's snapshot),
// then apply and re-compact.  Same decisions, same sweep count.
struct MisList {
  int count;      // entries in the current list
  int next;       // entries appended to the next list
  int undecided;  // global undecided count (== count between sweeps)
  int sweeps;
};
__global__ void k_mis_list_init(const int8_t* state, int64_t n, idx* list, MisList* ml) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n && state[i] == 0) list[atomicAdd(&ml->count, 1)] = static_cast<idx>(i);
}
__global__ void k_mis_2hop(const idx* __restrict__ rp, const idx* __restrict__ col,
                           const Tuple* cur, const idx* list, const MisList* ml, int8_t* dec) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (ml->undecided == 0 || t >= ml->count) return;
  const idx i = list[t];
  Tuple far = load_tuple(cur + i);
  for (idx a = rp[i] - 1; a < rp[i + 1]; ++a) {  // j = i, then the neighbours
    const idx j = a < rp[i] ? i : col[a];
    const Tuple tj = load_tuple(cur + j);
    if (tuple_less(far, tj)) far = tj;
    for (idx k = rp[j]; k < rp[j + 1]; ++k) {
      const Tuple tl = load_tuple(cur + col[k]);
      if (tuple_less(far, tl)) far = tl;
    }
  }
  dec[t] = (far.i == static_cast<int>(i)) ? 1 : (far.s == 1 ? -1 : 0);
}
__global__ void k_mis_list_apply(const idx* list, MisList* ml, const int8_t* dec, Tuple* cur,
                                 int8_t* state, idx* next_list) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (ml->undecided == 0 || t >= ml->count) return;
  const idx i = list[t];
  const int8_t d = dec[t];
  if (d != 0) {
    state[i] = d;
    cur[i].s = d;
  } else {
    next_list[atomicAdd(&ml->next, 1)] = i;
  }
}
__global__ void k_mis_list_swap(MisList* ml) {
  if (ml->undecided == 0) return;
  ml->sweeps += 1;
  ml->count = ml->next;
  ml->undecided = ml->next;
  ml->next = 0;
}

// ---- a7 aggregation ------------------------------------------------------------------------
// rep[i] = representative node of i's aggregate after pass 1 (roots: themselves).
__global__ void k_agg_pass1(const idx* rp, const idx* col, int64_t n, const int8_t* state,
                            idx* rep) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  idx r = -1;
  if (state[i] == 1) {
    r = static_cast<idx>(i);
  } else {
    for (idx k = rp[i]; k < rp[i + 1]; ++k) {
      const idx j = col[k];
      if (state[j] == 1) {
        r = j;
        break;
      }
    }
  }
  rep[i] = r;
}

__device__ inline double csr_at(const idx* rp, const idx* col, const double* val, idx i, idx j) {
  idx lo = rp[i], hi = rp[i + 1];
  while (lo < hi) {  // lower_bound (sparse.cpp:15-20)
    const idx mid = lo + ((hi - lo) >> 1);
    if (col[mid] < j)
      lo = mid + 1;
    else
      hi = mid;
  }
  return (lo < rp[i + 1] && col[lo] == j) ? val[lo] : 0.0;
}

// Pass 2 against the pass-1 snapshot (aggregation.cpp:118-136); leftovers become
// their own representative (aggregation.cpp:139-144).  Comparing representative node
// ids is equivalent to comparing the reference's pre-ids, which are root ranks.
__global__ void k_agg_pass2(const idx* srp, const idx* scol, const idx* arp, const idx* acol,
                            const double* aval, int64_t n, const idx* rep, idx* rep2,
                            idx* isrep) {
  const int64_t ii = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (ii >= n) return;
  const idx i = static_cast<idx>(ii);
  idx r = rep[i];
  if (r == -1) {
    idx best = -1;
    double best_w = -1.0;
    // A(i, j) by a merge walk of the sorted rows S_i and A_i (no search per neighbour);
    // A(j, i) by a lower_bound in row j (sparse.cpp:15-20)
    idx a = arp[i];
    const idx a1 = arp[i + 1];
    for (idx k = srp[i]; k < srp[i + 1]; ++k) {
      const idx j = scol[k];
      while (a < a1 && acol[a] < j) ++a;
      const idx ja = rep[j];
      if (ja == -1) continue;
      const double aij = (a < a1 && acol[a] == j) ? aval[a] : 0.0;
      const double w = dmax_ref(fabs(aij), fabs(csr_at(arp, acol, aval, j, i)));
      if (w > best_w || (w == best_w && ja < best)) {
        best_w = w;
        best = ja;
      }
    }
    r = best == -1 ? i : best;
  }
  rep2[i] = r;
  isrep[i] = (r == i) ? 1 : 0;
}

__global__ void k_agg_assign(const idx* rep2, const idx* rank, int64_t n, idx* assignment,
                             idx* representatives) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const idx r = rep2[i];
  assignment[i] = rank[r];
  if (r == static_cast<idx>(i)) representatives[rank[i]] = static_cast<idx>(i);
}

__global__ void k_group_scatter(const idx* assignment, int64_t n, const idx* off, idx* cursor,
                                idx* rows) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const idx a = assignment[i];
  rows[off[a] + atomicAdd(&cursor[a], 1)] = static_cast<idx>(i);
}

// ---- a8 transfer ---------------------------------------------------------------------------
// sq_J = sum_{i in J ascending} b_i*b_i (transfer.cpp:21-22); also counts the nonzero rows
__global__ void k_transfer_norms(const idx* goff, const idx* rows, const double* b, int64_t nc,
                                 double* coarse_b, idx* rcnt, int* bad_agg) {
  const int64_t J = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (J >= nc) return;
  double sq = 0.0;
  idx c = 0;
  for (idx m = goff[J]; m < goff[J + 1]; ++m) {
    const double bi = b[rows[m]];
    sq = __dadd_rn(sq, __dmul_rn(bi, bi));
    c += (bi != 0.0) ? 1 : 0;
  }
  if (!(sq > 0.0)) atomicMin(bad_agg, static_cast<int>(J));
  coarse_b[J] = __dsqrt_rn(sq);
  rcnt[J] = c;
}
__global__ void k_transfer_pval(const idx* assignment, const double* b, const double* coarse_b,
                                int64_t n, double* pval) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double bi = b[i];
  pval[i] = (bi != 0.0) ? __ddiv_rn(bi, coarse_b[assignment[i]]) : 0.0;
}
// R = P^T: rows = aggregates, entries = member rows with b_i != 0, ascending.
__global__ void k_transfer_R(const idx* goff, const idx* rows, const double* pval, int64_t nc,
                             const idx* rrp, idx* rcol, double* rval) {
  const int64_t J = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (J >= nc) return;
  idx p = rrp[J];
  for (idx m = goff[J]; m < goff[J + 1]; ++m) {
    const idx i = rows[m];
    const double w = pval[i];
    if (w != 0.0) {
      rcol[p] = i;
      rval[p] = w;
      ++p;
    }
  }
}

// ---- a9/a10 Galerkin -------------------------------------------------------------------------
__global__ void k_group_entry_counts(const idx* goff, const idx* rows, const idx* arp, int64_t nc,
                                     idx* ecnt) {
  const int64_t J = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (J >= nc) return;
  idx c = 0;
  for (idx m = goff[J]; m < goff[J + 1]; ++m) {
    const idx i = rows[m];
    c += arp[i + 1] - arp[i];
  }
  ecnt[J] = c;
}

constexpr int kGalWarps = 8;
constexpr int kGalCap = 192;     // tier 1: fine entries per coarse row, one warp, shared memory (5 CTAs per SM)
constexpr int kGalCapBig = 4096; // tier 2: one CTA per coarse row, shared memory (80 KB)
constexpr int kGalCapSmem = 2048;  // tier 2 rows staged in shared memory per launch
constexpr int kGalHash = 512;    // tier 2: distinct coarse columns per row (hash table slots)

// Member-parallel gather of coarse row I's fine entries into (key, k, row) slots:
// lanes own member rows, a warp scan of the row lengths gives each member its slot
// range, so slot order = (member row ascending, storage order) = global storage order.
// Tier 1 — warp per coarse row I: gather the fine entries of I's member rows, sort them
// by coarse column J with the gather position as the tie-break (= the reference's stable
// sort by key I*nc+J, galerkin.cpp:52-62) and emit entry / entry_row / sorted J; count
// the distinct J (coarse row length).  Rows longer than kGalCap go to tier 2.
// O(L) per row, no comparison sort:
//  1. gather, entry-parallel: member starts by a warp scan of the member lengths, every lane
//     resolves its entries' member by a binary search, so the acol / assignment loads of the
//     whole row are in flight together;
//  2. distinct J in a per-warp shared hash table with their counts; the (few) distinct J
//     ranked against each other; start offsets by a warp scan in J order;
//  3. stable scatter in gather order, 32 entries at a time: __match_any_sync groups equal J,
//     an entry's slot is the J's cursor plus its rank among the equal lanes before it.
constexpr int kGalHash1 = 128;     // tier 1 hash slots per warp (distinct J per coarse row <= L)
constexpr int kGalMembers1 = 64;   // tier 1 members per coarse row (aggregates are ~10-30 rows)
__global__ void __launch_bounds__(kGalWarps * 32)
    k_gal_symbolic(const idx* goff, const idx* rows, const idx* arp, const idx* acol,
                   const idx* assignment, int64_t nc, const idx* eoff, idx* entry, idx* entry_row,
                   idx* sorted_j, idx* cnnz, idx* big_list, int* big_count) {
  __shared__ idx s_j[kGalWarps][kGalCap], s_kk[kGalWarps][kGalCap], s_ri[kGalWarps][kGalCap];
  __shared__ idx s_moff[kGalWarps][kGalMembers1], s_mlo[kGalWarps][kGalMembers1],
      s_mrow[kGalWarps][kGalMembers1];
  __shared__ idx s_hj[kGalWarps][kGalHash1], s_hc[kGalWarps][kGalHash1];
  __shared__ idx s_dj[kGalWarps][kGalHash1], s_ds[kGalWarps][kGalHash1];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned kFull = 0xffffffffu;
  const int64_t I = static_cast<int64_t>(blockIdx.x) * kGalWarps + w;
  if (I >= nc) return;
  const idx base_e = eoff[I];
  const idx L = eoff[I + 1] - base_e;
  const idx m0 = goff[I], nm = goff[I + 1] - m0;
  if (L > kGalCap || nm > kGalMembers1) {
    if (lane == 0) big_list[atomicAdd(big_count, 1)] = static_cast<idx>(I);
    return;
  }
  idx* sj = s_j[w];
  idx* skk = s_kk[w];
  idx* sri = s_ri[w];
  idx* moff = s_moff[w];
  idx* mlo = s_mlo[w];
  idx* mrow = s_mrow[w];
  idx* hj = s_hj[w];
  idx* hc = s_hc[w];
  for (int q = lane; q < kGalHash1; q += 32) {
    hj[q] = -1;
    hc[q] = 0;
  }
  // ---- 1. gather ----
  idx run = 0;
  for (idx mb = 0; mb < nm; mb += 32) {
    const idx m = mb + lane;
    idx len = 0;
    if (m < nm) {
      const idx i = rows[m0 + m];
      const idx lo = arp[i];
      len = arp[i + 1] - lo;
      mlo[m] = lo;
      mrow[m] = i;
    }
    idx incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const idx t = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += t;
    }
    if (m < nm) moff[m] = run + incl - len;
    run += __shfl_sync(kFull, incl, 31);
  }
  __syncwarp();
  // the loads of all (up to kGalCap / 32) rounds are issued together: every entry's column,
  // then every column's aggregate (two dependent round trips for the row, not two per round)
  constexpr int kRounds = kGalCap / 32;
  idx kk[kRounds], cc[kRounds];
#pragma unroll
  for (int it = 0; it < kRounds; ++it) {
    const idx p = lane + 32 * it;
    kk[it] = 0;
    if (p < L) {
      idx lo = 0, hi = nm;  // the last member whose start is <= p
      while (hi - lo > 1) {
        const idx mid = (lo + hi) >> 1;
        if (moff[mid] <= p)
          lo = mid;
        else
          hi = mid;
      }
      kk[it] = mlo[lo] + (p - moff[lo]);
      skk[p] = kk[it];
      sri[p] = mrow[lo];
    }
  }
#pragma unroll
  for (int it = 0; it < kRounds; ++it)
    if (lane + 32 * it < L) cc[it] = acol[kk[it]];
#pragma unroll
  for (int it = 0; it < kRounds; ++it)
    if (lane + 32 * it < L) sj[lane + 32 * it] = assignment[cc[it]];
  __syncwarp();
  // ---- 2. distinct J, counts, starts ----
  bool over = false;
  for (idx p = lane; p < L; p += 32) {
    const idx J = sj[p];
    unsigned h = (static_cast<unsigned>(J) * 2654435761u) & (kGalHash1 - 1);
    int probes = 0;
    while (true) {
      const idx old = atomicCAS(&hj[h], -1, J);
      if (old == -1 || old == J) break;
      h = (h + 1) & (kGalHash1 - 1);
      if (++probes == kGalHash1) break;  // more distinct J than slots
    }
    if (probes == kGalHash1)
      over = true;
    else
      atomicAdd(&hc[h], 1);
  }
  if (__any_sync(kFull, over)) {  // a coarse row of > kGalHash1 columns: tier 2
    if (lane == 0) big_list[atomicAdd(big_count, 1)] = static_cast<idx>(I);
    return;
  }
  __syncwarp();
  // compact the occupied slots (slot order), then rank each distinct J among them
  idx* dj = s_dj[w];   // distinct J in slot order
  idx* ds = s_ds[w];   // their hash slots
  idx nd = 0;
  for (int q0 = 0; q0 < kGalHash1; q0 += 32) {
    const int q = q0 + lane;
    const bool occ = hj[q] != -1;
    const unsigned bal = __ballot_sync(kFull, occ);
    if (occ) {
      const idx at = nd + __popc(bal & ((1u << lane) - 1));
      dj[at] = hj[q];
      ds[at] = q;
    }
    nd += __popc(bal);
  }
  __syncwarp();
  // start of each distinct J = sum of the counts of the smaller J (nd is small: a coarse row)
  idx start[kGalHash1 / 32];
#pragma unroll
  for (int r = 0; r < kGalHash1 / 32; ++r) {
    const idx d = lane + 32 * r;
    start[r] = 0;
    if (d < nd) {
      const idx J = dj[d];
      for (idx e = 0; e < nd; ++e) start[r] += dj[e] < J ? hc[ds[e]] : 0;
    }
  }
  __syncwarp();
#pragma unroll
  for (int r = 0; r < kGalHash1 / 32; ++r)  // counts -> cursors
    if (lane + 32 * r < nd) hc[ds[lane + 32 * r]] = start[r];
  __syncwarp();
  // ---- 3. stable scatter in gather order ----
  for (idx pb = 0; pb < L; pb += 32) {
    const idx p = pb + lane;
    const bool act = p < L;
    const idx J = act ? sj[p] : -1 - lane;  // inactive lanes never match a real J
    unsigned h = (static_cast<unsigned>(J) * 2654435761u) & (kGalHash1 - 1);
    if (act)
      while (hj[h] != J) h = (h + 1) & (kGalHash1 - 1);
    const unsigned peers = __match_any_sync(kFull, J);
    const idx cur = act ? hc[h] : 0;
    const idx slot = cur + __popc(peers & ((1u << lane) - 1));
    if (act) {
      entry[base_e + slot] = skk[p];
      entry_row[base_e + slot] = sri[p];
      sorted_j[base_e + slot] = J;
    }
    __syncwarp();
    if (act && lane == __ffs(peers) - 1) hc[h] = cur + __popc(peers);
    __syncwarp();
  }
  if (lane == 0) cnnz[I] = nd;
}

// Tier 1 without a length cap — warp per coarse row I, nothing per entry kept in shared
// memory: pass A gathers J = assignment[acol[k]] for the row's entries (4 x 32 in flight per
// lane group) and counts the distinct J in a per-warp hash table; the distinct J are ranked
// into start offsets; pass B re-gathers the same entries (L1 / L2 hits) in gather order and
// scatters them stably (match_any rank + the J's cursor).  The same output as k_gal_symbolic
// for any L; rows with more than kGalMembersW members or kGalHashW / 2 distinct J go to tier 2.
constexpr int kGalMembersW = 128;
constexpr int kGalHashW = 256;
constexpr int kGalU = 4;  // 32-entry groups whose loads are issued together
__device__ __forceinline__ idx gal_member_of(const idx* moff, idx nm, idx p) {
  idx lo = 0, hi = nm;  // the last member whose start is <= p
  while (hi - lo > 1) {
    const idx mid = (lo + hi) >> 1;
    if (moff[mid] <= p)
      lo = mid;
    else
      hi = mid;
  }
  return lo;
}
__global__ void __launch_bounds__(kGalWarps * 32)
    k_gal_symbolic_w(const idx* goff, const idx* rows, const idx* arp, const idx* acol,
                     const idx* assignment, int64_t nc, const idx* eoff, idx* entry, idx* entry_row,
                     idx* sorted_j, idx* cnnz, idx* big_list, int* big_count) {
  __shared__ idx s_moff[kGalWarps][kGalMembersW + 1], s_mlo[kGalWarps][kGalMembersW],
      s_mrow[kGalWarps][kGalMembersW];
  __shared__ idx s_hj[kGalWarps][kGalHashW], s_hc[kGalWarps][kGalHashW];
  __shared__ idx s_ds[kGalWarps][kGalHashW / 2];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned kFull = 0xffffffffu;
  const int64_t I = static_cast<int64_t>(blockIdx.x) * kGalWarps + w;
  if (I >= nc) return;
  const idx base_e = eoff[I];
  const idx L = eoff[I + 1] - base_e;
  const idx m0 = goff[I], nm = goff[I + 1] - m0;
  if (nm > kGalMembersW) {
    if (lane == 0) big_list[atomicAdd(big_count, 1)] = static_cast<idx>(I);
    return;
  }
  idx* moff = s_moff[w];
  idx* mlo = s_mlo[w];
  idx* mrow = s_mrow[w];
  idx* hj = s_hj[w];
  idx* hc = s_hc[w];
  for (int q = lane; q < kGalHashW; q += 32) {
    hj[q] = -1;
    hc[q] = 0;
  }
  idx run = 0;
  for (idx mb = 0; mb < nm; mb += 32) {
    const idx m = mb + lane;
    idx len = 0;
    if (m < nm) {
      const idx i = rows[m0 + m];
      const idx lo = arp[i];
      len = arp[i + 1] - lo;
      mlo[m] = lo;
      mrow[m] = i;
    }
    idx incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const idx t = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += t;
    }
    if (m < nm) moff[m] = run + incl - len;
    run += __shfl_sync(kFull, incl, 31);
  }
  __syncwarp();
  // ---- A. distinct J and their counts ----
  bool over = false;
  for (idx pb = 0; pb < L; pb += 32 * kGalU) {
    idx J[kGalU];
#pragma unroll
    for (int u = 0; u < kGalU; ++u) {
      const idx p = pb + 32 * u + lane;
      J[u] = -1;
      if (p < L) {
        const idx m = gal_member_of(moff, nm, p);
        J[u] = acol[mlo[m] + (p - moff[m])];
      }
    }
#pragma unroll
    for (int u = 0; u < kGalU; ++u)
      if (J[u] >= 0) J[u] = assignment[J[u]];
#pragma unroll
    for (int u = 0; u < kGalU; ++u) {
      const idx Jv = pb + 32 * u + lane < L ? J[u] : -2 - lane;  // inactive lanes: unique keys
      const unsigned peers = __match_any_sync(kFull, Jv);
      if (Jv >= 0 && lane == __ffs(peers) - 1) {
        unsigned h = (static_cast<unsigned>(Jv) * 2654435761u) & (kGalHashW - 1);
        int probes = 0;
        while (true) {
          const idx old = atomicCAS(&hj[h], -1, Jv);
          if (old == -1 || old == Jv) break;
          h = (h + 1) & (kGalHashW - 1);
          if (++probes == kGalHashW) break;
        }
        if (probes == kGalHashW)
          over = true;
        else
          atomicAdd(&hc[h], static_cast<idx>(__popc(peers)));
      }
    }
  }
  __syncwarp();
  // the occupied slots, compacted (at most kGalHashW / 2 distinct J: the load factor)
  idx nd = 0;
  idx* ds = s_ds[w];
  for (int q0 = 0; q0 < kGalHashW; q0 += 32) {
    const bool occ = hj[q0 + lane] != -1;
    const unsigned bal = __ballot_sync(kFull, occ);
    const idx at = nd + __popc(bal & ((1u << lane) - 1));
    if (occ && at < kGalHashW / 2) ds[at] = q0 + lane;
    nd += __popc(bal);
  }
  if (__any_sync(kFull, over) || nd > kGalHashW / 2) {
    if (lane == 0) big_list[atomicAdd(big_count, 1)] = static_cast<idx>(I);
    return;
  }
  __syncwarp();
  // start of each distinct J = sum of the counts of the smaller J
  idx start[kGalHashW / 64];
#pragma unroll
  for (int r = 0; r < kGalHashW / 64; ++r) {
    const idx d = lane + 32 * r;
    start[r] = 0;
    if (d < nd) {
      const idx J = hj[ds[d]];
      for (idx e = 0; e < nd; ++e) {
        const idx se = ds[e];
        start[r] += hj[se] < J ? hc[se] : 0;
      }
    }
  }
  __syncwarp();
#pragma unroll
  for (int r = 0; r < kGalHashW / 64; ++r)  // counts -> cursors
    if (lane + 32 * r < nd) hc[ds[lane + 32 * r]] = start[r];
  __syncwarp();
  // ---- B. stable scatter in gather order ----
  for (idx pb = 0; pb < L; pb += 32 * kGalU) {
    idx K[kGalU], R[kGalU], J[kGalU];
#pragma unroll
    for (int u = 0; u < kGalU; ++u) {
      const idx p = pb + 32 * u + lane;
      K[u] = -1;
      R[u] = 0;
      if (p < L) {
        const idx m = gal_member_of(moff, nm, p);
        K[u] = mlo[m] + (p - moff[m]);
        R[u] = mrow[m];
      }
    }
#pragma unroll
    for (int u = 0; u < kGalU; ++u) J[u] = K[u] >= 0 ? acol[K[u]] : -1;
#pragma unroll
    for (int u = 0; u < kGalU; ++u)
      if (K[u] >= 0) J[u] = assignment[J[u]];
#pragma unroll
    for (int u = 0; u < kGalU; ++u) {
      if (pb + 32 * u >= L) break;  // warp-uniform
      const bool act = K[u] >= 0;
      const idx Jv = act ? J[u] : -2 - lane;
      unsigned h = (static_cast<unsigned>(Jv) * 2654435761u) & (kGalHashW - 1);
      if (act)
        while (hj[h] != Jv) h = (h + 1) & (kGalHashW - 1);
      const unsigned peers = __match_any_sync(kFull, Jv);
      const idx cur = act ? hc[h] : 0;
      const idx slot = cur + __popc(peers & ((1u << lane) - 1));
      if (act) {
        entry[base_e + slot] = K[u];
        entry_row[base_e + slot] = R[u];
        sorted_j[base_e + slot] = Jv;
      }
      __syncwarp();
      if (act && lane == __ffs(peers) - 1) hc[h] = cur + __popc(peers);
      __syncwarp();
    }
  }
  if (lane == 0) cnnz[I] = nd;
}

// Lean cache (a hierarchy's own setup): only what the numeric reduce and refresh_values read —
// coarse pattern and slot_of_csr — without the per-entry sorted arrays (entry, entry_row,
// segment_offsets: the standalone cache API builds those).  Two warp-per-coarse-row passes:
//  count: the distinct J of the row, sorted (rank = number of smaller J), into the row's
//         scratch range and its length into cnnz;
//  fill:  after the scan, the coarse columns and every fine entry's slot (crp[I] + rank of J).
// A row with more than kGalMembersW members or kLeanSlots distinct J sets *bad (the full path
// then runs instead).
constexpr int kLeanSlots = 64;   // = the row-walk numeric reduce's slots
constexpr int kLeanHash = 128;
__device__ __forceinline__ void gal_members(const idx* goff, const idx* rows, const idx* arp, int64_t I,
                                            int lane, idx* moff, idx* mlo, idx& nm_out,
                                            const double* pv = nullptr, double* mpv = nullptr) {
  const idx m0 = goff[I], nm = goff[I + 1] - m0;
  idx run = 0;
  for (idx mb = 0; mb < nm; mb += 32) {
    const idx m = mb + lane;
    idx len = 0;
    if (m < nm) {
      const idx i = rows[m0 + m];
      const idx lo = arp[i];
      len = arp[i + 1] - lo;
      mlo[m] = lo;
      if (mpv) mpv[m] = pv[i];
    }
    idx incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const idx t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    if (m < nm) moff[m] = run + incl - len;
    run += __shfl_sync(0xffffffffu, incl, 31);
  }
  nm_out = nm;
  __syncwarp();
}

__global__ void __launch_bounds__(kGalWarps * 32)
    k_gal_lean_count(const idx* goff, const idx* rows, const idx* arp, const idx* acol,
                     const idx* assignment, int64_t nc, const idx* eoff, idx* tmpj, idx* cnnz, int* bad) {
  __shared__ idx s_moff[kGalWarps][kGalMembersW], s_mlo[kGalWarps][kGalMembersW];
  __shared__ idx s_hj[kGalWarps][kLeanHash], s_dj[kGalWarps][kLeanSlots];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned kFull = 0xffffffffu;
  const int64_t I = static_cast<int64_t>(blockIdx.x) * kGalWarps + w;
  if (I >= nc) return;
  if (goff[I + 1] - goff[I] > kGalMembersW) {
    if (lane == 0) *bad = 1;
    return;
  }
  const idx base_e = eoff[I], L = eoff[I + 1] - base_e;
  idx* moff = s_moff[w];
  idx* mlo = s_mlo[w];
  idx* hj = s_hj[w];
  for (int q = lane; q < kLeanHash; q += 32) hj[q] = -1;
  idx nm;
  gal_members(goff, rows, arp, I, lane, moff, mlo, nm);
  bool over = false;
  for (idx pb = 0; pb < L; pb += 32 * kGalU) {
    idx J[kGalU];
#pragma unroll
    for (int u = 0; u < kGalU; ++u) {
      const idx p = pb + 32 * u + lane;
      J[u] = -1;
      if (p < L) {
        const idx m = gal_member_of(moff, nm, p);
        J[u] = acol[mlo[m] + (p - moff[m])];
      }
    }
#pragma unroll
    for (int u = 0; u < kGalU; ++u)
      if (J[u] >= 0) J[u] = assignment[J[u]];
#pragma unroll
    for (int u = 0; u < kGalU; ++u) {
      const idx Jv = pb + 32 * u + lane < L ? J[u] : -2 - lane;
      const unsigned peers = __match_any_sync(kFull, Jv);
      if (Jv >= 0 && lane == __ffs(peers) - 1) {
        unsigned h = (static_cast<unsigned>(Jv) * 2654435761u) & (kLeanHash - 1);
        int probes = 0;
        while (true) {
          const idx old = atomicCAS(&hj[h], -1, Jv);
          if (old == -1 || old == Jv) break;
          h = (h + 1) & (kLeanHash - 1);
          if (++probes == kLeanHash) {
            over = true;
            break;
          }
        }
      }
    }
  }
  __syncwarp();
  // the distinct J compacted; rank = number of smaller distinct J
  idx* dj = s_dj[w];
  idx nd = 0;
#pragma unroll
  for (int r = 0; r < kLeanHash / 32; ++r) {
    const idx J = hj[lane + 32 * r];
    const unsigned bal = __ballot_sync(kFull, J != -1);
    const idx at = nd + __popc(bal & ((1u << lane) - 1));
    if (J != -1 && at < kLeanSlots) dj[at] = J;
    nd += __popc(bal);
  }
  if (__any_sync(kFull, over) || nd > kLeanSlots) {
    if (lane == 0) *bad = 1;
    return;
  }
  __syncwarp();
  for (idx d = lane; d < nd; d += 32) {
    const idx J = dj[d];
    idx rank = 0;
    for (idx e = 0; e < nd; ++e) rank += dj[e] < J ? 1 : 0;
    tmpj[base_e + rank] = J;
  }
  if (lane == 0) cnnz[I] = nd;
}

__global__ void __launch_bounds__(kGalWarps * 32)
    k_gal_lean_fill(const idx* goff, const idx* rows, const idx* arp, const idx* acol,
                    const idx* assignment, int64_t nc, const idx* eoff, const idx* tmpj, const idx* crp,
                    idx* ccol, idx* slot_of_csr, const double* aval, const double* pv, double* out) {
  // with pv / out: also Ac = the row-walk numeric reduce (k_gal_numeric_walk's sums: products
  // added into their slot in gather order, equal-slot lanes of a round lowest lane first)
  __shared__ idx s_moff[kGalWarps][kGalMembersW], s_mlo[kGalWarps][kGalMembersW];
  __shared__ idx s_hj[kGalWarps][kLeanHash], s_hr[kGalWarps][kLeanHash];
  __shared__ double s_mpv[kGalWarps][kGalMembersW], s_acc[kGalWarps][kLeanSlots];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t I = static_cast<int64_t>(blockIdx.x) * kGalWarps + w;
  if (I >= nc) return;
  const idx base_e = eoff[I], L = eoff[I + 1] - base_e;
  const idx c0 = crp[I], nd = crp[I + 1] - c0;
  idx* moff = s_moff[w];
  idx* mlo = s_mlo[w];
  idx* hj = s_hj[w];
  idx* hr = s_hr[w];
  for (int q = lane; q < kLeanHash; q += 32) hj[q] = -1;
  __syncwarp();
  for (idx r = lane; r < nd; r += 32) {  // J -> rank (distinct J: plain inserts)
    const idx J = tmpj[base_e + r];
    ccol[c0 + r] = J;
    unsigned h = (static_cast<unsigned>(J) * 2654435761u) & (kLeanHash - 1);
    while (atomicCAS(&hj[h], -1, J) != -1) h = (h + 1) & (kLeanHash - 1);
    hr[h] = r;
  }
  const bool num = out != nullptr;
  double* mpv = s_mpv[w];
  double* acc = s_acc[w];
  if (num)
    for (int q = lane; q < kLeanSlots; q += 32) acc[q] = 0.0;
  idx nm;
  gal_members(goff, rows, arp, I, lane, moff, mlo, nm, pv, num ? mpv : nullptr);
  for (idx pb = 0; pb < L; pb += 32 * kGalU) {
    idx K[kGalU], J[kGalU], C[kGalU];
    double pm[kGalU];
#pragma unroll
    for (int u = 0; u < kGalU; ++u) {
      const idx p = pb + 32 * u + lane;
      K[u] = -1;
      pm[u] = 0.0;
      if (p < L) {
        const idx m = gal_member_of(moff, nm, p);
        K[u] = mlo[m] + (p - moff[m]);
        if (num) pm[u] = mpv[m];
      }
    }
#pragma unroll
    for (int u = 0; u < kGalU; ++u) C[u] = K[u] >= 0 ? acol[K[u]] : 0;
    double c[kGalU];
#pragma unroll
    for (int u = 0; u < kGalU; ++u) {
      J[u] = K[u] >= 0 ? assignment[C[u]] : 0;
      c[u] = (num && K[u] >= 0) ? __dmul_rn(__dmul_rn(pm[u], aval[K[u]]), pv[C[u]]) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < kGalU; ++u) {
      if (pb + 32 * u >= L) break;  // warp-uniform
      int r = -1 - lane;
      if (K[u] >= 0) {
        unsigned h = (static_cast<unsigned>(J[u]) * 2654435761u) & (kLeanHash - 1);
        while (hj[h] != J[u]) h = (h + 1) & (kLeanHash - 1);
        r = hr[h];
        slot_of_csr[K[u]] = c0 + r;
      }
      if (num) {
        const unsigned grp = __match_any_sync(0xffffffffu, r);
        const int rk = __popc(grp & ((1u << lane) - 1u));
        int mx = rk;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        for (int step = 0; step <= mx; ++step) {
          if (K[u] >= 0 && rk == step) acc[r] = __dadd_rn(acc[r], c[u]);
          __syncwarp();
        }
      }
    }
  }
  if (num) {
    __syncwarp();
    for (idx t = lane; t < nd; t += 32) out[c0 + t] = acc[t];
  }
}

// Tier 2 — one CTA (256 threads) per long coarse row (L > kGalCap gathered entries).
// Per-entry slots (J, k, row, hash slot, scratch) live in shared memory when L <= cap (the
// launch's largest L, at most kGalCapBig), else in global scratch at [base_e, base_e + L).
//  1. gather: entry-parallel over a member table (offsets by warp scan), so all 256 threads
//     load acol / assignment;
//  2. distinct coarse columns J in a shared hash table with per-J counts; ranks of the
//     distinct J; offsets by a warp scan;
//  3. one warp scatters the entries in gather order (match_any groups equal J, the group
//     leader advances the J's cursor) — the stable sort by (J, position) of
//     galerkin.cpp:52-62, in O(L).
// Fallback (hash overflow or more than kGalMembers members): the O(L^2) rank sort.
constexpr int kGalMembers = 512;
__global__ void __launch_bounds__(256)
    k_gal_symbolic_big(const idx* big_list, const idx* goff, const idx* rows, const idx* arp,
                       const idx* acol, const idx* assignment, const idx* eoff, int cap,
                       const int64_t* goff_big, idx* gscratch, idx* entry, idx* entry_row,
                       idx* sorted_j, idx* cnnz) {
  extern __shared__ idx big_smem[];
  __shared__ idx m_off[kGalMembers + 1], m_lo[kGalMembers], m_row[kGalMembers];
  __shared__ idx h_j[kGalHash], h_cnt[kGalHash], h_cur[kGalHash], d_slot[kGalHash];
  __shared__ idx w_cnt[8][kGalHash];  // per-warp counts, then cursors, of every J (step 3)
  __shared__ idx s_wsum[32];
  __shared__ int s_nd, s_over;
  const idx I = big_list[blockIdx.x];
  const idx base_e = eoff[I];
  const idx L = eoff[I + 1] - base_e;
  const bool in_smem = L <= cap;
  idx* base = in_smem ? big_smem : gscratch + 5 * goff_big[blockIdx.x];
  const idx stride = in_smem ? cap : L;
  idx* sJ = base;
  idx* skk = base + stride;
  idx* sri = base + 2 * stride;
  idx* sslot = base + 3 * stride;
  idx* stmp = base + 4 * stride;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const idx m0 = goff[I], m1 = goff[I + 1], nm = m1 - m0;

  // ---- 1. gather (gather position p = member ascending, storage order) ----
  if (nm <= kGalMembers) {
    for (idx m = threadIdx.x; m < nm; m += blockDim.x) {
      const idx i = rows[m0 + m];
      m_lo[m] = arp[i];
      m_row[m] = i;
      m_off[m + 1] = arp[i + 1] - arp[i];
    }
    __syncthreads();
    if (warp == 0) {  // exclusive scan of the member lengths: lane owns a contiguous run
      const idx per = (nm + 31) / 32;
      const idx b0 = lane * per, b1 = min(nm, b0 + per);
      idx loc = 0;
      for (idx m = b0; m < b1; ++m) loc += m_off[m + 1];
      idx incl = loc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const idx t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      idx run = incl - loc;
      for (idx m = b0; m < b1; ++m) {
        const idx len = m_off[m + 1];
        m_off[m] = run;  // m_off[m] becomes the start (m_off[m + 1] is read before written)
        run += len;
      }
      __syncwarp();
      if (lane == 31) m_off[nm] = incl;
    }
    __syncthreads();
    for (idx p = threadIdx.x; p < L; p += blockDim.x) {
      idx lo = 0, hi = nm;  // last member with m_off[m] <= p
      while (hi - lo > 1) {
        const idx mid = (lo + hi) >> 1;
        if (m_off[mid] <= p)
          lo = mid;
        else
          hi = mid;
      }
      const idx k = m_lo[lo] + (p - m_off[lo]);
      sJ[p] = assignment[acol[k]];
      skk[p] = k;
      sri[p] = m_row[lo];
    }
  } else {  // many members: member-parallel gather, block scan per batch
    __shared__ idx s_base;
    if (threadIdx.x == 0) s_base = 0;
    __syncthreads();
    for (idx mb = m0; mb < m1; mb += blockDim.x) {
      const idx m = mb + threadIdx.x;
      idx i = 0, lo = 0, len = 0;
      if (m < m1) {
        i = rows[m];
        lo = arp[i];
        len = arp[i + 1] - lo;
      }
      idx incl = len;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const idx t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      if (lane == 31) s_wsum[warp] = incl;
      __syncthreads();
      idx wbase = 0;
      for (int q = 0; q < warp; ++q) wbase += s_wsum[q];
      const idx off = s_base + wbase + incl - len;
      for (idx t = 0; t < len; ++t) {
        const idx k = lo + t, p = off + t;
        sJ[p] = assignment[acol[k]];
        skk[p] = k;
        sri[p] = i;
      }
      __syncthreads();
      if (threadIdx.x == 0) {
        idx tot = 0;
        for (int q = 0; q < 8; ++q) tot += s_wsum[q];
        s_base += tot;
      }
      __syncthreads();
    }
  }

  // ---- 2. distinct J and their counts ----
  for (int q = threadIdx.x; q < kGalHash; q += blockDim.x) {
    h_j[q] = -1;
    h_cnt[q] = 0;
  }
  if (threadIdx.x == 0) {
    s_nd = 0;
    s_over = 0;
  }
  __syncthreads();
  for (idx p = threadIdx.x; p < L; p += blockDim.x) {
    const idx J = sJ[p];
    unsigned h = (static_cast<unsigned>(J) * 2654435761u) & (kGalHash - 1);
    int probes = 0;
    while (true) {
      const idx old = atomicCAS(&h_j[h], -1, J);
      if (old == -1 || old == J) break;
      h = (h + 1) & (kGalHash - 1);
      if (++probes >= kGalHash) break;
    }
    if (probes >= kGalHash) {
      s_over = 1;
    } else {
      atomicAdd(&h_cnt[h], 1);
      sslot[p] = static_cast<idx>(h);
    }
  }
  __syncthreads();
  if (s_over) {  // fallback: rank sort by (J, p)
    for (idx q = threadIdx.x; q < L; q += blockDim.x) {
      const idx Jq = sJ[q];
      idx rank = 0;
      for (idx z = 0; z < L; ++z) {
        const idx Jz = sJ[z];
        rank += (Jz < Jq || (Jz == Jq && z < q)) ? 1 : 0;
      }
      entry[base_e + rank] = skk[q];
      entry_row[base_e + rank] = sri[q];
      sorted_j[base_e + rank] = Jq;
    }
    __syncthreads();
    idx c = 0;
    for (idx r = threadIdx.x; r < L; r += blockDim.x)
      c += (r == 0 || sorted_j[base_e + r] != sorted_j[base_e + r - 1]) ? 1 : 0;
    for (int o = 16; o > 0; o >>= 1) c += __shfl_down_sync(0xffffffffu, c, o);
    if (lane == 0) s_wsum[warp] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
      idx t = 0;
      for (int q = 0; q < 8; ++q) t += s_wsum[q];
      cnnz[I] = t;
    }
    return;
  }
  for (int q = threadIdx.x; q < kGalHash; q += blockDim.x)
    if (h_j[q] != -1) d_slot[atomicAdd(&s_nd, 1)] = q;
  __syncthreads();
  const int nd = s_nd;
  // rank of every distinct J (ascending): h_cur[rank] = slot
  for (int q = threadIdx.x; q < nd; q += blockDim.x) {
    const idx J = h_j[d_slot[q]];
    int r = 0;
    for (int z = 0; z < nd; ++z) r += (h_j[d_slot[z]] < J) ? 1 : 0;
    h_cur[r] = d_slot[q];
  }
  __syncthreads();
  if (warp == 0) {  // offsets in rank order -> d_slot[rank] = start; h_cnt[slot] = start
    const int per = (nd + 31) / 32;
    const int b0 = lane * per, b1 = min(nd, b0 + per);
    idx loc = 0;
    for (int r = b0; r < b1; ++r) loc += h_cnt[h_cur[r]];
    idx incl = loc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const idx t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    idx run = incl - loc;
    for (int r = b0; r < b1; ++r) {
      const idx sl = h_cur[r];
      const idx cnt = h_cnt[sl];
      d_slot[r] = run;  // start of run r
      h_cnt[sl] = run;  // cursor of slot sl
      run += cnt;
    }
  }
  __syncthreads();
  // ---- 3. stable scatter, all warps: warp w owns the w-th contiguous chunk of the gather
  //         order; per-warp counts per J, then per-warp bases (J's start + the counts of the
  //         earlier chunks), then each warp walks its chunk in order — lanes with the same J
  //         take consecutive positions (match_any), the group leader advances the cursor ----
  constexpr int kW = 8;
  const idx chunk = ((L + kW - 1) / kW + 31) & ~31;
  const idx c0 = warp * chunk, c1 = min(L, c0 + chunk);
  for (int q = threadIdx.x; q < kW * kGalHash; q += blockDim.x) (&w_cnt[0][0])[q] = 0;
  __syncthreads();
  for (idx c = c0; c < c1; c += 32) {
    const idx p = c + lane;
    const bool ok = p < c1;
    const idx sl = ok ? sslot[p] : -1 - lane;
    const unsigned grp = __match_any_sync(0xffffffffu, sl);
    if (ok && __popc(grp & ((1u << lane) - 1u)) == 0) w_cnt[warp][sl] += __popc(grp);
    __syncwarp();
  }
  __syncthreads();
  for (int q = threadIdx.x; q < kGalHash; q += blockDim.x) {
    if (h_j[q] == -1) continue;
    idx run = h_cnt[q];
    for (int w = 0; w < kW; ++w) {
      const idx t = w_cnt[w][q];
      w_cnt[w][q] = run;
      run += t;
    }
  }
  __syncthreads();
  for (idx c = c0; c < c1; c += 32) {
    const idx p = c + lane;
    const bool ok = p < c1;
    const idx sl = ok ? sslot[p] : -1 - lane;
    const unsigned grp = __match_any_sync(0xffffffffu, sl);
    const int rk = __popc(grp & ((1u << lane) - 1u));
    idx pos = 0;
    if (ok) pos = w_cnt[warp][sl] + rk;
    __syncwarp();
    if (ok && rk == 0) w_cnt[warp][sl] += __popc(grp);
    if (ok) stmp[pos] = p;
    __syncwarp();
  }
  __syncthreads();
  for (idx q = threadIdx.x; q < L; q += blockDim.x) {
    const idx p = stmp[q];
    entry[base_e + q] = skk[p];
    entry_row[base_e + q] = sri[p];
    sorted_j[base_e + q] = sJ[p];
  }
  if (threadIdx.x == 0) cnnz[I] = nd;
}

// scratch offsets of the rows that do not fit in shared memory (exclusive scan input)
__global__ void k_big_scratch_len(const idx* big_list, int nbig, const idx* eoff, int cap,
                                  int64_t* len) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= nbig) return;
  const idx I = big_list[t];
  const idx L = eoff[I + 1] - eoff[I];
  len[t] = L > cap ? L : 0;
}

__global__ void k_max_big_len(const idx* big_list, int nbig, const idx* eoff, int* out) {
  int m = 0;
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nbig; t += gridDim.x * blockDim.x) {
    const idx I = big_list[t];
    m = max(m, eoff[I + 1] - eoff[I]);
  }
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_down_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// ---- galerkin_direct: R*(A*P) in the reference spmm order (galerkin.cpp:33-36) ----------
//
// spmm(R, A) accumulates, for coarse row I, RA_Ij = sum over members i of I (ascending,
// P row non-empty) of p_i * a_ij, starting from 0 (sparse.cpp:102-120); spmm(RA, P) then
// accumulates Ac_IJ = sum over j ascending (P row j non-empty, agg(j) = J) of RA_Ij * p_j.
// Per coarse row we gather (key = J<<32 | j, value = p_i * a_ij) in member/storage order,
// rank-sort by key with the gather position as tie-break, and walk the sorted run
// sequentially — the exact association and order of the two CPU products.

// One coarse row's walk over sorted (key, value) arrays; writes (or counts) Ac entries.
__device__ inline idx gal_direct_walk(const unsigned long long* skey, const double* sval, idx L,
                                      const double* pval, idx* ccol, double* cval) {
  idx out = 0;
  idx p = 0;
  while (p < L) {
    const idx J = static_cast<idx>(skey[p] >> 32);
    double acc = 0.0;
    while (p < L && static_cast<idx>(skey[p] >> 32) == J) {
      const idx j = static_cast<idx>(skey[p] & 0xffffffffull);
      double raij = 0.0;
      while (p < L && skey[p] == ((static_cast<unsigned long long>(J) << 32) | static_cast<unsigned>(j))) {
        raij = __dadd_rn(raij, sval[p]);
        ++p;
      }
      acc = __dadd_rn(acc, __dmul_rn(raij, pval[j]));
    }
    if (ccol) {
      ccol[out] = J;
      cval[out] = acc;
    }
    ++out;
  }
  return out;
}

// mode 0: count coarse row lengths into cnnz; mode 1: fill at crp.  Warp per coarse row,
// rows with more than kGalCap gathered entries are deferred to the CTA kernel.
constexpr int kGalDirectWarps = 4;  // 4 warps x 256 x 32 B = 32 KB static smem
__global__ void __launch_bounds__(kGalDirectWarps * 32)
    k_gal_direct(const idx* goff, const idx* rows, const idx* arp, const idx* acol,
                 const double* aval, const idx* assignment, const double* pval, int64_t nc,
                 const idx* eoff, int mode, idx* cnnz, const idx* crp, idx* ccol, double* cval,
                 idx* big_list, int* big_count) {
  __shared__ unsigned long long s_key[kGalDirectWarps][kGalCap], s_skey[kGalDirectWarps][kGalCap];
  __shared__ double s_val[kGalDirectWarps][kGalCap], s_sval[kGalDirectWarps][kGalCap];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t I = static_cast<int64_t>(blockIdx.x) * kGalDirectWarps + w;
  if (I >= nc) return;
  if (eoff[I + 1] - eoff[I] > kGalCap) {
    if (lane == 0) big_list[atomicAdd(big_count, 1)] = static_cast<idx>(I);
    return;
  }
  // gather in (member ascending, storage order), skipping empty P rows on either side
  idx L = 0;
  for (idx m = goff[I]; m < goff[I + 1]; ++m) {
    const idx i = rows[m];
    const double pi = pval[i];
    if (pi == 0.0) continue;
    for (idx k0 = arp[i]; k0 < arp[i + 1]; k0 += 32) {
      const idx k = k0 + lane;
      bool keep = false;
      unsigned long long key = 0;
      double v = 0.0;
      if (k < arp[i + 1]) {
        const idx j = acol[k];
        if (pval[j] != 0.0) {
          keep = true;
          key = (static_cast<unsigned long long>(assignment[j]) << 32) | static_cast<unsigned>(j);
          v = __dmul_rn(pi, aval[k]);
        }
      }
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      if (keep) {
        const idx pos = L + __popc(bal & ((1u << lane) - 1u));
        s_key[w][pos] = key;
        s_val[w][pos] = v;
      }
      L += __popc(bal);
    }
  }
  __syncwarp();
  for (idx q = lane; q < L; q += 32) {  // stable rank: key, then gather position
    const unsigned long long key = s_key[w][q];
    idx rank = 0;
    for (idx z = 0; z < L; ++z) {
      const unsigned long long kz = s_key[w][z];
      rank += (kz < key || (kz == key && z < q)) ? 1 : 0;
    }
    s_skey[w][rank] = key;
    s_sval[w][rank] = s_val[w][q];
  }
  __syncwarp();
  if (lane == 0) {
    if (mode == 0)
      cnnz[I] = gal_direct_walk(s_skey[w], s_sval[w], L, pval, nullptr, nullptr);
    else
      gal_direct_walk(s_skey[w], s_sval[w], L, pval, ccol + crp[I], cval + crp[I]);
  }
}

// CTA per long coarse row, (key, value) staged in global scratch at [eoff[I], eoff[I+1]).
__global__ void __launch_bounds__(256)
    k_gal_direct_big(const idx* big_list, const idx* goff, const idx* rows, const idx* arp,
                     const idx* acol, const double* aval, const idx* assignment,
                     const double* pval, const idx* eoff, int mode, unsigned long long* gkey,
                     double* gval, unsigned long long* gskey, double* gsval, idx* cnnz,
                     const idx* crp, idx* ccol, double* cval) {
  __shared__ idx s_L;
  const idx I = big_list[blockIdx.x];
  const idx base = eoff[I];
  unsigned long long* key = gkey + base;
  double* val = gval + base;
  unsigned long long* skey = gskey + base;
  double* sval = gsval + base;
  if (threadIdx.x == 0) {  // sequential gather keeps member/storage order trivially
    idx L = 0;
    for (idx m = goff[I]; m < goff[I + 1]; ++m) {
      const idx i = rows[m];
      const double pi = pval[i];
      if (pi == 0.0) continue;
      for (idx k = arp[i]; k < arp[i + 1]; ++k) {
        const idx j = acol[k];
        if (pval[j] == 0.0) continue;
        key[L] = (static_cast<unsigned long long>(assignment[j]) << 32) | static_cast<unsigned>(j);
        val[L] = __dmul_rn(pi, aval[k]);
        ++L;
      }
    }
    s_L = L;
  }
  __syncthreads();
  const idx L = s_L;
  for (idx q = threadIdx.x; q < L; q += blockDim.x) {
    const unsigned long long kq = key[q];
    idx rank = 0;
    for (idx z = 0; z < L; ++z) rank += (key[z] < kq || (key[z] == kq && z < q)) ? 1 : 0;
    skey[rank] = kq;
    sval[rank] = val[q];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (mode == 0)
      cnnz[I] = gal_direct_walk(skey, sval, L, pval, nullptr, nullptr);
    else
      gal_direct_walk(skey, sval, L, pval, ccol + crp[I], cval + crp[I]);
  }
}

// Warp per coarse row: segment boundaries -> coarse columns, segment offsets, slot_of_csr.
__global__ void k_gal_fill(int64_t nc, const idx* eoff, const idx* sorted_j, const idx* entry,
                           const idx* crp, idx* ccol, idx* seg_off, idx* slot_of_csr) {
  const int64_t I = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (I >= nc) return;
  const idx base_e = eoff[I], L = eoff[I + 1] - base_e;
  idx carry = crp[I] - 1;
  for (idx b = 0; b < L; b += 32) {
    const idx r = b + lane;
    idx jc = 0;
    bool st = false;
    if (r < L) {
      jc = sorted_j[base_e + r];
      st = (r == 0) || jc != sorted_j[base_e + r - 1];
    }
    const unsigned bal = __ballot_sync(0xffffffffu, st);
    const idx seg = carry + __popc(bal & ((2u << lane) - 1u));
    if (r < L) {
      if (st) {
        ccol[seg] = jc;
        seg_off[seg] = base_e + r;
      }
      slot_of_csr[entry[base_e + r]] = seg;
    }
    carry += __popc(bal);
  }
}

// Ac[s] = sum over the segment, in stored order, of (pv[row] * a_e) * pv[col_e]
// (galerkin.cpp:128-135).
__global__ void k_gal_numeric(int64_t nnz_c, const idx* seg_off, const idx* entry,
                              const idx* entry_row, const idx* acol, const double* aval,
                              const double* pv, double* out) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= nnz_c) return;
  double acc = 0.0;
  for (idx p = seg_off[s]; p < seg_off[s + 1]; ++p) {
    const idx e = entry[p];
    acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(pv[entry_row[p]], aval[e]), pv[acol[e]]));
  }
  out[s] = acc;
}

__global__ void k_max_rowlen(const idx* rp, int64_t n, int* out) {
  int m = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    m = max(m, rp[i + 1] - rp[i]);
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_down_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// Row-walk numeric reduce (same sums as k_gal_numeric, different data path): a warp per coarse
// row walks its members ascending and each member's CSR row in order — contiguous reads of
// A and slot_of_csr instead of gathers through entry / entry_row — and adds every product into
// its slot in walk order (equal-slot lanes of one round add one after another, lowest lane
// first), which is the segment's stored order.  Coarse rows of <= 64 entries.
constexpr int kWalkWarps = 8, kWalkSlots = 64;
__global__ void __launch_bounds__(kWalkWarps * 32)
    k_gal_numeric_walk(int64_t nc, const idx* goff, const idx* grows, const idx* arp,
                       const idx* acol, const double* aval, const idx* slot_of_csr,
                       const double* pv, const idx* crp, double* out) {
  __shared__ double s_acc[kWalkWarps][kWalkSlots];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t I = static_cast<int64_t>(blockIdx.x) * kWalkWarps + w;
  if (I >= nc) return;
  double* acc = s_acc[w];
  const idx s0 = crp[I], ns = crp[I + 1] - s0;
  for (int t = lane; t < kWalkSlots; t += 32) acc[t] = 0.0;
  __syncwarp();
  for (idx mb = goff[I]; mb < goff[I + 1]; mb += 32) {
    const idx m = mb + lane;
    const int nm = static_cast<int>(min(static_cast<idx>(32), goff[I + 1] - mb));
    idx i = 0, lo = 0, len = 0;
    double pvi = 0.0;
    if (lane < nm) {
      i = grows[m];
      lo = arp[i];
      len = arp[i + 1] - lo;
      pvi = pv[i];
    }
    idx incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const idx t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const idx excl = incl - len;
    const idx T = __shfl_sync(0xffffffffu, incl, 31);
    for (idx pb = 0; pb < T; pb += 32) {
      const idx p = pb + lane;
      int a = 0, b = nm;  // last member with excl <= p
#pragma unroll
      for (int step = 0; step < 6; ++step) {
        const int mid = (a + b) >> 1;
        const idx em = __shfl_sync(0xffffffffu, excl, mid & 31);
        if (b - a > 1) {
          if (em <= p) a = mid;
          else b = mid;
        }
      }
      const idx mlo = __shfl_sync(0xffffffffu, lo, a);
      const idx mex = __shfl_sync(0xffffffffu, excl, a);
      const double mpv = __shfl_sync(0xffffffffu, pvi, a);
      int sl = -1 - lane;
      double c = 0.0;
      if (p < T) {
        const idx k = mlo + (p - mex);
        c = __dmul_rn(__dmul_rn(mpv, aval[k]), pv[acol[k]]);
        sl = slot_of_csr[k] - s0;
      }
      const unsigned grp = __match_any_sync(0xffffffffu, sl);
      const int rk = __popc(grp & ((1u << lane) - 1u));
      int mx = rk;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      for (int step = 0; step <= mx; ++step) {
        if (p < T && rk == step) acc[sl] = __dadd_rn(acc[sl], c);
        __syncwarp();
      }
    }
  }
  __syncwarp();
  for (idx t = lane; t < ns; t += 32) out[s0 + t] = acc[t];
}

__global__ void k_fingerprint(const idx* rowptr, int64_t n, const idx* col, int64_t nnz,
                              const idx* assignment, unsigned long long* out) {
  unsigned long long h = 0;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t total = (n + 1) + nnz + n;
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < total; t += stride) {
    unsigned long long v;
    if (t <= n)
      v = static_cast<unsigned long long>(rowptr[t]);
    else if (t <= n + nnz)
      v = static_cast<unsigned long long>(col[t - n - 1]);
    else
      v = static_cast<unsigned long long>(assignment[t - n - 1 - nnz]);
    h += hash_mix(hash_mix(static_cast<uint64_t>(t)) ^ v);
  }
  for (int o = 16; o > 0; o >>= 1) h += __shfl_down_sync(0xffffffffu, h, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, h);
}

}  // namespace

// ---- host drivers ---------------------------------------------------------------------------

DevCsrPtr classic_strength(const DevCsr& A, double alpha, int zero_diag_policy) {
  require(A.n_rows == A.n_cols, "strength: matrix must be square");
  return strength_rows(A, alpha, zero_diag_policy);
}

// Rows of a (possibly row-partitioned) operator whose owned columns are 0..n_rows-1 in
// local ids: the diagonal of row i is column i, halo columns never are.
namespace {
// one strength pass: CSR-stream staged when A has a row-block plan that fits, else thread-per-row
void strength_pass(const DevCsr& A, double alpha, int fail_zero, int mode, const idx* out_rowptr,
                   idx* out, int* bad) {
  const int64_t n = A.n_rows;
  if (n == 0) return;
  const int stage = ((A.smem_entries + 3) / 2) * 2 + 2;
  const size_t smem = static_cast<size_t>(stage) * (sizeof(double) + sizeof(idx));
  // staging pays for long rows only (measured: 27-point 8.5 -> 4.3 ms; 7- and 14-entry rows
  // are faster thread-per-row)
  const bool long_rows = A.nnz >= 20 * n;
  if (long_rows && A.rows_per_block > 0 && A.rows_per_block <= kStrThreads && smem <= 48 * 1024) {
    const int64_t nblocks = (n + A.rows_per_block - 1) / A.rows_per_block;
    static thread_local size_t cached_smem = 0;
    static thread_local int per_sm = 1;
    if (cached_smem != smem) {
      AGG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_strength_stream,
                                                             kStrThreads, smem));
      per_sm = std::max(1, per_sm);
      cached_smem = smem;
    }
    const int64_t grid = std::min<int64_t>(nblocks, static_cast<int64_t>(per_sm) * sm_count());
    AGG_LAUNCH(k_strength_stream, static_cast<unsigned>(grid), kStrThreads, smem, A.rowptr.get(),
               A.col.get(), A.val.get(), n, A.rows_per_block, nblocks, stage, alpha, fail_zero, mode,
               out_rowptr, out, bad);
    return;
  }
  AGG_LAUNCH(k_strength, grid_for(n, 256), 256, 0, A.rowptr.get(), A.col.get(), A.val.get(), n,
             alpha, fail_zero, mode, out_rowptr, out, bad);
}
}  // namespace

DevCsrPtr strength_rows(const DevCsr& A, double alpha, int zero_diag_policy) {
  require(alpha > 0.0 && alpha < 1.0, "strength: alpha must be in (0, 1)");
  const int64_t n = A.n_rows;
  auto C = std::make_shared<DevCsr>();
  C->n_rows = n;
  C->n_cols = A.n_cols;
  C->rowptr.resize(n + 1);
  DevBuf<idx> cnt(n);
  DevBuf<int> bad(1);
  fill_int(bad.get(), 1, INT32_MAX);
  strength_pass(A, alpha, zero_diag_policy, 0, nullptr, cnt.get(), bad.get());
  C->nnz = scan_to_offsets(cnt.get(), C->rowptr.get(), n);
  if (zero_diag_policy) {
    const int b = read_scalar(bad.get());
    if (b != INT32_MAX)
      throw Error("strength: zero or missing diagonal at row " + std::to_string(b));
  }
  C->col.resize(C->nnz);
  if (C->nnz > 0) strength_pass(A, alpha, 0, 1, C->rowptr.get(), C->col.get(), bad.get());
  return C;
}

void influence_and_symmetrize(const DevCsr& C, DevBuf<idx>& influence, DevCsrPtr& S) {
  require(C.n_rows == C.n_cols, "symmetrize: matrix must be square");
  const int64_t n = C.n_rows;
  influence.resize(n);
  S = std::make_shared<DevCsr>();
  S->n_rows = S->n_cols = n;
  S->rowptr.resize(n + 1);
  if (n == 0) {
    S->nnz = 0;
    fill_int(S->rowptr.get(), 1, 0);
    return;
  }
  DevBuf<idx> mirrored(n), ecnt(n), eoff(n + 1), scnt(n);
  DevBuf<int8_t> has_extra(n);
  DevBuf<unsigned long long> total(1);
  ecnt.zero();
  total.zero();
  const unsigned g = grid_for(n, 256);
  AGG_LAUNCH(k_sym_probe, g, 256, 0, C.rowptr.get(), C.col.get(), n, mirrored.get(), ecnt.get(),
             has_extra.get(), total.get());
  const unsigned long long ne = read_scalar(total.get());
  DevBuf<idx> ecol(static_cast<int64_t>(ne));
  if (ne > 0) {
    scan_to_offsets_async(ecnt.get(), eoff.get(), n);
    DevBuf<idx> cursor(n);
    cursor.zero();
    AGG_LAUNCH(k_sym_extras, g, 256, 0, C.rowptr.get(), C.col.get(), n, has_extra.get(), eoff.get(),
               cursor.get(), ecol.get());
  } else {
    eoff.zero();
  }
  AGG_LAUNCH(k_sym_counts, g, 256, 0, C.rowptr.get(), mirrored.get(), ecnt.get(), n,
             influence.get(), scnt.get());
  S->nnz = scan_to_offsets(scnt.get(), S->rowptr.get(), n);
  S->col.resize(S->nnz);
  if (S->nnz > 0)
    AGG_LAUNCH(k_sym_fill, g, 256, 0, C.rowptr.get(), C.col.get(), S->rowptr.get(), eoff.get(),
               ecnt.get(), ecol.get(), n, S->col.get());
}

Mis2Dev mis2(const DevCsr& S, const idx* influence, uint64_t seed) {
  require(S.n_rows == S.n_cols, "mis2: graph must be square");
  const int64_t n = S.n_rows;
  Mis2Dev res;
  res.state.resize(n);
  if (n == 0) return res;
  DevBuf<Tuple> cur(n), mid(n);
  DevBuf<MisCtl> ctl(1);
  MisCtl h0{static_cast<int>(n), 0, 0, 0};
  ctl.upload(&h0, 1);
  AGG_LAUNCH(k_mis_init, grid_for(n, 256), 256, 0, influence, n, seed, cur.get(), res.state.get());
  const unsigned g = grid_for(n, 256);
  const unsigned gp = grid_for(n, 256, 8 * int64_t{sm_count()});  // the sweeps' persistent grid
  // Sweeps are issued in batches; once every node is decided the kernels exit at entry,
  // so the device-side sweep counter matches the reference's loop count exactly.
  int batch = 8;
  while (true) {
    for (int b = 0; b < batch; ++b) {
      AGG_LAUNCH(k_mis_pass1, gp, 256, 0, S.rowptr.get(), S.col.get(), n, cur.get(), mid.get(), ctl.get());
      AGG_LAUNCH(k_mis_pass2, gp, 256, 0, S.rowptr.get(), S.col.get(), n, mid.get(), cur.get(),
                 res.state.get(), ctl.get());
    }
    const MisCtl h = read_scalar(ctl.get());
    if (h.sweeps > n) throw Error("mis2: failed to decide all nodes");
    if (h.undecided == 0) {
      res.sweeps = h.sweeps;
      return res;
    }
    batch = 4;
    if (static_cast<double>(h.undecided) < 0.25 * static_cast<double>(n)) {
      // late sweeps over the compact undecided list
      DevBuf<idx> la(h.undecided), lb(h.undecided);
      DevBuf<int8_t> dec(h.undecided);
      DevBuf<MisList> ml(1);
      MisList m0{0, 0, h.undecided, h.sweeps};
      ml.upload(&m0, 1);
      AGG_LAUNCH(k_mis_list_init, g, 256, 0, res.state.get(), n, la.get(), ml.get());
      const unsigned gl = grid_for(h.undecided, 128);
      idx* cur_list = la.get();
      idx* nxt_list = lb.get();
      while (true) {
        for (int b = 0; b < batch; ++b) {
          AGG_LAUNCH(k_mis_2hop, gl, 128, 0, S.rowptr.get(), S.col.get(), cur.get(), cur_list, ml.get(),
                     dec.get());
          AGG_LAUNCH(k_mis_list_apply, gl, 128, 0, cur_list, ml.get(), dec.get(), cur.get(),
                     res.state.get(), nxt_list);
          AGG_LAUNCH(k_mis_list_swap, 1, 1, 0, ml.get());
          std::swap(cur_list, nxt_list);
        }
        const MisList hm = read_scalar(ml.get());
        if (hm.sweeps > n) throw Error("mis2: failed to decide all nodes");
        if (hm.undecided == 0) {
          res.sweeps = hm.sweeps;
          return res;
        }
      }
    }
  }
  return res;
}

AggDev aggregate(const DevCsr& S, const DevCsr& A, const int8_t* state) {
  require(S.n_rows == S.n_cols && A.n_rows == A.n_cols && S.n_rows == A.n_rows,
          "aggregate: graph and matrix shapes disagree");
  const int64_t n = S.n_rows;
  AggDev agg;
  agg.n_fine = n;
  agg.assignment.resize(n);
  DevBuf<idx> rep(n), rep2(n), isrep(n), rank(n + 1);
  if (n > 0) {
    AGG_LAUNCH(k_agg_pass1, grid_for(n, 256), 256, 0, S.rowptr.get(), S.col.get(), n, state, rep.get());
    AGG_LAUNCH(k_agg_pass2, grid_for(n, 256), 256, 0, S.rowptr.get(), S.col.get(), A.rowptr.get(),
               A.col.get(), A.val.get(), n, rep.get(), rep2.get(), isrep.get());
  }
  agg.n_agg = scan_to_offsets(isrep.get(), rank.get(), n);
  agg.representatives.resize(agg.n_agg);
  if (n > 0)
    AGG_LAUNCH(k_agg_assign, grid_for(n, 256), 256, 0, rep2.get(), rank.get(), n,
               agg.assignment.get(), agg.representatives.get());
  build_groups(agg);
  return agg;
}

void build_groups(AggDev& agg) {
  const int64_t n = agg.n_fine, nc = agg.n_agg;
  DevBuf<idx> cnt(nc), tmp(n);
  cnt.zero();
  agg.agg_row_offsets.resize(nc + 1);
  agg.rows_by_coarse.resize(n);
  if (n > 0) AGG_LAUNCH(k_col_count, grid_for(n, 256), 256, 0, agg.assignment.get(), n, cnt.get());
  scan_to_offsets_async(cnt.get(), agg.agg_row_offsets.get(), nc);
  cnt.zero();
  if (n > 0)
    AGG_LAUNCH(k_group_scatter, grid_for(n, 256), 256, 0, agg.assignment.get(), n,
               agg.agg_row_offsets.get(), cnt.get(), tmp.get());
  segmented_sort(agg.agg_row_offsets.get(), nc, tmp.get(), agg.rows_by_coarse.get());
}

TransferDev build_transfer(const AggDev& agg, const double* fine_b) {
  const int64_t n = agg.n_fine, nc = agg.n_agg;
  TransferDev t;
  t.pval.resize(n);
  t.coarse_b.resize(nc);
  DevBuf<idx> rcnt(nc);
  DevBuf<int> bad(1);
  fill_int(bad.get(), 1, INT32_MAX);
  if (nc > 0)
    AGG_LAUNCH(k_transfer_norms, grid_for(nc, 256), 256, 0, agg.agg_row_offsets.get(),
               agg.rows_by_coarse.get(), fine_b, nc, t.coarse_b.get(), rcnt.get(), bad.get());
  t.R = std::make_shared<DevCsr>();
  t.R->n_rows = nc;
  t.R->n_cols = n;
  t.R->rowptr.resize(nc + 1);
  t.p_nnz = t.R->nnz = scan_to_offsets(rcnt.get(), t.R->rowptr.get(), nc);
  const int b = read_scalar(bad.get());
  if (b != INT32_MAX)
    throw Error("transfer: near-null-space vector vanishes on aggregate " + std::to_string(b));
  if (n > 0)
    AGG_LAUNCH(k_transfer_pval, grid_for(n, 256), 256, 0, agg.assignment.get(), fine_b,
               t.coarse_b.get(), n, t.pval.get());
  t.R->col.resize(t.R->nnz);
  t.R->val.resize(t.R->nnz);
  if (nc > 0)
    AGG_LAUNCH(k_transfer_R, grid_for(nc, 256), 256, 0, agg.agg_row_offsets.get(),
               agg.rows_by_coarse.get(), t.pval.get(), nc, t.R->rowptr.get(), t.R->col.get(),
               t.R->val.get());
  t.R->plan();
  return t;
}

namespace {
// the coarse-row walk's inputs shared by both cache builds: grouping copies and the longest row
void finish_cache(GalerkinDev& g, const DevCsr& A, const AggDev& agg) {
  const int64_t nc = g.n_coarse;
  g.group_offsets.resize(nc + 1);
  AGG_CUDA(cudaMemcpyAsync(g.group_offsets.get(), agg.agg_row_offsets.get(), sizeof(idx) * (nc + 1),
                           cudaMemcpyDeviceToDevice, stream()));
  g.group_rows.resize(A.n_rows);
  if (A.n_rows > 0)
    AGG_CUDA(cudaMemcpyAsync(g.group_rows.get(), agg.rows_by_coarse.get(), sizeof(idx) * A.n_rows,
                             cudaMemcpyDeviceToDevice, stream()));
  DevBuf<int> mr(1);
  mr.zero();
  if (nc > 0)
    AGG_LAUNCH(k_max_rowlen, grid_for(nc, 256, 4 * sm_count()), 256, 0, g.coarse_rowptr.get(), nc,
               mr.get());
  g.max_coarse_row = read_scalar(mr.get());
}
}  // namespace

GalerkinDev build_galerkin_cache(const DevCsr& A, const AggDev& agg, bool partial, bool fingerprint,
                                 bool lean, const double* pval, DevBuf<double>* values) {
  require(partial || A.n_rows == A.n_cols, "galerkin: matrix must be square");
  require(agg.n_fine == A.n_rows, "galerkin: aggregation size mismatch");
  const int64_t nc = agg.n_agg;
  GalerkinDev g;
  g.n_fine = A.n_rows;
  g.n_coarse = nc;
  g.nnz_fine = A.nnz;
  g.slot_of_csr.resize(A.nnz);
  DevBuf<idx> ecnt(nc), eoff(nc + 1), cnnz(nc);
  DevBuf<int> big_count(1);
  big_count.zero();
  if (nc > 0)
    AGG_LAUNCH(k_group_entry_counts, grid_for(nc, 256), 256, 0, agg.agg_row_offsets.get(),
               agg.rows_by_coarse.get(), A.rowptr.get(), nc, ecnt.get());
  const int64_t total = scan_to_offsets(ecnt.get(), eoff.get(), nc);
  require(partial || total == A.nnz, "galerkin: aggregation does not cover the matrix rows");
  // AGGMG_GAL_LEAN=0: the full cache in a hierarchy too (comparison runs)
  static const bool lean_on = [] {
    const char* e = std::getenv("AGGMG_GAL_LEAN");
    return !(e && e[0] == '0');
  }();
  if (lean && lean_on && !partial && nc > 0) {
    DevBuf<idx> tmpj(A.nnz);
    DevBuf<int> bad(1);
    bad.zero();
    const unsigned grid = static_cast<unsigned>((nc + kGalWarps - 1) / kGalWarps);
    AGG_LAUNCH(k_gal_lean_count, grid, kGalWarps * 32, 0, agg.agg_row_offsets.get(),
               agg.rows_by_coarse.get(), A.rowptr.get(), A.col.get(), agg.assignment.get(), nc,
               eoff.get(), tmpj.get(), cnnz.get(), bad.get());
    if (read_scalar(bad.get()) == 0) {
      g.lean = true;
      g.coarse_rowptr.resize(nc + 1);
      g.nnz_coarse = scan_to_offsets(cnnz.get(), g.coarse_rowptr.get(), nc);
      g.coarse_col.resize(g.nnz_coarse);
      if (values) values->resize(g.nnz_coarse);
      AGG_LAUNCH(k_gal_lean_fill, grid, kGalWarps * 32, 0, agg.agg_row_offsets.get(),
                 agg.rows_by_coarse.get(), A.rowptr.get(), A.col.get(), agg.assignment.get(), nc,
                 eoff.get(), tmpj.get(), g.coarse_rowptr.get(), g.coarse_col.get(), g.slot_of_csr.get(),
                 A.val.get(), pval, values ? values->get() : nullptr);
      finish_cache(g, A, agg);
      if (fingerprint) g.pattern_hash = pattern_fingerprint(A, agg.assignment.get());
      sync();  // tmpj dies here
      return g;
    }
  }
  g.entry.resize(A.nnz);
  g.entry_row.resize(A.nnz);
  DevBuf<idx> sorted_j(A.nnz), big_list(nc > 0 ? nc : 1);
  // AGGMG_GAL_TIER1=1: the length-capped tier 1 (comparison runs)
  static const bool capped_tier1 = [] {
    const char* e = std::getenv("AGGMG_GAL_TIER1");
    return e && e[0] == '1';
  }();
  const auto tier1 = capped_tier1 ? k_gal_symbolic : k_gal_symbolic_w;
  if (nc > 0)
    AGG_LAUNCH(tier1,
               static_cast<unsigned>((nc + kGalWarps - 1) / kGalWarps), kGalWarps * 32, 0,
               agg.agg_row_offsets.get(), agg.rows_by_coarse.get(), A.rowptr.get(), A.col.get(),
               agg.assignment.get(), nc, eoff.get(), g.entry.get(), g.entry_row.get(),
               sorted_j.get(), cnnz.get(), big_list.get(), big_count.get());
  const int nbig = read_scalar(big_count.get());
  if (nbig > 0) {
    DevBuf<int> maxlen(1);
    maxlen.zero();
    AGG_LAUNCH(k_max_big_len, grid_for(nbig, 256, 4 * sm_count()), 256, 0, big_list.get(), nbig,
               eoff.get(), maxlen.get());
    // rows up to 2048 entries in shared memory (three CTAs per SM); longer rows use global
    // scratch (measured on the 27-point operator: 4096 -> 2048 took the phase 29 -> 25 ms)
    const int cap = std::min(kGalCapSmem, read_scalar(maxlen.get()));
    const size_t smem = static_cast<size_t>(cap) * 5 * sizeof(idx);
    static std::atomic<unsigned long long> raised{0};  // the attribute is per device
    if (device_pending(raised)) {
      AGG_CUDA(cudaFuncSetAttribute(k_gal_symbolic_big, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    kGalCapBig * 5 * static_cast<int>(sizeof(idx))));
      mark_device(raised);
    }
    // global scratch only for the rows longer than the shared-memory capacity
    DevBuf<int64_t> blen(nbig), boff(nbig + 1);
    AGG_LAUNCH(k_big_scratch_len, grid_for(nbig, 256), 256, 0, big_list.get(), nbig, eoff.get(), cap,
               blen.get());
    int64_t big_total = 0;
    {
      std::vector<int64_t> h(nbig);
      blen.download(h.data(), nbig);
      sync();
      std::vector<int64_t> o(nbig + 1, 0);
      for (int t = 0; t < nbig; ++t) o[t + 1] = o[t] + h[t];
      big_total = o[nbig];
      boff.upload(o.data(), nbig + 1);
    }
    DevBuf<idx> scratch(std::max<int64_t>(1, 5 * big_total));
    AGG_LAUNCH(k_gal_symbolic_big, static_cast<unsigned>(nbig), 256, smem, big_list.get(),
               agg.agg_row_offsets.get(), agg.rows_by_coarse.get(), A.rowptr.get(), A.col.get(),
               agg.assignment.get(), eoff.get(), cap, boff.get(), scratch.get(), g.entry.get(),
               g.entry_row.get(), sorted_j.get(), cnnz.get());
  }
  g.coarse_rowptr.resize(nc + 1);
  g.nnz_coarse = scan_to_offsets(cnnz.get(), g.coarse_rowptr.get(), nc);
  g.coarse_col.resize(g.nnz_coarse);
  g.segment_offsets.resize(g.nnz_coarse + 1);
  if (nc > 0)
    AGG_LAUNCH(k_gal_fill, grid_for(nc * 32, 256), 256, 0, nc, eoff.get(), sorted_j.get(),
               g.entry.get(), g.coarse_rowptr.get(), g.coarse_col.get(), g.segment_offsets.get(),
               g.slot_of_csr.get());
  const idx nnz32 = static_cast<idx>(total);  // == A.nnz unless partial
  AGG_CUDA(cudaMemcpyAsync(g.segment_offsets.get() + g.nnz_coarse, &nnz32, sizeof(idx),
                           cudaMemcpyHostToDevice, stream()));
  sync();  // nnz32 lives on the host stack
  if (!partial) finish_cache(g, A, agg);
  if (!partial && fingerprint) g.pattern_hash = pattern_fingerprint(A, agg.assignment.get());
  return g;
}

DevCsrPtr coarse_from_cache(const GalerkinDev& g, DevBuf<double>&& values) {
  auto Ac = std::make_shared<DevCsr>();
  Ac->n_rows = Ac->n_cols = g.n_coarse;
  Ac->nnz = g.nnz_coarse;
  Ac->rowptr.resize(g.n_coarse + 1);
  Ac->col.resize(g.nnz_coarse);
  AGG_CUDA(cudaMemcpyAsync(Ac->rowptr.get(), g.coarse_rowptr.get(), sizeof(idx) * (g.n_coarse + 1),
                           cudaMemcpyDeviceToDevice, stream()));
  if (g.nnz_coarse > 0)
    AGG_CUDA(cudaMemcpyAsync(Ac->col.get(), g.coarse_col.get(), sizeof(idx) * g.nnz_coarse,
                             cudaMemcpyDeviceToDevice, stream()));
  Ac->val = std::move(values);
  Ac->plan();
  return Ac;
}

DevCsrPtr apply_galerkin_cache(const GalerkinDev& g, const DevCsr& A, const double* pval) {
  auto Ac = std::make_shared<DevCsr>();
  Ac->n_rows = Ac->n_cols = g.n_coarse;
  Ac->nnz = g.nnz_coarse;
  Ac->rowptr.resize(g.n_coarse + 1);
  Ac->col.resize(g.nnz_coarse);
  Ac->val.resize(g.nnz_coarse);
  AGG_CUDA(cudaMemcpyAsync(Ac->rowptr.get(), g.coarse_rowptr.get(), sizeof(idx) * (g.n_coarse + 1),
                           cudaMemcpyDeviceToDevice, stream()));
  if (g.nnz_coarse > 0) {
    AGG_CUDA(cudaMemcpyAsync(Ac->col.get(), g.coarse_col.get(), sizeof(idx) * g.nnz_coarse,
                             cudaMemcpyDeviceToDevice, stream()));
    require(!g.lean || g.max_coarse_row <= kWalkSlots, "galerkin: lean cache beyond the row walk");
    if (g.group_offsets.size() == g.n_coarse + 1 && g.max_coarse_row <= kWalkSlots)
      AGG_LAUNCH(k_gal_numeric_walk, static_cast<unsigned>((g.n_coarse + kWalkWarps - 1) / kWalkWarps),
                 kWalkWarps * 32, 0, g.n_coarse, g.group_offsets.get(), g.group_rows.get(),
                 A.rowptr.get(), A.col.get(), A.val.get(), g.slot_of_csr.get(), pval,
                 g.coarse_rowptr.get(), Ac->val.get());
    else
      AGG_LAUNCH(k_gal_numeric, grid_for(g.nnz_coarse, 256), 256, 0, g.nnz_coarse,
                 g.segment_offsets.get(), g.entry.get(), g.entry_row.get(), A.col.get(),
                 A.val.get(), pval, Ac->val.get());
  }
  Ac->plan();
  return Ac;
}

int64_t transfer_norms_groups(const idx* goff, const idx* rows, const double* b, int64_t nc,
                              double* coarse_b, idx* rcnt) {
  DevBuf<int> bad(1);
  fill_int(bad.get(), 1, INT32_MAX);
  if (nc > 0)
    AGG_LAUNCH(k_transfer_norms, grid_for(nc, 256), 256, 0, goff, rows, b, nc, coarse_b, rcnt, bad.get());
  const int v = read_scalar(bad.get());
  return v == INT32_MAX ? -1 : v;
}

void transfer_R_groups(const idx* goff, const idx* rows, const double* pval, int64_t nc,
                       const idx* rrp, idx* rcol, double* rval) {
  if (nc > 0)
    AGG_LAUNCH(k_transfer_R, grid_for(nc, 256), 256, 0, goff, rows, pval, nc, rrp, rcol, rval);
}

DevCsrPtr galerkin_direct(const DevCsr& A, const AggDev& agg, const double* pval) {
  require(A.n_rows == A.n_cols && agg.n_fine == A.n_rows, "galerkin: aggregation size mismatch");
  const int64_t nc = agg.n_agg;
  auto Ac = std::make_shared<DevCsr>();
  Ac->n_rows = Ac->n_cols = nc;
  Ac->rowptr.resize(nc + 1);
  DevBuf<idx> ecnt(nc), eoff(nc + 1), cnnz(nc), big_list(nc > 0 ? nc : 1);
  DevBuf<int> big_count(1);
  big_count.zero();
  if (nc > 0)
    AGG_LAUNCH(k_group_entry_counts, grid_for(nc, 256), 256, 0, agg.agg_row_offsets.get(),
               agg.rows_by_coarse.get(), A.rowptr.get(), nc, ecnt.get());
  scan_to_offsets_async(ecnt.get(), eoff.get(), nc);
  const unsigned grid = static_cast<unsigned>((nc + kGalDirectWarps - 1) / kGalDirectWarps);
  DevBuf<unsigned long long> gkey, gskey;
  DevBuf<double> gval, gsval;
  for (int mode = 0; mode < 2; ++mode) {
    big_count.zero();
    if (nc > 0)
      AGG_LAUNCH(k_gal_direct, grid, kGalDirectWarps * 32, 0, agg.agg_row_offsets.get(),
                 agg.rows_by_coarse.get(), A.rowptr.get(), A.col.get(), A.val.get(),
                 agg.assignment.get(), pval, nc, eoff.get(), mode, cnnz.get(), Ac->rowptr.get(),
                 Ac->col.get(), Ac->val.get(), big_list.get(), big_count.get());
    const int nbig = read_scalar(big_count.get());
    if (nbig > 0) {
      if (gkey.size() == 0) {
        gkey.resize(A.nnz);
        gskey.resize(A.nnz);
        gval.resize(A.nnz);
        gsval.resize(A.nnz);
      }
      AGG_LAUNCH(k_gal_direct_big, static_cast<unsigned>(nbig), 256, 0, big_list.get(),
                 agg.agg_row_offsets.get(), agg.rows_by_coarse.get(), A.rowptr.get(), A.col.get(),
                 A.val.get(), agg.assignment.get(), pval, eoff.get(), mode, gkey.get(), gval.get(),
                 gskey.get(), gsval.get(), cnnz.get(), Ac->rowptr.get(), Ac->col.get(),
                 Ac->val.get());
    }
    if (mode == 0) {
      Ac->nnz = scan_to_offsets(cnnz.get(), Ac->rowptr.get(), nc);
      Ac->col.resize(Ac->nnz);
      Ac->val.resize(Ac->nnz);
    }
  }
  Ac->plan();
  return Ac;
}

uint64_t pattern_fingerprint(const DevCsr& A, const idx* assignment) {
  DevBuf<unsigned long long> h(1);
  h.zero();
  AGG_LAUNCH(k_fingerprint, grid_for(A.n_rows + A.nnz + 1, 256, 4 * sm_count()), 256, 0,
             A.rowptr.get(), A.n_rows, A.col.get(), A.nnz, assignment, h.get());
  return read_scalar(h.get());
}

}  // namespace aggmg_b200
