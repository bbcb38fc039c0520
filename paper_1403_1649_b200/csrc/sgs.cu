// sgs.cu — symmetric Gauss-Seidel smoother (smoother.cpp:105-119), level-scheduled on the
// device and bit-identical to the reference's two sequential sweeps.
//
// Why it is exact.  Going forward, row i reads x_j for j < i after the sweep updated them
// and x_j for j > i before.  Each direction is run over a level schedule — level(i) = 1 +
// max level of the rows it reads updated values from — so every row it reads "new" is done
// before it; the values it reads "old" come from a buffer the sweep does not write (forward
// writes xn and reads old values from x; backward writes x and reads the forward output xn).
// Each row then computes the reference's own sequential sum in CSR order (diagonal skipped,
// no FMA), so no schedule changes a bit.
//
// Why it is fast.  The sweep is latency-bound: a level cannot start before the previous one
// is written.  Levels narrower than one CTA (2-D grids, every coarse level) run as one
// single-CTA kernel per run of levels, with the critical path kept on chip:
//   - slot data (row id, 1/A_ii, b, ELL codes and values) is staged into a shared-memory
//     slot ring by cp.async kAhead levels before it is swept;
//   - x values live in a shared-memory ring indexed by slot: new values are written there as
//     they are produced, old (input) values are staged by cp.async from a slot-ordered copy
//     kAhead + kOldReach levels ahead;
//   - each ELL entry carries a code chosen at setup: ring slot, or global old/new value when
//     the column is outside the run or the ring window (rare on grids).
// A level then costs a barrier plus a few shared-memory loads and the row's FP64 chain.
// Levels wider than a CTA run one launch each, a thread per row, from global memory.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "smoother.cuh"

namespace aggmg_b200 {
namespace {

constexpr uint32_t kOld = 0u, kNew = 1u << 30, kRing = 2u << 30;
constexpr uint32_t kKindMask = 3u << 30, kIdxMask = (1u << 30) - 1;
// ELL padding (rows shorter than the block): value +0 times the ring's +0 cell — s - (+0)
// is s for every s, so the run kernel sweeps all E entries without branches
constexpr int kWinCells = 8192;  // power of two: ring positions are masks
constexpr uint32_t kPad = kRing | static_cast<uint32_t>(kWinCells);
constexpr int kAhead = 3;           // levels of slot data staged ahead of the swept level
constexpr int kOldReach = 2;        // old values readable from the ring up to this many levels on
constexpr int kWin = kWinCells;     // x ring (doubles)
constexpr int kMaxRunLevels = 4096; // run offsets staged in shared memory

__host__ __device__ constexpr int cta_for(int E) { return E == 4 ? 512 : E == 8 ? 256 : 128; }
constexpr int back_window(int cta) { return kWin - (kAhead + kOldReach + 2) * cta; }

template <int E>
constexpr size_t run_smem() {
  constexpr size_t RS = (kAhead + 1) * cta_for(E);
  return sizeof(double) * (kWin + 2) + 16 * RS * (1 + E / 4 + E / 2) + sizeof(double) * RS +
         sizeof(int) * (kMaxRunLevels + 1);
}
static_assert(run_smem<4>() <= 227 * 1024 && run_smem<8>() <= 227 * 1024 &&
                  run_smem<16>() <= 227 * 1024,
              "sgs run kernel shared memory");

// Slot t in global memory: rec[t] = {row, off-diagonal count, 1/A_ii as two words}; ELL
// codes in E/4 uint4 chunks code[c*n + t], values in E/2 double2 chunks val[c*n + t] (so one
// 16-byte cp.async moves four codes or two values, and shared-memory reads are conflict-free).
struct SgsArgs {
  const int* rows;
  const int4* rec;
  const uint4* code;
  const double2* val;
  const idx* optr;
  const idx* ocol;
  const double* oval;
  int64_t n;
  const double* bp;  // b in slot order (run kernels)
  const double* xp;  // xc in slot order (run kernels)
  const double* b;   // natural order
  const double* xc;  // the sweep's old values (not written by this sweep)
  double* out;       // the sweep's new values
  int fwd;
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cpa8u(unsigned s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(g) : "memory");
}
__device__ __forceinline__ void cpa16u(unsigned s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(s), "l"(g) : "memory");
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cpa_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// where an ELL entry's x lives (generic address: the shared ring or global memory)
__device__ __forceinline__ const double* sgs_src(uint32_t c, const double* W, const SgsArgs& a) {
  const uint32_t k = c & kKindMask, j = c & kIdxMask;
  return k == kRing ? W + j : (k == kNew ? a.out : a.xc) + j;
}

// entries past the ELL block, in CSR order after it
__device__ __forceinline__ double sgs_overflow(double s, int i, int64_t t, const SgsArgs& a) {
  for (idx k = a.optr[t]; k < a.optr[t + 1]; ++k) {
    const int j = a.ocol[k];
    s = __dsub_rn(s, __dmul_rn(a.oval[k], (a.fwd ? j < i : j > i) ? a.out[j] : a.xc[j]));
  }
  return s;
}

template <int E>
__global__ void __launch_bounds__(cta_for(E), 1)
    k_sgs_run(SgsArgs a, const int* off_g, int64_t l0, int64_t l1, const int* pred) {
  if (pred && !*pred) return;
  constexpr int CTA = cta_for(E), RS = (kAhead + 1) * CTA, C4 = E / 4, C2 = E / 2;
  extern __shared__ __align__(16) unsigned char sm[];
  double* W = reinterpret_cast<double*>(sm);  // W[kWin] = +0: the padding entries' x
  int4* srec = reinterpret_cast<int4*>(W + kWin + 2);
  uint4* scode = reinterpret_cast<uint4*>(srec + RS);      // [C4][RS]
  double2* sval = reinterpret_cast<double2*>(scode + C4 * RS);  // [C2][RS]
  double* sb = reinterpret_cast<double*>(sval + C2 * RS);
  int* soff = reinterpret_cast<int*>(sb + RS);
  const int nl = static_cast<int>(l1 - l0), tid = threadIdx.x;
  for (int q = tid; q <= nl; q += CTA) soff[q] = off_g[l0 + q];
  if (tid == 0) W[kWin] = 0.0;
  __syncthreads();

  static_assert((RS & (RS - 1)) == 0 && (kWin & (kWin - 1)) == 0, "ring sizes");
  const unsigned uW = smem_u32(W), uRec = smem_u32(srec), uCode = smem_u32(scode),
                 uVal = smem_u32(sval), uB = smem_u32(sb);
  // stage level k's slots / old values: each thread moves its own slot
  auto stage_slots = [&](int s, int s_end) {
    if (s >= s_end) return;
    const unsigned r = static_cast<unsigned>(s) & (RS - 1);
    cpa16u(uRec + 16 * r, a.rec + s);
#pragma unroll
    for (int c = 0; c < C4; ++c) cpa16u(uCode + 16 * (c * RS + r), a.code + c * a.n + s);
#pragma unroll
    for (int c = 0; c < C2; ++c) cpa16u(uVal + 16 * (c * RS + r), a.val + c * a.n + s);
    cpa8u(uB + 8 * r, a.bp + s);
  };
  auto stage_x = [&](int s, int s_end) {
    if (s < s_end) cpa8u(uW + 8 * (static_cast<unsigned>(s) & (kWin - 1)), a.xp + s);
  };
  auto lo = [&](int k) { return k < nl ? soff[k] + tid : 0; };
  auto hi = [&](int k) { return k < nl ? soff[k + 1] : 0; };

  // cp.async group m carries level m's slots and level m+kOldReach's old values (group 0
  // also levels 0..kOldReach-1); groups 0..kAhead-1 are issued here, group k+kAhead at the
  // end of iteration k, so level k (group k, kAhead+k groups committed) waits with at most
  // kAhead-1 younger groups in flight
  for (int m = 0; m < kAhead; ++m) {
    if (m == 0)
      for (int q = 0; q < kOldReach; ++q) stage_x(lo(q), hi(q));
    stage_slots(lo(m), hi(m));
    stage_x(lo(m + kOldReach), hi(m + kOldReach));
    cpa_commit();
  }
  int t = soff[0] + tid, t_end = soff[1];
  for (int k = 0; k < nl; ++k) {
    // bounds of the levels staged at the end of this iteration (static shared data, read
    // before the barrier so the latency hides behind it)
    const int ss = lo(k + kAhead), se = hi(k + kAhead);
    const int xs = lo(k + kAhead + kOldReach), xe = hi(k + kAhead + kOldReach);
    cpa_wait<kAhead - 1>();
    __syncthreads();  // level k-1 written, level k's staged data visible, slot ring reusable
    if (t < t_end) {
      const int r = t & (RS - 1);
      const int4 rc = srec[r];
      uint32_t c[E];
#pragma unroll
      for (int q = 0; q < C4; ++q) {
        const uint4 u = scode[q * RS + r];
        c[4 * q] = u.x, c[4 * q + 1] = u.y, c[4 * q + 2] = u.z, c[4 * q + 3] = u.w;
      }
      // all E entries unconditionally: padding entries are 0 * (+0), an exact no-op.  Each x
      // is one shared load (the ring cell, or the +0 cell for global entries) plus a
      // predicated global load for entries outside the ring.
      double x[E];
#pragma unroll
      for (int e = 0; e < E; ++e) {
        const uint32_t kind = c[e] & kKindMask, j = c[e] & kIdxMask;
        const bool ring = kind == kRing;
        const double xr = W[ring ? j : kWin];
        double xg = 0.0;
        if (!ring) xg = (kind == kNew ? a.out : a.xc)[j];
        x[e] = ring ? xr : xg;
      }
      double s = sb[r];
#pragma unroll
      for (int q = 0; q < C2; ++q) {
        const double2 v = sval[q * RS + r];
        s = __dsub_rn(s, __dmul_rn(v.x, x[2 * q]));
        s = __dsub_rn(s, __dmul_rn(v.y, x[2 * q + 1]));
      }
      if (rc.y > E) s = sgs_overflow(s, rc.x, t, a);
      const double v = __dmul_rn(s, __hiloint2double(rc.w, rc.z));
      W[t & (kWin - 1)] = v;
      a.out[rc.x] = v;
    }
    stage_slots(ss, se);
    stage_x(xs, xe);
    cpa_commit();
    t = t_end + tid;
    t_end = soff[k + 2 <= nl ? k + 2 : nl];
  }
  cpa_wait<0>();
}

// One wide level, a thread per row, everything from global memory (codes are never kRing).
template <int E>
__global__ void k_sgs_level(SgsArgs a, int64_t begin, int64_t count, const int* pred) {
  if (pred && !*pred) return;
  const int64_t t = begin + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= begin + count) return;
  const int4 rc = a.rec[t];
  double s = a.b[rc.x];
#pragma unroll
  for (int q = 0; q < E / 4; ++q) {
    const uint4 u = a.code[q * a.n + t];
    const double2 v0 = a.val[2 * q * a.n + t], v1 = a.val[(2 * q + 1) * a.n + t];
    const uint32_t cc[4] = {u.x, u.y, u.z, u.w};
    const double vv[4] = {v0.x, v0.y, v1.x, v1.y};
#pragma unroll
    for (int e = 0; e < 4; ++e)
      if (4 * q + e < rc.y) s = __dsub_rn(s, __dmul_rn(vv[e], *sgs_src(cc[e], nullptr, a)));
  }
  if (rc.y > E) s = sgs_overflow(s, rc.x, t, a);
  a.out[rc.x] = __dmul_rn(s, __hiloint2double(rc.w, rc.z));
}

__global__ void k_sgs_permute(const int* rows, int64_t n, const double* b, const double* xc,
                              double* bp, double* xp, const int* pred) {
  if (pred && !*pred) return;
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int i = rows[t];
  bp[t] = b[i];
  xp[t] = xc[i];
}

__global__ void k_pack_rec(const int* rows, const int* lens, const double* inv, int64_t n,
                           int4* rec) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const double d = inv[rows[t]];
  rec[t] = make_int4(rows[t], lens[t], __double2loint(d), __double2hiint(d));
}

template <class T>
void put(DevBuf<T>& buf, const std::vector<T>& v) {
  buf.resize(static_cast<int64_t>(v.size()));
  buf.upload(v.data(), static_cast<int64_t>(v.size()));
}

void build_direction(const std::vector<idx>& rp, const std::vector<idx>& col,
                     const std::vector<double>& val, const double* inv_diag, int64_t n, bool fwd,
                     SgsDirection& d) {
  // levels: longest path over the rows read "new"
  std::vector<int> lvl(n, 0);
  int depth = n > 0 ? 1 : 0, max_len = 0;
  for (int64_t q = 0; q < n; ++q) {
    const int64_t i = fwd ? q : n - 1 - q;
    int m = -1, len = 0;
    for (idx k = rp[i]; k < rp[i + 1]; ++k) {
      const int64_t j = col[k];
      if (fwd ? j < i : j > i) m = std::max(m, lvl[j]);
      len += j != i;
    }
    lvl[i] = m + 1;
    depth = std::max(depth, m + 2);
    max_len = std::max(max_len, len);
  }
  const int E = max_len <= 4 ? 4 : max_len <= 8 ? 8 : 16;
  const int CTA = cta_for(E);
  d.ell = E;
  d.cta = CTA;
  d.h_offsets.assign(depth + 1, 0);
  for (int64_t i = 0; i < n; ++i) ++d.h_offsets[lvl[i] + 1];
  for (int l = 0; l < depth; ++l) d.h_offsets[l + 1] += d.h_offsets[l];
  std::vector<int> rows(n), slot(n), lens(n);
  {
    std::vector<int64_t> pos(d.h_offsets.begin(), d.h_offsets.end() - 1);
    for (int64_t i = 0; i < n; ++i) {
      slot[i] = static_cast<int>(pos[lvl[i]]++);
      rows[slot[i]] = static_cast<int>(i);
    }
  }
  // runs of narrow levels (at most kMaxRunLevels each); run id per level, -1 = wide
  d.runs.clear();
  std::vector<int> run_of(depth, -1);
  for (int l = 0; l < depth; ++l) {
    const bool narrow = d.h_offsets[l + 1] - d.h_offsets[l] <= CTA;
    auto& rs = d.runs;
    if (narrow && !rs.empty() && rs.back().narrow && rs.back().l1 == l &&
        rs.back().l1 - rs.back().l0 < kMaxRunLevels)
      rs.back().l1 = l + 1;
    else
      rs.push_back({l, l + 1, narrow});
    if (narrow) run_of[l] = static_cast<int>(rs.size()) - 1;
  }
  // per-slot ELL block with source codes, overflow CSR
  const int64_t back = back_window(CTA);
  std::vector<uint32_t> code(static_cast<size_t>(E) * n, kPad);
  std::vector<double> ev(static_cast<size_t>(E) * n, 0.0), ov;
  std::vector<idx> optr(n + 1, 0), oc;
  for (int64_t t = 0; t < n; ++t) {
    const int i = rows[t], li = lvl[i], run = run_of[li];
    int e = 0;
    for (idx k = rp[i]; k < rp[i + 1]; ++k) {
      const int j = col[k];
      if (j == i) continue;
      if (e < E) {
        const bool is_new = fwd ? j < i : j > i;
        const int lj = lvl[j], sj = slot[j];
        uint32_t c = (is_new ? kNew : kOld) | static_cast<uint32_t>(j);
        if (run >= 0 && run_of[lj] == run) {
          if (is_new ? (t - sj <= back) : (lj > li && lj <= li + kOldReach))
            c = kRing | static_cast<uint32_t>(sj % kWin);
        }
        code[(static_cast<size_t>(e / 4) * n + t) * 4 + e % 4] = c;
        ev[(static_cast<size_t>(e / 2) * n + t) * 2 + e % 2] = val[k];
      } else {
        oc.push_back(j);
        ov.push_back(val[k]);
      }
      ++e;
    }
    lens[t] = e;
    optr[t + 1] = static_cast<idx>(oc.size());
  }
  std::vector<int> offs(d.h_offsets.begin(), d.h_offsets.end());
  put(d.rows, rows);
  put(d.offsets, offs);
  put(d.code, code);
  put(d.val, ev);
  put(d.optr, optr);
  put(d.ocol, oc);
  put(d.oval, ov);
  DevBuf<int> dl(n);
  dl.upload(lens.data(), n);
  d.rec.resize(n);
  if (n > 0)
    AGG_LAUNCH(k_pack_rec, grid_for(n, 256), 256, 0, d.rows.get(), dl.get(), inv_diag, n,
               d.rec.get());
  AGG_CUDA(cudaStreamSynchronize(stream()));  // host staging vectors die here
}

template <int E>
void launch_run(const SgsArgs& a, const SgsDirection& d, const SgsDirection::Run& r,
                const int* pred) {
  static const bool attr = [] {
    AGG_CUDA(cudaFuncSetAttribute(k_sgs_run<E>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(run_smem<E>())));
    return true;
  }();
  (void)attr;
  AGG_LAUNCH(k_sgs_run<E>, 1, cta_for(E), run_smem<E>(), a, d.offsets.get(), r.l0, r.l1, pred);
}

template <int E>
void run_direction_t(const SgsDirection& d, const SgsArgs& a, const int* pred) {
  for (const auto& r : d.runs) {
    if (r.narrow) {
      launch_run<E>(a, d, r, pred);
    } else {
      const int64_t b0 = d.h_offsets[r.l0], cnt = d.h_offsets[r.l0 + 1] - b0;
      AGG_LAUNCH(k_sgs_level<E>, grid_for(cnt, 256), 256, 0, a, b0, cnt, pred);
    }
  }
}

void run_direction(const SgsDirection& d, const SmootherDev& s, int64_t n, const double* b,
                   const double* xc, double* out, bool fwd, const int* pred) {
  SgsArgs a{d.rows.get(), d.rec.get(), reinterpret_cast<const uint4*>(d.code.get()),
            reinterpret_cast<const double2*>(d.val.get()), d.optr.get(),
            d.ocol.get(), d.oval.get(), n, s.sgs_bp.get(), s.sgs_xp.get(), b, xc, out,
            fwd ? 1 : 0};
  bool any_run = false;
  for (const auto& r : d.runs) any_run |= r.narrow;
  if (any_run)
    AGG_LAUNCH(k_sgs_permute, grid_for(n, 256), 256, 0, d.rows.get(), n, b, xc, s.sgs_bp.get(),
               s.sgs_xp.get(), pred);
  if (d.ell == 4)
    run_direction_t<4>(d, a, pred);
  else if (d.ell == 8)
    run_direction_t<8>(d, a, pred);
  else
    run_direction_t<16>(d, a, pred);
}

}  // namespace

void build_sgs_schedule(const DevCsr& A, SmootherDev& s) {
  const int64_t n = A.n_rows;
  require(n < (int64_t{1} << 30), "smoother: the sgs schedule needs fewer than 2^30 rows");
  std::vector<idx> rp = A.rowptr.to_host(), col = A.col.to_host();
  std::vector<double> val = A.val.to_host();
  build_direction(rp, col, val, s.inv_diag.get(), n, true, s.sgs_fw);
  build_direction(rp, col, val, s.inv_diag.get(), n, false, s.sgs_bw);
  s.sgs_tmp.resize(n);
  s.sgs_bp.resize(n);
  s.sgs_xp.resize(n);
  if (std::getenv("AGGMG_SGS_INFO")) {
    for (const SgsDirection* d : {&s.sgs_fw, &s.sgs_bw}) {
      int64_t wide = 0;
      for (const auto& r : d->runs) wide += r.narrow ? 0 : 1;
      std::fprintf(stderr, "[sgs] n=%lld nnz=%lld %s depth=%zu ell=%d runs=%zu wide=%lld\n",
                   static_cast<long long>(n), static_cast<long long>(A.nnz),
                   d == &s.sgs_fw ? "fw" : "bw", d->h_offsets.size() - 1, d->ell, d->runs.size(),
                   static_cast<long long>(wide));
    }
  }
}

void smooth_sgs(const SmootherDev& s, const DevCsr& A, const double* b, double* x,
                const int* pred) {
  require(s.sgs_tmp.size() == A.n_rows && s.sgs_fw.rows.size() == A.n_rows,
          "smoother: sgs schedule missing");
  double* xn = s.sgs_tmp.get();
  run_direction(s.sgs_fw, s, A.n_rows, b, x, xn, true, pred);   // forward: x -> xn
  run_direction(s.sgs_bw, s, A.n_rows, b, xn, x, false, pred);  // backward: xn -> x
}

}  // namespace aggmg_b200
