// sparse.cu — device CSR, upload/validation, CSR-stream SpMV family, transpose and
// the device-side problem generators.
#include <atomic>
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "sparse.cuh"

namespace aggmg_b200 {

// ---- upload / validation ------------------------------------------------------------

namespace {

// Ordering checks on narrowed arrays (ranges were checked while narrowing on the host):
// row offsets non-decreasing and within [0, nnz]; columns strictly increasing per row.
__global__ void k_check_rows(const idx* rp, const idx* col, int64_t n_rows, int64_t nnz, int* bad_row,
                             int check_cols) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n_rows) return;
  const idx lo = rp[i], hi = rp[i + 1];
  if (hi < lo || lo < 0 || hi > nnz) {
    atomicMin(bad_row, static_cast<int>(i));
    return;
  }
  if (!check_cols) return;
  for (idx k = lo + 1; k < hi; ++k)
    if (col[k - 1] >= col[k]) {
      atomicMin(bad_row, static_cast<int>(i));
      return;
    }
}

__global__ void k_widen(const idx* in, int64_t* out, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i];
}

__global__ void k_max_row(const idx* rowptr, int64_t n, int* out) {
  int m = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    m = max(m, rowptr[i + 1] - rowptr[i]);
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_down_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// largest |col - row| over the entries (whether the columns fit 16-bit offsets)
__global__ void k_max_offset(const idx* rowptr, const idx* col, int64_t n, int* out) {
  int m = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    for (idx k = rowptr[i]; k < rowptr[i + 1]; ++k) m = max(m, abs(col[k] - static_cast<idx>(i)));
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_down_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

// largest staged span (e1 - (e0 & ~1)) over the row blocks of rpb rows
__global__ void k_max_block_span(const idx* rowptr, int64_t n, int rpb, int* out) {
  int m = 0;
  const int64_t nb = (n + rpb - 1) / rpb;
  for (int64_t b = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; b < nb;
       b += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r0 = b * rpb, r1 = min(r0 + rpb, n);
    m = max(m, rowptr[r1] - (rowptr[r0] & ~1));
  }
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_down_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) atomicMax(out, m);
}

}  // namespace

// ---- SELL-32 copy -------------------------------------------------------------------------
// SELL-C-sigma: inside every window of kSellSigma rows, rows ordered by descending length
// (stable), so the 32 rows of a slice have similar lengths and a warp idles less on the short
// ones (c2 level 1: 78% -> 95% of the slots are entries).  perm[q] = the row at position q.
constexpr int kSellSigma = 256;
__global__ void __launch_bounds__(kSellSigma) k_sell_sort_window(const idx* rowptr, int64_t n, idx* perm) {
  __shared__ idx len[kSellSigma];
  const int64_t w0 = static_cast<int64_t>(blockIdx.x) * kSellSigma;
  const int t = threadIdx.x;
  const int64_t r = w0 + t;
  const int cnt = static_cast<int>(min(static_cast<int64_t>(kSellSigma), n - w0));
  len[t] = r < n ? rowptr[r + 1] - rowptr[r] : -1;
  __syncthreads();
  if (t >= cnt) return;
  const idx l = len[t];
  int rank = 0;
  for (int j = 0; j < cnt; ++j) rank += (len[j] > l || (len[j] == l && j < t)) ? 1 : 0;
  perm[w0 + rank] = static_cast<idx>(r);
}

__global__ void k_slice_width(const idx* rowptr, int64_t n, int64_t nslices, int pad4, const idx* perm,
                              idx* w) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= nslices) return;
  idx m = 0;
  const int64_t r1 = min(n, 32 * (s + 1));
  for (int64_t q = 32 * s; q < r1; ++q) {
    const int64_t r = perm ? perm[q] : q;
    m = max(m, rowptr[r + 1] - rowptr[r]);
  }
  if (pad4) m = (m + 3) & ~3;  // packed dictionary codes: whole 4-slot groups per slice
  w[s] = 32 * m;
}
__global__ void k_sell_fill(const idx* rowptr, const idx* col, const double* val, int64_t n,
                            const idx* sptr, const idx* perm, idx* scol, double* sval, int with_cols,
                            unsigned char* slen, short* scol16) {
  const int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;  // position
  if (q >= n) return;
  const int64_t r = perm ? perm[q] : q;
  const idx base = sptr[q >> 5] + static_cast<idx>(q & 31), k0 = rowptr[r], len = rowptr[r + 1] - k0;
  slen[q] = static_cast<unsigned char>(len);
  for (idx k = 0; k < len; ++k) {
    if (with_cols) {
      if (scol16)
        scol16[base + 32 * k] = static_cast<short>(col[k0 + k] - static_cast<idx>(r));
      else
        scol[base + 32 * k] = col[k0 + k];
    }
    sval[base + 32 * k] = val[k0 + k];
  }
}

// ---- value dictionary (CSR-VI style) ----------------------------------------------------
// Hash set of the distinct value bit patterns: open addressing over kDictSlots, one CAS per
// new pattern.  A warp first groups equal patterns (__match_any_sync), so a stencil matrix
// costs a few probes per 32 values.  More than kDictMax patterns, or a value whose pattern is
// the empty marker, leaves the operator without a dictionary.
constexpr int kDictSlots = 1024;
constexpr int kDictMax = 256;
constexpr unsigned long long kDictEmpty = ~0ull;

__device__ __forceinline__ unsigned dict_hash(unsigned long long u) {
  u ^= u >> 33;
  u *= 0xff51afd7ed558ccdull;
  u ^= u >> 33;
  return static_cast<unsigned>(u) & (kDictSlots - 1);
}

// Each CTA keeps the patterns it has seen in a shared-memory copy of the set: a value already
// known to the CTA costs one shared probe; only patterns new to the CTA probe (and CAS into)
// the global set.  A stencil operator's ~10^8 values thus cost ~one global probe per distinct
// value per CTA.
__global__ void __launch_bounds__(256) k_dict_insert(const double* __restrict__ val, int64_t nnz,
                                                     unsigned long long* slots,
                                                     int* state /* [count, bad] */) {
  __shared__ unsigned long long seen[kDictSlots];
  for (int q = threadIdx.x; q < kDictSlots; q += blockDim.x) seen[q] = kDictEmpty;
  __syncthreads();
  volatile int* bad = state + 1;
  auto give_up = [&] {
    if (!*bad) atomicExch(state + 1, 1);
  };
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t start = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  // warp-uniform trip count, so every lane reaches the flag check; four values in flight
  constexpr int kU = 4;
  for (int64_t base = start - (threadIdx.x & 31); base < nnz; base += kU * stride) {
    if (__shfl_sync(0xffffffffu, *bad, 0)) return;  // > 256 patterns
    unsigned long long uu[kU];
    unsigned in = 0;
#pragma unroll
    for (int q = 0; q < kU; ++q) {
      const int64_t i = base + q * stride + (threadIdx.x & 31);
      in |= (i < nnz ? 1u : 0u) << q;
      uu[q] = i < nnz ? __double_as_longlong(val[i]) : 0ull;
    }
#pragma unroll
    for (int q = 0; q < kU; ++q) {
      // warp-uniform: every lane takes part in the match; lanes past the end hold a key no
      // value has (the empty marker) and do nothing else
      const bool act = (in >> q) & 1u;
      const unsigned long long u = act ? uu[q] : kDictEmpty;
      const unsigned peers = __match_any_sync(0xffffffffu, u);
      if (!act || (threadIdx.x & 31) != __ffs(peers) - 1) continue;  // one lane per pattern
      if (u == kDictEmpty) {
        give_up();
        continue;
      }
      // the CTA's copy is only a cache: short probe runs (a non-dictionary operator fills it
      // before the give-up is seen, and full-table probes would then cost O(slots) per value)
      constexpr int kLocalProbes = 8;
      unsigned h = dict_hash(u);
      bool known = false;
      for (int probe = 0; probe < kLocalProbes; ++probe, h = (h + 1) & (kDictSlots - 1)) {
        const unsigned long long cur = atomicCAS(seen + h, kDictEmpty, kDictEmpty);  // atomic read
        if (cur == u) {
          known = true;
          break;
        }
        if (cur == kDictEmpty) break;
      }
      if (known) continue;
      h = dict_hash(u);  // new to this CTA: the global set, then the CTA's copy
      for (int probe = 0;; ++probe, h = (h + 1) & (kDictSlots - 1)) {
        if (probe == kDictSlots || *bad) {  // full, or already lost: stop probing
          give_up();
          break;
        }
        const unsigned long long cur = slots[h];
        if (cur == u) break;
        if (cur != kDictEmpty) continue;
        const unsigned long long old = atomicCAS(slots + h, kDictEmpty, u);
        if (old == kDictEmpty) {
          if (atomicAdd(state, 1) >= kDictMax) give_up();
          break;
        }
        if (old == u) break;
      }
      h = dict_hash(u);
      for (int probe = 0; probe < kLocalProbes; ++probe, h = (h + 1) & (kDictSlots - 1)) {
        const unsigned long long old = atomicCAS(seen + h, kDictEmpty, u);
        if (old == kDictEmpty || old == u) break;
      }
    }
  }
}

// A thread per row writes its 4-slot groups whole: one int4 of columns and one 32-bit code
// word per group, so a warp's stores of a group are 512 and 128 contiguous bytes.  The
// dictionary's hash set is looked up from shared memory.
__global__ void __launch_bounds__(256)
    k_sell_codes(const idx* rowptr, const idx* col, const double* val, int64_t n, const idx* sptr,
                 const unsigned long long* __restrict__ slots,
                 const unsigned char* __restrict__ code_of_slot, unsigned char* scode, idx* pcol,
                 unsigned char* slen) {
  __shared__ unsigned long long s_slots[kDictSlots];
  __shared__ unsigned char s_code[kDictSlots];
  for (int q = threadIdx.x; q < kDictSlots; q += blockDim.x) {
    s_slots[q] = slots[q];
    s_code[q] = code_of_slot[q];
  }
  __syncthreads();
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const idx k0 = rowptr[r], len = rowptr[r + 1] - k0;
  slen[r] = static_cast<unsigned char>(len);
  // slots 4g..4g+3 of the row: int4 number sbase / 4 + 32 g + (r & 31) of the packed layout
  int4* pc4 = reinterpret_cast<int4*>(pcol + sptr[r >> 5]) + (r & 31);
  unsigned* cw = reinterpret_cast<unsigned*>(scode + sptr[r >> 5]) + (r & 31);
  for (idx g = 0; 4 * g < len; ++g) {
    int c[4] = {0, 0, 0, 0};
    unsigned w = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const idx k = 4 * g + j;
      if (k < len) {
        const unsigned long long u = __double_as_longlong(val[k0 + k]);
        unsigned h = dict_hash(u);
        while (s_slots[h] != u) h = (h + 1) & (kDictSlots - 1);  // present by construction
        w |= static_cast<unsigned>(s_code[h]) << (8 * j);
        c[j] = col[k0 + k];
      }
    }
    pc4[32 * g] = make_int4(c[0], c[1], c[2], c[3]);
    cw[32 * g] = w;
  }
}

// ---- row-pattern dictionary ------------------------------------------------------------
// A row's pattern = its length, column offsets from the diagonal position and value bit
// patterns.  Rows hash to 64 bits; a global open-addressing set keeps one representative
// row per hash (each CTA first checks a small shared cache of the hashes it has seen); the
// id pass then compares every row with its representative entry by entry, so a hash
// collision can only make the format give up, never change a value.
constexpr int kPatSlots = 8192;
constexpr int kPatMax = 4096;
constexpr int kPatW = 32;  // longest pattern
constexpr int kPatShortRow = 16;  // the format is tried for operators with rows up to this long
constexpr unsigned long long kPatEmpty = ~0ull;

__device__ __forceinline__ unsigned long long pat_mix(unsigned long long h, unsigned long long v) {
  h ^= v + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
  h *= 0xff51afd7ed558ccdull;
  return h ^ (h >> 29);
}
__device__ unsigned long long pat_hash_row(const idx* rowptr, const idx* col, const double* val, int64_t r) {
  const idx k0 = rowptr[r], k1 = rowptr[r + 1];
  unsigned long long h = pat_mix(0x5eedull, static_cast<unsigned long long>(k1 - k0));
  for (idx k = k0; k < k1; ++k) {
    h = pat_mix(h, static_cast<unsigned long long>(static_cast<long long>(col[k]) - r));
    h = pat_mix(h, static_cast<unsigned long long>(__double_as_longlong(val[k])));
  }
  return h == kPatEmpty ? kPatEmpty - 1 : h;
}

__global__ void __launch_bounds__(256) k_pat_insert(const idx* rowptr, const idx* col, const double* val,
                                                    int64_t n, unsigned long long* keys, int* reps,
                                                    unsigned long long* rowhash, int* state) {
  constexpr int kLocal = 256;
  __shared__ unsigned long long seen[kLocal];
  for (int q = threadIdx.x; q < kLocal; q += blockDim.x) seen[q] = kPatEmpty;
  __syncthreads();
  volatile int* bad = state + 1;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t base = static_cast<int64_t>(blockIdx.x) * blockDim.x; base < n; base += stride) {
    if (*bad) return;  // block-uniform: every thread reads the flag at the same trip
    const int64_t r = base + threadIdx.x;
    if (r >= n) continue;
    const unsigned long long h = pat_hash_row(rowptr, col, val, r);
    rowhash[r] = h;
    const unsigned lh = static_cast<unsigned>(h) & (kLocal - 1);
    // a one-way cache shared by the CTA (most rows repeat a recent pattern); atomic accesses:
    // a hit only skips a probe of a pattern that is already in the global set
    if (atomicCAS(seen + lh, h, h) == h) continue;
    unsigned s = static_cast<unsigned>(h >> 20) & (kPatSlots - 1);
    for (int probe = 0;; ++probe, s = (s + 1) & (kPatSlots - 1)) {
      if (probe == kPatSlots || *bad) {
        atomicExch(state + 1, 1);
        break;
      }
      const unsigned long long cur = keys[s];
      if (cur == h) break;
      if (cur != kPatEmpty) continue;
      const unsigned long long old = atomicCAS(keys + s, kPatEmpty, h);
      if (old == kPatEmpty) {
        reps[s] = static_cast<int>(r);
        if (atomicAdd(state, 1) >= kPatMax) atomicExch(state + 1, 1);
        break;
      }
      if (old == h) break;
    }
    atomicExch(seen + lh, h);
  }
}

// pattern tables from the representative rows (one thread per pattern)
__global__ void k_pat_tables(const idx* rowptr, const idx* col, const double* val, const int* rep_rows,
                             int npat, int w, unsigned char* plen, int* pdelta, double* pval) {
  const int p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= npat) return;
  const int64_t r = rep_rows[p];
  const idx k0 = rowptr[r], len = rowptr[r + 1] - k0;
  plen[p] = static_cast<unsigned char>(len);
  for (int j = 0; j < w; ++j) {
    pdelta[p * w + j] = j < len ? static_cast<int>(col[k0 + j] - r) : 0;
    pval[p * w + j] = j < len ? val[k0 + j] : 0.0;
  }
}

// id of every row, checked entry by entry against its pattern's table
__global__ void k_pat_assign(const idx* rowptr, const idx* col, const double* val, int64_t n,
                             const unsigned long long* keys, const unsigned short* slot_id,
                             const unsigned long long* rowhash, const unsigned char* plen,
                             const int* pdelta, const double* pval, int w, unsigned short* id,
                             int* bad) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const unsigned long long h = rowhash[r];
  unsigned s = static_cast<unsigned>(h >> 20) & (kPatSlots - 1);
  int probe = 0;
  while (keys[s] != h && probe < kPatSlots) s = (s + 1) & (kPatSlots - 1), ++probe;
  if (probe == kPatSlots) {
    *bad = 1;
    return;
  }
  const int p = slot_id[s];
  const idx k0 = rowptr[r], len = rowptr[r + 1] - k0;
  bool same = len == plen[p];
  for (idx j = 0; same && j < len; ++j)
    same = (col[k0 + j] - r == pdelta[p * w + j]) &&
           (__double_as_longlong(val[k0 + j]) == __double_as_longlong(pval[p * w + j]));
  if (!same) *bad = 1;  // a 64-bit hash collision: the format is not used
  id[r] = static_cast<unsigned short>(p);
}

constexpr int kStreamThreads = 256;
constexpr int kStreamTarget = 2048;  // staged products per row block (16 KB)

// Row-block plan: about kStreamTarget nonzeros per block (mean row length), staging
// sized to the largest actual block span so the shared-memory carve-out leaves L1
// room for the x gathers of the irregular coarse operators.
void DevCsr::plan() {
  max_row = 0;
  rows_per_block = 1;
  smem_entries = 8;
  if (n_rows == 0) return;
  DevBuf<int> m(1);
  m.zero();
  AGG_LAUNCH(k_max_row, grid_for(n_rows, 256, 4 * sm_count()), 256, 0, rowptr.get(), n_rows, m.get());
  max_row = read_scalar(m.get());
  const double mean = std::max(1.0, static_cast<double>(nnz) / static_cast<double>(n_rows));
  // AGGMG_STREAM_TARGET overrides the staged-products target (tuning experiments)
  static const double target = [] {
    const char* e = std::getenv("AGGMG_STREAM_TARGET");
    return e ? std::max(64.0, std::atof(e)) : static_cast<double>(kStreamTarget);
  }();
  int rpb = static_cast<int>(std::min<double>(kStreamThreads, std::max(1.0, target / mean)));
  while (true) {
    m.zero();
    AGG_LAUNCH(k_max_block_span, grid_for((n_rows + rpb - 1) / rpb, 256, 4 * sm_count()), 256, 0,
               rowptr.get(), n_rows, rpb, m.get());
    const int span = read_scalar(m.get());
    if (static_cast<int64_t>(span + 4) * 8 <= 200 * 1024 || rpb == 1) {
      rows_per_block = rpb;
      smem_entries = span + 4;
      break;
    }
    rpb = std::max(1, rpb / 2);
  }
  // rows longer than the opt-in shared-memory limit (~28k entries) are not supported
  require(static_cast<int64_t>(smem_entries) * 8 <= 227 * 1024,
          "spmv: a row has " + std::to_string(max_row) +
              " entries, beyond the CSR-stream staging capacity");
  // SELL-32 for large square operators with rows of 4-64 entries (AGGMG_SELL=0 disables).
  // Measured (tools/kernel_bench.py): 27-point level 0 0.72 -> 0.99 of peak, 7-point level 0
  // 0.88 -> 0.97, c2 level 1 (13.6 per row) 0.59 -> 0.69; the restriction R (gathers
  // dominate) and the L2-resident coarse levels are slower as SELL and keep CSR-stream.
  static const bool sell_on = [] {
    const char* e = std::getenv("AGGMG_SELL");
    return !(e && e[0] == '0');
  }();
  sell = false;
  static const double sell_min_mean = [] {
    const char* e = std::getenv("AGGMG_SELL_MIN_MEAN");
    return e ? std::atof(e) : 4.0;
  }();
  sell_short = mean < 10.0;
  // near-square: the operators, including a partitioned level's local rows (columns = owned +
  // halo); not the restriction (n_c x n)
  // (slot offsets are int32: every slice padded to the longest row must stay below 2^31)
  const bool fits = ((n_rows + 31) / 32) * 32 * static_cast<int64_t>(max_row) < INT32_MAX;
  // from 2^17 rows (c2 level 2 included: solve -1.3 ms for +1.1 ms of setup, c3 -2.4 ms net;
  // from 2^13 rows the small levels' SELL builds cost more than they save).
  // AGGMG_SELL_MIN_ROWS: tuning experiments
  static const int64_t sell_min_rows = [] {
    const char* e = std::getenv("AGGMG_SELL_MIN_ROWS");
    return e ? std::atoll(e) : (int64_t{1} << 17);
  }();
  // rectangular operators too (the restrictions R: c2 level-0 R 84 -> 59 us with the value
  // dictionary, solve -1.1 ms); AGGMG_SELL_RECT=0: square operators only
  static const bool sell_rect = [] {
    const char* e = std::getenv("AGGMG_SELL_RECT");
    return !(e && e[0] == '0');
  }();
  const bool shape_ok = sell_rect || (n_cols >= n_rows && n_cols <= n_rows + n_rows / 2);
  pat = false;
  pat_id.reset();
  if (sell_on && fits && shape_ok && mean >= sell_min_mean && n_rows >= sell_min_rows && max_row <= 64) {
    const int64_t ns = (n_rows + 31) / 32;
    DevBuf<idx> w(ns);
    DevBuf<unsigned long long> dslots;
    const bool dict = dict_scan(dslots);  // one scan, reused by build_codes below
    // stencil-like operators (a value dictionary and short rows) try the row patterns first
    // (measured: the 7-point level 0 sweeps 1.3-1.4x faster than the dictionary SELL copy;
    // the 27-point rows are slower through the pattern tables and keep SELL)
    const bool square = n_cols >= n_rows && n_cols <= n_rows + n_rows / 2;  // not a restriction
    if (dict && square && max_row <= kPatShortRow && build_patterns()) {
      sell_ptr.reset();
      sell_perm.reset();
      sell_len.reset();
      sell_col.reset();
      sell_val.reset();
      sell_code.reset();
      sell_pcol.reset();
      sell_vi = false;
      return;  // every SpMV epilogue runs on the row patterns
    }
    // the dictionary's packed layout pads slices to whole 4-slot groups; when that busts the
    // slot budget (rows of 4-5 entries pad to 8), the plain unpadded layout is tried next
    const bool fits4 = ns * 32 * int64_t{max_row + 3} < INT32_MAX;
    for (const bool pad4 : {dict && fits4, false}) {
      // the plain layout sorts rows by length inside windows (SELL-C-sigma) unless a row
      // sub-range will be launched on it (sell_sigma_ok = false: partitioned operators)
      if (!pad4 && sell_sigma_ok) {
        sell_perm.resize(n_rows);
        AGG_LAUNCH(k_sell_sort_window, static_cast<unsigned>((n_rows + kSellSigma - 1) / kSellSigma),
                   kSellSigma, 0, rowptr.get(), n_rows, sell_perm.get());
      } else {
        sell_perm.reset();
      }
      AGG_LAUNCH(k_slice_width, grid_for(ns, 256), 256, 0, rowptr.get(), n_rows, ns, pad4 ? 1 : 0,
                 sell_perm.size() ? sell_perm.get() : nullptr, w.get());
      sell_ptr.resize(ns + 1);
      sell_slots = scan_to_offsets(w.get(), sell_ptr.get(), ns);
      if (sell_slots <= static_cast<int64_t>((pad4 ? 1.75 : 1.5) * static_cast<double>(nnz)) + 32 * 64) {
        sell = true;
        sell_pad4 = pad4;
        break;
      }
      if (!pad4) break;
    }
    if (!sell) {
      sell_ptr.reset();
      sell_perm.reset();
      sell_len.reset();
    } else if (sell_pad4) {
      build_codes(dslots);
    } else {
      fill_plain();
    }
  }
}

// the distinct value patterns of val into slots (a kDictSlots hash set); false when there are
// more than kDictMax of them (or the dictionary is switched off: AGGMG_SELL_VI=0 /
// aggmg_set_value_dictionary(0))
std::atomic<int>& value_dictionary_switch() {
  static std::atomic<int> on{[] {
    const char* e = std::getenv("AGGMG_SELL_VI");
    return (e && e[0] == '0') ? 0 : 1;
  }()};
  return on;
}

bool DevCsr::dict_scan(DevBuf<unsigned long long>& slots) const {
  if (!value_dictionary_switch().load() || nnz == 0) return false;
  slots.resize(kDictSlots);
  AGG_CUDA(cudaMemsetAsync(slots.get(), 0xff, kDictSlots * sizeof(unsigned long long), stream()));
  DevBuf<int> state(2);
  state.zero();
  AGG_LAUNCH(k_dict_insert, grid_for(nnz, 256, 8 * sm_count()), 256, 0, val.get(), nnz, slots.get(),
             state.get());
  const std::vector<int> st = state.to_host();
  return st[1] == 0 && st[0] <= kDictMax;
}

// the plain SELL copy (4-byte column + 8-byte value per slot); drops the dictionary
void DevCsr::fill_plain() {
  sell_vi = false;
  sell_code.reset();
  sell_tab.reset();
  sell_pcol.reset();
  // (padding slots are never read: every row stops at its own length)
  // columns as 16-bit offsets from the row when every entry is within 32767 of its row (the
  // coarse operators of the structured problems: c2 / c3 level 1; AGGMG_SELL_D16=0: never)
  static const bool d16_on = [] {
    const char* e = std::getenv("AGGMG_SELL_D16");
    return !(e && e[0] == '0');
  }();
  sell_d16 = false;
  if (d16_on) {
    DevBuf<int> m(1);
    m.zero();
    AGG_LAUNCH(k_max_offset, grid_for(n_rows, 256, 8 * sm_count()), 256, 0, rowptr.get(), col.get(), n_rows,
               m.get());
    sell_d16 = read_scalar(m.get()) <= 32767;
  }
  if (sell_d16) {
    sell_col.reset();
    if (sell_col16.size() != sell_slots) sell_col16.resize(sell_slots);
  } else {
    sell_col16.reset();
    if (sell_col.size() != sell_slots) sell_col.resize(sell_slots);
  }
  if (sell_val.size() != sell_slots) sell_val.resize(sell_slots);
  sell_len.resize(n_rows);
  AGG_LAUNCH(k_sell_fill, grid_for(n_rows, 256), 256, 0, rowptr.get(), col.get(), val.get(), n_rows,
             sell_ptr.get(), sell_perm.size() ? sell_perm.get() : nullptr, sell_col.get(),
             sell_val.get(), 1, sell_len.get(), sell_d16 ? sell_col16.get() : nullptr);
}

// the dictionary copy (packed columns + one-byte codes) from the slots of a successful
// dict_scan; the plain copy is then not kept (the VI kernels never read it)
void DevCsr::build_codes(const DevBuf<unsigned long long>& slots) {
  const std::vector<unsigned long long> hs = slots.to_host();
  std::vector<double> tab;
  std::vector<unsigned char> code(kDictSlots, 0);
  for (int h = 0; h < kDictSlots; ++h) {
    if (hs[h] == kDictEmpty) continue;
    code[h] = static_cast<unsigned char>(tab.size());
    double v;
    std::memcpy(&v, &hs[h], sizeof v);
    tab.push_back(v);
  }
  tab.resize(kDictMax, 0.0);
  sell_tab.resize(kDictMax);
  sell_tab.upload(tab.data(), kDictMax);
  DevBuf<unsigned char> cos(kDictSlots);
  cos.upload(code.data(), kDictSlots);
  if (sell_code.size() != sell_slots) {
    sell_code.resize(sell_slots);
    sell_pcol.resize(sell_slots);
  }
  sell_len.resize(n_rows);
  AGG_LAUNCH(k_sell_codes, grid_for(n_rows, 256), 256, 0, rowptr.get(), col.get(), val.get(), n_rows,
             sell_ptr.get(), slots.get(), cos.get(), sell_code.get(), sell_pcol.get(), sell_len.get());
  sync();  // the temporaries above are freed on return
  sell_vi = true;
  sell_col.reset();
  sell_val.reset();
  sell_col16.reset();
  sell_d16 = false;
}

// AGGMG_PAT=0 / aggmg_set_row_patterns(0): no row-pattern format
std::atomic<int>& row_pattern_switch() {
  static std::atomic<int> on{[] {
    const char* e = std::getenv("AGGMG_PAT");
    return (e && e[0] == '0') ? 0 : 1;
  }()};
  return on;
}
bool pattern_format_on() { return row_pattern_switch().load() != 0; }

bool DevCsr::build_patterns() {
  pat = false;
  pat_id.reset();
  if (!pattern_format_on() || n_rows == 0 || max_row > kPatW || max_row == 0) return false;
  DevBuf<unsigned long long> keys(kPatSlots), rowhash(n_rows);
  DevBuf<int> reps(kPatSlots), state(2);
  AGG_CUDA(cudaMemsetAsync(keys.get(), 0xff, kPatSlots * sizeof(unsigned long long), stream()));
  state.zero();
  AGG_LAUNCH(k_pat_insert, grid_for(n_rows, 256, 8 * sm_count()), 256, 0, rowptr.get(), col.get(),
             val.get(), n_rows, keys.get(), reps.get(), rowhash.get(), state.get());
  const std::vector<int> st = state.to_host();
  if (st[1] != 0 || st[0] > kPatMax) return false;
  const std::vector<unsigned long long> hk = keys.to_host();
  const std::vector<int> hr = reps.to_host();
  std::vector<unsigned short> sid(kPatSlots, 0);
  std::vector<int> rep_rows;
  for (int q = 0; q < kPatSlots; ++q)
    if (hk[q] != kPatEmpty) {
      sid[q] = static_cast<unsigned short>(rep_rows.size());
      rep_rows.push_back(hr[q]);
    }
  const int npat = static_cast<int>(rep_rows.size());
  const int w = (max_row + 7) & ~7;  // whole 8-entry groups: the kernel loads them as vectors
  DevBuf<int> drep(npat);
  drep.upload(rep_rows.data(), npat);
  DevBuf<unsigned short> dsid(kPatSlots);
  dsid.upload(sid.data(), kPatSlots);
  pat_len.resize(npat);
  pat_delta.resize(static_cast<int64_t>(npat) * w);
  pat_val.resize(static_cast<int64_t>(npat) * w);
  AGG_LAUNCH(k_pat_tables, grid_for(npat, 128), 128, 0, rowptr.get(), col.get(), val.get(), drep.get(),
             npat, w, pat_len.get(), pat_delta.get(), pat_val.get());
  pat_id.resize(n_rows);
  DevBuf<int> bad(1);
  bad.zero();
  AGG_LAUNCH(k_pat_assign, grid_for(n_rows, 256), 256, 0, rowptr.get(), col.get(), val.get(), n_rows,
             keys.get(), dsid.get(), rowhash.get(), pat_len.get(), pat_delta.get(), pat_val.get(), w,
             pat_id.get(), bad.get());
  if (read_scalar(bad.get()) != 0) {
    pat_id.reset();
    return false;
  }
  pat_w = w;
  pat = true;
  return true;
}

void DevCsr::refresh_sell() {
  // new values: the same format decision as a fresh plan (row patterns, SELL with or without
  // the dictionary), so a refreshed operator runs exactly the kernels a new setup would
  if (n_rows == 0 || (!sell && !pat)) return;
  plan();
}

DevCsrPtr upload_csr(int64_t n_rows, int64_t n_cols, const int64_t* rowptr, const int64_t* col,
                     const double* val, bool validate) {
  require(n_rows >= 0 && n_cols >= 0, "negative dimensions");
  const int64_t nnz = rowptr[n_rows];
  if (validate) {
    require(rowptr[0] == 0, "row_offsets[0] must be 0");
    require(nnz >= 0, "row_offsets[n_rows] must equal nnz");
  }
  require(n_rows < (1LL << 31) - 1 && n_cols < (1LL << 31) - 1 && nnz < (1LL << 31) - 1,
          "matrix exceeds the int32 device index range (2^31 rows / nonzeros per GPU)");
  auto A = std::make_shared<DevCsr>();
  A->n_rows = n_rows;
  A->n_cols = n_cols;
  A->nnz = nnz;
  A->rowptr.resize(n_rows + 1);
  A->col.resize(nnz);
  A->val.resize(nnz);
  // indices are narrowed to int32 on the host while staging; range checks ride along,
  // ordering checks run on the device over the narrowed arrays
  DevBuf<int> bad(1);
  fill_int(bad.get(), 1, INT32_MAX);
  int64_t bad_rp = -1, bad_col = -1;
  host_to_device_narrow(A->rowptr.get(), rowptr, static_cast<size_t>(n_rows + 1), 0, nnz + 1, &bad_rp);
  host_to_device_narrow(A->col.get(), col, static_cast<size_t>(nnz), 0, validate ? n_cols : INT32_MAX,
                        &bad_col);
  if (nnz > 0) host_to_device_values(A->val.get(), val, static_cast<size_t>(nnz));
  if (n_rows > 0)
    AGG_LAUNCH(k_check_rows, grid_for(n_rows, 256), 256, 0, A->rowptr.get(), A->col.get(), n_rows,
               nnz, bad.get(), validate ? 1 : 0);
  int bad_row = read_scalar(bad.get());
  if (bad_rp >= 0) bad_row = std::min<int64_t>(bad_row, std::max<int64_t>(0, bad_rp - 1));
  if (bad_col >= 0 && bad_row != 0) {  // the row holding the first out-of-range column
    const int64_t r = std::upper_bound(rowptr, rowptr + n_rows + 1, bad_col) - rowptr - 1;
    bad_row = static_cast<int>(std::min<int64_t>(bad_row, std::max<int64_t>(0, r)));
  }
  if (bad_row != INT32_MAX) {
    // Reproduce the reference's first failing check for that row (sparse.cpp:29-38).
    const int64_t i = bad_row;
    if (rowptr[i] > rowptr[i + 1]) throw Error("row_offsets must be non-decreasing");
    if (rowptr[i] < 0 || rowptr[i + 1] > nnz) throw Error("row_offsets[n_rows] must equal nnz");
    for (int64_t k = rowptr[i]; k < rowptr[i + 1]; ++k) {
      if (col[k] < 0 || col[k] >= n_cols)
        throw Error("column index out of range in row " + std::to_string(i));
      if (k > rowptr[i] && col[k - 1] >= col[k])
        throw Error("columns must be strictly increasing in row " + std::to_string(i));
    }
  }
  A->plan();
  return A;
}

void download_csr(const DevCsr& A, int64_t* rowptr, int64_t* col, double* val) {
  DevBuf<int64_t> rp(A.n_rows + 1), c(A.nnz);
  AGG_LAUNCH(k_widen, grid_for(A.n_rows + 1, 256), 256, 0, A.rowptr.get(), rp.get(), A.n_rows + 1);
  if (A.nnz > 0) AGG_LAUNCH(k_widen, grid_for(A.nnz, 256), 256, 0, A.col.get(), c.get(), A.nnz);
  rp.download(rowptr, A.n_rows + 1);
  if (col) c.download(col, A.nnz);
  if (val) A.val.download(val, A.nnz);
  sync();
}

// ---- CSR-stream SpMV family ----------------------------------------------------------

namespace {

template <Epi E>
struct EpiTraits {
  static constexpr int np = (E == Epi::kSpmvDot1) ? 1
                            : (E == Epi::kSpmvDot2 || E == Epi::kJacobiDot2) ? 2
                            : (E == Epi::kSpmvDot3) ? 3 : 0;
};

// Persistent CSR-stream kernel: each CTA walks row blocks rb = blockIdx.x, +gridDim.x, ...
// For every row block, phase 1 streams the block's contiguous nonzero range with 128-bit
// loads and stages val * x[col] in shared memory; phase 2 sums each row sequentially in
// storage order and applies the epilogue.  Fused dot products accumulate per thread
// across row blocks and are reduced once per CTA (fixed grid => deterministic).
// Per-row epilogue of the SpMV family: y / residual / Jacobi / scaled output and the fused
// dot contributions, from the row's sequential sum.
// The row's epilogue operands (x_r, d_r, b_r, c_r, u_r as the epilogue needs them), loaded
// apart from the sum so the SELL kernels can issue them before the row's gathers.
struct EpiIn {
  double xr, d, b, c, u;
};
template <Epi E>
__device__ __forceinline__ EpiIn epi_load(const SpmvArgs& a, const double* __restrict__ x, int64_t rg) {
  constexpr int NP = EpiTraits<E>::np;
  EpiIn e{0.0, 0.0, 0.0, 0.0, 0.0};
  if constexpr (E == Epi::kJacobiDot2 || E == Epi::kJacobi) {
    e.xr = x[rg];
    e.d = a.d[rg];
    e.b = a.b[rg];
    if constexpr (E == Epi::kJacobiDot2) e.c = a.c[rg];
  } else if constexpr (E == Epi::kResidual) {
    e.b = a.b[rg];
  } else if constexpr (E == Epi::kResidualZero) {
    e.b = a.b[rg];
    e.d = a.d[rg];
  } else if constexpr (E == Epi::kSpmvZero || E == Epi::kScaleDiag) {
    e.d = a.d[rg];
  } else if constexpr (NP == 1) {
    e.u = a.u[rg];
  } else if constexpr (NP > 1) {
    if (a.dot_with_x) e.xr = x[rg];
    e.c = a.c[rg];
    if constexpr (NP == 3) e.u = a.u[rg];
  }
  return e;
}

template <Epi E>
__device__ __forceinline__ void row_epilogue_in(const SpmvArgs& a, const EpiIn& e, int64_t rg,
                                                double sum, double* v) {
  constexpr int NP = EpiTraits<E>::np;
  double yv = sum;
  if constexpr (E == Epi::kJacobiDot2) {
    yv = __dadd_rn(e.xr, __dmul_rn(e.d, __dsub_rn(e.b, sum)));
    a.y[rg] = yv;
  } else if constexpr (E == Epi::kSpmv || NP > 0) {
    a.y[rg] = sum;
  } else if constexpr (E == Epi::kResidual) {
    a.y[rg] = __dsub_rn(e.b, sum);
  } else if constexpr (E == Epi::kResidualZero) {
    a.y[rg] = __dsub_rn(e.b, sum);                          // r = b - A x1
    a.x_out[rg] = __dadd_rn(0.0, __dmul_rn(e.d, e.b));      // x1 = 0 + wd b
  } else if constexpr (E == Epi::kJacobi) {
    a.y[rg] = __dadd_rn(e.xr, __dmul_rn(e.d, __dsub_rn(e.b, sum)));
  } else if constexpr (E == Epi::kSpmvZero) {
    a.y[rg] = sum;
    a.x_out[rg] = __dadd_rn(0.0, __dmul_rn(e.d, sum));  // k_jacobi_zero's operation
  } else if constexpr (E == Epi::kScaleDiag) {
    a.y[rg] = __dmul_rn(sum, e.d);
  }
  if constexpr (E == Epi::kJacobiDot2) {
    v[0] = __dadd_rn(v[0], __dmul_rn(e.b, yv));  // r . z
    v[1] = __dadd_rn(v[1], __dmul_rn(e.c, yv));  // r_old . z
  } else if constexpr (NP > 0) {
    const double lhs = a.dot_with_x ? e.xr : sum;
    if constexpr (NP == 1) {
      v[0] = __dadd_rn(v[0], __dmul_rn(e.u, sum));
    } else if constexpr (NP == 2) {
      v[0] = __dadd_rn(v[0], __dmul_rn(lhs, sum));  // rho  = v.v (gmres) | c.v (cg)
      v[1] = __dadd_rn(v[1], __dmul_rn(lhs, e.c));  // alpha = v.rc       | c.rc
    } else {
      v[0] = __dadd_rn(v[0], __dmul_rn(lhs, e.u));  // gamma = w.v | d.v
      v[1] = __dadd_rn(v[1], __dmul_rn(lhs, sum));  // beta  = w.w | d.w
      v[2] = __dadd_rn(v[2], __dmul_rn(lhs, e.c));  // alpha2 = w.rt | d.rt
    }
  }
}

template <Epi E>
__device__ __forceinline__ void row_epilogue(const SpmvArgs& a, const double* __restrict__ x,
                                             int64_t rg, double sum, double* v) {
  row_epilogue_in<E>(a, epi_load<E>(a, x, rg), rg, sum, v);
}

template <Epi E>
__global__ void __launch_bounds__(kStreamThreads)
    k_csr_stream(const idx* __restrict__ rowptr, const idx* __restrict__ col,
                 const double* __restrict__ val, int64_t n_rows, int rpb, int64_t nblocks,
                 SpmvArgs a, double* partials, unsigned* ticket) {
  extern __shared__ __align__(16) double prod[];
  constexpr int NP = EpiTraits<E>::np;
  constexpr int NPX = NP > 0 ? NP : 1;
  __shared__ __align__(16) double red_smem[32 * 3 + 2];
  if (a.pred && !*a.pred) return;
  const double* __restrict__ x = a.x;
  double v[NPX];
#pragma unroll
  for (int k = 0; k < NPX; ++k) v[k] = 0.0;

  for (int64_t rb = blockIdx.x; rb < nblocks; rb += gridDim.x) {
    const int64_t r0 = rb * rpb;
    const int64_t r1 = min(r0 + static_cast<int64_t>(rpb), n_rows);
    const idx e0 = rowptr[r0], e1 = rowptr[r1];

    // Phase 1: stream the row block's nonzeros.  Thread t owns entry pairs
    // (ea + 2t + 512k, +1): 128-bit value loads, 64-bit column loads, both fully
    // coalesced; two pairs are issued before their gathers to keep 4 gathers in flight.
    // Products land in shared memory at [e - ea] (pairs 16-byte aligned, so the
    // 128-bit stores are bank-conflict free); slots outside [e0, e1) are never read.
    const idx ea = e0 & ~1;
    // two iterations unrolled: both pairs' loads issue before the first gathers (level-0
    // kernels +1-2 % of peak; 4 measured no better)
#pragma unroll 2
    for (idx e = ea + 2 * static_cast<idx>(threadIdx.x); e < e1; e += 4 * kStreamThreads) {
      const idx eb = e + 2 * kStreamThreads;
      const bool hb = eb < e1;
      const int2 ca = __ldcs(reinterpret_cast<const int2*>(col + e));
      const double2 va = __ldcs(reinterpret_cast<const double2*>(val + e));
      int2 cb = make_int2(0, 0);
      double2 vb = make_double2(0.0, 0.0);
      if (hb) {
        cb = __ldcs(reinterpret_cast<const int2*>(col + eb));
        vb = __ldcs(reinterpret_cast<const double2*>(val + eb));
      }
      const bool a0 = e >= e0, a1 = e + 1 < e1, b1 = hb && eb + 1 < e1;
      double xa0 = 0.0, xa1 = 0.0, xb0 = 0.0, xb1 = 0.0;
      if constexpr (E == Epi::kResidualZero) {
        // x = 0 + wd .* b evaluated on the fly for the gathered neighbours
        auto xz = [&](idx c) { return __dadd_rn(0.0, __dmul_rn(__ldg(a.d + c), __ldg(a.b + c))); };
        if (a0) xa0 = xz(ca.x);
        if (a1) xa1 = xz(ca.y);
        if (hb) xb0 = xz(cb.x);
        if (b1) xb1 = xz(cb.y);
      } else {
        if (a0) xa0 = __ldg(x + ca.x);
        if (a1) xa1 = __ldg(x + ca.y);
        if (hb) xb0 = __ldg(x + cb.x);
        if (b1) xb1 = __ldg(x + cb.y);
      }
      *reinterpret_cast<double2*>(prod + (e - ea)) =
          make_double2(__dmul_rn(va.x, xa0), __dmul_rn(va.y, xa1));
      if (hb)
        *reinterpret_cast<double2*>(prod + (eb - ea)) =
            make_double2(__dmul_rn(vb.x, xb0), __dmul_rn(vb.y, xb1));
    }
    __syncthreads();

    // Phase 2: one thread per row, sequential sum in storage order (sparse.cpp:58-61).
    const int64_t r = r0 + threadIdx.x;
    if (threadIdx.x < rpb && r < r1) {
      const idx s = rowptr[r] - ea, t = rowptr[r + 1] - ea;
      const int64_t rg = r + a.row_base;  // row index of the epilogue vectors
      double sum = 0.0;
      for (idx k = s; k < t; ++k) sum = __dadd_rn(sum, prod[k]);
      row_epilogue<E>(a, x, rg, sum, v);
    }
    __syncthreads();  // prod is reused by the next row block
  }
  if constexpr (NP > 0) {
    block_reduce<NPX>(v, red_smem);
    if (threadIdx.x == 0)
#pragma unroll
      for (int k = 0; k < NP; ++k) partials[blockIdx.x * NP + k] = v[k];
    finish_reduction<NPX>(partials, ticket, a.dots_out, red_smem);
  }
}

// SELL-32 SpMV family: a thread per row, a warp per slice; slot k of the 32 rows of a warp is
// one coalesced 256-byte load of values and 128 bytes of columns, no staging and no block
// barriers.  Each row sums its own entries in CSR order (the slot order), and the same
// epilogues apply: bit-identical to k_csr_stream.
// With the value dictionary (VI) a slot's value is one byte, its code into the operator's
// table of distinct values (shared memory); the value, and so every sum, is the same double.
// Tuning variants of the SELL kernels: g = 4-slot groups per step (VI layout), pf = the next
// step's columns / codes load under this step's gathers, pre = the row's epilogue operands
// load before its gathers, minb = __launch_bounds__ min blocks (caps registers for occupancy).
// Each (epilogue, layout) pair uses the variant sell_tune() picks (tools/kernel_bench.py over
// a sweep build: tools/build_variant.sh NAME -DAGGMG_SELL_SWEEP, AGGMG_SELL_TUNE=<variant>).
struct SellTune {
  int g, pf, pre, minb, legacy = 0;  // legacy: 4 slots per step, loads then gathers, no predication
};
constexpr SellTune kSellTunes[] = {
    {1, 0, 0, 1}, {1, 0, 0, 8}, {1, 1, 0, 8}, {1, 1, 1, 6}, {2, 1, 0, 1}, {1, 1, 1, 1},
    {2, 1, 1, 1}, {1, 1, 0, 6}, {2, 1, 0, 6}, {1, 0, 1, 8}, {1, 1, 0, 1}, {2, 1, 0, 4},
    {1, 0, 0, 1, 1}, {1, 0, 0, 8, 1}, {1, 0, 1, 1, 1}, {1, 0, 0, 6, 1},
};
constexpr int kSellTuneCount = sizeof(kSellTunes) / sizeof(kSellTunes[0]);
// measured on B200 (profiles/r02_sell_tune_sweep.txt, tools/kernel_bench.py at c2 and c4):
// the plain layout wants prefetch (short rows: with the epilogue preload at 6 CTAs per SM);
// the dictionary layout with short rows (7-point) wants 32 registers (8 CTAs per SM); with
// long rows (27-point) the plain-loop variants win, at 32 registers for the fused-dot
// epilogues and 2-group prefetch otherwise
constexpr int sell_tune(Epi e, bool vi, bool short_rows) {
  if (!vi) return short_rows ? 3 : 10;
  const bool dots = e == Epi::kSpmvDot1 || e == Epi::kSpmvDot2 || e == Epi::kSpmvDot3 ||
                    e == Epi::kJacobiDot2;
  if (short_rows) return e == Epi::kSpmvDot1 ? 2 : 1;
  return dots ? 13 : 4;
}

// D16 (plain layout only): columns stored as 16-bit offsets from the row
template <Epi E, bool VI, int T, bool D16 = false>
__global__ void __launch_bounds__(256, kSellTunes[T].minb)
    k_sell(const idx* __restrict__ rowptr, const idx* __restrict__ sptr, const idx* __restrict__ scol,
           const double* __restrict__ sval, const unsigned char* __restrict__ scode,
           const idx* __restrict__ pcol, const double* __restrict__ stab, const idx* __restrict__ perm,
           const unsigned char* __restrict__ slen, int64_t row0, int64_t n, SpmvArgs a,
           double* partials, unsigned* ticket, const short* __restrict__ scol16) {
  static_assert(!(VI && D16), "16-bit offsets only in the plain layout");
  constexpr int NP = EpiTraits<E>::np;
  constexpr int NPX = NP > 0 ? NP : 1;
  __shared__ __align__(16) double red_smem[32 * 3 + 2];
  __shared__ double s_tab[VI ? 256 : 1];
  if (a.pred && !*a.pred) return;
  if constexpr (VI) {
    s_tab[threadIdx.x] = stab[threadIdx.x];  // blockDim.x == 256 == the table size
    __syncthreads();
  }
  const double* __restrict__ x = a.x;
  double v[NPX];
#pragma unroll
  for (int k = 0; k < NPX; ++k) v[k] = 0.0;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  // positions [row0, row0 + n) (a sub-range of rows for the partitioned path's interior /
  // boundary split; SELL-C-sigma copies are only built where no sub-range is launched)
  for (int64_t q = row0 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < row0 + n;
       q += stride) {
    // the position's length and slice base and the row's epilogue operands are independent
    // loads: they all issue before the first column load (no rowptr round trip)
    const int64_t r = perm ? static_cast<int64_t>(__ldg(perm + q)) : q;
    const int len = slen[q];
    const idx sbase = sptr[q >> 5];
    constexpr SellTune tune = kSellTunes[T];
    EpiIn ein;
    if constexpr (tune.pre) ein = epi_load<E>(a, x, r);
    double sum = 0.0;
    if constexpr (VI && tune.legacy) {
      const unsigned* cw = reinterpret_cast<const unsigned*>(scode + sbase) + (q & 31);
      const int4* pc = reinterpret_cast<const int4*>(pcol + sbase) + (q & 31);
      for (int k = 0; k < len; k += 4) {
        const unsigned w = __ldcs(cw + 8 * k);  // + 32 (k / 4) words
        const int4 cq4 = __ldcs(pc + 8 * k);
        if (k + 4 <= len) {
          const double x0 = __ldg(x + cq4.x), x1 = __ldg(x + cq4.y), x2 = __ldg(x + cq4.z),
                       x3 = __ldg(x + cq4.w);
          sum = __dadd_rn(sum, __dmul_rn(s_tab[w & 255u], x0));
          sum = __dadd_rn(sum, __dmul_rn(s_tab[(w >> 8) & 255u], x1));
          sum = __dadd_rn(sum, __dmul_rn(s_tab[(w >> 16) & 255u], x2));
          sum = __dadd_rn(sum, __dmul_rn(s_tab[w >> 24], x3));
        } else {
          const idx cq[4] = {cq4.x, cq4.y, cq4.z, cq4.w};
#pragma unroll
          for (int j = 0; j < 3; ++j)
            if (j < len - k) sum = __dadd_rn(sum, __dmul_rn(s_tab[(w >> (8 * j)) & 255u], __ldg(x + cq[j])));
        }
      }
    } else if constexpr (!VI && tune.legacy) {
      const idx* c = scol + sbase + (q & 31);
      const double* vv = sval + sbase + (q & 31);
      int k = 0;
      for (; k + 4 <= len; k += 4) {
        const idx c0 = __ldcs(c + 32 * k), c1 = __ldcs(c + 32 * (k + 1)), c2 = __ldcs(c + 32 * (k + 2)),
                  c3 = __ldcs(c + 32 * (k + 3));
        const double v0 = __ldcs(vv + 32 * k), v1 = __ldcs(vv + 32 * (k + 1)),
                     v2 = __ldcs(vv + 32 * (k + 2)), v3 = __ldcs(vv + 32 * (k + 3));
        const double x0 = __ldg(x + c0), x1 = __ldg(x + c1), x2 = __ldg(x + c2), x3 = __ldg(x + c3);
        sum = __dadd_rn(sum, __dmul_rn(v0, x0));
        sum = __dadd_rn(sum, __dmul_rn(v1, x1));
        sum = __dadd_rn(sum, __dmul_rn(v2, x2));
        sum = __dadd_rn(sum, __dmul_rn(v3, x3));
      }
      for (; k < len; ++k) sum = __dadd_rn(sum, __dmul_rn(__ldcs(vv + 32 * k), __ldg(x + __ldcs(c + 32 * k))));
    } else if constexpr (VI) {
      // codes of slots k..k+3: one 32-bit word per row (the packed layout, sell_code)
      const unsigned* cw = reinterpret_cast<const unsigned*>(scode + sbase) + (q & 31);
      // columns in the same packing (sell_pcol): slots k..k+3 of a row are one int4
      const int4* pc = reinterpret_cast<const int4*>(pcol + sbase) + (q & 31);
      // G 4-slot groups per step; with pf the next step's codes and columns load under this
      // step's gathers
      constexpr int G = tune.g;
      unsigned w[G];
      int4 c[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        w[g] = 4 * g < len ? __ldcs(cw + 32 * g) : 0u;
        c[g] = 4 * g < len ? __ldcs(pc + 32 * g) : make_int4(0, 0, 0, 0);
      }
      for (int k = 0; k < len; k += 4 * G) {
        const int m = len - k;  // slots left in this row
        if (!tune.pf && k > 0) {
#pragma unroll
          for (int g = 0; g < G; ++g)
            if (4 * g < m) {
              w[g] = __ldcs(cw + 8 * (k + 4 * g));
              c[g] = __ldcs(pc + 8 * (k + 4 * g));
            }
        }
        double xs[4 * G];
        unsigned u[G];
#pragma unroll
        for (int g = 0; g < G; ++g) {
          u[g] = w[g];
          xs[4 * g] = 4 * g < m ? __ldg(x + c[g].x) : 0.0;
          xs[4 * g + 1] = 4 * g + 1 < m ? __ldg(x + c[g].y) : 0.0;
          xs[4 * g + 2] = 4 * g + 2 < m ? __ldg(x + c[g].z) : 0.0;
          xs[4 * g + 3] = 4 * g + 3 < m ? __ldg(x + c[g].w) : 0.0;
        }
#pragma unroll
        for (int g = 0; g < G; ++g)
          if (tune.pf && 4 * (G + g) < m) {
            w[g] = __ldcs(cw + 8 * (k + 4 * (G + g)));
            c[g] = __ldcs(pc + 8 * (k + 4 * (G + g)));
          }
#pragma unroll
        for (int j = 0; j < 4 * G; ++j)
          if (j < m) sum = __dadd_rn(sum, __dmul_rn(s_tab[(u[j >> 2] >> (8 * (j & 3))) & 255u], xs[j]));
      }
    } else {
      static_assert(!(D16 && tune.legacy), "16-bit offsets in the prefetching loop only");
      const idx* c = scol + sbase + (q & 31);
      const short* c16 = scol16 + sbase + (q & 31);
      const double* vv = sval + sbase + (q & 31);
      const idx ri = static_cast<idx>(r);
      auto ldc = [&](int off) -> idx {
        if constexpr (D16)
          return ri + static_cast<idx>(__ldcs(c16 + off));
        else
          return __ldcs(c + off);
      };
      // W = 4 g slots per step; the next step's columns and values load under this step's gathers
      constexpr int W = 4 * tune.g;
      idx cc[W];
      double vq[W];
#pragma unroll
      for (int j = 0; j < W; ++j) {
        cc[j] = j < len ? ldc(32 * j) : 0;
        vq[j] = j < len ? __ldcs(vv + 32 * j) : 0.0;
      }
      for (int k = 0; k < len; k += W) {
        const int m = len - k;
        if (!tune.pf && k > 0) {
#pragma unroll
          for (int j = 0; j < W; ++j) {
            cc[j] = j < m ? ldc(32 * (k + j)) : 0;
            vq[j] = j < m ? __ldcs(vv + 32 * (k + j)) : 0.0;
          }
        }
        double xs[W], vs[W];
#pragma unroll
        for (int j = 0; j < W; ++j) {
          xs[j] = j < m ? __ldg(x + cc[j]) : 0.0;
          vs[j] = vq[j];
        }
        if (tune.pf) {
#pragma unroll
          for (int j = 0; j < W; ++j) {
            cc[j] = j + W < m ? ldc(32 * (k + W + j)) : 0;
            vq[j] = j + W < m ? __ldcs(vv + 32 * (k + W + j)) : 0.0;
          }
        }
#pragma unroll
        for (int j = 0; j < W; ++j)
          if (j < m) sum = __dadd_rn(sum, __dmul_rn(vs[j], xs[j]));
      }
    }
    if constexpr (!tune.pre) ein = epi_load<E>(a, x, r);
    row_epilogue_in<E>(a, ein, r, sum, v);
  }
  if constexpr (NP > 0) {
    block_reduce<NPX>(v, red_smem);
    if (threadIdx.x == 0)
#pragma unroll
      for (int k = 0; k < NP; ++k) partials[blockIdx.x * NP + k] = v[k];
    finish_reduction<NPX>(partials, ticket, a.dots_out, red_smem);
  }
}

template <Epi E, bool VI, int T, bool D16 = false>
void launch_sell_t(const DevCsr& A, const SpmvArgs& a) {
  static std::atomic<int> per_sm_cache{0};
  int per_sm = per_sm_cache.load();
  if (!per_sm) {
    AGG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_sell<E, VI, T, D16>, 256, 0));
    per_sm = std::max(1, per_sm);
    per_sm_cache.store(per_sm);
  }
  const int64_t nrows = a.row_count >= 0 ? a.row_count : A.n_rows - a.row_base;
  const int64_t grid = std::min<int64_t>(grid_for(nrows, 256), static_cast<int64_t>(per_sm) * sm_count());
  const auto kern = k_sell<E, VI, T, D16>;
  AGG_LAUNCH(kern, static_cast<unsigned>(grid), 256, 0, A.rowptr.get(), A.sell_ptr.get(),
             A.sell_col.get(), A.sell_val.get(), A.sell_code.get(), A.sell_pcol.get(), A.sell_tab.get(),
             A.sell_perm.size() ? A.sell_perm.get() : nullptr, A.sell_len.get(), a.row_base, nrows, a,
             reduce_partials(), reduce_ticket(), A.sell_col16.get());
}

#ifdef AGGMG_SELL_SWEEP
// tuning build: AGGMG_SELL_TUNE=<variant> runs every SELL launch with that variant
template <Epi E, bool VI, int T = 0>
void launch_sell_sweep(const DevCsr& A, const SpmvArgs& a, int t) {
  if constexpr (T < kSellTuneCount) {
    if (t == T)
      launch_sell_t<E, VI, T>(A, a);
    else
      launch_sell_sweep<E, VI, T + 1>(A, a, t);
  }
}
int sell_sweep_variant() {
  static const int t = [] {
    const char* e = std::getenv("AGGMG_SELL_TUNE");
    return e ? std::atoi(e) : -1;
  }();
  return t;
}
#endif

template <Epi E, bool VI>
void launch_sell_v(const DevCsr& A, const SpmvArgs& a) {
#ifdef AGGMG_SELL_SWEEP
  if (sell_sweep_variant() >= 0 && !A.sell_d16) {
    launch_sell_sweep<E, VI>(A, a, sell_sweep_variant());
    return;
  }
#endif
  if constexpr (!VI) {
    if (A.sell_d16) {
      if (A.sell_short)
        launch_sell_t<E, false, sell_tune(E, false, true), true>(A, a);
      else
        launch_sell_t<E, false, sell_tune(E, false, false), true>(A, a);
      return;
    }
  }
  if (A.sell_short)
    launch_sell_t<E, VI, sell_tune(E, VI, true)>(A, a);
  else
    launch_sell_t<E, VI, sell_tune(E, VI, false)>(A, a);
}

template <Epi E>
void launch_sell(const DevCsr& A, const SpmvArgs& a) {
  if (A.sell_vi)
    launch_sell_v<E, true>(A, a);
  else
    launch_sell_v<E, false>(A, a);
}

// Row-pattern SpMV family: a thread per row reads its two-byte pattern id; the pattern's
// offsets and values come from the (L1-resident) tables, the x gathers and the epilogue as
// in k_sell.  Same products, same order: bit-identical to k_csr_stream / k_sell.
// __launch_bounds__ min blocks per epilogue (register caps; measured on the c2 level 0 with
// tools/kernel_bench.py: spmv / residual / Arnoldi 93-98 us at 5 CTAs per SM, the fused dots
// of the Jacobi sweep 125 us at 4, the plain Jacobi and PCG's SpMV + dot uncapped)
constexpr int pat_min_blocks(Epi e) {
  return (e == Epi::kSpmv || e == Epi::kResidual || e == Epi::kScaleDiag) ? 5
         : (e == Epi::kJacobiDot2 || e == Epi::kSpmvDot2 || e == Epi::kSpmvDot3) ? 4
                                                                                  : 1;
}
template <Epi E>
__global__ void __launch_bounds__(256, pat_min_blocks(E))
    k_pat(const unsigned short* __restrict__ pid, const unsigned char* __restrict__ plen,
          const int* __restrict__ pdelta, const double* __restrict__ pval, int w, int64_t row0,
          int64_t n, SpmvArgs a, double* partials, unsigned* ticket) {
  constexpr int NP = EpiTraits<E>::np;
  constexpr int NPX = NP > 0 ? NP : 1;
  __shared__ __align__(16) double red_smem[32 * 3 + 2];
  if (a.pred && !*a.pred) return;
  const double* __restrict__ x = a.x;
  double v[NPX];
#pragma unroll
  for (int k = 0; k < NPX; ++k) v[k] = 0.0;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  int64_t r = row0 + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  int p = r < row0 + n ? pid[r] : 0;
  for (; r < row0 + n; r += stride) {
    const int pn = r + stride < row0 + n ? pid[r + stride] : 0;  // the next row's id in flight
    const EpiIn ein = epi_load<E>(a, x, r);
    const int len = __ldg(plen + p);
    // the pattern's offsets and values: 8-entry groups as 16-byte loads (w is a multiple of 8)
    const int4* dl = reinterpret_cast<const int4*>(pdelta + p * w);
    const double2* vl = reinterpret_cast<const double2*>(pval + p * w);
    const int ri = static_cast<int>(r);  // operators are < 2^31 rows
    double sum = 0.0;
#pragma unroll 1
    for (int k = 0; k < len; k += 8) {
      const int4 d0 = __ldg(dl + k / 4), d1 = __ldg(dl + k / 4 + 1);
      const int dd[8] = {d0.x, d0.y, d0.z, d0.w, d1.x, d1.y, d1.z, d1.w};
      double xs[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) xs[j] = k + j < len ? __ldg(x + (ri + dd[j])) : 0.0;
      double vs[8];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const double2 t = __ldg(vl + k / 2 + j);
        vs[2 * j] = t.x;
        vs[2 * j + 1] = t.y;
      }
      // a group's slots past the row's length hold the value +0 and the x operand is +0, so
      // they add +0: the running sum, which starts at +0 and so is never -0 (round to
      // nearest), is unchanged bit for bit — no per-slot predicate on the chain
#pragma unroll
      for (int j = 0; j < 8; ++j) sum = __dadd_rn(sum, __dmul_rn(vs[j], xs[j]));
    }
    row_epilogue_in<E>(a, ein, r, sum, v);
    p = pn;
  }
  if constexpr (NP > 0) {
    block_reduce<NPX>(v, red_smem);
    if (threadIdx.x == 0)
#pragma unroll
      for (int k = 0; k < NP; ++k) partials[blockIdx.x * NP + k] = v[k];
    finish_reduction<NPX>(partials, ticket, a.dots_out, red_smem);
  }
}

template <Epi E>
void launch_pat(const DevCsr& A, const SpmvArgs& a) {
  static std::atomic<int> per_sm_cache{0};
  int per_sm = per_sm_cache.load();
  if (!per_sm) {
    AGG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_pat<E>, 256, 0));
    per_sm = std::max(1, per_sm);
    per_sm_cache.store(per_sm);
  }
  const int64_t nrows = a.row_count >= 0 ? a.row_count : A.n_rows - a.row_base;
  const int64_t grid = std::min<int64_t>(grid_for(nrows, 256), static_cast<int64_t>(per_sm) * sm_count());
  AGG_LAUNCH(k_pat<E>, static_cast<unsigned>(grid), 256, 0, A.pat_id.get(), A.pat_len.get(),
             A.pat_delta.get(), A.pat_val.get(), A.pat_w, a.row_base, nrows, a, reduce_partials(),
             reduce_ticket());
}

template <Epi E>
void launch_stream(const DevCsr& A, const SpmvArgs& a) {
  const int64_t nrows = a.row_count >= 0 ? a.row_count : A.n_rows - a.row_base;
  if (nrows <= 0) return;
  if constexpr (E != Epi::kResidualZero) {
    if (A.pat) {
      launch_pat<E>(A, a);
      return;
    }
    // short rows (7-point level 0): the Jacobi + PCG-dots sweep measured faster as CSR-stream
    // (0.845 vs 0.824 of peak), every other epilogue faster as SELL (0.95-0.97 vs 0.86-0.89)
    const bool skip = E == Epi::kJacobiDot2 && A.sell_short && !(A.sell_vi && fuse_dots_on_dictionary());
    if (A.sell && !skip) {
      launch_sell<E>(A, a);
      return;
    }
  }
  const int64_t nblocks = (nrows + A.rows_per_block - 1) / A.rows_per_block;
  const size_t smem = sizeof(double) * A.smem_entries;
  static std::atomic<unsigned long long> raised{0};
  if (smem > 48 * 1024 && device_pending(raised)) {
    AGG_CUDA(cudaFuncSetAttribute(k_csr_stream<E>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  226 * 1024));  // + the static reduction scratch <= 227 KB
    mark_device(raised);
  }
  // persistent grid: as many CTAs as can be co-resident
  static thread_local size_t cached_smem = 0;
  static thread_local int cached_per_sm = 0;
  if (cached_smem != smem) {
    int per_sm = 0;
    AGG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_csr_stream<E>,
                                                           kStreamThreads, smem));
    cached_per_sm = std::max(1, per_sm);
    cached_smem = smem;
  }
  const int64_t grid = std::min<int64_t>(nblocks, static_cast<int64_t>(cached_per_sm) * sm_count());
  AGG_LAUNCH(k_csr_stream<E>, static_cast<unsigned>(grid), kStreamThreads, smem,
             A.rowptr.get() + a.row_base, A.col.get(), A.val.get(), nrows, A.rows_per_block, nblocks,
             a, reduce_partials(), reduce_ticket());
}

}  // namespace

// AGGMG_DICT_DOTS=0: PCG's (r.z, r_old.z) as a separate pass even on a dictionary operator
bool fuse_dots_on_dictionary() {
  static const bool on = [] {
    const char* e = std::getenv("AGGMG_DICT_DOTS");
    return !(e && e[0] == '0');
  }();
  return on;
}

double spmv_bytes(const DevCsr& A, Epi epi) {
  const double n = static_cast<double>(A.n_rows), nnz = static_cast<double>(A.nnz);
  // the launch_stream dispatch: SELL with a value dictionary reads 4 + 1 bytes per entry
  const bool vi = A.sell && A.sell_vi && epi != Epi::kResidualZero &&
                  !(epi == Epi::kJacobiDot2 && A.sell_short && !fuse_dots_on_dictionary());
  const bool d16 = A.sell && A.sell_d16 && epi != Epi::kResidualZero &&
                   !(epi == Epi::kJacobiDot2 && A.sell_short);
  double b = (vi ? 5.0 : d16 ? 10.0 : 12.0) * nnz + 4.0 * (n + 1) + 8.0 * static_cast<double>(A.n_cols) +
             8.0 * n;
  // the row-pattern format: a two-byte pattern id per row (the tables are L1-resident)
  if (A.pat && epi != Epi::kResidualZero) b = 2.0 * n + 8.0 * static_cast<double>(A.n_cols) + 8.0 * n;
  switch (epi) {
    case Epi::kResidual: b += 8.0 * n; break;
    case Epi::kResidualZero: b += 8.0 * n + 16.0 * n; break;  // wd gathered, x1 written
    case Epi::kJacobi: b += 16.0 * n; break;
    case Epi::kScaleDiag: b += 8.0 * n; break;
    case Epi::kSpmvZero: b += 16.0 * n; break;
    case Epi::kSpmvDot1: b += 8.0 * n; break;
    case Epi::kSpmvDot2: b += 8.0 * n; break;
    case Epi::kSpmvDot3: b += 16.0 * n; break;
    case Epi::kJacobiDot2: b += 24.0 * n; break;
    default: break;
  }
  return b;
}

void spmv_run(const DevCsr& A, Epi epi, const SpmvArgs& a, int prof_family) {
  if (A.n_rows == 0) return;
  ProfileScope scope(prof_family, prof_family ? spmv_bytes(A, epi) : 0.0);
  switch (epi) {
    case Epi::kSpmv: launch_stream<Epi::kSpmv>(A, a); break;
    case Epi::kResidual: launch_stream<Epi::kResidual>(A, a); break;
    case Epi::kResidualZero: launch_stream<Epi::kResidualZero>(A, a); break;
    case Epi::kJacobi: launch_stream<Epi::kJacobi>(A, a); break;
    case Epi::kScaleDiag: launch_stream<Epi::kScaleDiag>(A, a); break;
    case Epi::kSpmvZero: launch_stream<Epi::kSpmvZero>(A, a); break;
    case Epi::kSpmvDot1: launch_stream<Epi::kSpmvDot1>(A, a); break;
    case Epi::kSpmvDot2: launch_stream<Epi::kSpmvDot2>(A, a); break;
    case Epi::kSpmvDot3: launch_stream<Epi::kSpmvDot3>(A, a); break;
    case Epi::kJacobiDot2: launch_stream<Epi::kJacobiDot2>(A, a); break;
  }
}

// ---- transpose ----------------------------------------------------------------------

namespace {
__global__ void k_count_cols(const idx* col, int64_t nnz, idx* cnt) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < nnz) atomicAdd(&cnt[col[k]], 1);
}
__global__ void k_scatter_transpose(const idx* rowptr, const idx* col, const double* val,
                                    int64_t n_rows, const idx* trow, idx* cursor, idx* tcol,
                                    double* tval) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n_rows) return;
  for (idx k = rowptr[i]; k < rowptr[i + 1]; ++k) {
    const idx j = col[k];
    const idx p = trow[j] + atomicAdd(&cursor[j], 1);
    tcol[p] = static_cast<idx>(i);
    if (tval) tval[p] = val[k];
  }
}
}  // namespace

DevCsrPtr transpose(const DevCsr& A) {
  auto T = std::make_shared<DevCsr>();
  T->n_rows = A.n_cols;
  T->n_cols = A.n_rows;
  T->nnz = A.nnz;
  T->rowptr.resize(A.n_cols + 1);
  T->col.resize(A.nnz);
  T->val.resize(A.nnz);
  DevBuf<idx> cnt(A.n_cols), tmpc(A.nnz);
  DevBuf<double> tmpv(A.nnz);
  cnt.zero();
  if (A.nnz > 0) AGG_LAUNCH(k_count_cols, grid_for(A.nnz, 256), 256, 0, A.col.get(), A.nnz, cnt.get());
  scan_to_offsets_async(cnt.get(), T->rowptr.get(), A.n_cols);
  cnt.zero();
  if (A.n_rows > 0)
    AGG_LAUNCH(k_scatter_transpose, grid_for(A.n_rows, 256), 256, 0, A.rowptr.get(), A.col.get(),
               A.val.get(), A.n_rows, T->rowptr.get(), cnt.get(), tmpc.get(), tmpv.get());
  segmented_sort(T->rowptr.get(), A.n_cols, tmpc.get(), T->col.get(), tmpv.get(), T->val.get());
  T->plan();
  return T;
}

// ---- generators ---------------------------------------------------------------------

namespace {

// Same stencil, ordering and arithmetic as poisson.cpp:32-75.
// Rows [row0, row0 + nrows) of the grid operator (the whole matrix: row0 = 0, nrows = n);
// output row t = global row row0 + t, columns global.
__global__ void k_poisson_count(int64_t nx, int64_t ny, int64_t nz, int64_t row0, int64_t nrows,
                                idx* cnt) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nrows) return;
  const int64_t r = row0 + t;
  const int64_t i = r % nx, j = (r / nx) % ny, k = r / (nx * ny);
  cnt[t] = 1 + (i > 0) + (i + 1 < nx) + (j > 0) + (j + 1 < ny) + (k > 0) + (k + 1 < nz);
}
__global__ void k_poisson_fill(int64_t nx, int64_t ny, int64_t nz, int64_t row0, int64_t nrows,
                               double cx, double cy, double cz, double diag, const idx* rowptr,
                               idx* col, double* val) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nrows) return;
  const int64_t r = row0 + t;
  const int64_t i = r % nx, j = (r / nx) % ny, k = r / (nx * ny);
  idx p = rowptr[t];
  auto put = [&](int64_t c, double v) {
    col[p] = static_cast<idx>(c);
    val[p] = v;
    ++p;
  };
  if (k > 0) put(r - nx * ny, cz);
  if (j > 0) put(r - nx, cy);
  if (i > 0) put(r - 1, cx);
  put(r, diag);
  if (i + 1 < nx) put(r + 1, cx);
  if (j + 1 < ny) put(r + nx, cy);
  if (k + 1 < nz) put(r + nx * ny, cz);
}

__device__ inline double jump_kappa(int64_t x, int64_t y, int64_t z, int64_t block, double jump) {
  return (((x / block) + (y / block) + (z / block)) & 1) ? jump : 1.0;
}

__global__ void k_jump27_count(int64_t nx, int64_t ny, int64_t nz, int64_t row0, int64_t nrows,
                               idx* cnt) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nrows) return;
  const int64_t r = row0 + t;
  const int64_t i = r % nx, j = (r / nx) % ny, k = r / (nx * ny);
  const int cxn = 1 + (i > 0) + (i + 1 < nx), cyn = 1 + (j > 0) + (j + 1 < ny),
            czn = 1 + (k > 0) + (k + 1 < nz);
  cnt[t] = cxn * cyn * czn;
}

// 27-point variable-coefficient operator: off-diagonal -kappa_ij with
// kappa_ij = 2 k_i k_j / (k_i + k_j); diagonal = sum over the 26 neighbour slots of
// kappa_ij (kappa_i for Dirichlet-eliminated slots), accumulated in slot order.
__global__ void k_jump27_fill(int64_t nx, int64_t ny, int64_t nz, int64_t row0, int64_t nrows,
                              double jump, int64_t block, const idx* rowptr, idx* col, double* val) {
  const int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (t >= nrows) return;
  const int64_t r = row0 + t;
  const int64_t i = r % nx, j = (r / nx) % ny, k = r / (nx * ny);
  const double ki = jump_kappa(i, j, k, block, jump);
  double diag = 0.0;
  idx p = rowptr[t];
  idx pdiag = -1;
  for (int dz = -1; dz <= 1; ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        const int64_t x = i + dx, y = j + dy, z = k + dz;
        const bool inside = x >= 0 && x < nx && y >= 0 && y < ny && z >= 0 && z < nz;
        if (dx == 0 && dy == 0 && dz == 0) {
          pdiag = p;
          col[p] = static_cast<idx>(r);
          ++p;
          continue;
        }
        if (!inside) {
          diag = __dadd_rn(diag, ki);
          continue;
        }
        const double kj = jump_kappa(x, y, z, block, jump);
        const double kij = __ddiv_rn(__dmul_rn(__dmul_rn(2.0, ki), kj), __dadd_rn(ki, kj));
        diag = __dadd_rn(diag, kij);
        col[p] = static_cast<idx>((z * ny + y) * nx + x);
        val[p] = -kij;
        ++p;
      }
  val[pdiag] = diag;
}

}  // namespace

DevCsrPtr generate_poisson_rows(int dims, int64_t nx, int64_t ny, int64_t nz, double eps,
                                int weak_axis, int64_t row0, int64_t nrows) {
  require(dims == 2 || dims == 3, "poisson: dims must be 2 or 3");
  if (dims == 2) nz = 1;
  require(nx >= 1 && ny >= 1 && nz >= 1, "poisson: grid extents must be positive");
  require(eps > 0.0, "poisson: epsilon must be positive");
  int weak = weak_axis < 0 ? (dims == 2 ? 1 : 2) : weak_axis;
  require(weak < dims, "poisson: weak axis " + std::to_string(weak) + " out of range for " +
                           std::to_string(dims) + "D");
  const int64_t n = nx * ny * nz;
  if (nrows < 0) nrows = n - row0;
  require(row0 >= 0 && row0 + nrows <= n, "poisson: row range outside the grid");
  const double cx = weak == 0 ? -eps : -1.0, cy = weak == 1 ? -eps : -1.0,
               cz = weak == 2 ? -eps : -1.0;
  const double diag = -2.0 * (cx + cy + (dims == 3 ? cz : 0.0));
  auto A = std::make_shared<DevCsr>();
  A->n_rows = nrows;
  A->n_cols = n;
  A->rowptr.resize(nrows + 1);
  DevBuf<idx> cnt(nrows);
  if (nrows > 0)
    AGG_LAUNCH(k_poisson_count, grid_for(nrows, 256), 256, 0, nx, ny, nz, row0, nrows, cnt.get());
  A->nnz = scan_to_offsets(cnt.get(), A->rowptr.get(), nrows);
  A->col.resize(A->nnz);
  A->val.resize(A->nnz);
  if (nrows > 0)
    AGG_LAUNCH(k_poisson_fill, grid_for(nrows, 256), 256, 0, nx, ny, nz, row0, nrows, cx, cy, cz,
               diag, A->rowptr.get(), A->col.get(), A->val.get());
  A->plan();
  return A;
}

DevCsrPtr generate_poisson_device(int dims, int64_t nx, int64_t ny, int64_t nz, double eps,
                                  int weak_axis) {
  return generate_poisson_rows(dims, nx, ny, nz, eps, weak_axis, 0, -1);
}

DevCsrPtr generate_jump27_rows(int64_t nx, int64_t ny, int64_t nz, double jump, int64_t block,
                               int64_t row0, int64_t nrows) {
  require(nx >= 1 && ny >= 1 && nz >= 1 && block >= 1, "jump27: extents must be positive");
  require(jump > 0.0, "jump27: jump must be positive");
  const int64_t n = nx * ny * nz;
  if (nrows < 0) nrows = n - row0;
  require(row0 >= 0 && row0 + nrows <= n, "jump27: row range outside the grid");
  auto A = std::make_shared<DevCsr>();
  A->n_rows = nrows;
  A->n_cols = n;
  A->rowptr.resize(nrows + 1);
  DevBuf<idx> cnt(nrows);
  if (nrows > 0)
    AGG_LAUNCH(k_jump27_count, grid_for(nrows, 256), 256, 0, nx, ny, nz, row0, nrows, cnt.get());
  A->nnz = scan_to_offsets(cnt.get(), A->rowptr.get(), nrows);
  A->col.resize(A->nnz);
  A->val.resize(A->nnz);
  if (nrows > 0)
    AGG_LAUNCH(k_jump27_fill, grid_for(nrows, 256), 256, 0, nx, ny, nz, row0, nrows, jump, block,
               A->rowptr.get(), A->col.get(), A->val.get());
  A->plan();
  return A;
}

DevCsrPtr generate_jump27_device(int64_t nx, int64_t ny, int64_t nz, double jump, int64_t block) {
  return generate_jump27_rows(nx, ny, nz, jump, block, 0, -1);
}

}  // namespace aggmg_b200
