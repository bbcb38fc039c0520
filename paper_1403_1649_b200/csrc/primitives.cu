// primitives.cu — scans, deterministic reductions, segmented rank sort.
#include <atomic>
#include "primitives.cuh"

#include "chunked.cuh"

namespace aggmg_b200 {

namespace {

constexpr int kScanBlock = 256;
constexpr int kScanItems = 8;
constexpr int kScanTile = kScanBlock * kScanItems;

// Exclusive scan of one 2048-element tile per block.  Loads are striped (coalesced),
// each thread scans 8 consecutive elements from shared memory, thread totals are
// combined with warp shuffles.  Writes the tile total to tile_sums[blockIdx.x].
__global__ void __launch_bounds__(kScanBlock) k_scan_tiles(const idx* in, idx* out, idx* tile_sums,
                                                           int64_t n) {
  __shared__ idx tile[kScanTile];
  __shared__ idx warp_tot[kScanBlock / 32];
  const int64_t base = static_cast<int64_t>(blockIdx.x) * kScanTile;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    const int64_t g = base + j * kScanBlock + threadIdx.x;
    tile[j * kScanBlock + threadIdx.x] = g < n ? in[g] : 0;
  }
  __syncthreads();
  idx local[kScanItems];
  idx run = 0;
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    local[j] = run;
    run += tile[threadIdx.x * kScanItems + j];
  }
  // inclusive warp scan of thread totals
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  idx incl = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    idx t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    idx w = lane < kScanBlock / 32 ? warp_tot[lane] : 0;
    idx wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      idx t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += t;
    }
    if (lane < kScanBlock / 32) warp_tot[lane] = wi - w;  // exclusive warp offsets
    if (lane == kScanBlock / 32 - 1) tile_sums[blockIdx.x] = wi;
  }
  __syncthreads();
  const idx off = warp_tot[warp] + (incl - run);
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) tile[threadIdx.x * kScanItems + j] = local[j] + off;
  __syncthreads();
#pragma unroll
  for (int j = 0; j < kScanItems; ++j) {
    const int64_t g = base + j * kScanBlock + threadIdx.x;
    if (g < n) out[g] = tile[j * kScanBlock + threadIdx.x];
  }
}

__global__ void k_add_tile_offsets(idx* out, const idx* tile_offsets, int64_t n) {
  const int64_t g = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (g < n) out[g] += tile_offsets[g / kScanTile];
}

// out[0..n) exclusive scan; *total = sum (device)
void scan_rec(const idx* in, idx* out, int64_t n, idx* total) {
  const int64_t nt = (n + kScanTile - 1) / kScanTile;
  if (nt <= 1) {
    AGG_LAUNCH(k_scan_tiles, 1, kScanBlock, 0, in, out, total, n);
    return;
  }
  DevBuf<idx> sums(nt);
  AGG_LAUNCH(k_scan_tiles, static_cast<unsigned>(nt), kScanBlock, 0, in, out, sums.get(), n);
  scan_rec(sums.get(), sums.get(), nt, total);
  AGG_LAUNCH(k_add_tile_offsets, grid_for(n, 256), 256, 0, out, sums.get(), n);
}

}  // namespace

void scan_to_offsets_async(const idx* counts, idx* offsets, int64_t n) {
  if (n == 0) {
    AGG_CUDA(cudaMemsetAsync(offsets, 0, sizeof(idx), stream()));
    return;
  }
  scan_rec(counts, offsets, n, offsets + n);
}

int64_t scan_to_offsets(const idx* counts, idx* offsets, int64_t n) {
  scan_to_offsets_async(counts, offsets, n);
  return read_scalar(offsets + n);
}

// ---- reductions ----------------------------------------------------------------

namespace {
constexpr int kRedBlock = 256;
struct RedScratch {
  double* partials = nullptr;
  unsigned* ticket = nullptr;
  int cap = 0;
  ~RedScratch() {
    if (partials) cudaFree(partials);
    if (ticket) cudaFree(ticket);
  }
};
RedScratch& red() {
  static thread_local RedScratch rs[2];  // [1]: kernels on a redirected (side) stream
  RedScratch& r = rs[stream_redirected() ? 1 : 0];
  if (!r.partials) {
    r.cap = 1 << 20;
    AGG_CUDA(cudaMalloc(&r.partials, sizeof(double) * 3 * r.cap));
    AGG_CUDA(cudaMalloc(&r.ticket, sizeof(unsigned) * 64));
    AGG_CUDA(cudaMemsetAsync(r.ticket, 0, sizeof(unsigned) * 64, stream()));
  }
  return r;
}

template <int NP>
__global__ void __launch_bounds__(kRedBlock) k_dot(DotArgs args, int64_t n, double* partials,
                                                   unsigned* ticket, double* out, const int* pred) {
  __shared__ double smem[32 * NP];
  if (pred && !*pred) return;
  double v[NP];
#pragma unroll
  for (int k = 0; k < NP; ++k) v[k] = 0.0;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  const int64_t npair = n >> 1;  // 128-bit loads; the odd tail element handled once below
  for (int64_t q = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; q < npair; q += stride) {
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      const double2 a = reinterpret_cast<const double2*>(args.a[k])[q];
      const double2 b = reinterpret_cast<const double2*>(args.b[k])[q];
      v[k] = __dadd_rn(v[k], __dmul_rn(a.x, b.x));
      v[k] = __dadd_rn(v[k], __dmul_rn(a.y, b.y));
    }
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0)
#pragma unroll
    for (int k = 0; k < NP; ++k) v[k] = __dadd_rn(v[k], __dmul_rn(args.a[k][n - 1], args.b[k][n - 1]));
  block_reduce<NP>(v, smem);
  if (threadIdx.x == 0)
#pragma unroll
    for (int k = 0; k < NP; ++k) partials[blockIdx.x * NP + k] = v[k];
  finish_reduction<NP>(partials, ticket, out, smem);
}
}  // namespace

unsigned reduce_grid(int64_t n) {
  const int64_t want = (n + kRedBlock * 8 - 1) / (kRedBlock * 8);
  const int64_t cap = 8 * static_cast<int64_t>(sm_count());
  return static_cast<unsigned>(std::max<int64_t>(1, std::min(want, cap)));
}
double* reduce_partials() { return red().partials; }
unsigned* reduce_ticket() { return red().ticket; }

namespace {
std::atomic<bool> g_exact{false};  // read by rank threads, written by the host API
template <int NP>
void dot_exact(const DotArgs& args, int64_t n, double* out, const int* pred) {
  DotOp<NP> op;
  for (int k = 0; k < NP; ++k) {
    op.a[k] = args.a[k];
    op.b[k] = args.b[k];
  }
  op.pred = pred;
  launch_chunked<NP>(op, n, out);
}
}  // namespace

bool exact_reductions() { return g_exact.load(); }
void set_exact_reductions(bool on) { g_exact.store(on); }

void dot_device(const DotArgs& args, int64_t n, double* out, const int* pred, int exact) {
  if (exact == 1 || (exact < 0 && g_exact.load())) {
    switch (args.np) {
      case 1: dot_exact<1>(args, n, out, pred); return;
      case 2: dot_exact<2>(args, n, out, pred); return;
      case 3: dot_exact<3>(args, n, out, pred); return;
      default: throw Error("dot_device: np must be 1..3");
    }
  }
  RedScratch& r = red();
  const unsigned g = reduce_grid(n);
  switch (args.np) {
    case 1: AGG_LAUNCH(k_dot<1>, g, kRedBlock, 0, args, n, r.partials, r.ticket, out, pred); break;
    case 2: AGG_LAUNCH(k_dot<2>, g, kRedBlock, 0, args, n, r.partials, r.ticket, out, pred); break;
    case 3: AGG_LAUNCH(k_dot<3>, g, kRedBlock, 0, args, n, r.partials, r.ticket, out, pred); break;
    default: throw Error("dot_device: np must be 1..3");
  }
}

double dot_host(const double* a, const double* b, int64_t n, int exact) {
  DevBuf<double> out(1);
  DotArgs d{};
  d.a[0] = a;
  d.b[0] = b;
  d.np = 1;
  dot_device(d, n, out.get(), nullptr, exact);
  return read_scalar(out.get());
}

// ---- segmented sort --------------------------------------------------------------

namespace {
// Warp per segment; rank of a key = number of smaller keys in its segment (keys are
// unique).  Segment keys are read through L1 as broadcast loads.
__global__ void k_segsort(const idx* offsets, int64_t nseg, const idx* kin, idx* kout,
                          const double* vin, double* vout) {
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= nseg) return;
  const idx lo = offsets[warp], hi = offsets[warp + 1];
  const idx L = hi - lo;
  for (idx e = lane; e < L; e += 32) {
    const idx key = kin[lo + e];
    idx rank = 0;
    for (idx q = 0; q < L; ++q) rank += (kin[lo + q] < key) ? 1 : 0;
    kout[lo + rank] = key;
    if (vout) vout[lo + rank] = vin[lo + e];
  }
}
}  // namespace

namespace {
constexpr int kSmallSeg = 16;
// Thread per segment for short segments (insertion sort in registers); longer segments
// are listed for the warp kernel.
__global__ void k_segsort_small(const idx* offsets, int64_t nseg, const idx* kin, idx* kout,
                                const double* vin, double* vout, idx* long_list, int* n_long) {
  const int64_t s = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (s >= nseg) return;
  const idx lo = offsets[s], L = offsets[s + 1] - lo;
  if (L > kSmallSeg) {
    long_list[atomicAdd(n_long, 1)] = static_cast<idx>(s);
    return;
  }
  idx k[kSmallSeg];
  double v[kSmallSeg];
#pragma unroll
  for (int q = 0; q < kSmallSeg; ++q) {
    if (q < L) {
      k[q] = kin[lo + q];
      if (vout) v[q] = vin[lo + q];
    }
  }
  for (int q = 1; q < L; ++q) {
    const idx kq = k[q];
    const double vq = vout ? v[q] : 0.0;
    int z = q - 1;
    while (z >= 0 && k[z] > kq) {
      k[z + 1] = k[z];
      if (vout) v[z + 1] = v[z];
      --z;
    }
    k[z + 1] = kq;
    if (vout) v[z + 1] = vq;
  }
  for (int q = 0; q < L; ++q) {
    kout[lo + q] = k[q];
    if (vout) vout[lo + q] = v[q];
  }
}

__global__ void k_segsort_list(const idx* list, const int* n_list, const idx* offsets,
                               const idx* kin, idx* kout, const double* vin, double* vout) {
  const int64_t w = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= *n_list) return;
  const idx s = list[w];
  const idx lo = offsets[s], L = offsets[s + 1] - lo;
  for (idx e = lane; e < L; e += 32) {
    const idx key = kin[lo + e];
    idx rank = 0;
    for (idx q = 0; q < L; ++q) rank += (kin[lo + q] < key) ? 1 : 0;
    kout[lo + rank] = key;
    if (vout) vout[lo + rank] = vin[lo + e];
  }
}
}  // namespace

void segmented_sort(const idx* offsets, int64_t nseg, const idx* kin, idx* kout, const double* vin,
                    double* vout) {
  if (nseg <= 0) return;
  DevBuf<idx> list(nseg);
  DevBuf<int> n_long(1);
  n_long.zero();
  AGG_LAUNCH(k_segsort_small, grid_for(nseg, 128), 128, 0, offsets, nseg, kin, kout, vin, vout,
             list.get(), n_long.get());
  const int nl = read_scalar(n_long.get());
  if (nl > 0)
    AGG_LAUNCH(k_segsort_list, grid_for(static_cast<int64_t>(nl) * 32, 256), 256, 0, list.get(),
               n_long.get(), offsets, kin, kout, vin, vout);
}

// ---- helpers -----------------------------------------------------------------------

namespace {
__global__ void k_fill_int(idx* p, int64_t n, idx v) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}
__global__ void k_fill_double(double* p, int64_t n, double v) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}
}  // namespace

void fill_int(idx* p, int64_t n, idx v) {
  if (n > 0) AGG_LAUNCH(k_fill_int, grid_for(n, 256), 256, 0, p, n, v);
}
void fill_double(double* p, int64_t n, double v) {
  if (n > 0) AGG_LAUNCH(k_fill_double, grid_for(n, 256), 256, 0, p, n, v);
}
void copy_double(double* dst, const double* src, int64_t n) {
  if (n > 0)
    AGG_CUDA(cudaMemcpyAsync(dst, src, sizeof(double) * n, cudaMemcpyDeviceToDevice, stream()));
}

}  // namespace aggmg_b200
