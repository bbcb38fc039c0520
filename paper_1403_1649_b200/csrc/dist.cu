// dist.cu — halo plans, halo exchange, request/reply and gathers of the row-partitioned path.
#include <algorithm>
#include <cub/cub.cuh>

#include "dist.cuh"
#include "primitives.cuh"

namespace aggmg_b200 {

// ---- partitions -----------------------------------------------------------------------

int Partition::owner(int64_t g) const {
  // last r with off[r] <= g (ranks may own zero rows)
  auto it = std::upper_bound(off.begin(), off.end(), g);
  int r = static_cast<int>(it - off.begin()) - 1;
  const int nr = static_cast<int>(off.size()) - 1;
  while (r < nr - 1 && off[r + 1] <= g) ++r;
  return std::max(0, std::min(r, nr - 1));
}

Partition Partition::even(int64_t n, int nranks, int64_t align) {
  Partition p;
  p.off.resize(nranks + 1);
  const int64_t units = (n + align - 1) / align;
  for (int r = 0; r <= nranks; ++r) p.off[r] = std::min(n, (units * r / nranks) * align);
  p.off[nranks] = n;
  return p;
}

Partition Partition::from_counts(const std::vector<int64_t>& counts) {
  Partition p;
  p.off.assign(counts.size() + 1, 0);
  for (size_t r = 0; r < counts.size(); ++r) p.off[r + 1] = p.off[r] + counts[r];
  return p;
}

namespace {

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
  while (lo < hi) {  // last r with off[r] <= g, skipping empty ranks
    const int mid = (lo + hi + 1) >> 1;
    if (p.off[mid] <= g)
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

__global__ void k_flag_off(const idx* g, int64_t m, int64_t c0, int64_t c1, idx* flag) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const int64_t v = g[k];
  flag[k] = (v < c0 || v >= c1) ? 1 : 0;
}
__global__ void k_compact(const idx* g, const idx* flag, const idx* pos, int64_t m, idx* out) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < m && flag[k]) out[pos[k]] = g[k];
}
__global__ void k_sub(idx* x, int64_t m, int64_t c0) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < m) x[k] = static_cast<idx>(x[k] - c0);
}
__global__ void k_check_range(const idx* x, int64_t m, int64_t n, int* bad) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < m && (x[k] < 0 || x[k] >= n)) atomicExch(bad, 1);
}
__global__ void k_localize(const idx* g, int64_t m, int64_t c0, int64_t nloc, const idx* halo,
                           int64_t nhalo, idx* out, int* bad) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const int64_t v = g[k];
  if (v >= c0 && v < c0 + nloc) {
    out[k] = static_cast<idx>(v - c0);
    return;
  }
  int64_t lo = 0, hi = nhalo;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (halo[mid] < v)
      lo = mid + 1;
    else
      hi = mid;
  }
  if (lo < nhalo && halo[lo] == v) {
    out[k] = static_cast<idx>(nloc + lo);
  } else {
    out[k] = 0;
    atomicExch(bad, 1);
  }
}
__global__ void k_globalize(const idx* l, int64_t m, int64_t c0, int64_t nloc, const idx* halo,
                            idx* out) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= m) return;
  const idx c = l[k];
  out[k] = c < nloc ? static_cast<idx>(c + c0) : halo[c - nloc];
}

template <class T>
__global__ void k_pack(const T* x, const idx* sidx, int64_t m, T* buf) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < m) buf[k] = x[sidx[k]];
}
__global__ void k_unpack_add(const idx* buf, const idx* sidx, int64_t m, idx* x) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < m) atomicAdd(&x[sidx[k]], buf[k]);
}

__global__ void k_owner_of(const idx* q, int64_t m, PartDev p, unsigned* own, idx* perm) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k >= m) return;
  own[k] = static_cast<unsigned>(dev_owner(p, q[k]));
  perm[k] = static_cast<idx>(k);
}
__global__ void k_gather_idx(const idx* q, const idx* perm, int64_t m, idx* out) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < m) out[k] = q[perm[k]];
}
template <class T>
__global__ void k_answer(const T* table, const idx* req, int64_t m, int64_t row0, T* out) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < m) out[k] = table[req[k] - row0];
}
template <class T>
__global__ void k_unpermute(const T* in, const idx* perm, int64_t m, T* out) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < m) out[perm[k]] = in[k];
}
__global__ void k_count_owner(const unsigned* own, int64_t m, int64_t* cnt) {
  const int64_t k = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (k < m) atomicAdd(reinterpret_cast<unsigned long long*>(&cnt[own[k]]), 1ull);
}

// rows holding a halo column (col >= nloc); lo = 1 + last such row below mid, hi = first at or
// above mid
__global__ void k_interior_bounds(const idx* rp, const idx* col, int64_t n, int64_t nloc,
                                  int64_t mid, unsigned long long* lo_hi) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  bool halo = false;
  for (idx k = rp[i]; k < rp[i + 1] && !halo; ++k) halo = col[k] >= nloc;
  if (!halo) return;
  if (i < mid)
    atomicMax(&lo_hi[0], static_cast<unsigned long long>(i + 1));
  else
    atomicMin(&lo_hi[1], static_cast<unsigned long long>(i));
}
__global__ void k_sum_parts(const double* parts, int np, int nparts, double* out) {
  const int k = threadIdx.x;
  if (k >= np) return;
  double s = parts[k];
  for (int p = 1; p < nparts; ++p) s = __dadd_rn(s, parts[p * 3 + k]);
  out[k] = s;
}

template <class F>
void cub_call(F&& f) {  // two-phase CUB call with a pooled temporary
  size_t bytes = 0;
  AGG_CUDA(f(nullptr, bytes));
  DevBuf<char> tmp(static_cast<int64_t>(std::max<size_t>(bytes, 1)));
  AGG_CUDA(f(tmp.get(), bytes));
}

}  // namespace

// ---- plans ------------------------------------------------------------------------------

void build_halo_plan(Comm& comm, const Partition& cols, const idx* gcols, int64_t m, HaloPlan& plan) {
  const int me = comm.rank(), P = comm.size();
  plan.col0 = cols.begin(me);
  plan.nloc = cols.count(me);
  // unique off-slab columns, ascending
  DevBuf<idx> flag(m), pos(m + 1);
  int64_t noff = 0;
  if (m > 0) {
    AGG_LAUNCH(k_flag_off, grid_for(m, 256), 256, 0, gcols, m, plan.col0, plan.col0 + plan.nloc,
               flag.get());
    noff = scan_to_offsets(flag.get(), pos.get(), m);
  }
  DevBuf<idx> off(noff), sorted(noff);
  if (noff > 0) {
    AGG_LAUNCH(k_compact, grid_for(m, 256), 256, 0, gcols, flag.get(), pos.get(), m, off.get());
    const int nbits = 64 - __builtin_clzll(static_cast<unsigned long long>(std::max<int64_t>(cols.n(), 2)));
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortKeys(t, b, off.get(), sorted.get(), static_cast<int>(noff), 0,
                                            nbits, stream());
    });
  }
  plan.halo_gid.resize(noff);
  DevBuf<int> nuniq(1);
  nuniq.zero();
  if (noff > 0)
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceSelect::Unique(t, b, sorted.get(), plan.halo_gid.get(), nuniq.get(),
                                       static_cast<int>(noff), stream());
    });
  plan.nhalo = read_scalar(nuniq.get());
  std::vector<idx> hg(plan.nhalo);
  if (plan.nhalo) plan.halo_gid.download(hg.data(), plan.nhalo);
  sync();
  // halo slots per owner (contiguous: slabs are contiguous and slots ascending)
  std::vector<int64_t> want(P, 0);
  plan.recv_peer.clear();
  plan.recv_off.clear();
  plan.recv_cnt.clear();
  for (int q = 0; q < P; ++q) {
    const int64_t lo = std::lower_bound(hg.begin(), hg.end(), cols.begin(q)) - hg.begin();
    const int64_t hi = std::lower_bound(hg.begin(), hg.end(), cols.begin(q) + cols.count(q)) - hg.begin();
    want[q] = hi - lo;
    if (hi > lo) {
      require(q != me, "halo plan: owned column classified as halo");
      plan.recv_peer.push_back(q);
      plan.recv_off.push_back(lo);
      plan.recv_cnt.push_back(hi - lo);
    }
  }
  // who wants what from me
  const std::vector<int64_t> all = comm.allgather_host(want);  // all[r * P + q]: r wants from q
  plan.send_peer.clear();
  plan.send_off.clear();
  plan.send_cnt.clear();
  int64_t ns = 0;
  for (int r = 0; r < P; ++r) {
    const int64_t c = all[static_cast<size_t>(r) * P + me];
    if (c > 0) {
      plan.send_peer.push_back(r);
      plan.send_off.push_back(ns);
      plan.send_cnt.push_back(c);
      ns += c;
    }
  }
  plan.nsend = ns;
  plan.send_idx.resize(ns);
  std::vector<CommMsg> sends, recvs;
  for (size_t k = 0; k < plan.recv_peer.size(); ++k)
    sends.push_back({plan.recv_peer[k], plan.halo_gid.get() + plan.recv_off[k],
                     sizeof(idx) * plan.recv_cnt[k]});
  for (size_t k = 0; k < plan.send_peer.size(); ++k)
    recvs.push_back({plan.send_peer[k], plan.send_idx.get() + plan.send_off[k],
                     sizeof(idx) * plan.send_cnt[k]});
  comm.exchange(sends, recvs);
  if (ns > 0) {
    AGG_LAUNCH(k_sub, grid_for(ns, 256), 256, 0, plan.send_idx.get(), ns, plan.col0);
    DevBuf<int> bad(1);
    bad.zero();
    AGG_LAUNCH(k_check_range, grid_for(ns, 256), 256, 0, plan.send_idx.get(), ns, plan.nloc, bad.get());
    require(read_scalar(bad.get()) == 0, "halo plan: a peer requested a row this rank does not own");
  }
  plan.sendbuf.resize(std::max<int64_t>(ns, 1) * 16);
}

void localize_cols(const HaloPlan& plan, const idx* gcols, int64_t m, idx* lcols, const char* err) {
  if (m <= 0) return;
  DevBuf<int> bad(1);
  bad.zero();
  AGG_LAUNCH(k_localize, grid_for(m, 256), 256, 0, gcols, m, plan.col0, plan.nloc,
             plan.halo_gid.get(), plan.nhalo, lcols, bad.get());
  require(read_scalar(bad.get()) == 0, err);
}

void globalize_cols(const HaloPlan& plan, const idx* lcols, int64_t m, idx* gcols) {
  if (m <= 0) return;
  AGG_LAUNCH(k_globalize, grid_for(m, 256), 256, 0, lcols, m, plan.col0, plan.nloc,
             plan.halo_gid.get(), gcols);
}

template <class T>
void halo_update_on(Comm& comm, const HaloPlan& plan, T* x, cudaStream_t st) {
  static_assert(sizeof(T) <= 16, "halo element too large");
  if (comm.size() == 1) return;
  T* buf = reinterpret_cast<T*>(plan.sendbuf.get());
  if (plan.nsend > 0) {
    k_pack<T><<<grid_for(plan.nsend, 256), 256, 0, st>>>(x, plan.send_idx.get(), plan.nsend, buf);
    note_launch();
    check_launch(__FILE__, __LINE__);
  }
  std::vector<CommMsg> sends, recvs;
  for (size_t k = 0; k < plan.send_peer.size(); ++k)
    sends.push_back({plan.send_peer[k], buf + plan.send_off[k], sizeof(T) * plan.send_cnt[k]});
  for (size_t k = 0; k < plan.recv_peer.size(); ++k)
    recvs.push_back({plan.recv_peer[k], x + plan.nloc + plan.recv_off[k], sizeof(T) * plan.recv_cnt[k]});
  comm.exchange(sends, recvs, st);
}
template void halo_update_on<double>(Comm&, const HaloPlan&, double*, cudaStream_t);

template <class T>
void halo_update(Comm& comm, const HaloPlan& plan, T* x) {
  halo_update_on<T>(comm, plan, x, stream());
}
template void halo_update<double>(Comm&, const HaloPlan&, double*);
template void halo_update<idx>(Comm&, const HaloPlan&, idx*);
template void halo_update<int8_t>(Comm&, const HaloPlan&, int8_t*);
template void halo_update<double2>(Comm&, const HaloPlan&, double2*);

void halo_reverse_add(Comm& comm, const HaloPlan& plan, idx* x) {
  if (comm.size() == 1) return;
  idx* buf = reinterpret_cast<idx*>(plan.sendbuf.get());
  std::vector<CommMsg> sends, recvs;
  for (size_t k = 0; k < plan.recv_peer.size(); ++k)
    sends.push_back({plan.recv_peer[k], x + plan.nloc + plan.recv_off[k], sizeof(idx) * plan.recv_cnt[k]});
  for (size_t k = 0; k < plan.send_peer.size(); ++k)
    recvs.push_back({plan.send_peer[k], buf + plan.send_off[k], sizeof(idx) * plan.send_cnt[k]});
  comm.exchange(sends, recvs);
  if (plan.nsend > 0)
    AGG_LAUNCH(k_unpack_add, grid_for(plan.nsend, 256), 256, 0, buf, plan.send_idx.get(), plan.nsend, x);
}

// ---- request / reply -----------------------------------------------------------------------

template <class T>
DevBuf<T> alltoallv(Comm& comm, const T* sendbuf, const std::vector<int64_t>& cnt,
                    std::vector<int64_t>* recv_cnt) {
  const int me = comm.rank(), P = comm.size();
  const std::vector<int64_t> all = comm.allgather_host(cnt);  // all[r * P + q]: r sends to q
  std::vector<int64_t> rc(P), roff(P + 1, 0), soff(P + 1, 0);
  for (int r = 0; r < P; ++r) {
    rc[r] = all[static_cast<size_t>(r) * P + me];
    roff[r + 1] = roff[r] + rc[r];
    soff[r + 1] = soff[r] + cnt[r];
  }
  DevBuf<T> out(roff[P]);
  std::vector<CommMsg> s, rv;
  for (int q = 0; q < P; ++q) {
    if (cnt[q]) s.push_back({q, const_cast<T*>(sendbuf) + soff[q], sizeof(T) * cnt[q]});
    if (rc[q]) rv.push_back({q, out.get() + roff[q], sizeof(T) * rc[q]});
  }
  comm.exchange(s, rv);
  if (recv_cnt) *recv_cnt = rc;
  return out;
}

template <class T>
void fetch_remote(Comm& comm, const Partition& part, const T* table, const idx* q, int64_t m, T* out) {
  const int me = comm.rank(), P = comm.size();
  const PartDev pd = part_dev(part);
  DevBuf<unsigned> own(m), own_s(m);
  DevBuf<idx> perm(m), perm_s(m), req(m);
  DevBuf<int64_t> cnt_d(P);
  cnt_d.zero();
  if (m > 0) {
    AGG_LAUNCH(k_owner_of, grid_for(m, 256), 256, 0, q, m, pd, own.get(), perm.get());
    AGG_LAUNCH(k_count_owner, grid_for(m, 256), 256, 0, own.get(), m, cnt_d.get());
    const int nbits = std::max(1, 32 - __builtin_clz(static_cast<unsigned>(P)));
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairs(t, b, own.get(), own_s.get(), perm.get(), perm_s.get(),
                                             static_cast<int>(m), 0, nbits, stream());
    });
    AGG_LAUNCH(k_gather_idx, grid_for(m, 256), 256, 0, q, perm_s.get(), m, req.get());
  }
  std::vector<int64_t> cnt(P);
  cnt_d.download(cnt.data(), P);
  sync();
  std::vector<int64_t> rc;
  DevBuf<idx> incoming = alltoallv<idx>(comm, req.get(), cnt, &rc);
  int64_t nin = 0;
  for (int64_t c : rc) nin += c;
  DevBuf<T> answers(nin);
  if (nin > 0)
    AGG_LAUNCH(k_answer<T>, grid_for(nin, 256), 256, 0, table, incoming.get(), nin, part.begin(me),
               answers.get());
  // send the answers back: what I received from r goes back to r
  DevBuf<T> replies = alltoallv<T>(comm, answers.get(), rc);
  if (m > 0)
    AGG_LAUNCH(k_unpermute<T>, grid_for(m, 256), 256, 0, replies.get(), perm_s.get(), m, out);
}
template void fetch_remote<double>(Comm&, const Partition&, const double*, const idx*, int64_t, double*);
template void fetch_remote<idx>(Comm&, const Partition&, const idx*, const idx*, int64_t, idx*);
template DevBuf<idx> alltoallv<idx>(Comm&, const idx*, const std::vector<int64_t>&, std::vector<int64_t>*);
template DevBuf<double> alltoallv<double>(Comm&, const double*, const std::vector<int64_t>&,
                                          std::vector<int64_t>*);
template DevBuf<double2> alltoallv<double2>(Comm&, const double2*, const std::vector<int64_t>&,
                                            std::vector<int64_t>*);
template DevBuf<int2> alltoallv<int2>(Comm&, const int2*, const std::vector<int64_t>&,
                                      std::vector<int64_t>*);
template DevBuf<int4> alltoallv<int4>(Comm&, const int4*, const std::vector<int64_t>&,
                                      std::vector<int64_t>*);

// ---- distributed matrices -------------------------------------------------------------------

DistCsrPtr make_dist(Comm& comm, const Partition& rows, const Partition& cols, DevCsr& gA,
                     const char* err) {
  auto M = std::make_shared<DistCsr>();
  M->rows = rows;
  M->cols = cols;
  build_halo_plan(comm, cols, gA.col.get(), gA.nnz, M->halo);
  M->A.n_rows = gA.n_rows;
  M->A.nnz = gA.nnz;
  M->A.n_cols = M->halo.nloc + M->halo.nhalo;
  M->A.rowptr = std::move(gA.rowptr);
  M->A.val = std::move(gA.val);
  M->A.col.resize(gA.nnz);
  localize_cols(M->halo, gA.col.get(), gA.nnz, M->A.col.get(), err);
  gA.col.reset();
  M->A.sell_sigma_ok = false;  // dist_spmv launches row sub-ranges
  M->A.plan();
  // overlap window: rows without halo columns around the middle of the slab
  const int64_t n = M->A.n_rows;
  M->int_lo = M->int_hi = 0;
  if (M->halo.nhalo > 0 && n > 0) {
    DevBuf<unsigned long long> lh(2);
    const unsigned long long init[2] = {0ull, static_cast<unsigned long long>(n)};
    lh.upload(init, 2);
    AGG_LAUNCH(k_interior_bounds, grid_for(n, 256), 256, 0, M->A.rowptr.get(), M->A.col.get(), n,
               M->halo.nloc, n / 2, lh.get());
    unsigned long long h[2];
    lh.download(h, 2);
    sync();
    const int64_t rpb = std::max(1, M->A.rows_per_block);
    const int64_t lo = (static_cast<int64_t>(h[0]) + rpb - 1) / rpb * rpb;
    const int64_t hi = static_cast<int64_t>(h[1]) / rpb * rpb;
    if (hi - lo >= std::max<int64_t>(rpb, n / 8)) {  // worth a split
      M->int_lo = lo;
      M->int_hi = hi;
    }
  }
  return M;
}

void dist_spmv(Comm& comm, const DistCsr& M, Epi epi, const SpmvArgs& a, int prof) {
  if (comm.size() == 1 || M.int_hi <= M.int_lo) {
    halo_update<double>(comm, M.halo, const_cast<double*>(a.x));
    spmv_run(M.A, epi, a, prof);
    return;
  }
  // exchange on the side stream, ordered after everything that produced a.x
  cudaStream_t side = side_stream();
  cudaEvent_t ready, landed;
  AGG_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
  AGG_CUDA(cudaEventCreateWithFlags(&landed, cudaEventDisableTiming));
  AGG_CUDA(cudaEventRecord(ready, stream()));
  AGG_CUDA(cudaStreamWaitEvent(side, ready, 0));
  halo_update_on<double>(comm, M.halo, const_cast<double*>(a.x), side);
  AGG_CUDA(cudaEventRecord(landed, side));
  const bool dots = a.dots_out != nullptr;
  DevBuf<double> parts(dots ? 9 : 0);
  // one timing scope over all parts: the effective time of the operator incl. any halo wait
  ProfileScope scope(prof, prof ? spmv_bytes(M.A, epi) : 0.0);
  auto part = [&](int64_t base, int64_t count, int slot) {
    if (count <= 0) {
      if (dots) AGG_CUDA(cudaMemsetAsync(parts.get() + 3 * slot, 0, 3 * sizeof(double), stream()));
      return;
    }
    SpmvArgs s = a;
    s.row_base = base;
    s.row_count = count;
    if (dots) s.dots_out = parts.get() + 3 * slot;
    spmv_run(M.A, epi, s);
  };
  part(M.int_lo, M.int_hi - M.int_lo, 0);  // interior: no halo column
  AGG_CUDA(cudaStreamWaitEvent(stream(), landed, 0));
  part(0, M.int_lo, 1);
  part(M.int_hi, M.A.n_rows - M.int_hi, 2);
  if (dots) {
    const int np = epi == Epi::kSpmvDot1 ? 1 : epi == Epi::kSpmvDot3 ? 3 : 2;
    AGG_LAUNCH(k_sum_parts, 1, 32, 0, parts.get(), np, 3, a.dots_out);
  }
  cudaEventDestroy(ready);
  cudaEventDestroy(landed);
}

DevBuf<idx> global_cols(const DistCsr& M) {
  DevBuf<idx> g(M.A.nnz);
  globalize_cols(M.halo, M.A.col.get(), M.A.nnz, g.get());
  return g;
}

namespace {
__global__ void k_row_len(const idx* rp, int64_t n, idx* len) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) len[i] = rp[i + 1] - rp[i];
}
}  // namespace

namespace {
// root >= 0: the matrix assembled on that rank only; root < 0: on every rank
DevCsrPtr gather_csr(Comm& comm, const DistCsr& M, int root) {
  const int me = comm.rank(), P = comm.size();
  const bool all = root < 0;
  const std::vector<int64_t> nnz_all = comm.allgather_host({M.A.nnz});
  DevBuf<idx> gcol = global_cols(M);
  DevBuf<idx> len(M.A.n_rows);
  if (M.A.n_rows > 0)
    AGG_LAUNCH(k_row_len, grid_for(M.A.n_rows, 256), 256, 0, M.A.rowptr.get(), M.A.n_rows, len.get());
  DevCsrPtr G;
  std::vector<CommMsg> s, r;
  for (int q = 0; q < P; ++q) {
    if (!all && q != root) continue;
    s.push_back({q, len.get(), sizeof(idx) * M.A.n_rows});
    s.push_back({q, gcol.get(), sizeof(idx) * M.A.nnz});
    s.push_back({q, M.A.val.get(), sizeof(double) * M.A.nnz});
  }
  DevBuf<idx> all_len;
  if (all || me == root) {
    const int64_t n = M.rows.n();
    int64_t nnz = 0;
    for (int64_t c : nnz_all) nnz += c;
    G = std::make_shared<DevCsr>();
    G->n_rows = n;
    G->n_cols = M.cols.n();
    G->nnz = nnz;
    G->rowptr.resize(n + 1);
    G->col.resize(nnz);
    G->val.resize(nnz);
    all_len.resize(n);
    int64_t eo = 0;
    for (int q = 0; q < P; ++q) {
      r.push_back({q, all_len.get() + M.rows.begin(q), sizeof(idx) * M.rows.count(q)});
      r.push_back({q, G->col.get() + eo, sizeof(idx) * nnz_all[q]});
      r.push_back({q, G->val.get() + eo, sizeof(double) * nnz_all[q]});
      eo += nnz_all[q];
    }
  }
  comm.exchange(s, r);
  if (all || me == root) {
    scan_to_offsets(all_len.get(), G->rowptr.get(), G->n_rows);
    G->plan();
  }
  return G;
}
}  // namespace

DevCsrPtr gather_to_root(Comm& comm, const DistCsr& M, int root) { return gather_csr(comm, M, root); }
DevCsrPtr gather_to_all(Comm& comm, const DistCsr& M) { return gather_csr(comm, M, -1); }

void allgather_vector(Comm& comm, const Partition& part, const double* x_loc, double* x_all) {
  const int P = comm.size();
  std::vector<CommMsg> s, r;
  for (int q = 0; q < P; ++q) {
    s.push_back({q, const_cast<double*>(x_loc), sizeof(double) * part.count(comm.rank())});
    r.push_back({q, x_all + part.begin(q), sizeof(double) * part.count(q)});
  }
  comm.exchange(s, r);
}

void gather_vector(Comm& comm, const Partition& part, const double* x_loc, double* x_root, int root) {
  const int me = comm.rank(), P = comm.size();
  std::vector<CommMsg> s, r;
  s.push_back({root, const_cast<double*>(x_loc), sizeof(double) * part.count(me)});
  if (me == root)
    for (int q = 0; q < P; ++q) r.push_back({q, x_root + part.begin(q), sizeof(double) * part.count(q)});
  comm.exchange(s, r);
}

void scatter_vector(Comm& comm, const Partition& part, const double* x_root, double* x_loc, int root) {
  const int me = comm.rank(), P = comm.size();
  std::vector<CommMsg> s, r;
  if (me == root)
    for (int q = 0; q < P; ++q)
      s.push_back({q, const_cast<double*>(x_root) + part.begin(q), sizeof(double) * part.count(q)});
  r.push_back({root, x_loc, sizeof(double) * part.count(me)});
  comm.exchange(s, r);
}

}  // namespace aggmg_b200
