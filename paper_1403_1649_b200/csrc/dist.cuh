// dist.cuh — row-partitioned operators for the multi-GPU path.
//
// Every level above the agglomeration threshold is split into contiguous row slabs, one per
// rank.  A rank stores its rows with LOCAL column ids: owned column g -> g - col0, every
// other column -> nloc + h, h its slot in the sorted list of halo columns.  Entries keep the
// global ascending order inside each row, so the CSR-stream kernels sum every row in the
// reference's order and the partitioned results are bit-identical to the one-GPU ones.
//
// A HaloPlan is the communication schedule of one column space: which of my owned entries
// each peer needs (send list) and where the peers' entries land (halo slots, grouped by
// owner because halo slots are sorted by global id and slabs are contiguous).
#pragma once

#include <memory>
#include <vector>

#include "comm.cuh"
#include "sparse.cuh"

namespace aggmg_b200 {

// Contiguous block partition of [0, n): rank r owns [off[r], off[r+1]).
struct Partition {
  std::vector<int64_t> off;
  int64_t n() const { return off.empty() ? 0 : off.back(); }
  int64_t begin(int r) const { return off[r]; }
  int64_t count(int r) const { return off[r + 1] - off[r]; }
  int owner(int64_t g) const;  // host binary search
  static Partition even(int64_t n, int nranks, int64_t align = 1);
  static Partition from_counts(const std::vector<int64_t>& counts);
};

struct HaloPlan {
  int64_t nloc = 0, col0 = 0;  // owned range of the column space
  int64_t nhalo = 0, nsend = 0;
  std::vector<int> recv_peer;        // peers I receive from (ascending)
  std::vector<int64_t> recv_off, recv_cnt;  // halo slots [off, off+cnt) per recv peer
  std::vector<int> send_peer;
  std::vector<int64_t> send_off, send_cnt;  // send_idx[off, off+cnt) per send peer
  DevBuf<idx> send_idx;   // owned local indices to pack
  DevBuf<idx> halo_gid;   // global id of every halo slot (ascending)
  mutable DevBuf<char> sendbuf;  // staging, 16 bytes per send entry
};

// Builds the plan for the column ids gcols[0..m) (global, any order, may repeat).
void build_halo_plan(Comm& comm, const Partition& cols, const idx* gcols, int64_t m, HaloPlan& plan);
// Global -> local column ids (owned: g - col0, halo: nloc + slot).  A column that is
// neither owned nor in the plan raises `err` (checked on the device, reported on the host).
void localize_cols(const HaloPlan& plan, const idx* gcols, int64_t m, idx* lcols, const char* err);
// local -> global
void globalize_cols(const HaloPlan& plan, const idx* lcols, int64_t m, idx* gcols);

// x[nloc + h] <- owner's x for every halo slot (x has nloc + nhalo entries).
template <class T>
void halo_update(Comm& comm, const HaloPlan& plan, T* x);
template <class T>
void halo_update_on(Comm& comm, const HaloPlan& plan, T* x, cudaStream_t st);
// owner's x[i] += x[nloc + h] for every halo slot h that refers to i (integer counts).
void halo_reverse_add(Comm& comm, const HaloPlan& plan, idx* x);

// One-shot request / reply: for every global id q[k] (owned by some rank), fetch
// table[q - begin(owner)] from the owner's device table.  Replies arrive in request order.
template <class T>
void fetch_remote(Comm& comm, const Partition& part, const T* table, const idx* q, int64_t m,
                  T* out);
// Variable-size all-to-all of POD records: sendbuf is grouped by destination rank with
// counts cnt[r]; returns the received records grouped by source rank (rank order).
template <class T>
DevBuf<T> alltoallv(Comm& comm, const T* sendbuf, const std::vector<int64_t>& cnt,
                    std::vector<int64_t>* recv_cnt = nullptr);

// Row-partitioned CSR (square operators, R and P): local rows, local column ids.
// [int_lo, int_hi) is a run of rows without halo columns, aligned to the CSR-stream row
// blocks: those rows are computed while the halo exchange is in flight (empty: no overlap).
struct DistCsr {
  Partition rows, cols;
  DevCsr A;  // n_rows = rows.count(me), n_cols = nloc_cols + nhalo
  HaloPlan halo;
  int64_t int_lo = 0, int_hi = 0;
};

// y-side of a CSR-stream kernel on a row-partitioned operator: the halo of a.x is exchanged
// on a side stream while the interior rows run, then the boundary rows; fused dots are
// combined as interior + low + high partials (deterministic).
void dist_spmv(Comm& comm, const DistCsr& M, Epi epi, const SpmvArgs& a, int prof = 0);
using DistCsrPtr = std::shared_ptr<DistCsr>;

// Wraps rows [row0, row0 + nloc) given with GLOBAL column ids (gA.col) into a DistCsr.
DistCsrPtr make_dist(Comm& comm, const Partition& rows, const Partition& cols, DevCsr& gA,
                     const char* err = "distributed setup requires a structurally symmetric matrix");
// Global column id of every stored entry (device array of A.nnz).
DevBuf<idx> global_cols(const DistCsr& M);

// Gathers a row-partitioned matrix (global cols) / vector onto rank `root` as one DevCsr.
DevCsrPtr gather_to_root(Comm& comm, const DistCsr& M, int root);
DevCsrPtr gather_to_all(Comm& comm, const DistCsr& M);  // the same matrix on every rank
// x_all[part.begin(q) + i] = rank q's x_loc[i] on every rank
void allgather_vector(Comm& comm, const Partition& part, const double* x_loc, double* x_all);
void gather_vector(Comm& comm, const Partition& part, const double* x_loc, double* x_root, int root);
void scatter_vector(Comm& comm, const Partition& part, const double* x_root, double* x_loc, int root);

}  // namespace aggmg_b200
