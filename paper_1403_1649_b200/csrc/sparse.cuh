// sparse.cuh — device CSR and the CSR-stream SpMV family.
//
// Layout in HBM: row_offsets int32[n+1], col int32[nnz], val f64[nnz].
//
// SpMV = "CSR-stream with shared-memory staging": a block owns a run of
// rows_per_block consecutive rows; its threads stream the run's contiguous
// val/col range with 128-bit loads (2 doubles + 4 int32 per thread-step), multiply by
// the gathered x and stage the products in shared memory; then one thread per row sums
// its products sequentially in storage order.  That is exactly the reference's
// row-sequential `sum += a * x` (sparse.cpp:57-62), so every SpMV-family kernel is
// bit-identical to the CPU oracle (built without FMA).
#pragma once

#include <atomic>
#include <memory>

#include "primitives.cuh"

namespace aggmg_b200 {

struct DevCsr {
  int64_t n_rows = 0, n_cols = 0, nnz = 0;
  DevBuf<idx> rowptr, col;
  DevBuf<double> val;
  int max_row = 0;         // longest row
  int rows_per_block = 0;  // CSR-stream plan
  int smem_entries = 0;
  // SELL-32 copy for operators with longer rows (sparse.cu): slice s = rows [32s, 32s+32),
  // slot k of its row r at sell_ptr[s] + 32k + (r & 31) — the row's k-th CSR entry
  bool sell = false;
  bool sell_short = false;  // mean row length < 10
  DevBuf<idx> sell_ptr, sell_col;
  DevBuf<double> sell_val;
  // SELL-C-sigma (plain layout only): position q of the copy holds row sell_perm[q], rows sorted
  // by length inside windows of 256 (empty = identity).  Partitioned operators keep the identity
  // (their interior / boundary launches address row sub-ranges): sell_sigma_ok = false.
  DevBuf<idx> sell_perm;
  bool sell_sigma_ok = true;
  // value dictionary (operators with <= 256 distinct values, e.g. stencil matrices): slot k's
  // value is sell_tab[sell_code[slot]] — the same double, one byte per entry instead of eight
  bool sell_vi = false;
  bool sell_pad4 = false;  // slice widths are whole 4-slot groups (the packed code layout)
  DevBuf<unsigned char> sell_code;  // byte of slot k of row r: slice base + 32(k & ~3) + 4(r & 31) + (k & 3)
  DevBuf<double> sell_tab;
  DevBuf<idx> sell_pcol;  // the columns in sell_code's packing (int4 per 4 slots of a row)
  // length of the row at position q (<= 64): the SELL kernels read it beside the slice base,
  // so a row's column loads wait on no rowptr / perm round trip
  DevBuf<unsigned char> sell_len;
  // plain layout with every column within 32767 of its row: 16-bit offsets instead of columns
  bool sell_d16 = false;
  DevBuf<short> sell_col16;

  // Row-pattern dictionary (stencil-like operators: at most kPatMax distinct rows up to the
  // diagonal shift): row r's entries are (r + pat_delta[p][j], pat_val[p][j]), j < pat_len[p],
  // p = pat_id[r] — two bytes per row instead of a column and a value code per entry.  Same
  // values in the same order: every sum bit-identical to CSR / SELL.
  bool pat = false;
  int pat_w = 0;  // table row width (the longest pattern)
  DevBuf<unsigned short> pat_id;
  DevBuf<unsigned char> pat_len;
  DevBuf<int> pat_delta;
  DevBuf<double> pat_val;
  bool build_patterns();  // false (and no pattern format) beyond kPatMax patterns
  void plan();          // computes max_row / rows_per_block, builds the SELL copy (synchronises)
  int64_t sell_slots = 0;  // padded slot count of the SELL layout
  void refresh_sell();  // after val changed in place: rebuild the SELL copy (dictionary or plain)
  bool dict_scan(DevBuf<unsigned long long>& slots) const;
  void fill_plain();
  void build_codes(const DevBuf<unsigned long long>& slots);
};
using DevCsrPtr = std::shared_ptr<DevCsr>;

// Upload a host int64 CSR; validates canonical form on the device with the
// reference's messages (sparse.cpp:22-39).
DevCsrPtr upload_csr(int64_t n_rows, int64_t n_cols, const int64_t* rowptr, const int64_t* col,
                     const double* val, bool validate);
// Download to host int64 arrays (caller allocates).
void download_csr(const DevCsr& A, int64_t* rowptr, int64_t* col, double* val);

// ---- SpMV epilogues ---------------------------------------------------------------
enum class Epi {
  kSpmv,       // y = A x
  kResidual,   // y = b - A x
  kResidualZero,  // x_out = 0 + wd .* b ; y = b - A x_out  (first sweep from x = 0 fused)
  kJacobi,     // y = x + wd .* (b - A x)          (wd = omega * inv_diag)
  kScaleDiag,  // y = (A x) .* d                   (Arnoldi, smoother.cpp:53-54)
  kSpmvDot2,   // y = A x ; dots (y.y, y.c) [gmres inner] or (x.y, x.c) [cg inner]
  kSpmvDot3,   // y = A x ; dots (y.u, y.y, y.c) [gmres] or (x.u, x.y, x.c) [cg]
  kSpmvDot1,   // y = A x ; dot (u . y)
  kJacobiDot2, // y = x + wd .* (b - A x) ; dots (b . y, c . y)  (PCG's r.z, r_old.z fused)
  kSpmvZero,   // y = A x ; x_out = 0 + d .* y  (restriction + the next level's zero-guess sweep)
};

struct SpmvArgs {
  const double* x = nullptr;
  double* y = nullptr;
  double* x_out = nullptr;     // kResidualZero: the smoothed iterate
  const double* b = nullptr;   // residual / jacobi rhs
  const double* d = nullptr;   // wd (jacobi) or inv_diag (scale)
  const double* c = nullptr;   // second dot operand
  const double* u = nullptr;   // third dot operand
  int dot_with_x = 0;          // cg-style inner products use x instead of y
  double* dots_out = nullptr;  // device slots for the dot results
  const int* pred = nullptr;   // device predicate: skip the launch body when *pred == 0
  // rows [row_base, row_base + row_count) only (row_count < 0: to the end); row_base must be a
  // multiple of A.rows_per_block so the row blocks coincide with the plan's
  int64_t row_base = 0;
  int64_t row_count = -1;
};

void spmv_run(const DevCsr& A, Epi epi, const SpmvArgs& a, int prof_family = 0);

inline void spmv(const DevCsr& A, const double* x, double* y, const int* pred = nullptr) {
  SpmvArgs a;
  a.x = x;
  a.y = y;
  a.pred = pred;
  spmv_run(A, Epi::kSpmv, a);
}

// Transpose with values; output rows sorted (sparse.cpp:133-151).
DevCsrPtr transpose(const DevCsr& A);

// device Poisson / 27-point generators (poisson.cpp:15-77 semantics)
DevCsrPtr generate_poisson_device(int dims, int64_t nx, int64_t ny, int64_t nz, double eps,
                                  int weak_axis);
DevCsrPtr generate_jump27_device(int64_t nx, int64_t ny, int64_t nz, double jump, int64_t block);
// Rows [row0, row0 + nrows) only (nrows < 0: to the end), global column ids; n_cols = n.
DevCsrPtr generate_poisson_rows(int dims, int64_t nx, int64_t ny, int64_t nz, double eps,
                                int weak_axis, int64_t row0, int64_t nrows);
DevCsrPtr generate_jump27_rows(int64_t nx, int64_t ny, int64_t nz, double jump, int64_t block,
                               int64_t row0, int64_t nrows);

double spmv_bytes(const DevCsr& A, Epi epi);
// the fused damped-Jacobi + PCG dots sweep runs on a value-dictionary SELL copy (latency-bound:
// the two extra streams ride along); false = the plain sweep and a separate dot pass
bool fuse_dots_on_dictionary();

// process-wide switch of the SELL value dictionary (default on; AGGMG_SELL_VI=0 starts it off);
// takes effect for operators planned (or refreshed) afterwards
std::atomic<int>& value_dictionary_switch();
std::atomic<int>& row_pattern_switch();

}  // namespace aggmg_b200
