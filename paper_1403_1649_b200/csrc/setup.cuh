// setup.cuh — the AMG setup kernels, bit-exact with the
// reference's `reuse_caches=true` path.
#pragma once

#include <vector>

#include "sparse.cuh"

namespace aggmg_b200 {

// a3: classic strength (strength.cpp:28-72).  Pattern only (values not stored on device).
DevCsrPtr classic_strength(const DevCsr& A, double alpha, int zero_diag_policy);
// Same kernel on the local rows of a row-partitioned operator (local column ids).
DevCsrPtr strength_rows(const DevCsr& A, double alpha, int zero_diag_policy);
// a4 + a5: influence counts (column counts of C) and S = pattern(C u C^T).
void influence_and_symmetrize(const DevCsr& C, DevBuf<idx>& influence, DevCsrPtr& S);

// a6: MIS(2) (aggregation.cpp:45-86).  state[i] in {+1,-1}.
struct Mis2Dev {
  DevBuf<int8_t> state;
  int sweeps = 0;
};
Mis2Dev mis2(const DevCsr& S, const idx* influence, uint64_t seed);

// a7: aggregation (aggregation.cpp:88-159).
struct AggDev {
  int64_t n_fine = 0, n_agg = 0;
  DevBuf<idx> assignment;       // fine -> aggregate
  DevBuf<idx> representatives;  // aggregate -> representative node
  // grouping of fine rows by aggregate, ascending inside a group (galerkin.cpp:87-94)
  DevBuf<idx> agg_row_offsets;  // n_agg + 1
  DevBuf<idx> rows_by_coarse;   // n_fine
};
AggDev aggregate(const DevCsr& S, const DevCsr& A, const int8_t* state);
void build_groups(AggDev& agg);  // agg_row_offsets / rows_by_coarse from assignment

// a8: transfer (transfer.cpp:15-49).  pval[i] = P value of row i (0 for empty rows);
// coarse_b[J] = ||b restricted to J||; R = P^T as CSR (rows ascending fine index).
struct TransferDev {
  DevBuf<double> pval;
  DevBuf<double> coarse_b;
  DevCsrPtr R;
  int64_t p_nnz = 0;
};
TransferDev build_transfer(const AggDev& agg, const double* fine_b);
// The same kernels over explicit member groups (goff / rows index b and pval): returns the
// first aggregate whose norm vanishes, or -1.
int64_t transfer_norms_groups(const idx* goff, const idx* rows, const double* b, int64_t nc,
                              double* coarse_b, idx* rcnt);
void transfer_R_groups(const idx* goff, const idx* rows, const double* pval, int64_t nc,
                       const idx* rrp, idx* rcol, double* rval);

// a9/a10: Galerkin cache and numeric reduce (galerkin.cpp:38-137).
struct GalerkinDev {
  int64_t n_fine = 0, n_coarse = 0, nnz_fine = 0, nnz_coarse = 0;
  DevBuf<idx> coarse_rowptr, coarse_col;
  DevBuf<idx> entry, entry_row, segment_offsets, slot_of_csr;
  DevBuf<idx> group_offsets, group_rows;  // copy of the aggregate grouping (not for partial
                                          // caches): the row-walk numeric reduce
  int max_coarse_row = 0;
  uint64_t pattern_hash = 0;
  bool lean = false;  // entry / entry_row / segment_offsets not built (max_coarse_row <= 64)
};
// partial: the groups cover only some rows of A (rows of other groups, and halo rows, are
// skipped; the row-partitioned setup's extended row set) — no coverage check, no fingerprint.
// fingerprint: the pattern hash apply_galerkin_cache checks for a caller-supplied A (galerkin.cpp:
// 18-29, 101-103); a hierarchy applies its cache to its own stored operator and skips it.
// lean: a hierarchy's own cache — only the coarse pattern and slot_of_csr when every coarse row
// fits the row-walk reduce (the per-entry sorted arrays are for the standalone cache API)
// values (lean path only): also the coarse values for P weights pval (the numeric reduce fused
// into the fill pass); left empty when the full path ran
GalerkinDev build_galerkin_cache(const DevCsr& A, const AggDev& agg, bool partial = false,
                                 bool fingerprint = true, bool lean = false,
                                 const double* pval = nullptr, DevBuf<double>* values = nullptr);
// the coarse operator of a cache and its values
DevCsrPtr coarse_from_cache(const GalerkinDev& g, DevBuf<double>&& values);
// Ac values for the cached pattern.  pval: per fine row P weight.
DevCsrPtr apply_galerkin_cache(const GalerkinDev& g, const DevCsr& A, const double* pval);
uint64_t pattern_fingerprint(const DevCsr& A, const idx* assignment);

// galerkin_direct (galerkin.cpp:33-36): R*(A*P) for P = one entry per row (pval) and
// R = P^T, summed in the association and order of the reference's two spmm calls.
DevCsrPtr galerkin_direct(const DevCsr& A, const AggDev& agg, const double* pval);

}  // namespace aggmg_b200
