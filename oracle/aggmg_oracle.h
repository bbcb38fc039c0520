/*
 * aggmg_oracle.h — TEST INFRASTRUCTURE.  CPU restatement of the reference aggmg
 * algorithm (/root/reference/proj/core) in plain C, used only by tests/, smoke() and
 * bench.py's cpu_baseline leg as the checker.  Never linked into the product.
 *
 * Every function mirrors the same-named entry point of include/aggmg_b200.h with the
 * prefix aggmg_oracle_ and the same argument meaning; opaque handles are void*.
 * Pinned against the reference itself (oracle/_ref, tests/test_oracle.py) and the
 * committed golden fixtures (tests/golden/).
 */
#ifndef AGGMG_ORACLE_H
#define AGGMG_ORACLE_H

#include "../include/aggmg_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* aggmg_oracle_last_error(void);
void aggmg_oracle_csr_free(aggmg_csr* m);
void aggmg_oracle_set_num_threads(int n);
int aggmg_oracle_num_threads(void);
int aggmg_oracle_generate_poisson(int dims, int64_t nx, int64_t ny, int64_t nz, double eps,
                                  int weak_axis, aggmg_csr* A);
int aggmg_oracle_generate_jump27(int64_t nx, int64_t ny, int64_t nz, double jump, int64_t block,
                                 aggmg_csr* A);
int aggmg_oracle_spmv(const aggmg_csr* A, const double* x, double* y);
int aggmg_oracle_transpose(const aggmg_csr* A, aggmg_csr* T);
int aggmg_oracle_dot(int64_t n, const double* a, const double* b, double* out);
int aggmg_oracle_norm2(int64_t n, const double* a, double* out);
int aggmg_oracle_axpy(int64_t n, double a, const double* x, double* y);
int aggmg_oracle_scale(int64_t n, double a, double* x);
int aggmg_oracle_classic_strength(const aggmg_csr* A, double alpha, int policy, aggmg_csr* C);
int aggmg_oracle_influence_counts(const aggmg_csr* C, int64_t* counts);
int aggmg_oracle_symmetrize_pattern(const aggmg_csr* C, aggmg_csr* S);
int aggmg_oracle_mis2(const aggmg_csr* S, const int64_t* influence, uint64_t seed, int8_t* state,
                      int64_t* n_roots, int32_t* sweeps);
int aggmg_oracle_aggregate(const aggmg_csr* S, const aggmg_csr* A, const int8_t* state,
                           int64_t* assignment, int64_t* representatives, int64_t* n_aggregates);
int aggmg_oracle_build_transfer(int64_t n, int64_t nc, const int64_t* assignment,
                                const double* fine_b, aggmg_csr* P, aggmg_csr* R, double* coarse_b);
int aggmg_oracle_galerkin_direct(const aggmg_csr* R, const aggmg_csr* A, const aggmg_csr* P,
                                 aggmg_csr* Ac);
int aggmg_oracle_build_galerkin_cache(const aggmg_csr* A, int64_t nc, const int64_t* assignment,
                                      void** out);
int aggmg_oracle_galerkin_cache_info(const void* c, int64_t* n_fine, int64_t* n_coarse,
                                     int64_t* nnz_fine, int64_t* nnz_coarse);
int aggmg_oracle_galerkin_cache_export(const void* c, int64_t* coarse_row_offsets,
                                       int64_t* coarse_col_indices, int64_t* entry,
                                       int64_t* entry_row, int64_t* segment_offsets,
                                       int64_t* slot_of_csr, int64_t* rows_by_coarse,
                                       int64_t* agg_row_offsets);
int aggmg_oracle_apply_galerkin_cache(const void* c, const aggmg_csr* A, const aggmg_csr* P,
                                      aggmg_csr* Ac);
void aggmg_oracle_galerkin_cache_free(void* c);
int aggmg_oracle_setup_smoother(const aggmg_csr* A, int kind, int m, uint64_t seed,
                                double* inv_diag, double* omega, double* rho);
int aggmg_oracle_smooth(int kind, const double* inv_diag, double omega, const aggmg_csr* A,
                        const double* b, double* x);
int aggmg_oracle_hessenberg_eigenvalues(int64_t n, const double* H, double* re, double* im);
int aggmg_oracle_setup_hierarchy(const aggmg_csr* A0, const double* B0,
                                 const aggmg_setup_config* cfg, void** out);
int aggmg_oracle_refresh_values(void* h, const double* values, int64_t count);
void aggmg_oracle_hierarchy_free(void* h);
int64_t aggmg_oracle_hierarchy_n_levels(const void* h);
int aggmg_oracle_hierarchy_level_size(const void* h, int64_t k, int64_t* n, int64_t* nnz);
int aggmg_oracle_hierarchy_level_A(const void* h, int64_t k, aggmg_csr* A);
int aggmg_oracle_hierarchy_level_P(const void* h, int64_t k, aggmg_csr* P);
int aggmg_oracle_hierarchy_level_R(const void* h, int64_t k, aggmg_csr* R);
int aggmg_oracle_hierarchy_level_B(const void* h, int64_t k, double* B);
int aggmg_oracle_hierarchy_level_aggregation(const void* h, int64_t k, int64_t* assignment,
                                             int64_t* n_aggregates, int32_t* mis_sweeps);
int aggmg_oracle_hierarchy_level_smoother(const void* h, int64_t k, double* omega, double* rho,
                                          double* inv_diag);
int64_t aggmg_oracle_hierarchy_n_warnings(const void* h);
const char* aggmg_oracle_hierarchy_warning(const void* h, int64_t i);
int aggmg_oracle_vcycle(const void* h, int64_t k, const double* b, double* x);
int aggmg_oracle_kcycle(const void* h, const aggmg_cycle_config* cfg, int64_t k, const double* b,
                        double* x);
int aggmg_oracle_apply_preconditioner(const void* h, const aggmg_cycle_config* cfg,
                                      const double* r, double* z);
int aggmg_oracle_pcg(const aggmg_csr* A, const double* b, const double* x0, const void* M,
                     const aggmg_cycle_config* cycle, const aggmg_solver_config* cfg, double* x,
                     aggmg_solve_report* rep);
int aggmg_oracle_fgmres(const aggmg_csr* A, const double* b, const double* x0, const void* M,
                        const aggmg_cycle_config* cycle, const aggmg_solver_config* cfg,
                        double* x, aggmg_solve_report* rep);
int aggmg_oracle_setup_and_solve(const aggmg_csr* A, const double* b, const double* B0,
                                 const double* x0, const aggmg_setup_config* setup,
                                 const aggmg_cycle_config* cycle,
                                 const aggmg_solver_config* solver, double* x,
                                 aggmg_solve_report* rep);

#ifdef __cplusplus
}
#endif

#endif
