/*
 * aggmg_b200.h — C-ABI drop-in boundary of the B200-native unsmoothed-aggregation AMG.
 *
 * Every entry point replaces one public function of the reference C++ library
 * `aggmg` (/root/reference/proj/core/include/aggmg/...).  The reference has no FFI of
 * its own; these signatures are what a ctypes / cgo / JNI binding of that C++ API
 * would bind: plain pointers and sizes, int64 host indices (reference types.hpp:12),
 * fp64 values (types.hpp:16), no C++ or torch types.
 *
 * Conventions
 *   - Every function returns AGGMG_OK (0) on success.  Failures that the reference
 *     reports as `aggmg::Error` (error.hpp:14-27) return AGGMG_ERR and leave the same
 *     message text in aggmg_last_error() (tests grep the reference substrings:
 *     "rebuild", "too large", "row i", "use fgmres", "length", "aggregate", "pivot",
 *     "diagonal", "outside shape").  CUDA failures return AGGMG_ERR_CUDA.
 *   - Host arrays in, host arrays out.  The computation runs on the current CUDA
 *     device through hand-written sm_100a kernels; there is no CPU fallback.
 *   - Output matrices are library-allocated aggmg_csr values; release them with
 *     aggmg_csr_free().
 *   - Results are independent of the device count and launch configuration (the
 *     reference's thread-count invariance, parallel.hpp:25-27).
 */
#ifndef AGGMG_B200_H
#define AGGMG_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define AGGMG_OK 0
#define AGGMG_ERR 1
#define AGGMG_ERR_CUDA 2

/* ---- value types --------------------------------------------------------- */

/* Canonical CSR (reference sparse.hpp:18-47): row_offsets[n_rows+1], strictly
 * increasing columns per row.  As an input the arrays are borrowed; as an output
 * they are owned by the library until aggmg_csr_free(). */
typedef struct aggmg_csr {
  int64_t n_rows;
  int64_t n_cols;
  int64_t nnz;
  int64_t* row_offsets;
  int64_t* col_indices;
  double* values;
} aggmg_csr;

/* enums mirror the reference values */
enum { AGGMG_ZERO_DIAG_POSITIVE = 0, AGGMG_ZERO_DIAG_FAIL = 1 };           /* strength.hpp:15 */
enum { AGGMG_SMOOTHER_JACOBI = 0, AGGMG_SMOOTHER_DAMPED_JACOBI = 1,
       AGGMG_SMOOTHER_SGS = 2 };                                          /* smoother.hpp:13 */
enum { AGGMG_CYCLE_V = 0, AGGMG_CYCLE_K = 1, AGGMG_CYCLE_HYBRID = 2 };     /* cycles.hpp:11 */
enum { AGGMG_INNER_CG = 0, AGGMG_INNER_GMRES = 1 };                       /* cycles.hpp:12 */
enum { AGGMG_SOLVER_FGMRES = 0, AGGMG_SOLVER_PCG = 1 };                   /* krylov.hpp:14 */

/* SetupConfig, reference hierarchy.hpp:30-38 (same defaults via aggmg_setup_config_default). */
typedef struct aggmg_setup_config {
  double alpha;            /* 0.25 */
  int64_t coarse_size_max; /* 600 */
  int32_t max_levels;      /* 25 */
  int32_t smoother;        /* AGGMG_SMOOTHER_DAMPED_JACOBI */
  int32_t arnoldi_m;       /* 5 */
  int32_t reuse_caches;    /* 0; coarse values always follow the cached segment order */
  uint64_t seed;           /* 42 */
} aggmg_setup_config;

/* CycleConfig, reference cycles.hpp:17-22. */
typedef struct aggmg_cycle_config {
  int32_t kind;     /* AGGMG_CYCLE_HYBRID */
  int32_t k_levels; /* 2 */
  double t;         /* 0.25 */
  int32_t inner;    /* AGGMG_INNER_GMRES */
} aggmg_cycle_config;

/* SolverConfig, reference krylov.hpp:16-21. */
typedef struct aggmg_solver_config {
  int32_t method;    /* AGGMG_SOLVER_FGMRES */
  double tol;        /* 1e-6 */
  int32_t max_iters; /* 200 */
  int32_t restart;   /* 30 */
} aggmg_solver_config;

/* SolveReport, reference krylov.hpp:23-30.  The caller provides `history` with
 * room for history_capacity doubles (max_iters + 1 always suffices); the library
 * writes history_length entries. */
typedef struct aggmg_solve_report {
  int32_t converged;
  int32_t iterations;
  double* history;
  int64_t history_capacity;
  int64_t history_length;
  double setup_seconds; /* filled by aggmg_setup_and_solve only */
  double solve_seconds;
  char note[256];
} aggmg_solve_report;

typedef struct aggmg_hierarchy aggmg_hierarchy;           /* Hierarchy, hierarchy.hpp:40-48 */
typedef struct aggmg_galerkin_cache aggmg_galerkin_cache; /* GalerkinCache, galerkin.hpp:25-45 */
typedef struct aggmg_dmatrix aggmg_dmatrix;               /* device-resident CSR (no reference analogue) */

/* ---- library state --------------------------------------------------------- */

const char* aggmg_version(void);                 /* types.hpp:18 */
const char* aggmg_last_error(void);              /* message of the last failing call (thread-local) */
int aggmg_init(int device);                      /* select device, create stream + memory pool */
int aggmg_synchronize(void);
void aggmg_set_num_threads(int n);               /* parallel.hpp:27 — accepted, no effect on results */
int aggmg_num_threads(void);                     /* parallel.hpp:29 — reports the SM count */
int64_t aggmg_kernel_launches(void);             /* number of kernels this library has launched */
/* Solve-phase dot products in the reference's 8192-chunk sequential order (1) or as
 * deterministic tree reductions (0, default).  Setup (Arnoldi omega) and aggmg_dot /
 * aggmg_norm2 always use the reference order (vector_ops.hpp:16-40).  Set to 1 BEFORE setup
 * and the hierarchy also keeps the reference's coarsest LU factors (dense.cpp:16-79) for a
 * substitution in the reference's order: solves are then bit-identical to the reference
 * (slower: 1.3-1.7x per step on the bench configs). */
void aggmg_set_exact_reductions(int on);
int aggmg_exact_reductions(void);
/* The SELL-32 copy of a large operator stores its values as one-byte codes into a table of
 * its distinct values when there are <= 256 of them (stencil matrices; same doubles, same
 * results).  on = 0 keeps plain fp64 values: operators planned or refreshed afterwards use the
 * 12-byte-per-entry layout (the variable-coefficient case; bench.py's no-dictionary line). */
void aggmg_set_value_dictionary(int on);
/* A large operator with a value dictionary and rows of <= 16 entries whose rows repeat a few
 * patterns (offsets from the diagonal position and values: stencil matrices) is stored as a
 * two-byte pattern id per row plus the pattern tables (same doubles, same order, same
 * results).  on = 0: operators planned or refreshed afterwards keep the SELL-32 copy. */
void aggmg_set_row_patterns(int on);
void aggmg_setup_config_default(aggmg_setup_config* c);
void aggmg_cycle_config_default(aggmg_cycle_config* c);
void aggmg_solver_config_default(aggmg_solver_config* c);
void aggmg_csr_free(aggmg_csr* m);

/* ---- L1 sparse / vector kernels (sparse.hpp, vector_ops.hpp) ---------------- */

int aggmg_spmv(const aggmg_csr* A, const double* x, double* y);            /* sparse.hpp:70-71 */
int aggmg_transpose(const aggmg_csr* A, aggmg_csr* T);                     /* sparse.hpp:78 */
int aggmg_dot(int64_t n, const double* a, const double* b, double* out);  /* vector_ops.hpp:20 */
int aggmg_norm2(int64_t n, const double* a, double* out);                 /* vector_ops.hpp:42 */
int aggmg_axpy(int64_t n, double a, const double* x, double* y);          /* vector_ops.hpp:45 */
int aggmg_scale(int64_t n, double a, double* x);                          /* vector_ops.hpp:50 */

/* ---- L2 setup components ----------------------------------------------------- */

/* strength.hpp:22-23 / strength.cpp:28-72 */
int aggmg_classic_strength(const aggmg_csr* A, double alpha, int zero_diag_policy, aggmg_csr* C);
/* strength.hpp:27 / strength.cpp:74-78; counts has C->n_cols entries */
int aggmg_influence_counts(const aggmg_csr* C, int64_t* counts);
/* strength.hpp:31 / strength.cpp:80-111 */
int aggmg_symmetrize_pattern(const aggmg_csr* C, aggmg_csr* S);
/* aggregation.hpp:28-29 / aggregation.cpp:45-86.  state[n] in {+1,-1}; roots are the
 * nodes with state +1, ascending. */
int aggmg_mis2(const aggmg_csr* S, const int64_t* influence, uint64_t seed, int8_t* state,
               int64_t* n_roots, int32_t* sweeps);
/* aggregation.hpp:45 / aggregation.cpp:88-159.  representatives has room for n. */
int aggmg_aggregate(const aggmg_csr* S, const aggmg_csr* A, const int8_t* state,
                    int64_t* assignment, int64_t* representatives, int64_t* n_aggregates);
/* transfer.hpp:24 / transfer.cpp:15-49 */
int aggmg_build_transfer(int64_t n_fine, int64_t n_aggregates, const int64_t* assignment,
                         const double* fine_b, aggmg_csr* P, aggmg_csr* R, double* coarse_b);
/* galerkin.hpp:16 — explicit R*A*P (two row-wise products, sparse.cpp:71-131 order) */
int aggmg_galerkin_direct(const aggmg_csr* R, const aggmg_csr* A, const aggmg_csr* P,
                          aggmg_csr* Ac);
/* galerkin.hpp:47 / galerkin.cpp:38-96 */
int aggmg_build_galerkin_cache(const aggmg_csr* A, int64_t n_aggregates, const int64_t* assignment,
                               aggmg_galerkin_cache** out);
/* sizes of the cache arrays: nnz_fine = entry length, nnz_coarse = segments */
int aggmg_galerkin_cache_info(const aggmg_galerkin_cache* c, int64_t* n_fine, int64_t* n_coarse,
                              int64_t* nnz_fine, int64_t* nnz_coarse);
/* copies the GalerkinCache fields (galerkin.hpp:29-44) to caller arrays; any pointer may be NULL */
int aggmg_galerkin_cache_export(const aggmg_galerkin_cache* c, int64_t* coarse_row_offsets,
                                int64_t* coarse_col_indices, int64_t* entry, int64_t* entry_row,
                                int64_t* segment_offsets, int64_t* slot_of_csr,
                                int64_t* rows_by_coarse, int64_t* agg_row_offsets);
/* galerkin.hpp:52-53 / galerkin.cpp:98-137 */
int aggmg_apply_galerkin_cache(const aggmg_galerkin_cache* c, const aggmg_csr* A,
                               const aggmg_csr* P, aggmg_csr* Ac);
void aggmg_galerkin_cache_free(aggmg_galerkin_cache* c);
/* smoother.hpp:31-32 / smoother.cpp:86-99; inv_diag has n entries (may be NULL) */
int aggmg_setup_smoother(const aggmg_csr* A, int kind, int arnoldi_m, uint64_t seed,
                         double* inv_diag, double* omega, double* rho_est);
/* smoother.hpp:37 / smoother.cpp:101-124; x is updated in place */
int aggmg_smooth(int kind, const double* inv_diag, double omega, const aggmg_csr* A,
                 const double* b, double* x);
/* dense.hpp:45 / dense.cpp:104-212 (host routine used by the smoother setup) */
int aggmg_hessenberg_eigenvalues(int64_t n, const double* H_row_major, double* re, double* im);

/* ---- L3 hierarchy ---------------------------------------------------------------- */

/* hierarchy.hpp:57 / hierarchy.cpp:34-88 */
int aggmg_setup_hierarchy(const aggmg_csr* A0, const double* B0, const aggmg_setup_config* cfg,
                          aggmg_hierarchy** out);
/* hierarchy.hpp:64 / hierarchy.cpp:90-104, in place on h.  The reference takes the
 * Hierarchy by value; a caller that keeps the old hierarchy clones it first (the C++ drop-in
 * does so whenever its handle is shared).  A level-0 operator shared with a device matrix
 * (aggmg_setup_hierarchy_device) is copied, never rewritten. */
int aggmg_refresh_values(aggmg_hierarchy* h, const double* new_values, int64_t count);
/* deep copy of a hierarchy (every level in HBM; Hierarchy's copy semantics) */
int aggmg_hierarchy_clone(const aggmg_hierarchy* h, aggmg_hierarchy** out);
void aggmg_hierarchy_free(aggmg_hierarchy* h);
int64_t aggmg_hierarchy_n_levels(const aggmg_hierarchy* h);                 /* hierarchy.hpp:46 */
int aggmg_hierarchy_level_size(const aggmg_hierarchy* h, int64_t k, int64_t* n, int64_t* nnz);
int aggmg_hierarchy_level_A(const aggmg_hierarchy* h, int64_t k, aggmg_csr* A); /* Level::A */
int aggmg_hierarchy_level_P(const aggmg_hierarchy* h, int64_t k, aggmg_csr* P); /* Level::P */
int aggmg_hierarchy_level_R(const aggmg_hierarchy* h, int64_t k, aggmg_csr* R); /* Level::R */
int aggmg_hierarchy_level_B(const aggmg_hierarchy* h, int64_t k, double* B);    /* Level::B */
/* aggregation of level k -> k+1 (GalerkinCache::assignment) and its MIS sweeps */
int aggmg_hierarchy_level_aggregation(const aggmg_hierarchy* h, int64_t k, int64_t* assignment,
                                      int64_t* n_aggregates, int32_t* mis_sweeps);
/* Level::smoother (smoother.hpp:18-24); inv_diag may be NULL */
int aggmg_hierarchy_level_smoother(const aggmg_hierarchy* h, int64_t k, double* omega,
                                   double* rho_est, double* inv_diag);
int64_t aggmg_hierarchy_n_warnings(const aggmg_hierarchy* h);              /* Hierarchy::warnings */
const char* aggmg_hierarchy_warning(const aggmg_hierarchy* h, int64_t i);
/* hierarchy.hpp:78 */
int aggmg_hierarchy_report(const aggmg_hierarchy* h, double* grid_complexity,
                           double* operator_complexity);
/* device time of the last setup (ms) split into phases */
int aggmg_hierarchy_setup_ms(const aggmg_hierarchy* h, double* total_ms);

/* ---- L4 cycles --------------------------------------------------------------- */

int aggmg_vcycle(const aggmg_hierarchy* h, int64_t k, const double* b, double* x);   /* cycles.hpp:28 */
int aggmg_kcycle(const aggmg_hierarchy* h, const aggmg_cycle_config* cfg, int64_t k,
                 const double* b, double* x);                                      /* cycles.hpp:37 */
int aggmg_apply_preconditioner(const aggmg_hierarchy* h, const aggmg_cycle_config* cfg,
                               const double* r, double* z);                        /* cycles.hpp:42 */

/* ---- L4 Krylov --------------------------------------------------------------- */

/* krylov.hpp:43-50.  M == NULL is the identity preconditioner (krylov.cpp:23-25);
 * otherwise M is apply_preconditioner(M, cycle, .) exactly as the reference CLI wires it
 * (aggmg_main.cpp:194-196). */
int aggmg_pcg(const aggmg_csr* A, const double* b, const double* x0, const aggmg_hierarchy* M,
              const aggmg_cycle_config* cycle, const aggmg_solver_config* cfg, double* x,
              aggmg_solve_report* report);
int aggmg_fgmres(const aggmg_csr* A, const double* b, const double* x0, const aggmg_hierarchy* M,
                 const aggmg_cycle_config* cycle, const aggmg_solver_config* cfg, double* x,
                 aggmg_solve_report* report);

/* krylov.hpp:38-50 with an arbitrary host preconditioner (the reference's
 * std::function<Vector(const Vector&)>, e.g. the CLI's lambda aggmg_main.cpp:194-196 or the
 * Jacobi preconditioner of test_krylov.cpp:129-156).  The Krylov loop stays on the device;
 * each application copies r (n doubles) to the host, calls M(r, z, n, user) and copies z back.
 * M returns 0 on success; nonzero aborts the solve with AGGMG_ERR ("preconditioner callback
 * failed").  M == NULL is the identity. */
typedef int (*aggmg_precond_fn)(const double* r, double* z, int64_t n, void* user);
int aggmg_pcg_cb(const aggmg_csr* A, const double* b, const double* x0, aggmg_precond_fn M,
                 void* user, const aggmg_solver_config* cfg, double* x, aggmg_solve_report* report);
int aggmg_fgmres_cb(const aggmg_csr* A, const double* b, const double* x0, aggmg_precond_fn M,
                    void* user, const aggmg_solver_config* cfg, double* x,
                    aggmg_solve_report* report);

/* One call = reference CLI `solve` pipeline (aggmg_main.cpp:163-210): setup_hierarchy(A, B0)
 * then pcg/fgmres(A, b, x0) preconditioned by the hierarchy.  B0/x0 may be NULL (ones / zeros).
 * Host buffers in and out; this is the end-to-end entry point bench.py times. */
int aggmg_setup_and_solve(const aggmg_csr* A, const double* b, const double* B0, const double* x0,
                          const aggmg_setup_config* setup, const aggmg_cycle_config* cycle,
                          const aggmg_solver_config* solver, double* x,
                          aggmg_solve_report* report);

/* ---- inputs (poisson.hpp) ------------------------------------------------------ */

/* poisson.hpp:17-26 / poisson.cpp:15-77, host generator */
int aggmg_generate_poisson(int dims, int64_t nx, int64_t ny, int64_t nz, double epsilon,
                           int weak_axis, aggmg_csr* A);
/* poisson.hpp:30 / poisson.cpp:81-87: x_i = uniform_sym(seed, i) in (-1, 1) */
int aggmg_random_vector(int64_t n, uint64_t seed, double* x);
/* 27-point variable-coefficient diffusion with coefficient jumps (BASELINE config 4;
 * no reference generator exists, definition in DESIGN.md) */
int aggmg_generate_jump27(int64_t nx, int64_t ny, int64_t nz, double jump, int64_t block,
                          aggmg_csr* A);

/* ---- device-resident path (inputs already in HBM; no reference analogue) ----------- */

int aggmg_dmatrix_from_host(const aggmg_csr* A, aggmg_dmatrix** out);
/* same matrix as aggmg_generate_poisson, generated directly in HBM */
int aggmg_dmatrix_poisson(int dims, int64_t nx, int64_t ny, int64_t nz, double epsilon,
                          int weak_axis, aggmg_dmatrix** out);
int aggmg_dmatrix_jump27(int64_t nx, int64_t ny, int64_t nz, double jump, int64_t block,
                         aggmg_dmatrix** out);
int aggmg_dmatrix_size(const aggmg_dmatrix* A, int64_t* n_rows, int64_t* nnz);
/* 1 in *sell when the operator carries a SELL-32 copy (large operators, 4-64 entries per row:
 * its SpMV-family kernels run sliced-ELL), 2 when that copy also stores its values as one-byte
 * codes into a table of the <= 256 distinct values (stencil operators), 3 when the operator is
 * stored as row-pattern ids (stencil operators with <= 16 entries per row and <= 4096
 * distinct rows up to the diagonal shift: aggmg_set_row_patterns), else 0 (CSR-stream) */
int aggmg_dmatrix_format(const aggmg_dmatrix* A, int* sell);
int aggmg_dmatrix_to_host(const aggmg_dmatrix* A, aggmg_csr* out);
void aggmg_dmatrix_free(aggmg_dmatrix* A);
/* setup_hierarchy on a device matrix (B0 = ones); the hierarchy shares A's storage.  Level 0's
 * kernel layout (its SELL-32 copy and value dictionary) is rebuilt as part of the setup. */
int aggmg_setup_hierarchy_device(const aggmg_dmatrix* A0, const aggmg_setup_config* cfg,
                                 aggmg_hierarchy** out);
/* device view of level k's operator (which = 0) or restriction R (which = 1); shares storage */
int aggmg_hierarchy_level_dmatrix(const aggmg_hierarchy* h, int64_t k, int which,
                                  aggmg_dmatrix** out);
/* pcg/fgmres on level 0 of h with b = ones, x0 = 0, everything resident in HBM;
 * x (host, may be NULL) receives the solution */
int aggmg_solve_device(const aggmg_hierarchy* h, const aggmg_cycle_config* cycle,
                       const aggmg_solver_config* cfg, double* x, aggmg_solve_report* report);

/* ---- row-partitioned multi-GPU path (no reference analogue: the reference
 * is single-process OpenMP, parallel.hpp:40-74) --------------------------------------------
 * Fine levels are split into contiguous row slabs, one per rank; levels at or below
 * `agglomerate_rows` are gathered onto rank 0.  Every call below is COLLECTIVE over the
 * communicator (all ranks call it in the same order).  Setup artefacts equal the one-GPU
 * hierarchy bit for bit; solve scalars are summed over ranks in rank order. */
typedef struct aggmg_comm aggmg_comm;
typedef struct aggmg_dist_matrix aggmg_dist_matrix;
typedef struct aggmg_dist_hierarchy aggmg_dist_hierarchy;

/* one process per GPU over NCCL: rank 0 creates the id, the launcher broadcasts it;
 * call aggmg_init(local_device) first */
int aggmg_comm_nccl_unique_id(char id[128]);
int aggmg_comm_init_nccl(int rank, int nranks, const char id[128], aggmg_comm** out);
/* R ranks as R threads of this process (devices[r] per rank, may repeat): fn(comm, rank,
 * user) runs on every rank thread; returns the first non-zero fn result (or an error). */
typedef int (*aggmg_rank_fn)(aggmg_comm* comm, int rank, void* user);
int aggmg_comm_run_threads(int nranks, const int* devices, aggmg_rank_fn fn, void* user);
int aggmg_comm_barrier(aggmg_comm* c);  /* host + device barrier over the ranks */
int aggmg_comm_rank(const aggmg_comm* c);
int aggmg_comm_size(const aggmg_comm* c);
const char* aggmg_comm_kind(const aggmg_comm* c);
void aggmg_comm_free(aggmg_comm* c);

/* this rank's rows [row0, row0 + rows->n_rows) of an n_global x n_global matrix, global
 * column ids (canonical rows) */
int aggmg_dist_matrix_from_host(aggmg_comm* c, int64_t n_global, int64_t row0,
                                const aggmg_csr* rows, aggmg_dist_matrix** out);
/* ---- Matrix Market I/O (matrix_market.hpp:23-35) ----------------------------------------
 * Reader: the reference's file semantics and error messages ("matrix market: line L: ...");
 * data lines parsed on all host cores, CSR assembled on the device.  Writers: 17 significant
 * digits, byte-identical to the reference's. */
int aggmg_read_matrix_market_file(const char* path, int allow_pattern, aggmg_csr* A);
int aggmg_read_matrix_market(const char* text, int64_t size, int allow_pattern, aggmg_csr* A);
int aggmg_write_matrix_market_file(const char* path, const aggmg_csr* A);
/* x may be NULL to query the length n */
int aggmg_read_vector_market_file(const char* path, double* x, int64_t capacity, int64_t* n);
int aggmg_write_vector_market_file(const char* path, const double* x, int64_t n);

/* host rows [row0, row0 + nrows) of the generator matrices (global column ids): one rank's
 * slab as a host input for aggmg_dist_matrix_from_host */
int aggmg_generate_poisson_rows(int dims, int64_t nx, int64_t ny, int64_t nz, double epsilon,
                                int weak_axis, int64_t row0, int64_t nrows, aggmg_csr* A);
int aggmg_generate_jump27_rows(int64_t nx, int64_t ny, int64_t nz, double jump, int64_t block,
                               int64_t row0, int64_t nrows, aggmg_csr* A);
/* generated in HBM on every rank (even row partition) — poisson.cpp:15-77 / DESIGN.md §7 */
int aggmg_dist_matrix_poisson(aggmg_comm* c, int dims, int64_t nx, int64_t ny, int64_t nz,
                              double epsilon, int weak_axis, aggmg_dist_matrix** out);
int aggmg_dist_matrix_jump27(aggmg_comm* c, int64_t nx, int64_t ny, int64_t nz, double jump,
                             int64_t block, aggmg_dist_matrix** out);
int aggmg_dist_matrix_info(const aggmg_dist_matrix* A, int64_t* n_global, int64_t* row0,
                           int64_t* n_local, int64_t* nnz_local);
/* this rank's rows: 1 = SELL-32 copy, 2 = SELL-32 with the value dictionary, 3 = row-pattern
 * ids, 0 = CSR-stream */
int aggmg_dist_matrix_format(const aggmg_dist_matrix* A, int* sell);
void aggmg_dist_matrix_free(aggmg_dist_matrix* A);

/* setup_hierarchy (hierarchy.hpp:57) over the ranks; B0_local (host, this rank's rows) may be
 * NULL = ones; agglomerate_rows <= 0 picks the default (max(coarse_size_max, 2^22): coarse levels below ~4 M rows are
 * latency-bound, one GPU runs them faster than exchanging halos for them) */
int aggmg_dist_setup(aggmg_comm* c, const aggmg_dist_matrix* A0, const double* B0_local,
                     const aggmg_setup_config* cfg, int64_t agglomerate_rows,
                     aggmg_dist_hierarchy** out);
/* pcg/fgmres (krylov.hpp:43-50) preconditioned by the partitioned cycle, x0 = 0;
 * b_local (host) NULL = ones; x_local (host) may be NULL */
int aggmg_dist_solve(aggmg_dist_hierarchy* h, const aggmg_cycle_config* cycle,
                     const aggmg_solver_config* cfg, const double* b_local, double* x_local,
                     aggmg_solve_report* report);
/* refresh_values (hierarchy.hpp:64) over the ranks: new values of this rank's level-0 rows
 * (same pattern); needs a hierarchy set up with reuse_caches */
int aggmg_dist_refresh_values(aggmg_dist_hierarchy* h, const double* new_values_local,
                              int64_t count);
/* z = M r on this rank's rows (apply_preconditioner, cycles.hpp:42) */
int aggmg_dist_apply_preconditioner(aggmg_dist_hierarchy* h, const aggmg_cycle_config* cycle,
                                    const double* r_local, double* z_local);
int aggmg_dist_hierarchy_info(const aggmg_dist_hierarchy* h, int64_t* n_levels,
                              int64_t* n_distributed, double* setup_ms);
int aggmg_dist_hierarchy_level_size(const aggmg_dist_hierarchy* h, int64_t k, int64_t* n,
                                    int64_t* nnz);
/* level k's artefacts gathered on rank 0 (global numbering; other ranks receive nothing):
 * operator, aggregation (assignment[n_k], mis sweeps), P values (pval[n_k]), B[n_k], omega */
int aggmg_dist_hierarchy_level_A(aggmg_dist_hierarchy* h, int64_t k, aggmg_csr* A);
int aggmg_dist_hierarchy_level_transfer(aggmg_dist_hierarchy* h, int64_t k, int64_t* assignment,
                                        double* pval, int32_t* mis_sweeps);
int aggmg_dist_hierarchy_level_B(aggmg_dist_hierarchy* h, int64_t k, double* B);
int aggmg_dist_hierarchy_level_omega(aggmg_dist_hierarchy* h, int64_t k, double* omega);
int64_t aggmg_dist_hierarchy_n_warnings(const aggmg_dist_hierarchy* h);
const char* aggmg_dist_hierarchy_warning(const aggmg_dist_hierarchy* h, int64_t i);
void aggmg_dist_hierarchy_free(aggmg_dist_hierarchy* h);

/* ---- measurement ------------------------------------------------------------------ */

/* Per-kernel-family CUDA-event timing on the library stream.  mask has bit (1 << f) set
 * for every timed family f (0 = off); ids in DESIGN.md (1 = level-0 damped-Jacobi sweep,
 * 2 = level-0 SpMV / residual). */
int aggmg_profile_enable(int mask);
int aggmg_profile_read(int family, double* total_ms, int64_t* launches, double* bytes);
/* device time on the library stream between the two calls (ms) */
int aggmg_timer_start(void);
int aggmg_timer_stop(double* ms);
/* dot_device micro-benchmark: np products over n elements, exact = reference chunk order */
int aggmg_bench_dot(int64_t n, int np, int exact, int reps, double* avg_ms);
/* SpMV micro-benchmark on a device matrix: average ms per launch over `reps` launches */
int aggmg_bench_spmv(const aggmg_dmatrix* A, int reps, double* avg_ms, double* bytes);
/* same for one CSR-stream variant: 0 spmv, 1 residual, 2 fused zero-guess Jacobi+residual,
 * 3 damped-Jacobi sweep, 4 spmv + dot, 5 spmv scaled by the inverse diagonal,
 * 6 damped-Jacobi sweep + the two fused PCG dots, 7 one level-scheduled symmetric Gauss-Seidel
 * smooth (forward + backward) */
int aggmg_bench_kernel(const aggmg_dmatrix* A, int kind, int reps, double* avg_ms, double* bytes);

#ifdef __cplusplus
}
#endif

#endif /* AGGMG_B200_H */
