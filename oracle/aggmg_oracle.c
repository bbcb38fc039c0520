/*
 * aggmg_oracle.c — TEST INFRASTRUCTURE ONLY (see aggmg_oracle.h).
 *
 * Plain-C, single-threaded restatement of the reference aggmg setup/solve path
 * (/root/reference/proj/core/src).  Each function cites the reference lines it restates.
 * Arithmetic follows the reference's evaluation order and is compiled with
 * -ffp-contract=off (the reference is built without -march, hence without FMA), so the
 * setup artefacts are bit-identical and the solve histories identical up to the
 * Hessenberg eigen-solver's last bits.  Only tests/, smoke() and bench.py's cpu_baseline
 * leg load this library, always as the checker.
 */
#define _POSIX_C_SOURCE 200809L
#include "aggmg_oracle.h"

#include <math.h>
#include <setjmp.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>

/* ---- errors (reference error.hpp:14-27) --------------------------------------------- */

static _Thread_local char g_err[512];
static _Thread_local jmp_buf* g_jb;

static void fail(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof g_err, fmt, ap);
  va_end(ap);
  longjmp(*g_jb, 1);
}
#define API_BEGIN                 \
  jmp_buf jb_;                    \
  jmp_buf* prev_jb_ = g_jb;       \
  g_jb = &jb_;                    \
  if (setjmp(jb_)) {              \
    g_jb = prev_jb_;              \
    return AGGMG_ERR;             \
  }
#define API_END          \
  g_jb = prev_jb_;       \
  g_err[0] = 0;          \
  return AGGMG_OK;

static void* xmalloc(size_t n) {
  void* p = malloc(n ? n : 1);
  if (!p) fail("oracle: out of memory");
  return p;
}
static void* xcalloc(size_t n, size_t s) {
  void* p = calloc(n ? n : 1, s ? s : 1);
  if (!p) fail("oracle: out of memory");
  return p;
}

const char* aggmg_oracle_last_error(void) { return g_err; }
void aggmg_oracle_set_num_threads(int n) { (void)n; }
int aggmg_oracle_num_threads(void) { return 1; }

/* ---- CSR helpers (reference sparse.hpp:18-47) ---------------------------------------- */

static void csr_alloc(aggmg_csr* m, int64_t rows, int64_t cols, int64_t nnz) {
  m->n_rows = rows;
  m->n_cols = cols;
  m->nnz = nnz;
  m->row_offsets = xcalloc((size_t)rows + 1, sizeof(int64_t));
  m->col_indices = xmalloc(sizeof(int64_t) * (size_t)nnz);
  m->values = xmalloc(sizeof(double) * (size_t)nnz);
}
void aggmg_oracle_csr_free(aggmg_csr* m) {
  if (!m) return;
  free(m->row_offsets);
  free(m->col_indices);
  free(m->values);
  m->row_offsets = NULL;
  m->col_indices = NULL;
  m->values = NULL;
}
static int64_t nnz_of(const aggmg_csr* m) { return m->row_offsets[m->n_rows]; }
static void csr_copy(aggmg_csr* dst, const aggmg_csr* src) {
  const int64_t nnz = nnz_of(src);
  csr_alloc(dst, src->n_rows, src->n_cols, nnz);
  memcpy(dst->row_offsets, src->row_offsets, sizeof(int64_t) * (size_t)(src->n_rows + 1));
  memcpy(dst->col_indices, src->col_indices, sizeof(int64_t) * (size_t)nnz);
  if (src->values)
    memcpy(dst->values, src->values, sizeof(double) * (size_t)nnz);
  else
    for (int64_t k = 0; k < nnz; ++k) dst->values[k] = 1.0;
}
static void csr_empty(aggmg_csr* m) { csr_alloc(m, 0, 0, 0); }

/* value at (i, j), 0 when absent: binary search (sparse.cpp:15-20) */
static double csr_at(const aggmg_csr* A, int64_t i, int64_t j) {
  int64_t lo = A->row_offsets[i], hi = A->row_offsets[i + 1];
  const int64_t end = hi;
  while (lo < hi) {
    const int64_t mid = lo + (hi - lo) / 2;
    if (A->col_indices[mid] < j)
      lo = mid + 1;
    else
      hi = mid;
  }
  return (lo < end && A->col_indices[lo] == j) ? A->values[lo] : 0.0;
}

/* canonical-form check (sparse.cpp:22-39) */
static void csr_validate(const aggmg_csr* A) {
  if (A->n_rows < 0 || A->n_cols < 0) fail("negative dimensions");
  if (A->row_offsets[0] != 0) fail("row_offsets[0] must be 0");
  for (int64_t i = 0; i < A->n_rows; ++i) {
    if (A->row_offsets[i] > A->row_offsets[i + 1]) fail("row_offsets must be non-decreasing");
    for (int64_t k = A->row_offsets[i]; k < A->row_offsets[i + 1]; ++k) {
      if (A->col_indices[k] < 0 || A->col_indices[k] >= A->n_cols)
        fail("column index out of range in row %lld", (long long)i);
      if (k > A->row_offsets[i] && A->col_indices[k - 1] >= A->col_indices[k])
        fail("columns must be strictly increasing in row %lld", (long long)i);
    }
  }
}

/* ---- counter RNG (rng.hpp:14-34) ---------------------------------------------------- */

static uint64_t hash_mix(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}
static double u01(uint64_t seed, uint64_t c) {
  const uint64_t bits = hash_mix(hash_mix(seed) ^ c) >> 11;
  return ((double)bits + 0.5) * 0x1.0p-53;
}
static double usym(uint64_t seed, uint64_t c) { return 2.0 * u01(seed, c) - 1.0; }
static uint64_t level_seed(uint64_t seed, int64_t level, uint64_t tag) { /* hierarchy.cpp:25-27 */
  return hash_mix(hash_mix(seed ^ tag) ^ (uint64_t)level);
}

/* ---- vector ops: fixed 8192-element chunks (vector_ops.hpp:16-52) ---------------------- */

enum { CHUNK = 8192 };
static double vdot(int64_t n, const double* a, const double* b) {
  if (n <= CHUNK) {
    double s = 0.0;
    for (int64_t i = 0; i < n; ++i) s += a[i] * b[i];
    return s;
  }
  double total = 0.0;
  for (int64_t lo = 0; lo < n; lo += CHUNK) {
    const int64_t hi = lo + CHUNK < n ? lo + CHUNK : n;
    double s = 0.0;
    for (int64_t i = lo; i < hi; ++i) s += a[i] * b[i];
    total += s;
  }
  return total;
}
static double vnorm(int64_t n, const double* a) { return sqrt(vdot(n, a, a)); }
static void vaxpy(int64_t n, double a, const double* x, double* y) {
  for (int64_t i = 0; i < n; ++i) y[i] += a * x[i];
}
static void vscale(int64_t n, double a, double* x) {
  for (int64_t i = 0; i < n; ++i) x[i] *= a;
}
static double* vdup(int64_t n, const double* x) {
  double* y = xmalloc(sizeof(double) * (size_t)n);
  memcpy(y, x, sizeof(double) * (size_t)n);
  return y;
}

/* ---- sparse kernels ------------------------------------------------------------------- */

/* y = A x, row-sequential sums (sparse.cpp:52-63) */
static void spmv(const aggmg_csr* A, const double* x, double* y) {
  for (int64_t i = 0; i < A->n_rows; ++i) {
    double s = 0.0;
    for (int64_t k = A->row_offsets[i]; k < A->row_offsets[i + 1]; ++k)
      s += A->values[k] * x[A->col_indices[k]];
    y[i] = s;
  }
}

/* counting-sort transpose, rows stay sorted (sparse.cpp:133-151) */
static void transpose(const aggmg_csr* A, aggmg_csr* T) {
  const int64_t nnz = nnz_of(A);
  csr_alloc(T, A->n_cols, A->n_rows, nnz);
  for (int64_t k = 0; k < nnz; ++k) T->row_offsets[A->col_indices[k] + 1]++;
  for (int64_t j = 0; j < A->n_cols; ++j) T->row_offsets[j + 1] += T->row_offsets[j];
  int64_t* next = xmalloc(sizeof(int64_t) * (size_t)(A->n_cols + 1));
  memcpy(next, T->row_offsets, sizeof(int64_t) * (size_t)(A->n_cols + 1));
  for (int64_t i = 0; i < A->n_rows; ++i)
    for (int64_t k = A->row_offsets[i]; k < A->row_offsets[i + 1]; ++k) {
      const int64_t p = next[A->col_indices[k]]++;
      T->col_indices[p] = i;
      T->values[p] = A->values ? A->values[k] : 1.0;
    }
  free(next);
}

static int cmp_i64(const void* a, const void* b) {
  const int64_t x = *(const int64_t*)a, y = *(const int64_t*)b;
  return (x > y) - (x < y);
}

/* C = A B: accumulation in A's row-entry order, touched columns emitted sorted
 * (sparse.cpp:71-131) */
static void spmm(const aggmg_csr* A, const aggmg_csr* B, aggmg_csr* Cm) {
  if (A->n_cols != B->n_rows)
    fail("spmm: inner dimensions differ (%lld vs %lld)", (long long)A->n_cols, (long long)B->n_rows);
  int64_t* mark = xmalloc(sizeof(int64_t) * (size_t)(B->n_cols + 1));
  double* acc = xcalloc((size_t)B->n_cols + 1, sizeof(double));
  int64_t* touched = xmalloc(sizeof(int64_t) * (size_t)(B->n_cols + 1));
  int64_t* rownnz = xcalloc((size_t)A->n_rows + 1, sizeof(int64_t));
  for (int64_t j = 0; j < B->n_cols; ++j) mark[j] = -1;
  for (int64_t i = 0; i < A->n_rows; ++i)
    for (int64_t ka = A->row_offsets[i]; ka < A->row_offsets[i + 1]; ++ka) {
      const int64_t k = A->col_indices[ka];
      for (int64_t kb = B->row_offsets[k]; kb < B->row_offsets[k + 1]; ++kb)
        if (mark[B->col_indices[kb]] != i) {
          mark[B->col_indices[kb]] = i;
          rownnz[i]++;
        }
    }
  int64_t total = 0;
  for (int64_t i = 0; i < A->n_rows; ++i) total += rownnz[i];
  csr_alloc(Cm, A->n_rows, B->n_cols, total);
  for (int64_t i = 0; i < A->n_rows; ++i) Cm->row_offsets[i + 1] = Cm->row_offsets[i] + rownnz[i];
  for (int64_t j = 0; j < B->n_cols; ++j) mark[j] = -1;
  for (int64_t i = 0; i < A->n_rows; ++i) {
    int64_t nt = 0;
    for (int64_t ka = A->row_offsets[i]; ka < A->row_offsets[i + 1]; ++ka) {
      const int64_t k = A->col_indices[ka];
      const double av = A->values[ka];
      for (int64_t kb = B->row_offsets[k]; kb < B->row_offsets[k + 1]; ++kb) {
        const int64_t j = B->col_indices[kb];
        if (mark[j] != i) {
          mark[j] = i;
          acc[j] = 0.0;
          touched[nt++] = j;
        }
        acc[j] += av * B->values[kb];
      }
    }
    qsort(touched, (size_t)nt, sizeof(int64_t), cmp_i64);
    int64_t out = Cm->row_offsets[i];
    for (int64_t t = 0; t < nt; ++t) {
      Cm->col_indices[out] = touched[t];
      Cm->values[out] = acc[touched[t]];
      ++out;
    }
  }
  free(mark);
  free(acc);
  free(touched);
  free(rownnz);
}

/* ---- problem generators (poisson.cpp:15-77; jump27 per DESIGN.md §7) ------------------- */

static void gen_poisson(int dims, int64_t nx, int64_t ny, int64_t nz, double eps, int weak,
                        aggmg_csr* A) {
  if (dims != 2 && dims != 3) fail("poisson: dims must be 2 or 3");
  if (dims == 2) nz = 1;
  if (nx < 1 || ny < 1 || nz < 1) fail("poisson: grid extents must be positive");
  if (!(eps > 0.0)) fail("poisson: epsilon must be positive");
  if (weak < 0) weak = dims == 2 ? 1 : 2;
  if (weak >= dims) fail("poisson: weak axis %d out of range for %dD", weak, dims);
  const double cx = weak == 0 ? -eps : -1.0, cy = weak == 1 ? -eps : -1.0,
               cz = weak == 2 ? -eps : -1.0;
  const double diag = -2.0 * (cx + cy + (dims == 3 ? cz : 0.0));
  const int64_t n = nx * ny * nz;
  csr_alloc(A, n, n, n * (dims == 3 ? 7 : 5));
  int64_t p = 0;
  for (int64_t r = 0; r < n; ++r) {
    const int64_t i = r % nx, j = (r / nx) % ny, k = r / (nx * ny);
#define PUT(c, v) (A->col_indices[p] = (c), A->values[p] = (v), ++p)
    if (k > 0) PUT(r - nx * ny, cz);
    if (j > 0) PUT(r - nx, cy);
    if (i > 0) PUT(r - 1, cx);
    PUT(r, diag);
    if (i + 1 < nx) PUT(r + 1, cx);
    if (j + 1 < ny) PUT(r + nx, cy);
    if (k + 1 < nz) PUT(r + nx * ny, cz);
#undef PUT
    A->row_offsets[r + 1] = p;
  }
  A->nnz = p;
}

static double kappa27(int64_t x, int64_t y, int64_t z, int64_t block, double jump) {
  return (((x / block) + (y / block) + (z / block)) & 1) ? jump : 1.0;
}
static void gen_jump27(int64_t nx, int64_t ny, int64_t nz, double jump, int64_t block,
                       aggmg_csr* A) {
  if (nx < 1 || ny < 1 || nz < 1 || block < 1) fail("jump27: extents must be positive");
  const int64_t n = nx * ny * nz;
  csr_alloc(A, n, n, n * 27);
  int64_t p = 0;
  for (int64_t r = 0; r < n; ++r) {
    const int64_t i = r % nx, j = (r / nx) % ny, k = r / (nx * ny);
    const double ki = kappa27(i, j, k, block, jump);
    double diag = 0.0;
    int64_t pd = -1;
    for (int dz = -1; dz <= 1; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          const int64_t x = i + dx, y = j + dy, z = k + dz;
          if (dx == 0 && dy == 0 && dz == 0) {
            pd = p;
            A->col_indices[p++] = r;
            continue;
          }
          if (x < 0 || x >= nx || y < 0 || y >= ny || z < 0 || z >= nz) {
            diag = diag + ki;
            continue;
          }
          const double kj = kappa27(x, y, z, block, jump);
          const double kij = ((2.0 * ki) * kj) / (ki + kj);
          diag = diag + kij;
          A->col_indices[p] = (z * ny + y) * nx + x;
          A->values[p++] = -kij;
        }
    A->values[pd] = diag;
    A->row_offsets[r + 1] = p;
  }
  A->nnz = p;
}

/* ---- strength (strength.cpp:16-111) --------------------------------------------------- */

static void strength(const aggmg_csr* A, double alpha, int fail_zero, aggmg_csr* Cm) {
  if (A->n_rows != A->n_cols) fail("strength: matrix must be square");
  if (!(alpha > 0.0 && alpha < 1.0)) fail("strength: alpha must be in (0, 1)");
  const int64_t n = A->n_rows;
  int64_t* cnt = xcalloc((size_t)n + 1, sizeof(int64_t));
  double* sg = xmalloc(sizeof(double) * (size_t)(n + 1));
  double* thr = xmalloc(sizeof(double) * (size_t)(n + 1));
  int64_t total = 0;
  for (int64_t i = 0; i < n; ++i) {
    const double d = csr_at(A, i, i);
    double s;
    if (d == 0.0) {
      if (fail_zero) fail("strength: zero or missing diagonal at row %lld", (long long)i);
      s = 1.0;
    } else {
      s = d > 0.0 ? 1.0 : -1.0;
    }
    double m = 0.0;
    for (int64_t k = A->row_offsets[i]; k < A->row_offsets[i + 1]; ++k) {
      if (A->col_indices[k] == i) continue;
      const double v = -s * A->values[k];
      if (m < v) m = v;
    }
    sg[i] = s;
    thr[i] = alpha * m;
    if (m > 0.0)
      for (int64_t k = A->row_offsets[i]; k < A->row_offsets[i + 1]; ++k)
        if (A->col_indices[k] != i && -s * A->values[k] > thr[i]) cnt[i]++;
    total += cnt[i];
  }
  csr_alloc(Cm, n, n, total);
  for (int64_t i = 0; i < n; ++i) Cm->row_offsets[i + 1] = Cm->row_offsets[i] + cnt[i];
  for (int64_t i = 0; i < n; ++i) {
    int64_t p = Cm->row_offsets[i];
    if (cnt[i] == 0) continue;
    for (int64_t k = A->row_offsets[i]; k < A->row_offsets[i + 1]; ++k)
      if (A->col_indices[k] != i && -sg[i] * A->values[k] > thr[i]) {
        Cm->col_indices[p] = A->col_indices[k];
        Cm->values[p] = 1.0;
        ++p;
      }
  }
  free(cnt);
  free(sg);
  free(thr);
}

static void influence(const aggmg_csr* Cm, int64_t* counts) { /* strength.cpp:74-78 */
  memset(counts, 0, sizeof(int64_t) * (size_t)Cm->n_cols);
  for (int64_t k = 0; k < nnz_of(Cm); ++k) counts[Cm->col_indices[k]]++;
}

/* S = pattern(C u C^T), sorted merge per row (strength.cpp:80-111) */
static void symmetrize(const aggmg_csr* Cm, aggmg_csr* S) {
  if (Cm->n_rows != Cm->n_cols) fail("symmetrize: matrix must be square");
  aggmg_csr T;
  transpose(Cm, &T);
  const int64_t n = Cm->n_rows;
  int64_t* cnt = xcalloc((size_t)n + 1, sizeof(int64_t));
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1) {
      int64_t total = 0;
      for (int64_t i = 0; i < n; ++i) total += cnt[i];
      csr_alloc(S, n, n, total);
      for (int64_t i = 0; i < n; ++i) S->row_offsets[i + 1] = S->row_offsets[i] + cnt[i];
    }
    for (int64_t i = 0; i < n; ++i) {
      int64_t a = Cm->row_offsets[i], ae = Cm->row_offsets[i + 1];
      int64_t b = T.row_offsets[i], be = T.row_offsets[i + 1];
      int64_t c = 0;
      while (a < ae || b < be) {
        int64_t j;
        if (b >= be || (a < ae && Cm->col_indices[a] <= T.col_indices[b])) {
          j = Cm->col_indices[a];
          if (b < be && T.col_indices[b] == j) ++b;
          ++a;
        } else {
          j = T.col_indices[b++];
        }
        if (pass == 1) {
          S->col_indices[S->row_offsets[i] + c] = j;
          S->values[S->row_offsets[i] + c] = 1.0;
        }
        ++c;
      }
      cnt[i] = c;
    }
  }
  free(cnt);
  aggmg_oracle_csr_free(&T);
}

/* ---- MIS(2) (aggregation.cpp:19-86) ----------------------------------------------------- */

typedef struct {
  int8_t s;
  double v;
  int64_t i;
} Tup;
static int tup_less(const Tup* a, const Tup* b) {
  if (a->s != b->s) return a->s < b->s;
  if (a->v != b->v) return a->v < b->v;
  return a->i < b->i;
}
static void propagate(const aggmg_csr* S, const Tup* in, Tup* out) {
  for (int64_t i = 0; i < S->n_rows; ++i) {
    Tup best = in[i];
    for (int64_t k = S->row_offsets[i]; k < S->row_offsets[i + 1]; ++k)
      if (tup_less(&best, &in[S->col_indices[k]])) best = in[S->col_indices[k]];
    out[i] = best;
  }
}
static int mis2(const aggmg_csr* S, const int64_t* infl, uint64_t seed, int8_t* state) {
  if (S->n_rows != S->n_cols) fail("mis2: graph must be square");
  const int64_t n = S->n_rows;
  Tup* cur = xmalloc(sizeof(Tup) * (size_t)(n + 1));
  Tup* mid = xmalloc(sizeof(Tup) * (size_t)(n + 1));
  Tup* far = xmalloc(sizeof(Tup) * (size_t)(n + 1));
  for (int64_t i = 0; i < n; ++i) {
    state[i] = 0;
    cur[i].s = 0;
    cur[i].v = (double)infl[i] + u01(seed, (uint64_t)i);
    cur[i].i = i;
  }
  int sweeps = 0;
  int64_t undecided = n;
  while (undecided > 0) {
    if (sweeps > n) fail("mis2: failed to decide all nodes");
    propagate(S, cur, mid);
    propagate(S, mid, far);
    for (int64_t i = 0; i < n; ++i) {
      if (state[i] != 0) continue;
      if (far[i].i == i) {
        state[i] = 1;
        --undecided;
      } else if (far[i].s == 1) {
        state[i] = -1;
        --undecided;
      }
    }
    for (int64_t i = 0; i < n; ++i) cur[i].s = state[i];
    ++sweeps;
  }
  free(cur);
  free(mid);
  free(far);
  return sweeps;
}

/* ---- aggregation (aggregation.cpp:88-159) ------------------------------------------------- */

static int64_t aggregate(const aggmg_csr* S, const aggmg_csr* A, const int8_t* state,
                         int64_t* assignment, int64_t* reps_out) {
  if (!(S->n_rows == S->n_cols && A->n_rows == A->n_cols && S->n_rows == A->n_rows))
    fail("aggregate: graph and matrix shapes disagree");
  const int64_t n = S->n_rows;
  int64_t* reps = xmalloc(sizeof(int64_t) * (size_t)(n + 1));
  int64_t nr = 0;
  for (int64_t i = 0; i < n; ++i) {
    assignment[i] = -1;
    if (state[i] == 1) reps[nr++] = i;
  }
  for (int64_t a = 0; a < nr; ++a) assignment[reps[a]] = a;
  for (int64_t i = 0; i < n; ++i) { /* pass 1 */
    if (state[i] == 1) continue;
    for (int64_t k = S->row_offsets[i]; k < S->row_offsets[i + 1]; ++k)
      if (state[S->col_indices[k]] == 1) {
        assignment[i] = assignment[S->col_indices[k]];
        break;
      }
  }
  int64_t* pass2 = xmalloc(sizeof(int64_t) * (size_t)(n + 1));
  for (int64_t i = 0; i < n; ++i) { /* pass 2 against the pass-1 snapshot */
    pass2[i] = -1;
    if (assignment[i] != -1) continue;
    int64_t best = -1;
    double bw = -1.0;
    for (int64_t k = S->row_offsets[i]; k < S->row_offsets[i + 1]; ++k) {
      const int64_t j = S->col_indices[k], ja = assignment[j];
      if (ja == -1) continue;
      const double w1 = fabs(csr_at(A, i, j)), w2 = fabs(csr_at(A, j, i));
      const double w = w1 < w2 ? w2 : w1;
      if (w > bw || (w == bw && ja < best)) {
        bw = w;
        best = ja;
      }
    }
    pass2[i] = best;
  }
  for (int64_t i = 0; i < n; ++i)
    if (assignment[i] == -1 && pass2[i] != -1) assignment[i] = pass2[i];
  for (int64_t i = 0; i < n; ++i)
    if (assignment[i] == -1) {
      assignment[i] = nr;
      reps[nr++] = i;
    }
  /* renumber by representative node (reps are distinct node ids) */
  int64_t* rank_of_node = xmalloc(sizeof(int64_t) * (size_t)(n + 1));
  char* isrep = xcalloc((size_t)n + 1, 1);
  for (int64_t a = 0; a < nr; ++a) isrep[reps[a]] = 1;
  int64_t r = 0;
  for (int64_t i = 0; i < n; ++i)
    if (isrep[i]) {
      rank_of_node[i] = r;
      if (reps_out) reps_out[r] = i;
      ++r;
    }
  int64_t* rank = xmalloc(sizeof(int64_t) * (size_t)(nr + 1));
  for (int64_t a = 0; a < nr; ++a) rank[a] = rank_of_node[reps[a]];
  for (int64_t i = 0; i < n; ++i) assignment[i] = rank[assignment[i]];
  free(reps);
  free(pass2);
  free(rank_of_node);
  free(isrep);
  free(rank);
  return nr;
}

/* ---- transfer (transfer.cpp:15-49) -------------------------------------------------------- */

static void build_transfer(int64_t n, int64_t nc, const int64_t* a, const double* b,
                           aggmg_csr* P, aggmg_csr* R, double* cb) {
  double* sq = xcalloc((size_t)nc + 1, sizeof(double));
  for (int64_t i = 0; i < n; ++i) sq[a[i]] += b[i] * b[i];
  for (int64_t J = 0; J < nc; ++J) {
    if (!(sq[J] > 0.0))
      fail("transfer: near-null-space vector vanishes on aggregate %lld", (long long)J);
    cb[J] = sqrt(sq[J]);
  }
  int64_t nnz = 0;
  for (int64_t i = 0; i < n; ++i) nnz += b[i] != 0.0;
  csr_alloc(P, n, nc, nnz);
  int64_t p = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (b[i] != 0.0) {
      P->col_indices[p] = a[i];
      P->values[p] = b[i] / cb[a[i]];
      ++p;
    }
    P->row_offsets[i + 1] = p;
  }
  transpose(P, R);
  free(sq);
}

/* ---- Galerkin (galerkin.cpp:18-137) --------------------------------------------------------- */

typedef struct {
  int64_t n_fine, n_coarse, nnz;
  uint64_t hash;
  int64_t* assignment;
  aggmg_csr coarse; /* pattern only */
  int64_t *entry, *entry_row, *seg, *slot, *rbc, *aro;
  int64_t nseg;
} GCache;

static uint64_t mix_words(uint64_t h, const int64_t* v, int64_t n) {
  for (int64_t i = 0; i < n; ++i) h = hash_mix(h ^ (uint64_t)v[i]);
  return h;
}
static uint64_t fingerprint(const aggmg_csr* A, const int64_t* a) {
  uint64_t h = 0x9e3779b97f4a7c15ULL;
  h = mix_words(h, A->row_offsets, A->n_rows + 1);
  h = mix_words(h, A->col_indices, nnz_of(A));
  return mix_words(h, a, A->n_rows);
}

/* stable merge sort of idx[] by key[idx] */
static void msort(int64_t* idx, int64_t* tmp, int64_t n, const int64_t* key) {
  for (int64_t w = 1; w < n; w *= 2) {
    for (int64_t lo = 0; lo < n; lo += 2 * w) {
      const int64_t mid = lo + w < n ? lo + w : n, hi = lo + 2 * w < n ? lo + 2 * w : n;
      int64_t i = lo, j = mid, o = lo;
      while (i < mid && j < hi) tmp[o++] = (key[idx[j]] < key[idx[i]]) ? idx[j++] : idx[i++];
      while (i < mid) tmp[o++] = idx[i++];
      while (j < hi) tmp[o++] = idx[j++];
    }
    memcpy(idx, tmp, sizeof(int64_t) * (size_t)n);
  }
}

static GCache* build_cache(const aggmg_csr* A, int64_t nc, const int64_t* a) {
  if (A->n_rows != A->n_cols) fail("galerkin: matrix must be square");
  const int64_t n = A->n_rows, nnz = nnz_of(A);
  GCache* c = xcalloc(1, sizeof(GCache));
  c->n_fine = n;
  c->n_coarse = nc;
  c->nnz = nnz;
  c->assignment = xmalloc(sizeof(int64_t) * (size_t)(n + 1));
  memcpy(c->assignment, a, sizeof(int64_t) * (size_t)n);
  c->hash = fingerprint(A, a);
  int64_t* key = xmalloc(sizeof(int64_t) * (size_t)(nnz + 1));
  int64_t* row = xmalloc(sizeof(int64_t) * (size_t)(nnz + 1));
  c->entry = xmalloc(sizeof(int64_t) * (size_t)(nnz + 1));
  c->entry_row = xmalloc(sizeof(int64_t) * (size_t)(nnz + 1));
  for (int64_t i = 0; i < n; ++i)
    for (int64_t k = A->row_offsets[i]; k < A->row_offsets[i + 1]; ++k) {
      c->entry[k] = k;
      row[k] = i;
      key[k] = a[i] * nc + a[A->col_indices[k]];
    }
  int64_t* tmp = xmalloc(sizeof(int64_t) * (size_t)(nnz + 1));
  msort(c->entry, tmp, nnz, key);
  free(tmp);
  for (int64_t k = 0; k < nnz; ++k) c->entry_row[k] = row[c->entry[k]];
  int64_t nseg = 0;
  for (int64_t k = 0; k < nnz; ++k)
    if (k + 1 == nnz || key[c->entry[k + 1]] != key[c->entry[k]]) ++nseg;
  c->nseg = nseg;
  csr_alloc(&c->coarse, nc, nc, nseg);
  c->seg = xmalloc(sizeof(int64_t) * (size_t)(nseg + 1));
  c->seg[0] = 0;
  int64_t s = 0;
  for (int64_t k = 0; k < nnz; ++k)
    if (k + 1 == nnz || key[c->entry[k + 1]] != key[c->entry[k]]) {
      c->seg[s + 1] = k + 1;
      c->coarse.col_indices[s] = key[c->entry[k]] % nc;
      c->coarse.row_offsets[key[c->entry[k]] / nc + 1]++;
      ++s;
    }
  for (int64_t I = 0; I < nc; ++I) c->coarse.row_offsets[I + 1] += c->coarse.row_offsets[I];
  c->slot = xmalloc(sizeof(int64_t) * (size_t)(nnz + 1));
  for (int64_t q = 0; q < nseg; ++q)
    for (int64_t k = c->seg[q]; k < c->seg[q + 1]; ++k) c->slot[c->entry[k]] = q;
  c->aro = xcalloc((size_t)nc + 1, sizeof(int64_t));
  for (int64_t i = 0; i < n; ++i) c->aro[a[i] + 1]++;
  for (int64_t I = 0; I < nc; ++I) c->aro[I + 1] += c->aro[I];
  c->rbc = xmalloc(sizeof(int64_t) * (size_t)(n + 1));
  int64_t* cur = xmalloc(sizeof(int64_t) * (size_t)(nc + 1));
  memcpy(cur, c->aro, sizeof(int64_t) * (size_t)(nc + 1));
  for (int64_t i = 0; i < n; ++i) c->rbc[cur[a[i]]++] = i;
  free(cur);
  free(key);
  free(row);
  return c;
}

static void gcache_free(GCache* c) {
  if (!c) return;
  free(c->assignment);
  aggmg_oracle_csr_free(&c->coarse);
  free(c->entry);
  free(c->entry_row);
  free(c->seg);
  free(c->slot);
  free(c->rbc);
  free(c->aro);
  free(c);
}

static void apply_cache(const GCache* c, const aggmg_csr* A, const aggmg_csr* P, aggmg_csr* Ac) {
  if (P->n_rows != c->n_fine || P->n_cols != c->n_coarse)
    fail("galerkin cache: prolongator shape changed; rebuild the cache");
  if (A->n_rows != c->n_fine || nnz_of(A) != c->nnz || fingerprint(A, c->assignment) != c->hash)
    fail("galerkin cache: fine matrix pattern changed; rebuild the cache");
  double* pv = xcalloc((size_t)c->n_fine + 1, sizeof(double));
  for (int64_t i = 0; i < c->n_fine; ++i) {
    const int64_t w = P->row_offsets[i + 1] - P->row_offsets[i];
    if (w > 1) fail("galerkin cache: prolongator row %lld has more than one entry", (long long)i);
    if (w == 1) {
      if (P->col_indices[P->row_offsets[i]] != c->assignment[i])
        fail("galerkin cache: prolongator disagrees with the cached aggregation");
      pv[i] = P->values[P->row_offsets[i]];
    }
  }
  csr_copy(Ac, &c->coarse);
  for (int64_t q = 0; q < c->nseg; ++q) Ac->values[q] = 0.0;
  for (int64_t I = 0; I < c->n_coarse; ++I)
    for (int64_t t = c->aro[I]; t < c->aro[I + 1]; ++t) {
      const int64_t i = c->rbc[t];
      const double wi = pv[i];
      for (int64_t e = A->row_offsets[i]; e < A->row_offsets[i + 1]; ++e)
        Ac->values[c->slot[e]] += wi * A->values[e] * pv[A->col_indices[e]];
    }
  free(pv);
}

/* ---- dense: LU + Hessenberg eigenvalues (dense.cpp:24-212) ------------------------------------ */

typedef struct {
  int64_t n;
  double* lu;
  int64_t* perm;
} Lu;

static void lu_factor(Lu* f, double* a, int64_t n) {
  f->n = n;
  f->lu = a;
  f->perm = xmalloc(sizeof(int64_t) * (size_t)(n + 1));
  for (int64_t i = 0; i < n; ++i) f->perm[i] = i;
  for (int64_t k = 0; k < n; ++k) {
    int64_t piv = k;
    double best = fabs(a[k * n + k]);
    for (int64_t i = k + 1; i < n; ++i)
      if (fabs(a[i * n + k]) > best) {
        best = fabs(a[i * n + k]);
        piv = i;
      }
    if (best == 0.0) fail("lu_factor: zero pivot at index %lld", (long long)k);
    if (piv != k) {
      for (int64_t j = 0; j < n; ++j) {
        const double t = a[k * n + j];
        a[k * n + j] = a[piv * n + j];
        a[piv * n + j] = t;
      }
      const int64_t t = f->perm[k];
      f->perm[k] = f->perm[piv];
      f->perm[piv] = t;
    }
    const double inv = 1.0 / a[k * n + k];
    for (int64_t i = k + 1; i < n; ++i) {
      const double m = a[i * n + k] * inv;
      a[i * n + k] = m;
      for (int64_t j = k + 1; j < n; ++j) a[i * n + j] -= m * a[k * n + j];
    }
  }
}
static void lu_solve(const Lu* f, const double* b, double* x) {
  const int64_t n = f->n;
  for (int64_t i = 0; i < n; ++i) {
    double s = b[f->perm[i]];
    for (int64_t j = 0; j < i; ++j) s -= f->lu[i * n + j] * x[j];
    x[i] = s;
  }
  for (int64_t i = n - 1; i >= 0; --i) {
    double s = x[i];
    for (int64_t j = i + 1; j < n; ++j) s -= f->lu[i * n + j] * x[j];
    x[i] = s / f->lu[i * n + i];
  }
}

/* Eigenvalues of a small upper-Hessenberg matrix by the reference's Francis
 * double-shift QR (dense.cpp:81-212), restated operation for operation so the spectral
 * radius, and hence omega, is bit-identical: trailing deflation at 1e-14, 1x1 and 2x2
 * blocks resolved in closed form, Householder bulge chase, final Givens, exceptional
 * shift every 20 iterations.  a is row-major n x n and is destroyed; eigenvalues are
 * appended to (wr, wi) in deflation order. */
static void eig2(double a, double b, double c, double d, double* wr, double* wi, int* ne) {
  const double tr = a + d, det = a * d - b * c;
  const double disc = tr * tr / 4.0 - det;
  if (disc >= 0.0) {
    const double r = sqrt(disc);
    wr[*ne] = tr / 2.0 + r; wi[(*ne)++] = 0.0;
    wr[*ne] = tr / 2.0 - r; wi[(*ne)++] = 0.0;
  } else {
    const double r = sqrt(-disc);
    wr[*ne] = tr / 2.0; wi[(*ne)++] = r;
    wr[*ne] = tr / 2.0; wi[(*ne)++] = -r;
  }
}

static void hqr(double* a, int n, double* wr, double* wi) {
#define H(i, j) a[(i) * n + (j)]
  int ne = 0, hi = n - 1, stuck = 0, total = 0;
  const int budget = 30 * n + 100;
  while (hi >= 0) {
    if (!(total++ < budget)) fail("hessenberg_eigenvalues: QR iteration did not converge");
    int lo = hi;
    for (; lo > 0; --lo) {
      const double sc = fabs(H(lo - 1, lo - 1)) + fabs(H(lo, lo));
      if (fabs(H(lo, lo - 1)) <= 1e-14 * (sc > 0.0 ? sc : 1.0)) {
        H(lo, lo - 1) = 0.0;
        break;
      }
    }
    if (lo == hi) {
      wr[ne] = H(hi, hi);
      wi[ne++] = 0.0;
      hi -= 1;
      stuck = 0;
      continue;
    }
    if (lo == hi - 1) {
      eig2(H(lo, lo), H(lo, hi), H(hi, lo), H(hi, hi), wr, wi, &ne);
      hi -= 2;
      stuck = 0;
      continue;
    }
    double s = H(hi - 1, hi - 1) + H(hi, hi);
    double t = H(hi - 1, hi - 1) * H(hi, hi) - H(hi - 1, hi) * H(hi, hi - 1);
    if (++stuck % 20 == 0) {
      const double w = fabs(H(hi, hi - 1)) + fabs(H(hi - 1, hi - 2));
      s = 1.5 * w;
      t = w * w;
    }
    double x = H(lo, lo) * H(lo, lo) + H(lo, lo + 1) * H(lo + 1, lo) - s * H(lo, lo) + t;
    double y = H(lo + 1, lo) * (H(lo, lo) + H(lo + 1, lo + 1) - s);
    double z = H(lo + 2, lo + 1) * H(lo + 1, lo);
    for (int k = lo; k <= hi - 2; ++k) {
      double al = sqrt(x * x + y * y + z * z);
      if (al != 0.0) {
        if (x > 0.0) al = -al;
        const double v0 = x - al;
        const double bt = 2.0 / (v0 * v0 + y * y + z * z);
        for (int j = (k > lo ? k - 1 : lo); j <= hi; ++j) {
          double d = v0 * H(k, j) + y * H(k + 1, j) + z * H(k + 2, j);
          d *= bt;
          H(k, j) -= d * v0;
          H(k + 1, j) -= d * y;
          H(k + 2, j) -= d * z;
        }
        const int last = k + 3 < hi ? k + 3 : hi;
        for (int i = lo; i <= last; ++i) {
          double d = v0 * H(i, k) + y * H(i, k + 1) + z * H(i, k + 2);
          d *= bt;
          H(i, k) -= d * v0;
          H(i, k + 1) -= d * y;
          H(i, k + 2) -= d * z;
        }
      }
      x = H(k + 1, k);
      y = H(k + 2, k);
      z = (k + 3 <= hi) ? H(k + 3, k) : 0.0;
    }
    const int k = hi - 1;
    const double r = hypot(x, y);
    if (r > 0.0) {
      const double c = x / r, sn = y / r;
      for (int j = k - 1; j <= hi; ++j) {
        const double t1 = H(k, j), t2 = H(k + 1, j);
        H(k, j) = c * t1 + sn * t2;
        H(k + 1, j) = -sn * t1 + c * t2;
      }
      for (int i = lo; i <= hi; ++i) {
        const double t1 = H(i, k), t2 = H(i, k + 1);
        H(i, k) = c * t1 + sn * t2;
        H(i, k + 1) = -sn * t1 + c * t2;
      }
    }
  }
#undef H
}

/* ---- smoother (smoother.cpp:21-124) ------------------------------------------------------------- */

typedef struct {
  int kind;
  double* inv_diag;
  double omega, rho;
} Smoother;

static double estimate_rho(const aggmg_csr* A, const double* inv, int m, uint64_t seed) {
  const int64_t n = A->n_rows;
  if (m > n) m = (int)n;
  double** V = xcalloc((size_t)m + 1, sizeof(double*));
  V[0] = xmalloc(sizeof(double) * (size_t)(n + 1));
  for (int64_t i = 0; i < n; ++i) V[0][i] = usym(seed, (uint64_t)i);
  const double qn = vnorm(n, V[0]);
  if (!(qn > 0.0)) fail("smoother: degenerate start vector");
  vscale(n, 1.0 / qn, V[0]);
  double* Hm = xcalloc((size_t)(m + 1) * (size_t)m + 1, sizeof(double)); /* (m+1) x m row-major */
  int m_eff = m, nv = 1;
  double* w = xmalloc(sizeof(double) * (size_t)(n + 1));
  for (int j = 0; j < m; ++j) {
    spmv(A, V[j], w);
    for (int64_t i = 0; i < n; ++i) w[i] *= inv[i];
    double h_scale = 0.0;
    for (int i = 0; i <= j; ++i) {
      const double h = vdot(n, V[i], w) / vdot(n, V[i], V[i]);
      Hm[i * m + j] = h;
      vaxpy(n, -h, V[i], w);
      if (h_scale < fabs(h)) h_scale = fabs(h);
    }
    const double hj = vnorm(n, w);
    if (hj <= 1e-12 * (h_scale > 1.0 ? h_scale : 1.0)) {
      m_eff = j + 1;
      break;
    }
    Hm[(j + 1) * m + j] = hj;
    if (j + 1 < m) {
      V[nv] = vdup(n, w);
      vscale(n, 1.0 / hj, V[nv]);
      ++nv;
    }
  }
  double* sq = xmalloc(sizeof(double) * (size_t)(m_eff * m_eff + 1));
  for (int i = 0; i < m_eff; ++i)
    for (int j = 0; j < m_eff; ++j) sq[i * m_eff + j] = Hm[i * m + j];
  double wr[8], wi[8];
  hqr(sq, m_eff, wr, wi);
  double rho = 0.0;
  for (int i = 0; i < m_eff; ++i) {
    const double mag = hypot(wr[i], wi[i]);
    if (rho < mag) rho = mag;
  }
  if (!(rho > 0.0)) fail("smoother: spectral radius estimate collapsed to zero");
  for (int i = 0; i < nv; ++i) free(V[i]);
  free(V);
  free(Hm);
  free(w);
  free(sq);
  return rho;
}

static void setup_smoother(const aggmg_csr* A, int kind, int m, uint64_t seed, Smoother* s) {
  if (A->n_rows != A->n_cols) fail("smoother: matrix must be square");
  if (m < 1 || m > 5) fail("smoother: arnoldi_m must be in [1, 5]");
  s->kind = kind;
  s->inv_diag = xmalloc(sizeof(double) * (size_t)(A->n_rows + 1));
  for (int64_t i = 0; i < A->n_rows; ++i) {
    const double d = csr_at(A, i, i);
    if (d == 0.0) fail("smoother: zero diagonal at row %lld", (long long)i);
    s->inv_diag[i] = 1.0 / d;
  }
  s->omega = 1.0;
  s->rho = 1.0;
  if (kind == AGGMG_SMOOTHER_DAMPED_JACOBI) {
    s->rho = estimate_rho(A, s->inv_diag, m, seed);
    s->omega = (4.0 / 3.0) / s->rho;
  }
}

static void smooth(const Smoother* s, const aggmg_csr* A, const double* b, double* x) {
  const int64_t n = A->n_rows;
  if (s->kind == AGGMG_SMOOTHER_SGS) {
    for (int pass = 0; pass < 2; ++pass)
      for (int64_t t = 0; t < n; ++t) {
        const int64_t i = pass == 0 ? t : n - 1 - t;
        double sum = b[i];
        for (int64_t k = A->row_offsets[i]; k < A->row_offsets[i + 1]; ++k)
          if (A->col_indices[k] != i) sum -= A->values[k] * x[A->col_indices[k]];
        x[i] = sum * s->inv_diag[i];
      }
    return;
  }
  const double omega = s->kind == AGGMG_SMOOTHER_JACOBI ? 1.0 : s->omega;
  double* r = xmalloc(sizeof(double) * (size_t)(n + 1));
  spmv(A, x, r);
  for (int64_t i = 0; i < n; ++i) x[i] += omega * s->inv_diag[i] * (b[i] - r[i]);
  free(r);
}

/* ---- hierarchy (hierarchy.cpp:23-104) ------------------------------------------------------------ */

typedef struct {
  aggmg_csr A, P, R;
  double* B;
  Smoother sm;
  int has_sm;
  int64_t* assignment;
  int64_t n_agg;
  int sweeps;
  GCache* cache;
} OLevel;

typedef struct {
  OLevel* lv;
  int64_t nl;
  Lu lu;
  aggmg_setup_config cfg;
  char** warn;
  int64_t nwarn;
} OHier;

static const uint64_t kMisTag = 0x6d697332, kSmoothTag = 0x736d6f6f;

static void factor_coarsest(OHier* h) {
  const aggmg_csr* A = &h->lv[h->nl - 1].A;
  const int64_t nL = A->n_rows;
  const int64_t cap = h->cfg.coarse_size_max > 5000 ? h->cfg.coarse_size_max : 5000;
  if (nL > cap) fail("setup: coarsest level has %lld unknowns, too large for a dense solve", (long long)nL);
  double* d = xcalloc((size_t)(nL * nL) + 1, sizeof(double));
  for (int64_t i = 0; i < nL; ++i)
    for (int64_t k = A->row_offsets[i]; k < A->row_offsets[i + 1]; ++k)
      d[i * nL + A->col_indices[k]] = A->values[k];
  if (h->lu.lu) {
    free(h->lu.lu);
    free(h->lu.perm);
  }
  lu_factor(&h->lu, d, nL);
}

static OHier* setup_hierarchy(const aggmg_csr* A0, const double* B0, const aggmg_setup_config* c) {
  csr_validate(A0);
  if (A0->n_rows != A0->n_cols) fail("setup: matrix must be square");
  const int64_t n0 = A0->n_rows;
  if (!(vnorm(n0, B0) > 0.0)) fail("setup: near-null-space vector is zero");
  if (c->coarse_size_max < 1) fail("setup: coarse_size_max must be at least 1");
  if (c->max_levels < 1) fail("setup: max_levels must be at least 1");
  OHier* h = xcalloc(1, sizeof(OHier));
  h->cfg = *c;
  h->lv = xcalloc((size_t)c->max_levels + 1, sizeof(OLevel));
  csr_copy(&h->lv[0].A, A0);
  h->lv[0].B = vdup(n0, B0);
  h->nl = 1;
  while (h->lv[h->nl - 1].A.n_rows > c->coarse_size_max && h->nl < c->max_levels) {
    const int64_t k = h->nl - 1;
    OLevel* f = &h->lv[k];
    const int64_t n = f->A.n_rows;
    aggmg_csr Cm, S;
    strength(&f->A, c->alpha, 0, &Cm);
    int64_t* infl = xmalloc(sizeof(int64_t) * (size_t)(n + 1));
    influence(&Cm, infl);
    symmetrize(&Cm, &S);
    int8_t* state = xmalloc((size_t)n + 1);
    const int sweeps = mis2(&S, infl, level_seed(c->seed, k, kMisTag), state);
    int64_t* a = xmalloc(sizeof(int64_t) * (size_t)(n + 1));
    const int64_t nc = aggregate(&S, &f->A, state, a, NULL);
    aggmg_oracle_csr_free(&Cm);
    aggmg_oracle_csr_free(&S);
    free(infl);
    free(state);
    if ((double)nc >= 0.95 * (double)n) {
      char buf[256];
      snprintf(buf, sizeof buf,
               "coarsening stalled at level %lld (%lld -> %lld aggregates); solving this level directly",
               (long long)k, (long long)n, (long long)nc);
      h->warn = realloc(h->warn, sizeof(char*) * (size_t)(h->nwarn + 1));
      h->warn[h->nwarn++] = strdup(buf);
      free(a);
      break;
    }
    OLevel* nx = &h->lv[k + 1];
    nx->B = xmalloc(sizeof(double) * (size_t)(nc + 1));
    build_transfer(n, nc, a, f->B, &f->P, &f->R, nx->B);
    if (c->reuse_caches) {
      f->cache = build_cache(&f->A, nc, a);
      apply_cache(f->cache, &f->A, &f->P, &nx->A);
    } else {
      aggmg_csr RA;
      spmm(&f->R, &f->A, &RA);
      spmm(&RA, &f->P, &nx->A);
      aggmg_oracle_csr_free(&RA);
    }
    setup_smoother(&f->A, c->smoother, c->arnoldi_m, level_seed(c->seed, k, kSmoothTag), &f->sm);
    f->has_sm = 1;
    f->assignment = a;
    f->n_agg = nc;
    f->sweeps = sweeps;
    h->nl++;
  }
  factor_coarsest(h);
  return h;
}

static void hier_free(OHier* h) {
  if (!h) return;
  for (int64_t k = 0; k < h->nl; ++k) {
    OLevel* L = &h->lv[k];
    aggmg_oracle_csr_free(&L->A);
    if (L->P.row_offsets) aggmg_oracle_csr_free(&L->P);
    if (L->R.row_offsets) aggmg_oracle_csr_free(&L->R);
    free(L->B);
    free(L->sm.inv_diag);
    free(L->assignment);
    gcache_free(L->cache);
  }
  for (int64_t i = 0; i < h->nwarn; ++i) free(h->warn[i]);
  free(h->warn);
  free(h->lv);
  free(h->lu.lu);
  free(h->lu.perm);
  free(h);
}

/* ---- cycles (cycles.cpp:16-146) ---------------------------------------------------------------- */

static int accelerated(const aggmg_cycle_config* c, int64_t k) {
  if (c->kind == AGGMG_CYCLE_K) return 1;
  if (c->kind == AGGMG_CYCLE_HYBRID) return k < c->k_levels;
  return 0;
}
static void kcyc(const OHier* h, const aggmg_cycle_config* c, int64_t k, const double* b, double* x);
static void vcyc(const OHier* h, int64_t k, const double* b, double* x);
static void inner(const OHier* h, const aggmg_cycle_config* c, int64_t k, const double* b, double* x) {
  if (accelerated(c, k))
    kcyc(h, c, k, b, x);
  else
    vcyc(h, k, b, x);
}
static double* restrict_residual(const OLevel* L, const double* b, const double* x) {
  const int64_t n = L->A.n_rows;
  double* r = xmalloc(sizeof(double) * (size_t)(n + 1));
  spmv(&L->A, x, r);
  for (int64_t i = 0; i < n; ++i) r[i] = b[i] - r[i];
  double* rc = xmalloc(sizeof(double) * (size_t)(L->R.n_rows + 1));
  spmv(&L->R, r, rc);
  free(r);
  return rc;
}
static void prolong_add(const aggmg_csr* P, const double* xc, double* x) {
  for (int64_t i = 0; i < P->n_rows; ++i) {
    double s = 0.0;
    for (int64_t k = P->row_offsets[i]; k < P->row_offsets[i + 1]; ++k)
      s += P->values[k] * xc[P->col_indices[k]];
    x[i] += s;
  }
}
static void vcyc(const OHier* h, int64_t k, const double* b, double* x) {
  if (k == h->nl - 1) {
    lu_solve(&h->lu, b, x);
    return;
  }
  const OLevel* L = &h->lv[k];
  smooth(&L->sm, &L->A, b, x);
  double* rc = restrict_residual(L, b, x);
  const int64_t nc = L->R.n_rows;
  double* xc = xcalloc((size_t)nc + 1, sizeof(double));
  if (k + 1 == h->nl - 1)
    lu_solve(&h->lu, rc, xc);
  else
    vcyc(h, k + 1, rc, xc);
  prolong_add(&L->P, xc, x);
  smooth(&L->sm, &L->A, b, x);
  free(rc);
  free(xc);
}
static void kcyc(const OHier* h, const aggmg_cycle_config* c, int64_t k, const double* b, double* x) {
  if (k == h->nl - 1) {
    lu_solve(&h->lu, b, x);
    return;
  }
  const OLevel* L = &h->lv[k];
  smooth(&L->sm, &L->A, b, x);
  double* rc = restrict_residual(L, b, x);
  const int64_t nc = L->R.n_rows;
  double* xc = xcalloc((size_t)nc + 1, sizeof(double));
  if (k + 1 == h->nl - 1) {
    lu_solve(&h->lu, rc, xc);
  } else {
    const aggmg_csr* Ac = &h->lv[k + 1].A;
    double* cv = xcalloc((size_t)nc + 1, sizeof(double));
    inner(h, c, k + 1, rc, cv);
    double* v = xmalloc(sizeof(double) * (size_t)(nc + 1));
    spmv(Ac, cv, v);
    const int cg = c->inner == AGGMG_INNER_CG;
    const double rho1 = cg ? vdot(nc, cv, v) : vdot(nc, v, v);
    const double alpha1 = cg ? vdot(nc, cv, rc) : vdot(nc, v, rc);
    if (rho1 == 0.0) {
      fprintf(stderr, "kcycle: zero curvature at level %lld, keeping the unscaled correction\n",
              (long long)(k + 1));
      memcpy(xc, cv, sizeof(double) * (size_t)nc);
    } else {
      const double s1 = alpha1 / rho1;
      double* rt = vdup(nc, rc);
      vaxpy(nc, -s1, v, rt);
      if (vnorm(nc, rt) <= c->t * vnorm(nc, rc)) {
        memcpy(xc, cv, sizeof(double) * (size_t)nc);
        vscale(nc, s1, xc);
      } else {
        double* d = xcalloc((size_t)nc + 1, sizeof(double));
        inner(h, c, k + 1, rt, d);
        double* w = xmalloc(sizeof(double) * (size_t)(nc + 1));
        spmv(Ac, d, w);
        const double gamma = cg ? vdot(nc, d, v) : vdot(nc, w, v);
        const double beta = cg ? vdot(nc, d, w) : vdot(nc, w, w);
        const double alpha2 = cg ? vdot(nc, d, rt) : vdot(nc, w, rt);
        const double rho2 = beta - gamma * gamma / rho1;
        memcpy(xc, cv, sizeof(double) * (size_t)nc);
        if (rho2 == 0.0) {
          fprintf(stderr,
                  "kcycle: singular inner Gram matrix at level %lld, keeping the one-step correction\n",
                  (long long)(k + 1));
          vscale(nc, s1, xc);
        } else {
          vscale(nc, s1 - gamma * alpha2 / (rho1 * rho2), xc);
          vaxpy(nc, alpha2 / rho2, d, xc);
        }
        free(d);
        free(w);
      }
      free(rt);
    }
    free(cv);
    free(v);
  }
  prolong_add(&L->P, xc, x);
  smooth(&L->sm, &L->A, b, x);
  free(rc);
  free(xc);
}

static void precond(const OHier* h, const aggmg_cycle_config* c, const double* r, double* z) {
  memset(z, 0, sizeof(double) * (size_t)h->lv[0].A.n_rows);
  inner(h, c, 0, r, z);
}

/* ---- Krylov (krylov.cpp:36-201) ------------------------------------------------------------------- */

typedef struct {
  int converged, iterations;
  double* hist;
  int64_t nh, caph;
  char note[256];
  double seconds;
} Rep;

static void push(Rep* r, double v) {
  if (r->nh == r->caph) {
    r->caph = r->caph ? 2 * r->caph : 64;
    r->hist = realloc(r->hist, sizeof(double) * (size_t)r->caph);
  }
  r->hist[r->nh++] = v;
}
static void apply_m(const OHier* M, const aggmg_cycle_config* c, const double* r, double* z,
                    int64_t n) {
  if (M)
    precond(M, c, r, z);
  else
    memcpy(z, r, sizeof(double) * (size_t)n);
}
static double now_s(void) {
  struct timespec ts;
  clock_gettime(CLOCK_MONOTONIC, &ts);
  return (double)ts.tv_sec + 1e-9 * (double)ts.tv_nsec;
}
static void true_res(const aggmg_csr* A, const double* b, const double* x, double* r) {
  spmv(A, x, r);
  for (int64_t i = 0; i < A->n_rows; ++i) r[i] = b[i] - r[i];
}

static void pcg_solve(const aggmg_csr* A, const double* b, double* x, const OHier* M,
                      const aggmg_cycle_config* cc, const aggmg_solver_config* cfg, Rep* rep) {
  if (A->n_rows != A->n_cols) fail("pcg: matrix must be square");
  if (!(cfg->tol > 0.0)) fail("pcg: tol must be positive");
  const double t0 = now_s();
  const int64_t n = A->n_rows;
  const double nb = vnorm(n, b);
  if (nb == 0.0) {
    memset(x, 0, sizeof(double) * (size_t)n);
    rep->converged = 1;
    push(rep, 0.0);
    return;
  }
  const double target = cfg->tol * nb;
  double* r = xmalloc(sizeof(double) * (size_t)(n + 1));
  double* z = xmalloc(sizeof(double) * (size_t)(n + 1));
  double* Ap = xmalloc(sizeof(double) * (size_t)(n + 1));
  double* rold = xmalloc(sizeof(double) * (size_t)(n + 1));
  true_res(A, b, x, r);
  double res = vnorm(n, r);
  push(rep, res);
  apply_m(M, cc, r, z, n);
  double* p = vdup(n, z);
  double rz = vdot(n, r, z);
  while (res > target && rep->iterations < cfg->max_iters) {
    spmv(A, p, Ap);
    const double pAp = vdot(n, p, Ap);
    if (!(pAp > 0.0)) fail("pcg: non-positive curvature (matrix not positive definite); use fgmres");
    const double alpha = rz / pAp;
    vaxpy(n, alpha, p, x);
    memcpy(rold, r, sizeof(double) * (size_t)n);
    vaxpy(n, -alpha, Ap, r);
    rep->iterations++;
    res = vnorm(n, r);
    push(rep, res);
    if (res <= target) break;
    apply_m(M, cc, r, z, n);
    const double rz_new = vdot(n, r, z);
    const double beta = (rz_new - vdot(n, rold, z)) / rz;
    for (int64_t i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
    rz = rz_new;
  }
  rep->converged = res <= target;
  rep->seconds = now_s() - t0;
  free(r);
  free(z);
  free(Ap);
  free(rold);
  free(p);
}

static void fgmres_solve(const aggmg_csr* A, const double* b, double* x, const OHier* M,
                         const aggmg_cycle_config* cc, const aggmg_solver_config* cfg, Rep* rep) {
  if (A->n_rows != A->n_cols) fail("fgmres: matrix must be square");
  if (!(cfg->tol > 0.0)) fail("fgmres: tol must be positive");
  if (cfg->restart < 1) fail("fgmres: restart must be at least 1");
  const double t0 = now_s();
  const int64_t n = A->n_rows;
  const int m = cfg->restart;
  const double nb = vnorm(n, b);
  if (nb == 0.0) {
    memset(x, 0, sizeof(double) * (size_t)n);
    rep->converged = 1;
    push(rep, 0.0);
    return;
  }
  const double target = cfg->tol * nb;
  double* r = xmalloc(sizeof(double) * (size_t)(n + 1));
  true_res(A, b, x, r);
  double beta = vnorm(n, r);
  push(rep, beta);
  double** V = xcalloc((size_t)m + 2, sizeof(double*));
  double** Z = xcalloc((size_t)m + 1, sizeof(double*));
  for (int i = 0; i <= m; ++i) V[i] = xmalloc(sizeof(double) * (size_t)(n + 1));
  for (int i = 0; i < m; ++i) Z[i] = xmalloc(sizeof(double) * (size_t)(n + 1));
  double* Hc = xmalloc(sizeof(double) * (size_t)((m + 1) * m)); /* column-major, ld m+1 */
#define HH(i, j) Hc[(j) * (m + 1) + (i)]
  double* cs = xmalloc(sizeof(double) * (size_t)m);
  double* sn = xmalloc(sizeof(double) * (size_t)m);
  double* g = xmalloc(sizeof(double) * (size_t)(m + 1));
  double* y = xmalloc(sizeof(double) * (size_t)(m + 1));
  double* w = xmalloc(sizeof(double) * (size_t)(n + 1));
  double prev = beta;
  while (beta > target && rep->iterations < cfg->max_iters) {
    memcpy(V[0], r, sizeof(double) * (size_t)n);
    vscale(n, 1.0 / beta, V[0]);
    for (int i = 0; i <= m; ++i) g[i] = 0.0;
    g[0] = beta;
    for (int i = 0; i < (m + 1) * m; ++i) Hc[i] = 0.0;
    int j = 0;
    for (; j < m && rep->iterations < cfg->max_iters; ++j) {
      apply_m(M, cc, V[j], Z[j], n);
      spmv(A, Z[j], w);
      for (int i = 0; i <= j; ++i) {
        HH(i, j) = vdot(n, V[i], w);
        vaxpy(n, -HH(i, j), V[i], w);
      }
      HH(j + 1, j) = vnorm(n, w);
      const int breakdown = HH(j + 1, j) == 0.0;
      if (!breakdown) {
        memcpy(V[j + 1], w, sizeof(double) * (size_t)n);
        vscale(n, 1.0 / HH(j + 1, j), V[j + 1]);
      }
      for (int i = 0; i < j; ++i) {
        const double t = cs[i] * HH(i, j) + sn[i] * HH(i + 1, j);
        HH(i + 1, j) = -sn[i] * HH(i, j) + cs[i] * HH(i + 1, j);
        HH(i, j) = t;
      }
      const double den = hypot(HH(j, j), HH(j + 1, j));
      if (den == 0.0) {
        cs[j] = 1.0;
        sn[j] = 0.0;
      } else {
        cs[j] = HH(j, j) / den;
        sn[j] = HH(j + 1, j) / den;
      }
      HH(j, j) = cs[j] * HH(j, j) + sn[j] * HH(j + 1, j);
      HH(j + 1, j) = 0.0;
      g[j + 1] = -sn[j] * g[j];
      g[j] = cs[j] * g[j];
      rep->iterations++;
      push(rep, fabs(g[j + 1]));
      if (fabs(g[j + 1]) <= target || breakdown) {
        ++j;
        break;
      }
    }
    for (int i = j - 1; i >= 0; --i) {
      double s = g[i];
      for (int l = i + 1; l < j; ++l) s -= HH(i, l) * y[l];
      y[i] = s / HH(i, i);
    }
    for (int i = 0; i < j; ++i) vaxpy(n, y[i], Z[i], x);
    true_res(A, b, x, r);
    beta = vnorm(n, r);
    rep->hist[rep->nh - 1] = beta;
    if (beta > target && beta >= prev && j == m)
      snprintf(rep->note, sizeof rep->note, "stagnation: no residual decrease over a full restart cycle");
    prev = beta;
  }
#undef HH
  rep->converged = beta <= target;
  rep->seconds = now_s() - t0;
  for (int i = 0; i <= m; ++i) free(V[i]);
  for (int i = 0; i < m; ++i) free(Z[i]);
  free(V);
  free(Z);
  free(Hc);
  free(cs);
  free(sn);
  free(g);
  free(y);
  free(w);
  free(r);
}

static void fill_rep(const Rep* r, aggmg_solve_report* out) {
  if (!out) return;
  out->converged = r->converged;
  out->iterations = r->iterations;
  out->history_length = r->nh;
  if (out->history)
    for (int64_t i = 0; i < r->nh && i < out->history_capacity; ++i) out->history[i] = r->hist[i];
  out->solve_seconds = r->seconds;
  snprintf(out->note, sizeof out->note, "%s", r->note);
}

/* ---- C-ABI ------------------------------------------------------------------------------------------ */

int aggmg_oracle_generate_poisson(int dims, int64_t nx, int64_t ny, int64_t nz, double eps,
                                  int weak, aggmg_csr* A) {
  API_BEGIN
  gen_poisson(dims, nx, ny, nz, eps, weak, A);
  API_END
}
int aggmg_oracle_generate_jump27(int64_t nx, int64_t ny, int64_t nz, double jump, int64_t block,
                                 aggmg_csr* A) {
  API_BEGIN
  gen_jump27(nx, ny, nz, jump, block, A);
  API_END
}
int aggmg_oracle_spmv(const aggmg_csr* A, const double* x, double* y) {
  API_BEGIN
  spmv(A, x, y);
  API_END
}
int aggmg_oracle_transpose(const aggmg_csr* A, aggmg_csr* T) {
  API_BEGIN
  transpose(A, T);
  API_END
}
int aggmg_oracle_dot(int64_t n, const double* a, const double* b, double* out) {
  API_BEGIN
  *out = vdot(n, a, b);
  API_END
}
int aggmg_oracle_norm2(int64_t n, const double* a, double* out) {
  API_BEGIN
  *out = vnorm(n, a);
  API_END
}
int aggmg_oracle_axpy(int64_t n, double a, const double* x, double* y) {
  API_BEGIN
  vaxpy(n, a, x, y);
  API_END
}
int aggmg_oracle_scale(int64_t n, double a, double* x) {
  API_BEGIN
  vscale(n, a, x);
  API_END
}
int aggmg_oracle_classic_strength(const aggmg_csr* A, double alpha, int policy, aggmg_csr* Cm) {
  API_BEGIN
  strength(A, alpha, policy, Cm);
  API_END
}
int aggmg_oracle_influence_counts(const aggmg_csr* Cm, int64_t* counts) {
  API_BEGIN
  influence(Cm, counts);
  API_END
}
int aggmg_oracle_symmetrize_pattern(const aggmg_csr* Cm, aggmg_csr* S) {
  API_BEGIN
  symmetrize(Cm, S);
  API_END
}
int aggmg_oracle_mis2(const aggmg_csr* S, const int64_t* infl, uint64_t seed, int8_t* state,
                      int64_t* n_roots, int32_t* sweeps) {
  API_BEGIN
  const int sw = mis2(S, infl, seed, state);
  int64_t nr = 0;
  for (int64_t i = 0; i < S->n_rows; ++i) nr += state[i] == 1;
  if (n_roots) *n_roots = nr;
  if (sweeps) *sweeps = sw;
  API_END
}
int aggmg_oracle_aggregate(const aggmg_csr* S, const aggmg_csr* A, const int8_t* state,
                           int64_t* assignment, int64_t* reps, int64_t* n_agg) {
  API_BEGIN
  *n_agg = aggregate(S, A, state, assignment, reps);
  API_END
}
int aggmg_oracle_build_transfer(int64_t n, int64_t nc, const int64_t* a, const double* b,
                                aggmg_csr* P, aggmg_csr* R, double* cb) {
  API_BEGIN
  aggmg_csr Pl, Rl;
  double* cbl = xmalloc(sizeof(double) * (size_t)(nc + 1));
  build_transfer(n, nc, a, b, &Pl, &Rl, cbl);
  if (P) *P = Pl; else aggmg_oracle_csr_free(&Pl);
  if (R) *R = Rl; else aggmg_oracle_csr_free(&Rl);
  if (cb) memcpy(cb, cbl, sizeof(double) * (size_t)nc);
  free(cbl);
  API_END
}
int aggmg_oracle_galerkin_direct(const aggmg_csr* R, const aggmg_csr* A, const aggmg_csr* P,
                                 aggmg_csr* Ac) {
  API_BEGIN
  aggmg_csr RA;
  spmm(R, A, &RA);
  spmm(&RA, P, Ac);
  aggmg_oracle_csr_free(&RA);
  API_END
}
int aggmg_oracle_build_galerkin_cache(const aggmg_csr* A, int64_t nc, const int64_t* a, void** out) {
  API_BEGIN
  *out = build_cache(A, nc, a);
  API_END
}
int aggmg_oracle_galerkin_cache_info(const void* cp, int64_t* nf, int64_t* nc, int64_t* nnzf,
                                     int64_t* nnzc) {
  const GCache* c = cp;
  if (nf) *nf = c->n_fine;
  if (nc) *nc = c->n_coarse;
  if (nnzf) *nnzf = c->nnz;
  if (nnzc) *nnzc = c->nseg;
  return AGGMG_OK;
}
static void cp64(int64_t* dst, const int64_t* src, int64_t n) {
  if (dst && n > 0) memcpy(dst, src, sizeof(int64_t) * (size_t)n);
}
int aggmg_oracle_galerkin_cache_export(const void* cp, int64_t* cro, int64_t* cci, int64_t* entry,
                                       int64_t* entry_row, int64_t* seg, int64_t* slot,
                                       int64_t* rbc, int64_t* aro) {
  const GCache* c = cp;
  cp64(cro, c->coarse.row_offsets, c->n_coarse + 1);
  cp64(cci, c->coarse.col_indices, c->nseg);
  cp64(entry, c->entry, c->nnz);
  cp64(entry_row, c->entry_row, c->nnz);
  cp64(seg, c->seg, c->nseg + 1);
  cp64(slot, c->slot, c->nnz);
  cp64(rbc, c->rbc, c->n_fine);
  cp64(aro, c->aro, c->n_coarse + 1);
  return AGGMG_OK;
}
int aggmg_oracle_apply_galerkin_cache(const void* c, const aggmg_csr* A, const aggmg_csr* P,
                                      aggmg_csr* Ac) {
  API_BEGIN
  apply_cache(c, A, P, Ac);
  API_END
}
void aggmg_oracle_galerkin_cache_free(void* c) { gcache_free(c); }

int aggmg_oracle_setup_smoother(const aggmg_csr* A, int kind, int m, uint64_t seed, double* inv,
                                double* omega, double* rho) {
  API_BEGIN
  Smoother s = {0};
  setup_smoother(A, kind, m, seed, &s);
  if (inv) memcpy(inv, s.inv_diag, sizeof(double) * (size_t)A->n_rows);
  if (omega) *omega = s.omega;
  if (rho) *rho = s.rho;
  free(s.inv_diag);
  API_END
}
int aggmg_oracle_smooth(int kind, const double* inv, double omega, const aggmg_csr* A,
                        const double* b, double* x) {
  API_BEGIN
  Smoother s = {kind, (double*)inv, omega, 1.0};
  smooth(&s, A, b, x);
  API_END
}
int aggmg_oracle_hessenberg_eigenvalues(int64_t n, const double* Hin, double* re, double* im) {
  API_BEGIN
  double* a = vdup(n * n, Hin);
  hqr(a, (int)n, re, im);
  free(a);
  API_END
}

int aggmg_oracle_setup_hierarchy(const aggmg_csr* A0, const double* B0,
                                 const aggmg_setup_config* cfg, void** out) {
  API_BEGIN
  aggmg_setup_config c;
  if (cfg) {
    c = *cfg;
  } else {
    c.alpha = 0.25;
    c.coarse_size_max = 600;
    c.max_levels = 25;
    c.smoother = AGGMG_SMOOTHER_DAMPED_JACOBI;
    c.arnoldi_m = 5;
    c.reuse_caches = 0;
    c.seed = 42;
  }
  double* ones = NULL;
  if (!B0) {
    ones = xmalloc(sizeof(double) * (size_t)(A0->n_rows + 1));
    for (int64_t i = 0; i < A0->n_rows; ++i) ones[i] = 1.0;
    B0 = ones;
  }
  *out = setup_hierarchy(A0, B0, &c);
  free(ones);
  API_END
}
int aggmg_oracle_refresh_values(void* hp, const double* values, int64_t count) {
  API_BEGIN
  OHier* h = hp;
  if (!h->cfg.reuse_caches) fail("refresh: hierarchy was built without caches");
  if (count != nnz_of(&h->lv[0].A)) fail("refresh: value count does not match the level-0 pattern");
  memcpy(h->lv[0].A.values, values, sizeof(double) * (size_t)count);
  for (int64_t k = 0; k + 1 < h->nl; ++k) {
    OLevel* f = &h->lv[k];
    aggmg_oracle_csr_free(&h->lv[k + 1].A);
    apply_cache(f->cache, &f->A, &f->P, &h->lv[k + 1].A);
    free(f->sm.inv_diag);
    setup_smoother(&f->A, h->cfg.smoother, h->cfg.arnoldi_m, level_seed(h->cfg.seed, k, kSmoothTag),
                   &f->sm);
  }
  factor_coarsest(h);
  API_END
}
void aggmg_oracle_hierarchy_free(void* h) { hier_free(h); }
int64_t aggmg_oracle_hierarchy_n_levels(const void* h) { return ((const OHier*)h)->nl; }
int aggmg_oracle_hierarchy_level_size(const void* hp, int64_t k, int64_t* n, int64_t* nnz) {
  const OHier* h = hp;
  if (n) *n = h->lv[k].A.n_rows;
  if (nnz) *nnz = nnz_of(&h->lv[k].A);
  return AGGMG_OK;
}
int aggmg_oracle_hierarchy_level_A(const void* hp, int64_t k, aggmg_csr* A) {
  API_BEGIN
  csr_copy(A, &((const OHier*)hp)->lv[k].A);
  API_END
}
int aggmg_oracle_hierarchy_level_P(const void* hp, int64_t k, aggmg_csr* P) {
  API_BEGIN
  const OLevel* L = &((const OHier*)hp)->lv[k];
  if (L->P.row_offsets)
    csr_copy(P, &L->P);
  else
    csr_empty(P);
  API_END
}
int aggmg_oracle_hierarchy_level_R(const void* hp, int64_t k, aggmg_csr* R) {
  API_BEGIN
  const OLevel* L = &((const OHier*)hp)->lv[k];
  if (L->R.row_offsets)
    csr_copy(R, &L->R);
  else
    csr_empty(R);
  API_END
}
int aggmg_oracle_hierarchy_level_B(const void* hp, int64_t k, double* B) {
  const OLevel* L = &((const OHier*)hp)->lv[k];
  memcpy(B, L->B, sizeof(double) * (size_t)L->A.n_rows);
  return AGGMG_OK;
}
int aggmg_oracle_hierarchy_level_aggregation(const void* hp, int64_t k, int64_t* a, int64_t* nc,
                                             int32_t* sweeps) {
  API_BEGIN
  const OLevel* L = &((const OHier*)hp)->lv[k];
  if (!L->assignment) fail("hierarchy: the coarsest level has no aggregation");
  cp64(a, L->assignment, L->A.n_rows);
  if (nc) *nc = L->n_agg;
  if (sweeps) *sweeps = L->sweeps;
  API_END
}
int aggmg_oracle_hierarchy_level_smoother(const void* hp, int64_t k, double* omega, double* rho,
                                          double* inv) {
  const OLevel* L = &((const OHier*)hp)->lv[k];
  if (omega) *omega = L->has_sm ? L->sm.omega : 1.0;
  if (rho) *rho = L->has_sm ? L->sm.rho : 1.0;
  if (inv && L->has_sm) memcpy(inv, L->sm.inv_diag, sizeof(double) * (size_t)L->A.n_rows);
  return AGGMG_OK;
}
int64_t aggmg_oracle_hierarchy_n_warnings(const void* hp) { return ((const OHier*)hp)->nwarn; }
const char* aggmg_oracle_hierarchy_warning(const void* hp, int64_t i) {
  return ((const OHier*)hp)->warn[i];
}
int aggmg_oracle_vcycle(const void* hp, int64_t k, const double* b, double* x) {
  API_BEGIN
  vcyc(hp, k, b, x);
  API_END
}
int aggmg_oracle_kcycle(const void* hp, const aggmg_cycle_config* c, int64_t k, const double* b,
                        double* x) {
  API_BEGIN
  kcyc(hp, c, k, b, x);
  API_END
}
int aggmg_oracle_apply_preconditioner(const void* hp, const aggmg_cycle_config* c, const double* r,
                                      double* z) {
  API_BEGIN
  precond(hp, c, r, z);
  API_END
}

static int krylov(const aggmg_csr* A, const double* b, const double* x0, const void* M,
                  const aggmg_cycle_config* cc, const aggmg_solver_config* cfg, double* x,
                  aggmg_solve_report* out, int use_pcg) {
  Rep rep;
  memset(&rep, 0, sizeof rep);
  API_BEGIN
  memcpy(x, x0, sizeof(double) * (size_t)A->n_rows);
  if (use_pcg)
    pcg_solve(A, b, x, M, cc, cfg, &rep);
  else
    fgmres_solve(A, b, x, M, cc, cfg, &rep);
  fill_rep(&rep, out);
  free(rep.hist);
  API_END
}
int aggmg_oracle_pcg(const aggmg_csr* A, const double* b, const double* x0, const void* M,
                     const aggmg_cycle_config* cc, const aggmg_solver_config* cfg, double* x,
                     aggmg_solve_report* rep) {
  return krylov(A, b, x0, M, cc, cfg, x, rep, 1);
}
int aggmg_oracle_fgmres(const aggmg_csr* A, const double* b, const double* x0, const void* M,
                        const aggmg_cycle_config* cc, const aggmg_solver_config* cfg, double* x,
                        aggmg_solve_report* rep) {
  return krylov(A, b, x0, M, cc, cfg, x, rep, 0);
}
int aggmg_oracle_setup_and_solve(const aggmg_csr* A, const double* b, const double* B0,
                                 const double* x0, const aggmg_setup_config* setup,
                                 const aggmg_cycle_config* cycle,
                                 const aggmg_solver_config* solver, double* x,
                                 aggmg_solve_report* rep) {
  const double t0 = now_s();
  void* h = NULL;
  int rc = aggmg_oracle_setup_hierarchy(A, B0, setup, &h);
  if (rc) return rc;
  const double ts = now_s() - t0;
  double* z0 = NULL;
  if (!x0) {
    z0 = calloc((size_t)A->n_rows + 1, sizeof(double));
    x0 = z0;
  }
  rc = krylov(A, b, x0, h, cycle, solver, x, rep, solver->method == AGGMG_SOLVER_PCG);
  free(z0);
  hier_free(h);
  if (rep) rep->setup_seconds = ts;
  return rc;
}
