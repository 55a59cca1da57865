/*
 * sl_oracle.c — CPU restatement of the reference's hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library, and
 * only as the checker or the CPU baseline — never as the product path.
 *
 * Each function restates, in plain C, what the reference interpreter computes
 * for one BASELINE pattern (reference = /root/reference/pkg/src/sparselevels,
 * a pure-Python package; there is no compiled reference to build):
 *   - evaluation order and association      engine.py:520-534
 *   - scatter output: zero-fill, then +=     engine.py:303, :320
 *   - gather-append output: extend 0.0, +=   engine.py:387-413
 *   - level functions                        levels.py:215-333
 *   - loop orders per pattern                lattice.py:346-552
 * The restatement is pinned against golden vectors produced by running the
 * reference itself (tests/golden/make_golden.py).
 *
 * Every reduction also returns sum|term| per output component, the scale of
 * the condition-scaled tolerance |gpu - ref| <= 1e-12 * max(|ref|, sum|terms|).
 *
 * The *_mt variants partition OUTPUT ROWS (slices) across OpenMP threads, so
 * each component is still accumulated by one thread in the reference order:
 * they are bit-identical to the single-threaded functions.  They exist only
 * as the multi-core CPU baseline.
 *
 * Build: make -C oracle   (gcc -O2 -ffp-contract=off -fopenmp)
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define EMPTY (-1)

static int clamp_threads(int t) {
#ifdef _OPENMP
  if (t <= 0) t = omp_get_max_threads();
  return t;
#else
  (void)t;
  return 1;
#endif
}

/* ------------------------------------------------------------------------
 * SpMV, COO-SoA: run_fused over the i(+)j chain, one scatter per stored entry
 * (engine.py:636-713 with _needs_grouping False for scatter, :726-728),
 * _ScatterWriter: vals zero-filled (:303), vals[pos] += a*x (:320). */
void or_spmv_coo(int64_t nrows, int64_t nnz, const int32_t* rows, const int32_t* cols,
                 const double* vals, const double* x, double* y, double* absy) {
  for (int64_t r = 0; r < nrows; ++r) { y[r] = 0.0; if (absy) absy[r] = 0.0; }
  for (int64_t e = 0; e < nnz; ++e) {
    const double t = vals[e] * x[cols[e]];
    y[rows[e]] = y[rows[e]] + t;
    if (absy) absy[rows[e]] += fabs(t);
  }
}

/* Row-sorted COO split at row boundaries: each thread owns whole rows. */
void or_spmv_coo_mt(int64_t nrows, int64_t nnz, const int32_t* rows, const int32_t* cols,
                    const double* vals, const double* x, double* y, int nthreads) {
  nthreads = clamp_threads(nthreads);
#pragma omp parallel for num_threads(nthreads) schedule(static)
  for (int64_t r = 0; r < nrows; ++r) y[r] = 0.0;
#pragma omp parallel num_threads(nthreads)
  {
#ifdef _OPENMP
    const int t = omp_get_thread_num(), T = omp_get_num_threads();
#else
    const int t = 0, T = 1;
#endif
    int64_t b = nnz * t / T, e = nnz * (t + 1) / T;
    while (b > 0 && b < nnz && rows[b] == rows[b - 1]) ++b;   /* snap to row start */
    while (e > 0 && e < nnz && rows[e] == rows[e - 1]) ++e;
    for (int64_t q = b; q < e; ++q) y[rows[q]] = y[rows[q]] + vals[q] * x[cols[q]];
  }
}

/* ------------------------------------------------------------------------
 * SpMV, CSR: run_node(i) over dense A0, run_node(j) over A1 with x located;
 * total = ((0.0 + t1) + t2) + ... (engine.py:591-634). */
void or_spmv_csr(int64_t nrows, const int32_t* pos, const int32_t* crd, const double* vals,
                 const double* x, double* y, double* absy) {
  for (int64_t r = 0; r < nrows; ++r) {
    double acc = 0.0, a = 0.0;
    for (int64_t p = pos[r]; p < pos[r + 1]; ++p) {
      const double t = vals[p] * x[crd[p]];
      acc = acc + t;
      a += fabs(t);
    }
    y[r] = acc;
    if (absy) absy[r] = a;
  }
}

void or_spmv_csr_mt(int64_t nrows, const int32_t* pos, const int32_t* crd, const double* vals,
                    const double* x, double* y, int nthreads) {
  nthreads = clamp_threads(nthreads);
#pragma omp parallel for num_threads(nthreads) schedule(static, 1024)
  for (int64_t r = 0; r < nrows; ++r) {
    double acc = 0.0;
    for (int64_t p = pos[r]; p < pos[r + 1]; ++p) acc = acc + vals[p] * x[crd[p]];
    y[r] = acc;
  }
}

/* ------------------------------------------------------------------------
 * SpMV, ELL: order (slot, i, j); for each slot s, each row i: y[i] += a*x at
 * position s*N + i (levels.py:230), padding (col 0, 0.0) included. */
void or_spmv_ell(int64_t nrows, int32_t nslots, const int32_t* crd, const double* vals,
                 const double* x, double* y, double* absy) {
  for (int64_t r = 0; r < nrows; ++r) { y[r] = 0.0; if (absy) absy[r] = 0.0; }
  for (int32_t s = 0; s < nslots; ++s)
    for (int64_t i = 0; i < nrows; ++i) {
      const int64_t p = (int64_t)s * nrows + i;
      const double t = vals[p] * x[crd[p]];
      y[i] = y[i] + t;
      if (absy) absy[i] += fabs(t);
    }
}

void or_spmv_ell_mt(int64_t nrows, int32_t nslots, const int32_t* crd, const double* vals,
                    const double* x, double* y, int nthreads) {
  nthreads = clamp_threads(nthreads);
#pragma omp parallel for num_threads(nthreads) schedule(static, 1024)
  for (int64_t i = 0; i < nrows; ++i) {
    double acc = 0.0;
    for (int32_t s = 0; s < nslots; ++s) {
      const int64_t p = (int64_t)s * nrows + i;
      acc = acc + vals[p] * x[crd[p]];
    }
    y[i] = acc;
  }
}

/* ------------------------------------------------------------------------
 * SpMV, DIA: order (diag, i, j); i ranges over the range level's bounds
 * [max(0,-off), min(N, M-off)) (levels.py:220-222); column i + off
 * (levels.py:256). */
void or_spmv_dia(int64_t nrows, int64_t ncols, int32_t ndiag, const int32_t* offs,
                 const double* vals, const double* x, double* y, double* absy) {
  for (int64_t r = 0; r < nrows; ++r) { y[r] = 0.0; if (absy) absy[r] = 0.0; }
  for (int32_t d = 0; d < ndiag; ++d) {
    const int64_t off = offs[d];
    const int64_t lo = off < 0 ? -off : 0;
    const int64_t hi = nrows < ncols - off ? nrows : ncols - off;
    for (int64_t i = lo; i < hi; ++i) {
      const double t = vals[(int64_t)d * nrows + i] * x[i + off];
      y[i] = y[i] + t;
      if (absy) absy[i] += fabs(t);
    }
  }
}

void or_spmv_dia_mt(int64_t nrows, int64_t ncols, int32_t ndiag, const int32_t* offs,
                    const double* vals, const double* x, double* y, int nthreads) {
  nthreads = clamp_threads(nthreads);
#pragma omp parallel for num_threads(nthreads) schedule(static, 4096)
  for (int64_t i = 0; i < nrows; ++i) {
    double acc = 0.0;
    for (int32_t d = 0; d < ndiag; ++d) {
      const int64_t j = i + offs[d];
      if (j >= 0 && j < ncols) acc = acc + vals[(int64_t)d * nrows + i] * x[j];
    }
    y[i] = acc;
  }
}

/* ------------------------------------------------------------------------
 * Hashed level locate / insert (levels.py:270-280, 312-333). */
static int64_t hashed_locate1(int64_t parent, int64_t c, int64_t w, const int32_t* crd) {
  const int64_t base = parent * w;
  for (int64_t step = 0; step < w; ++step) {
    const int64_t p = base + (c + step) % w;
    if (crd[p] == c) return p;
    if (crd[p] == EMPTY) return -1;
  }
  return -1;
}

void or_hashed_locate(int64_t nq, const int32_t* parent, const int32_t* coord, int64_t w,
                      const int32_t* crd, int32_t* out_pos, uint8_t* out_found) {
  for (int64_t q = 0; q < nq; ++q) {
    const int64_t p = hashed_locate1(parent ? parent[q] : 0, coord[q], w, crd);
    out_pos[q] = (int32_t)p;
    out_found[q] = p >= 0;
  }
}

/* Sequential insertion in query order; returns 0, or 4 (segment full). */
int or_hashed_insert(int64_t nq, const int32_t* parent, const int32_t* coord, int64_t w,
                     int32_t* crd) {
  for (int64_t q = 0; q < nq; ++q) {
    const int64_t base = (parent ? parent[q] : 0) * w;
    const int64_t c = coord[q];
    int64_t step = 0;
    for (; step < w; ++step) {
      const int64_t p = base + (c + step) % w;
      if (crd[p] == c) break;
      if (crd[p] == EMPTY) { crd[p] = (int32_t)c; break; }
    }
    if (step == w) return 4;
  }
  return 0;
}

/* SpMV CSR x hash-vector: x located per stored entry (engine.py:558-572);
 * a miss matches no case and contributes nothing (engine.py:618-624). */
void or_spmv_csr_hashx(int64_t nrows, const int32_t* pos, const int32_t* crd,
                       const double* vals, int64_t w, const int32_t* xcrd, const double* xvals,
                       double* y, double* absy) {
  for (int64_t r = 0; r < nrows; ++r) {
    double acc = 0.0, a = 0.0;
    for (int64_t p = pos[r]; p < pos[r + 1]; ++p) {
      const int64_t s = hashed_locate1(0, crd[p], w, xcrd);
      if (s < 0) continue;
      const double t = vals[p] * xvals[s];
      acc = acc + t;
      a += fabs(t);
    }
    y[r] = acc;
    if (absy) absy[r] = a;
  }
}

void or_spmv_csr_hashx_mt(int64_t nrows, const int32_t* pos, const int32_t* crd,
                          const double* vals, int64_t w, const int32_t* xcrd,
                          const double* xvals, double* y, int nthreads) {
  nthreads = clamp_threads(nthreads);
#pragma omp parallel for num_threads(nthreads) schedule(static, 1024)
  for (int64_t r = 0; r < nrows; ++r) {
    double acc = 0.0;
    for (int64_t p = pos[r]; p < pos[r + 1]; ++p) {
      const int64_t s = hashed_locate1(0, crd[p], w, xcrd);
      if (s >= 0) acc = acc + vals[p] * xvals[s];
    }
    y[r] = acc;
  }
}

/* ------------------------------------------------------------------------
 * C = A + B -> CSR.  Row-wise union merge, as engine.py:591-634 runs the
 * j-lattice {A1,B1} -> {A1} -> {B1} over one shared pair of streams: visit
 * the minimum coordinate; both present -> a + b, else the copy.  B's
 * duplicate (i,j) entries are grouped (Grouped, engine.py:107-149) and summed
 * by Python's sum() (engine.py:524-527) — on the CPython 3.12 the reference
 * runs on, Neumaier-compensated (py_sum below).  The gather
 * writer appends 0.0 then += (0.0 + value) (engine.py:404, :413, :625-631),
 * so the stored value is 0.0 + e.  B rows come from b_pos (CSR) or from the
 * row-sorted b_rows (COO).  Returns nnz(C). */
static void b_row_range(int64_t r, const int32_t* b_pos, const int32_t* b_rows, int64_t b_nnz,
                        int64_t* lo, int64_t* hi, int64_t* cursor) {
  if (b_pos) { *lo = b_pos[r]; *hi = b_pos[r + 1]; return; }
  int64_t q = *cursor;
  while (q < b_nnz && b_rows[q] < r) ++q;
  *lo = q;
  while (q < b_nnz && b_rows[q] == r) ++q;
  *hi = q;
  *cursor = q;
}

/* CPython 3.12 builtin sum() over floats (bltinmodule.c builtin_sum_impl):
 * f = 0 + v[0] (int 0 + float), then for each x: t = f + x,
 * c += |f| >= |x| ? (f - t) + x : (x - t) + f, f = t; returns f + c when c is
 * nonzero and finite, else f. */
double or_py_sum(const double* v, int64_t n) {
  double f = 0.0 + v[0], c = 0.0;
  for (int64_t u = 1; u < n; ++u) {
    const double x = v[u], t = f + x;
    if (fabs(f) >= fabs(x)) c += (f - t) + x; else c += (x - t) + f;
    f = t;
  }
  return (c != 0.0 && isfinite(c)) ? f + c : f;
}

static int64_t add_row(int64_t alo, int64_t ahi, const int32_t* a_crd, const double* a_vals,
                       int64_t blo, int64_t bhi, const int32_t* b_cols, const double* b_vals,
                       int32_t* c_crd, double* c_vals) {
  int64_t n = 0, pa = alo, pb = blo;
  while (pa < ahi || pb < bhi) {
    const int64_t ca = pa < ahi ? a_crd[pa] : INT64_MAX;
    const int64_t cb = pb < bhi ? b_cols[pb] : INT64_MAX;
    const int64_t c = ca < cb ? ca : cb;
    double e;
    int have_a = 0, have_b = 0;
    double a = 0.0, b = 0.0;
    if (ca == c) { a = a_vals[pa++]; have_a = 1; }
    if (cb == c) {
      /* group duplicates of c in B */
      int64_t q = pb + 1;
      while (q < bhi && b_cols[q] == c) ++q;
      b = q - pb == 1 ? b_vals[pb] : or_py_sum(b_vals + pb, q - pb);
      pb = q;
      have_b = 1;
    }
    e = have_a && have_b ? a + b : (have_a ? a : b);
    if (c_crd) { c_crd[n] = (int32_t)c; c_vals[n] = 0.0 + e; }
    ++n;
  }
  return n;
}

int64_t or_add_csr(int64_t nrows, const int32_t* a_pos, const int32_t* a_crd,
                   const double* a_vals, int64_t b_nnz, const int32_t* b_pos,
                   const int32_t* b_rows, const int32_t* b_cols, const double* b_vals,
                   int32_t* c_pos, int32_t* c_crd, double* c_vals) {
  int64_t cursor = 0, n = 0;
  c_pos[0] = 0;
  for (int64_t r = 0; r < nrows; ++r) {
    int64_t blo, bhi;
    b_row_range(r, b_pos, b_rows, b_nnz, &blo, &bhi, &cursor);
    n += add_row(a_pos[r], a_pos[r + 1], a_crd, a_vals, blo, bhi, b_cols, b_vals,
                 c_crd ? c_crd + n : NULL, c_vals ? c_vals + n : NULL);
    c_pos[r + 1] = (int32_t)n;
  }
  return n;
}

/* Two-pass multi-threaded variant (count, scan, fill): bit-identical. */
int64_t or_add_csr_mt(int64_t nrows, const int32_t* a_pos, const int32_t* a_crd,
                      const double* a_vals, int64_t b_nnz, const int32_t* b_pos,
                      const int32_t* b_rows, const int32_t* b_cols, const double* b_vals,
                      int32_t* c_pos, int32_t* c_crd, double* c_vals, int nthreads) {
  nthreads = clamp_threads(nthreads);
  int32_t* bp = NULL;
  if (!b_pos) {
    bp = (int32_t*)malloc(sizeof(int32_t) * (size_t)(nrows + 1));
    /* row pointer of the row-sorted COO: first q with rows[q] >= r */
#pragma omp parallel for num_threads(nthreads) schedule(static, 4096)
    for (int64_t r = 0; r <= nrows; ++r) {
      int64_t lo = 0, hi = b_nnz;
      while (lo < hi) { const int64_t mid = (lo + hi) / 2; if (b_rows[mid] < r) lo = mid + 1; else hi = mid; }
      bp[r] = (int32_t)lo;
    }
    b_pos = bp;
  }
  c_pos[0] = 0;
#pragma omp parallel for num_threads(nthreads) schedule(static, 4096)
  for (int64_t r = 0; r < nrows; ++r)
    c_pos[r + 1] = (int32_t)add_row(a_pos[r], a_pos[r + 1], a_crd, a_vals, b_pos[r], b_pos[r + 1],
                                    b_cols, b_vals, NULL, NULL);
  for (int64_t r = 0; r < nrows; ++r) c_pos[r + 1] += c_pos[r];
#pragma omp parallel for num_threads(nthreads) schedule(static, 4096)
  for (int64_t r = 0; r < nrows; ++r)
    add_row(a_pos[r], a_pos[r + 1], a_crd, a_vals, b_pos[r], b_pos[r + 1], b_cols, b_vals,
            c_crd + c_pos[r], c_vals + c_pos[r]);
  free(bp);
  return c_pos[nrows];
}

/* ------------------------------------------------------------------------
 * MTTKRP A(i,r) = X(i,j,k) * B(j,r) * C(k,r): loop order (i, j, k, r),
 * scatter at depth 3, term = (x * B[j,r]) * C[k,r] (engine.py:528-529,
 * Mul(Mul(X,B),C)).  COO-3 and CSF store the same lexicographic order. */
void or_mttkrp_coo3(int64_t I, int32_t R, int64_t nnz, const int32_t* ii, const int32_t* jj,
                    const int32_t* kk, const double* vals, const double* B, const double* C,
                    double* A, double* absA) {
  memset(A, 0, sizeof(double) * (size_t)(I * R));
  if (absA) memset(absA, 0, sizeof(double) * (size_t)(I * R));
  for (int64_t e = 0; e < nnz; ++e) {
    const double v = vals[e];
    const double* b = B + (int64_t)jj[e] * R;
    const double* c = C + (int64_t)kk[e] * R;
    double* a = A + (int64_t)ii[e] * R;
    for (int32_t r = 0; r < R; ++r) {
      const double t = (v * b[r]) * c[r];
      a[r] = a[r] + t;
      if (absA) absA[(int64_t)ii[e] * R + r] += fabs(t);
    }
  }
}

/* Slice-partitioned (whole i-rows per thread, nnz-balanced): bit-identical. */
void or_mttkrp_coo3_mt(int64_t I, int32_t R, int64_t nnz, const int32_t* ii, const int32_t* jj,
                       const int32_t* kk, const double* vals, const double* B, const double* C,
                       double* A, int nthreads) {
  nthreads = clamp_threads(nthreads);
#pragma omp parallel for num_threads(nthreads) schedule(static)
  for (int64_t q = 0; q < I * R; ++q) A[q] = 0.0;
#pragma omp parallel num_threads(nthreads)
  {
#ifdef _OPENMP
    const int t = omp_get_thread_num(), T = omp_get_num_threads();
#else
    const int t = 0, T = 1;
#endif
    int64_t b = nnz * t / T, e = nnz * (t + 1) / T;
    while (b > 0 && b < nnz && ii[b] == ii[b - 1]) ++b;
    while (e > 0 && e < nnz && ii[e] == ii[e - 1]) ++e;
    for (int64_t q = b; q < e; ++q) {
      const double v = vals[q];
      const double* bb = B + (int64_t)jj[q] * R;
      const double* cc = C + (int64_t)kk[q] * R;
      double* a = A + (int64_t)ii[q] * R;
      for (int32_t r = 0; r < R; ++r) a[r] = a[r] + (v * bb[r]) * cc[r];
    }
  }
}

void or_mttkrp_csf(int64_t I, int32_t R, int64_t nslices, const int32_t* crd0,
                   const int32_t* pos1, const int32_t* crd1, const int32_t* pos2,
                   const int32_t* crd2, const double* vals, const double* B, const double* C,
                   double* A, double* absA) {
  memset(A, 0, sizeof(double) * (size_t)(I * R));
  if (absA) memset(absA, 0, sizeof(double) * (size_t)(I * R));
  for (int64_t s = 0; s < nslices; ++s) {
    double* a = A + (int64_t)crd0[s] * R;
    double* aa = absA ? absA + (int64_t)crd0[s] * R : NULL;
    for (int64_t f = pos1[s]; f < pos1[s + 1]; ++f) {
      const double* b = B + (int64_t)crd1[f] * R;
      for (int64_t p = pos2[f]; p < pos2[f + 1]; ++p) {
        const double* c = C + (int64_t)crd2[p] * R;
        const double v = vals[p];
        for (int32_t r = 0; r < R; ++r) {
          const double t = (v * b[r]) * c[r];
          a[r] = a[r] + t;
          if (aa) aa[r] += fabs(t);
        }
      }
    }
  }
}

void or_mttkrp_csf_mt(int64_t I, int32_t R, int64_t nslices, const int32_t* crd0,
                      const int32_t* pos1, const int32_t* crd1, const int32_t* pos2,
                      const int32_t* crd2, const double* vals, const double* B, const double* C,
                      double* A, int nthreads) {
  nthreads = clamp_threads(nthreads);
#pragma omp parallel for num_threads(nthreads) schedule(static)
  for (int64_t q = 0; q < I * R; ++q) A[q] = 0.0;
#pragma omp parallel for num_threads(nthreads) schedule(dynamic, 1)
  for (int64_t s = 0; s < nslices; ++s) {
    double* a = A + (int64_t)crd0[s] * R;
    for (int64_t f = pos1[s]; f < pos1[s + 1]; ++f) {
      const double* b = B + (int64_t)crd1[f] * R;
      for (int64_t p = pos2[f]; p < pos2[f + 1]; ++p) {
        const double* c = C + (int64_t)crd2[p] * R;
        const double v = vals[p];
        for (int32_t r = 0; r < R; ++r) a[r] = a[r] + (v * b[r]) * c[r];
      }
    }
  }
}

/* ------------------------------------------------------------------------
 * SpMV CSR x sparse-vector (compressed, ordered, unique: formats.py
 * "sparse-vector").  The j-lattice of a product is the intersection {A1, x1}:
 * merge_visits (engine.py:211-225) walks both sorted streams and the case
 * body runs only where both are present, in ascending j (run_node,
 * engine.py:591-634); the scatter writer adds each term to y(i) from +0.0. */
void or_spmv_csr_spx(int64_t nrows, const int32_t* pos, const int32_t* crd, const double* vals,
                     int64_t xnnz, const int32_t* xcrd, const double* xvals, double* y,
                     double* absy) {
  for (int64_t r = 0; r < nrows; ++r) {
    double acc = 0.0, a = 0.0;
    int64_t q = 0;
    for (int64_t p = pos[r]; p < pos[r + 1]; ++p) {
      while (q < xnnz && xcrd[q] < crd[p]) ++q;
      if (q == xnnz) break;
      if (xcrd[q] != crd[p]) continue;
      const double t = vals[p] * xvals[q];
      acc = acc + t;
      a += fabs(t);
    }
    y[r] = acc;
    if (absy) absy[r] = a;
  }
}

/* SpMM Y(i,k) = A(i,j) * X(j,k): A CSR, X and Y dense-2 (row-major).  Loop
 * nest (i, j, k) with Y located densely (engine.py:591-634, scatter writer
 * :281-320): each Y(i,k) receives A(i,j) * X(j,k) for the row's j in storage
 * order, accumulated from +0.0.  Y has nrows * K entries. */
void or_spmm_csr(int64_t nrows, int64_t K, const int32_t* pos, const int32_t* crd,
                 const double* vals, const double* X, double* Y, double* absY) {
  for (int64_t q = 0; q < nrows * K; ++q) {
    Y[q] = 0.0;
    if (absY) absY[q] = 0.0;
  }
  for (int64_t r = 0; r < nrows; ++r) {
    double* yr = Y + r * K;
    for (int64_t p = pos[r]; p < pos[r + 1]; ++p) {
      const double a = vals[p];
      const double* xr = X + (int64_t)crd[p] * K;
      for (int64_t k = 0; k < K; ++k) {
        const double t = a * xr[k];
        yr[k] = yr[k] + t;
        if (absY) absY[r * K + k] += fabs(t);
      }
    }
  }
}

void or_spmm_csr_mt(int64_t nrows, int64_t K, const int32_t* pos, const int32_t* crd,
                    const double* vals, const double* X, double* Y, int nthreads) {
  nthreads = clamp_threads(nthreads);
#pragma omp parallel for num_threads(nthreads) schedule(static, 256)
  for (int64_t r = 0; r < nrows; ++r) {
    double* yr = Y + r * K;
    for (int64_t k = 0; k < K; ++k) yr[k] = 0.0;
    for (int64_t p = pos[r]; p < pos[r + 1]; ++p) {
      const double a = vals[p];
      const double* xr = X + (int64_t)crd[p] * K;
      for (int64_t k = 0; k < K; ++k) yr[k] = yr[k] + a * xr[k];
    }
  }
}

/* ------------------------------------------------------------------------
 * TTV Y(i,j) = X(i,j,k) * v(k), X CSF: loop nest (i, j, k) (engine.py:591-634);
 * each (i, j) fiber's products accumulate from +0.0 in storage order.
 * Dense output (I x J, absent fibers 0.0) via the scatter writer; the CSR
 * output (gather writer, engine.py:330-434) stores the same fiber sums
 * (0.0 then += each product) with pos over i and crd = the fibers' j. */
void or_ttv_csf(int64_t nslices, const int32_t* crd0, const int32_t* pos1, const int32_t* crd1,
                const int32_t* pos2, const int32_t* crd2, const double* vals, const double* v,
                double* fiber_sums, double* abs_sums) {
  for (int64_t s = 0; s < nslices; ++s)
    for (int64_t f = pos1[s]; f < pos1[s + 1]; ++f) {
      double acc = 0.0, a = 0.0;
      for (int64_t p = pos2[f]; p < pos2[f + 1]; ++p) {
        const double t = vals[p] * v[crd2[p]];
        acc = acc + t;
        a += fabs(t);
      }
      fiber_sums[f] = acc;
      if (abs_sums) abs_sums[f] = a;
    }
  (void)crd0;
  (void)crd1;
}

/* TTM Y(i,j,r) = X(i,j,k) * U(k,r), X CSF, U and Y dense: loop nest
 * (i, j, k, r); each Y(i,j,r) accumulates the fiber's products x * U(k,r)
 * from +0.0 in storage order.  Writes one R-row per fiber. */
void or_ttm_csf(int64_t nslices, int32_t R, const int32_t* pos1, const int32_t* pos2,
                const int32_t* crd2, const double* vals, const double* U, double* fiber_rows) {
  for (int64_t s = 0; s < nslices; ++s)
    for (int64_t f = pos1[s]; f < pos1[s + 1]; ++f) {
      double* y = fiber_rows + f * R;
      for (int32_t r = 0; r < R; ++r) y[r] = 0.0;
      for (int64_t p = pos2[f]; p < pos2[f + 1]; ++p) {
        const double x = vals[p];
        const double* u = U + (int64_t)crd2[p] * R;
        for (int32_t r = 0; r < R; ++r) y[r] = y[r] + x * u[r];
      }
    }
}

/* INNERPROD a() = X(i,j,k) * Z(i,j,k), both COO-3 sorted lexicographically:
 * the product's lattice at every level is the intersection (merge_visits,
 * engine.py:211-225), and each loop level reduces into its own temporary
 * before adding it to the parent's (run_node, engine.py:591-634): per (i, j)
 * fiber the k products from +0.0, per slice i the fiber sums from +0.0, then
 * the slice sums from +0.0 — verified bit for bit against the reference's
 * evaluate() (tests/golden/widen.npz).  Returns the sum; *abs_sum = sum |x z|. */
double or_inner_coo3(int64_t nx, const int32_t* xi, const int32_t* xj, const int32_t* xk,
                     const double* xv, int64_t nz, const int32_t* zi, const int32_t* zj,
                     const int32_t* zk, const double* zv, double* abs_sum) {
  double total = 0.0, slice = 0.0, fiber = 0.0, a = 0.0;
  int64_t cur_i = -1, cur_j = -1;
  int64_t p = 0, q = 0;
  while (p < nx && q < nz) {
    const int c = xi[p] != zi[q] ? (xi[p] < zi[q] ? -1 : 1)
                : xj[p] != zj[q] ? (xj[p] < zj[q] ? -1 : 1)
                : xk[p] != zk[q] ? (xk[p] < zk[q] ? -1 : 1) : 0;
    if (c < 0) { ++p; continue; }
    if (c > 0) { ++q; continue; }
    if (xi[p] != cur_i || xj[p] != cur_j) {
      if (cur_i >= 0) slice = slice + fiber;
      fiber = 0.0;
      if (xi[p] != cur_i) {
        if (cur_i >= 0) total = total + slice;
        slice = 0.0;
      }
      cur_i = xi[p];
      cur_j = xj[p];
    }
    /* both streams are Grouped (engine.py:107-149): a repeated coordinate is
     * one visit whose value is Python's sum() over its run (engine.py:527) */
    int64_t p2 = p + 1, q2 = q + 1;
    while (p2 < nx && xi[p2] == xi[p] && xj[p2] == xj[p] && xk[p2] == xk[p]) ++p2;
    while (q2 < nz && zi[q2] == zi[q] && zj[q2] == zj[q] && zk[q2] == zk[q]) ++q2;
    const double gx = p2 - p == 1 ? xv[p] : or_py_sum(xv + p, p2 - p);
    const double gz = q2 - q == 1 ? zv[q] : or_py_sum(zv + q, q2 - q);
    const double t = gx * gz;
    fiber = fiber + t;
    for (int64_t u = p; u < p2; ++u)
      for (int64_t w = q; w < q2; ++w) a += fabs(xv[u] * zv[w]);
    p = p2;
    q = q2;
  }
  if (cur_i >= 0) {
    slice = slice + fiber;
    total = total + slice;
  }
  if (abs_sum) *abs_sum = a;
  return total;
}

int or_num_threads(void) { return clamp_threads(0); }
