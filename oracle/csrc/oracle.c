/* CPU ORACLE -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, obviously-correct fp64 reference for the multigrid hot path of
 * arXiv 2405.05047 (PAPER.md "P:n" = line n).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load this library.
 * It shares no code with the CUDA library (paper_2405_05047_b200/csrc).
 *
 * Conventions: block-CSR (BSR) with bs x bs row-major fp64 blocks, int64
 * row_ptr and int64 block columns; vectors node-major [n*bs].
 * Every row is summed sequentially in CSR order; compiled with
 * -ffp-contract=off (no FMA); OpenMP only distributes independent rows, so
 * results are bit-identical for any thread count.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef int64_t i64;

/* y = alpha * A x + beta * y   ("alpha op(A) x + beta y", op = identity).
 * beta == 0 overwrites y without reading it. */
void or_bsr_spmv(i64 n, int bs, const i64 *rp, const i64 *col, const double *val,
                 double alpha, const double *x, double beta, double *y) {
#pragma omp parallel for schedule(static)
  for (i64 i = 0; i < n; ++i) {
    double acc[8];
    for (int r = 0; r < bs; ++r) acc[r] = 0.0;
    for (i64 k = rp[i]; k < rp[i + 1]; ++k) {
      const double *blk = val + (size_t)k * bs * bs;
      const double *xj = x + (size_t)col[k] * bs;
      for (int r = 0; r < bs; ++r)
        for (int c = 0; c < bs; ++c) acc[r] += blk[r * bs + c] * xj[c];
    }
    for (int r = 0; r < bs; ++r) {
      double v = alpha * acc[r];
      y[i * bs + r] = (beta == 0.0) ? v : v + beta * y[i * bs + r];
    }
  }
}

/* r = b - A x  (Alg. gmg Step 2 residual) */
void or_bsr_residual(i64 n, int bs, const i64 *rp, const i64 *col, const double *val,
                     const double *x, const double *b, double *r) {
#pragma omp parallel for schedule(static)
  for (i64 i = 0; i < n; ++i) {
    double acc[8];
    for (int q = 0; q < bs; ++q) acc[q] = 0.0;
    for (i64 k = rp[i]; k < rp[i + 1]; ++k) {
      const double *blk = val + (size_t)k * bs * bs;
      const double *xj = x + (size_t)col[k] * bs;
      for (int q = 0; q < bs; ++q)
        for (int c = 0; c < bs; ++c) acc[q] += blk[q * bs + c] * xj[c];
    }
    for (int q = 0; q < bs; ++q) r[i * bs + q] = b[i * bs + q] - acc[q];
  }
}

/* Gauss-Jordan inverse of one bs x bs block with partial pivoting (max |a|,
 * ties -> lowest row).  Returns 0, or -5 if a pivot is exactly zero. */
static int gj_inverse(int bs, const double *a_in, double *inv) {
  double a[64], e[64];
  memcpy(a, a_in, sizeof(double) * bs * bs);
  for (int r = 0; r < bs; ++r)
    for (int c = 0; c < bs; ++c) e[r * bs + c] = (r == c) ? 1.0 : 0.0;
  for (int k = 0; k < bs; ++k) {
    int p = k;
    for (int r = k + 1; r < bs; ++r)
      if (fabs(a[r * bs + k]) > fabs(a[p * bs + k])) p = r;
    if (a[p * bs + k] == 0.0) return -5;
    if (p != k)
      for (int c = 0; c < bs; ++c) {
        double t = a[k * bs + c]; a[k * bs + c] = a[p * bs + c]; a[p * bs + c] = t;
        t = e[k * bs + c]; e[k * bs + c] = e[p * bs + c]; e[p * bs + c] = t;
      }
    double piv = a[k * bs + k];
    for (int c = 0; c < bs; ++c) { a[k * bs + c] /= piv; e[k * bs + c] /= piv; }
    for (int r = 0; r < bs; ++r) {
      if (r == k) continue;
      double f = a[r * bs + k];
      if (f == 0.0) continue;
      for (int c = 0; c < bs; ++c) { a[r * bs + c] -= f * a[k * bs + c]; e[r * bs + c] -= f * e[k * bs + c]; }
    }
  }
  memcpy(inv, e, sizeof(double) * bs * bs);
  return 0;
}

/* D^{-1}: inverse of every diagonal block A_ii (block-Jacobi S).
 * Returns 0, -3 if a row has no diagonal block, -5 if a block is singular. */
int or_block_diag_inverse(i64 n, int bs, const i64 *rp, const i64 *col, const double *val, double *dinv) {
  int status = 0;
  for (i64 i = 0; i < n; ++i) {
    i64 kd = -1;
    for (i64 k = rp[i]; k < rp[i + 1]; ++k)
      if (col[k] == i) { kd = k; break; }
    if (kd < 0) { status = -3; continue; }
    if (gj_inverse(bs, val + (size_t)kd * bs * bs, dinv + (size_t)i * bs * bs) != 0) status = -5;
  }
  return status;
}

/* One damped block-Jacobi sweep  x_out = x + omega * D^{-1} (b - A x)
 * (S = D^{-1}).  x_out must not alias x. */
void or_jacobi_sweep(i64 n, int bs, const i64 *rp, const i64 *col, const double *val,
                     const double *dinv, double omega, const double *x, const double *b, double *x_out) {
#pragma omp parallel for schedule(static)
  for (i64 i = 0; i < n; ++i) {
    double t[8];
    for (int q = 0; q < bs; ++q) t[q] = 0.0;
    for (i64 k = rp[i]; k < rp[i + 1]; ++k) {
      const double *blk = val + (size_t)k * bs * bs;
      const double *xj = x + (size_t)col[k] * bs;
      for (int q = 0; q < bs; ++q)
        for (int c = 0; c < bs; ++c) t[q] += blk[q * bs + c] * xj[c];
    }
    for (int q = 0; q < bs; ++q) t[q] = b[i * bs + q] - t[q];
    const double *D = dinv + (size_t)i * bs * bs;
    for (int q = 0; q < bs; ++q) {
      double s = 0.0;
      for (int c = 0; c < bs; ++c) s += D[q * bs + c] * t[c];
      x_out[i * bs + q] = x[i * bs + q] + omega * s;
    }
  }
}

/* y = P x (accumulate = 0) or y += P x (accumulate = 1) for a transfer matrix
 * P (n_rows x n_cols CSR, weights_per_entry wpe in {1, bs}): component c of
 * row i is  sum_t w[t*wpe + (wpe>1 ? c : 0)] * x[col[t]*bs + c]. */
void or_transfer(i64 n_rows, int bs, const i64 *rp, const i64 *col, const double *w, int wpe,
                 const double *x, double *y, int accumulate) {
#pragma omp parallel for schedule(static)
  for (i64 i = 0; i < n_rows; ++i) {
    double acc[8];
    for (int c = 0; c < bs; ++c) acc[c] = 0.0;
    for (i64 t = rp[i]; t < rp[i + 1]; ++t)
      for (int c = 0; c < bs; ++c) acc[c] += w[t * wpe + (wpe > 1 ? c : 0)] * x[col[t] * bs + c];
    for (int c = 0; c < bs; ++c) y[i * bs + c] = accumulate ? y[i * bs + c] + acc[c] : acc[c];
  }
}

/* Stable counting-sort transpose of a CSR matrix (R = P^T).
 * out_rp has n_cols+1 entries; entries of each output row appear in
 * ascending original row order. */
void or_csr_transpose(i64 n_rows, i64 n_cols, const i64 *rp, const i64 *col, const double *w, int wpe,
                      i64 *out_rp, i64 *out_col, double *out_w) {
  for (i64 j = 0; j <= n_cols; ++j) out_rp[j] = 0;
  for (i64 t = 0; t < rp[n_rows]; ++t) out_rp[col[t] + 1]++;
  for (i64 j = 0; j < n_cols; ++j) out_rp[j + 1] += out_rp[j];
  i64 *pos = malloc(sizeof(i64) * (size_t)(n_cols + 1));
  memcpy(pos, out_rp, sizeof(i64) * (size_t)(n_cols + 1));
  for (i64 i = 0; i < n_rows; ++i)
    for (i64 t = rp[i]; t < rp[i + 1]; ++t) {
      i64 d = pos[col[t]]++;
      out_col[d] = i;
      for (int q = 0; q < wpe; ++q) out_w[d * wpe + q] = w[t * wpe + q];
    }
  free(pos);
}

/* Dense LU with partial pivoting (max |a|, ties -> lowest row), in place,
 * row-major n x n.  Returns 0 or -5 on an exactly zero pivot. */
int or_lu_factor(i64 n, double *a, i64 *piv) {
  for (i64 k = 0; k < n; ++k) {
    i64 p = k;
    for (i64 r = k + 1; r < n; ++r)
      if (fabs(a[r * n + k]) > fabs(a[p * n + k])) p = r;
    piv[k] = p;
    if (a[p * n + k] == 0.0) return -5;
    if (p != k)
      for (i64 c = 0; c < n; ++c) { double t = a[k * n + c]; a[k * n + c] = a[p * n + c]; a[p * n + c] = t; }
    for (i64 r = k + 1; r < n; ++r) {
      double f = a[r * n + k] / a[k * n + k];
      a[r * n + k] = f;
      if (f == 0.0) continue;
      for (i64 c = k + 1; c < n; ++c) a[r * n + c] -= f * a[k * n + c];
    }
  }
  return 0;
}

/* Solve A x = b with the factors of or_lu_factor (x may alias b). */
void or_lu_solve(i64 n, const double *lu, const i64 *piv, const double *b, double *x) {
  if (x != b) memcpy(x, b, sizeof(double) * (size_t)n);
  for (i64 k = 0; k < n; ++k)
    if (piv[k] != k) { double t = x[k]; x[k] = x[piv[k]]; x[piv[k]] = t; }
  for (i64 r = 0; r < n; ++r) {
    double s = x[r];
    for (i64 c = 0; c < r; ++c) s -= lu[r * n + c] * x[c];
    x[r] = s;
  }
  for (i64 r = n - 1; r >= 0; --r) {
    double s = x[r];
    for (i64 c = r + 1; c < n; ++c) s -= lu[r * n + c] * x[c];
    x[r] = s / lu[r * n + r];
  }
}

/* Sequential dot product sum_i a_i b_i (GMRES MGS). */
double or_dot(i64 n, const double *a, const double *b) {
  double s = 0.0;
  for (i64 i = 0; i < n; ++i) s += a[i] * b[i];
  return s;
}
