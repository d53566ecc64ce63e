// Host-side setup of libmgb200.so: validation, the SELL-32-sigma device
// layout, R = P^T, inverse diagonal blocks, coarse dense inverse, and the
// multi-GPU column localisation.  No CUDA calls here (CPU-testable through the
// mgi_* exports of include/mg_internal.h).  Independent of oracle/.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
#include <vector>

#include "../../include/mg.h"
#include "../../include/mg_internal.h"

namespace {
constexpr int kSlice = 32;  // rows per slice = lanes per warp

inline void put_entry(double *val, int64_t e, int lane, int vpe, const double *src) {
  // chunked layout, see mg_internal.h
  double *base = val + (e - lane) * vpe;
  const int half = vpe / 2;
  for (int j = 0; j < half; ++j) {
    base[64 * j + 2 * lane + 0] = src ? src[2 * j + 0] : 0.0;
    base[64 * j + 2 * lane + 1] = src ? src[2 * j + 1] : 0.0;
  }
  if (vpe & 1) base[64 * half + lane] = src ? src[vpe - 1] : 0.0;
}

// fp32 layout: 4-float (16-byte) chunks, then vpe % 4 single-float planes
inline void put_entry(float *val, int64_t e, int lane, int vpe, const double *src) {
  float *base = val + (e - lane) * vpe;
  const int q = vpe / 4;
  for (int j = 0; j < q; ++j)
    for (int t = 0; t < 4; ++t) base[128 * j + 4 * lane + t] = src ? float(src[4 * j + t]) : 0.0f;
  for (int k = 0; k < vpe % 4; ++k) base[128 * q + 32 * k + lane] = src ? float(src[4 * q + k]) : 0.0f;
}

// Gauss-Jordan with partial pivoting on one bs x bs block (bs <= 8).
int gj_block(int bs, const double *a_in, double *out) {
  double a[64], inv[64];
  std::memcpy(a, a_in, sizeof(double) * bs * bs);
  for (int i = 0; i < bs * bs; ++i) inv[i] = 0.0;
  for (int i = 0; i < bs; ++i) inv[i * bs + i] = 1.0;
  for (int k = 0; k < bs; ++k) {
    int p = k;
    double best = std::fabs(a[k * bs + k]);
    for (int r = k + 1; r < bs; ++r) {
      double v = std::fabs(a[r * bs + k]);
      if (v > best) { best = v; p = r; }
    }
    if (!(best > 0.0)) return MG_ERR_SINGULAR;
    if (p != k)
      for (int c = 0; c < bs; ++c) {
        std::swap(a[k * bs + c], a[p * bs + c]);
        std::swap(inv[k * bs + c], inv[p * bs + c]);
      }
    const double d = a[k * bs + k];
    for (int c = 0; c < bs; ++c) { a[k * bs + c] /= d; inv[k * bs + c] /= d; }
    for (int r = 0; r < bs; ++r) {
      if (r == k) continue;
      const double f = a[r * bs + k];
      if (f == 0.0) continue;
      for (int c = 0; c < bs; ++c) {
        a[r * bs + c] -= f * a[k * bs + c];
        inv[r * bs + c] -= f * inv[k * bs + c];
      }
    }
  }
  for (int i = 0; i < bs * bs; ++i)
    if (!std::isfinite(inv[i])) return MG_ERR_SINGULAR;
  std::memcpy(out, inv, sizeof(double) * bs * bs);
  return 0;
}
}  // namespace

extern "C" {

int mgi_validate_csr(int64_t n, int64_t n_cols, const int64_t *rp, const int64_t *col,
                     const double *val, int64_t vpe, int need_diag, int64_t diag_offset) {
  if (n < 0 || !rp) return MG_ERR_INVALID_ARG;
  if (rp[0] != 0) return MG_ERR_STRUCTURE;
  int bad = 0, nonfinite = 0;
#pragma omp parallel for schedule(static) reduction(| : bad, nonfinite)
  for (int64_t i = 0; i < n; ++i) {
    const int64_t a = rp[i], b = rp[i + 1];
    if (b < a) { bad |= 1; continue; }
    bool diag = false;
    for (int64_t k = a; k < b; ++k) {
      const int64_t c = col[k];
      if (c < 0 || c >= n_cols || (k > a && c <= col[k - 1])) bad |= 1;
      if (c == diag_offset + i) diag = true;
    }
    if (need_diag && !diag) bad |= 1;
    if (val)
      for (int64_t t = a * vpe; t < b * vpe; ++t)
        if (!std::isfinite(val[t])) nonfinite |= 1;
  }
  if (bad) return MG_ERR_STRUCTURE;
  if (nonfinite) return MG_ERR_NONFINITE;
  return 0;
}

int mgi_sell_size(int64_t n, const int64_t *rp, int sigma, int64_t *n_slices, int64_t *n_entries) {
  if (n < 0 || sigma < kSlice || sigma % kSlice) return MG_ERR_INVALID_ARG;
  const int64_t ns = (n + kSlice - 1) / kSlice;
  const int64_t nw = (n + sigma - 1) / sigma;
  int64_t total = 0;
#pragma omp parallel for schedule(static) reduction(+ : total)
  for (int64_t w = 0; w < nw; ++w) {
    const int64_t r0 = w * sigma, r1 = std::min<int64_t>(n, r0 + sigma);
    std::vector<int64_t> len(r1 - r0);
    for (int64_t i = r0; i < r1; ++i) len[i - r0] = rp[i + 1] - rp[i];
    std::sort(len.begin(), len.end(), std::greater<int64_t>());
    for (size_t s = 0; s < len.size(); s += kSlice) total += len[s] * kSlice;
  }
  *n_slices = ns;
  *n_entries = total;
  return 0;
}

}  // extern "C" (template helpers below)

template <class T>
int sell_fill(int64_t n, const int64_t *rp, const int64_t *col_in, const double *val_in, int vpe, int sigma,
              int64_t *slice_ptr, int32_t *perm, int32_t *col, T *val) {
  if (n < 0 || sigma < kSlice || sigma % kSlice || vpe < 1) return MG_ERR_INVALID_ARG;
  if (n >= (int64_t(1) << 31)) return MG_ERR_DIMENSION;
  const int64_t ns = (n + kSlice - 1) / kSlice;
  const int64_t nw = (n + sigma - 1) / sigma;
  // 1. permutation: stable sort by length (descending) inside each window
#pragma omp parallel for schedule(static)
  for (int64_t w = 0; w < nw; ++w) {
    const int64_t r0 = w * sigma, r1 = std::min<int64_t>(n, r0 + sigma);
    std::vector<int32_t> idx(r1 - r0);
    std::iota(idx.begin(), idx.end(), int32_t(r0));
    std::stable_sort(idx.begin(), idx.end(), [&](int32_t a, int32_t b) {
      return (rp[a + 1] - rp[a]) > (rp[b + 1] - rp[b]);
    });
    std::copy(idx.begin(), idx.end(), perm + r0);
  }
  for (int64_t t = n; t < ns * kSlice; ++t) perm[t] = -1;
  // 2. slice pointers
  slice_ptr[0] = 0;
  for (int64_t s = 0; s < ns; ++s) {
    const int32_t r = perm[s * kSlice];
    const int64_t len = r >= 0 ? rp[r + 1] - rp[r] : 0;
    slice_ptr[s + 1] = slice_ptr[s] + len * kSlice;
  }
  // 3. entries
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t s = 0; s < ns; ++s) {
    const int64_t len = (slice_ptr[s + 1] - slice_ptr[s]) / kSlice;
    for (int lane = 0; lane < kSlice; ++lane) {
      const int32_t r = perm[s * kSlice + lane];
      const int64_t rl = r >= 0 ? rp[r + 1] - rp[r] : 0;
      for (int64_t k = 0; k < len; ++k) {
        const int64_t e = slice_ptr[s] + k * kSlice + lane;
        if (k < rl) {
          col[e] = int32_t(col_in[rp[r] + k]);
          if (val) put_entry(val, e, lane, vpe, val_in + (rp[r] + k) * vpe);
        } else {
          // padding: zero value at a valid column (the row's last real column,
          // or 0 for empty rows / padding lanes) -- valid for rectangular P, R too
          col[e] = rl > 0 ? int32_t(col_in[rp[r] + rl - 1]) : 0;
          if (val) put_entry(val, e, lane, vpe, nullptr);
        }
      }
    }
  }
  return 0;
}

extern "C" {

int mgi_sell_fill(int64_t n, const int64_t *rp, const int64_t *col_in, const double *val_in, int vpe, int sigma,
                  int64_t *slice_ptr, int32_t *perm, int32_t *col, double *val) {
  return sell_fill<double>(n, rp, col_in, val_in, vpe, sigma, slice_ptr, perm, col, val);
}

int mgi_sell_fill_f32(int64_t n, const int64_t *rp, const int64_t *col_in, const double *val_in, int vpe, int sigma,
                      int64_t *slice_ptr, int32_t *perm, int32_t *col, float *val) {
  return sell_fill<float>(n, rp, col_in, val_in, vpe, sigma, slice_ptr, perm, col, val);
}

int mgi_tsell_size(int64_t n, const int64_t *rp, int C, int sigma, int64_t *n_slices, int64_t *n_entries) {
  if (n < 0 || C < 1 || C > 32 || sigma < C || sigma % C) return MG_ERR_INVALID_ARG;
  const int64_t ns = (n + C - 1) / C;
  const int64_t nw = (n + sigma - 1) / sigma;
  int64_t total = 0;
#pragma omp parallel for schedule(static) reduction(+ : total)
  for (int64_t w = 0; w < nw; ++w) {
    const int64_t r0 = w * sigma, r1 = std::min<int64_t>(n, r0 + sigma);
    std::vector<int64_t> len(r1 - r0);
    for (int64_t i = r0; i < r1; ++i) len[i - r0] = rp[i + 1] - rp[i];
    std::sort(len.begin(), len.end(), std::greater<int64_t>());
    for (size_t s = 0; s < len.size(); s += size_t(C)) total += len[s] * C;
  }
  *n_slices = ns;
  *n_entries = total;
  return 0;
}

int mgi_tsell_fill(int64_t n, const int64_t *rp, const int64_t *col_in, const double *w_in, int wpe, int C, int sigma,
                   int64_t *slice_ptr, int32_t *perm, int32_t *col, float *w) {
  if (n < 0 || C < 1 || C > 32 || sigma < C || sigma % C || wpe < 1) return MG_ERR_INVALID_ARG;
  if (n >= (int64_t(1) << 31)) return MG_ERR_DIMENSION;
  const int64_t nnz = rp[n];
  for (int64_t t = 0; t < nnz * wpe; ++t)
    if (double(float(w_in[t])) != w_in[t]) return 2;  // not exact in fp32: caller keeps the fp64 layout
  const int64_t ns = (n + C - 1) / C;
  const int64_t nw = (n + sigma - 1) / sigma;
#pragma omp parallel for schedule(static)
  for (int64_t wi = 0; wi < nw; ++wi) {
    const int64_t r0 = wi * sigma, r1 = std::min<int64_t>(n, r0 + sigma);
    std::vector<int32_t> idx(r1 - r0);
    std::iota(idx.begin(), idx.end(), int32_t(r0));
    std::stable_sort(idx.begin(), idx.end(), [&](int32_t a, int32_t b) {
      return (rp[a + 1] - rp[a]) > (rp[b + 1] - rp[b]);
    });
    std::copy(idx.begin(), idx.end(), perm + r0);
  }
  for (int64_t t = n; t < ns * C; ++t) perm[t] = -1;
  slice_ptr[0] = 0;
  for (int64_t s = 0; s < ns; ++s) {
    const int32_t r = perm[s * C];
    slice_ptr[s + 1] = slice_ptr[s] + (r >= 0 ? rp[r + 1] - rp[r] : 0) * C;
  }
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t s = 0; s < ns; ++s) {
    const int64_t len = (slice_ptr[s + 1] - slice_ptr[s]) / C;
    for (int q = 0; q < C; ++q) {
      const int32_t r = perm[s * C + q];
      const int64_t rl = r >= 0 ? rp[r + 1] - rp[r] : 0;
      for (int64_t k = 0; k < len; ++k) {
        const int64_t e = slice_ptr[s] + k * C + q;
        const bool real = k < rl;
        col[e] = real ? int32_t(col_in[rp[r] + k]) : (rl > 0 ? int32_t(col_in[rp[r] + rl - 1]) : 0);
        for (int t = 0; t < wpe; ++t) w[e * wpe + t] = real ? float(w_in[(rp[r] + k) * wpe + t]) : 0.0f;
      }
    }
  }
  return 0;
}

int mgi_sell_entry_map(int64_t n, const int64_t *rp, const int64_t *slice_ptr, const int32_t *perm, int64_t *map,
                       int32_t *row_pos) {
  const int64_t ns = (n + kSlice - 1) / kSlice;
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t s = 0; s < ns; ++s)
    for (int lane = 0; lane < kSlice; ++lane) {
      const int32_t r = perm[s * kSlice + lane];
      if (r < 0) continue;
      if (row_pos) row_pos[r] = int32_t(s * kSlice + lane);
      for (int64_t k = 0; k < rp[r + 1] - rp[r]; ++k) map[rp[r] + k] = slice_ptr[s] + k * kSlice + lane;
    }
  return 0;
}

int mgi_csr_transpose(int64_t n_rows, int64_t n_cols, const int64_t *rp, const int64_t *col,
                      const double *w, int wpe, int64_t *orp, int64_t *ocol, double *ow) {
  if (n_rows < 0 || n_cols < 0 || wpe < 1) return MG_ERR_INVALID_ARG;
  std::fill(orp, orp + n_cols + 1, int64_t(0));
  const int64_t nnz = rp[n_rows];
  for (int64_t t = 0; t < nnz; ++t) {
    if (col[t] < 0 || col[t] >= n_cols) return MG_ERR_STRUCTURE;
    orp[col[t] + 1]++;
  }
  for (int64_t j = 0; j < n_cols; ++j) orp[j + 1] += orp[j];
  std::vector<int64_t> next(orp, orp + n_cols);
  for (int64_t i = 0; i < n_rows; ++i)
    for (int64_t t = rp[i]; t < rp[i + 1]; ++t) {
      const int64_t d = next[col[t]]++;
      ocol[d] = i;
      for (int q = 0; q < wpe; ++q) ow[d * wpe + q] = w[t * wpe + q];
    }
  return 0;
}

int mgi_block_diag_inverse(int64_t n, int bs, const int64_t *rp, const int64_t *col,
                           const double *val, double *dinv) {
  if (bs < 1 || bs > 8) return MG_ERR_INVALID_ARG;
  int status = 0;
#pragma omp parallel for schedule(static) reduction(min : status)
  for (int64_t i = 0; i < n; ++i) {
    int64_t kd = -1;
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k)
      if (col[k] == i) { kd = k; break; }
    if (kd < 0) { status = std::min(status, int(MG_ERR_STRUCTURE)); continue; }
    const int st = gj_block(bs, val + kd * bs * bs, dinv + i * bs * bs);
    if (st) status = std::min(status, st);
  }
  return status;
}

int mgi_dense_inverse(int64_t N, double *a, double *inv) {
  if (N < 1) return MG_ERR_INVALID_ARG;
  for (int64_t i = 0; i < N * N; ++i) inv[i] = 0.0;
  for (int64_t i = 0; i < N; ++i) inv[i * N + i] = 1.0;
  for (int64_t k = 0; k < N; ++k) {
    int64_t p = k;
    double best = std::fabs(a[k * N + k]);
    for (int64_t r = k + 1; r < N; ++r) {
      const double v = std::fabs(a[r * N + k]);
      if (v > best) { best = v; p = r; }
    }
    if (!(best > 0.0)) return MG_ERR_SINGULAR;
    if (p != k) {
      std::swap_ranges(a + k * N, a + (k + 1) * N, a + p * N);
      std::swap_ranges(inv + k * N, inv + (k + 1) * N, inv + p * N);
    }
    const double d = a[k * N + k];
    for (int64_t c = 0; c < N; ++c) { a[k * N + c] /= d; inv[k * N + c] /= d; }
    const double *ak = a + k * N;
    const double *ik = inv + k * N;
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < N; ++r) {
      if (r == k) continue;
      const double f = a[r * N + k];
      if (f == 0.0) continue;
      double *ar = a + r * N;
      double *ir = inv + r * N;
      for (int64_t c = k; c < N; ++c) ar[c] -= f * ak[c];
      for (int64_t c = 0; c < N; ++c) ir[c] -= f * ik[c];
    }
  }
  for (int64_t i = 0; i < N * N; ++i)
    if (!std::isfinite(inv[i])) return MG_ERR_SINGULAR;
  return 0;
}

int mgi_bsr_to_dense(int64_t n, int bs, const int64_t *rp, const int64_t *col, const double *val,
                     double *dense) {
  const int64_t N = n * bs;
  std::fill(dense, dense + N * N, 0.0);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k)
      for (int r = 0; r < bs; ++r)
        for (int c = 0; c < bs; ++c)
          dense[(i * bs + r) * N + col[k] * bs + c] += val[(k * bs + r) * bs + c];
  return 0;
}

int mgi_localize_columns(int64_t n_rows, int64_t row_begin, int64_t row_end, const int64_t *rp, const int64_t *col,
                         int64_t *local_col, int64_t *ghosts, int64_t *n_ghost) {
  const int64_t n = row_end - row_begin;
  if (n < 0 || n_rows < 0) return MG_ERR_INVALID_ARG;
  const int64_t nnz = rp[n_rows];
  int64_t ng = 0;
  for (int64_t t = 0; t < nnz; ++t)
    if (col[t] < row_begin || col[t] >= row_end) ghosts[ng++] = col[t];
  std::sort(ghosts, ghosts + ng);
  ng = std::unique(ghosts, ghosts + ng) - ghosts;
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < nnz; ++t) {
    const int64_t c = col[t];
    if (c >= row_begin && c < row_end) local_col[t] = c - row_begin;
    else local_col[t] = n + (std::lower_bound(ghosts, ghosts + ng, c) - ghosts);
  }
  *n_ghost = ng;
  return 0;
}

int mgi_owner(int64_t g, const int64_t *bounds, int nranks) {
  return int(std::upper_bound(bounds, bounds + nranks + 1, g) - bounds) - 1;
}

int mgi_assemble_routed_rows(int64_t m, const int64_t *J, const int64_t *i, const double *w, int wpe, int64_t r0,
                             int64_t nr, int64_t *orp, int64_t *ocol, double *ow) {
  std::fill(orp, orp + nr + 1, int64_t(0));
  for (int64_t t = 0; t < m; ++t) {
    if (J[t] < r0 || J[t] >= r0 + nr) return MG_ERR_STRUCTURE;
    orp[J[t] - r0 + 1]++;
  }
  for (int64_t j = 0; j < nr; ++j) orp[j + 1] += orp[j];
  std::vector<int64_t> next(orp, orp + nr);
  for (int64_t t = 0; t < m; ++t) {
    const int64_t d = next[J[t] - r0]++;
    ocol[d] = i[t];
    for (int q = 0; q < wpe; ++q) ow[d * wpe + q] = w[t * wpe + q];
  }
  return 0;
}

}  // extern "C"
