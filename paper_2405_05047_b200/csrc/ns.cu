// The explicit pressure-correction Navier-Stokes time step of Alg. 2
// on the device: the C ABI of include/ns.h.
//
// B200-first structure: the velocity state lives in ONE
// 32-byte record per velocity node, (u_1, u_2, u_3, p_hat) with
// p_hat = Pi (p + q), so every neighbour gather of the momentum kernel is a
// single sector.  Step 1 is ONE kernel over the SELL-32 velocity pattern with
// four values per entry (K_v, C_x, C_y, C_z): the node-wise products of
// Eq. `tp` are formed on the fly from the gathered record and
// folded into the C_d products (Eq. `multC`), together with the viscous term,
// the pressure gradient C_c p_hat (= G_c (p + q) for the nested Q1-iso-Q2 pair),
// the lumped-mass inverse and the Dirichlet values -- the paper's mom-rhs-nonlin,
// mom-rhs-p, mom-rhs-visc and mom-solve (Table `ns`) in one pass.
// Step 2's divergence G^T u is a warp-per-row CSR product over the pressure
// rows; Step 3 is elementwise plus the zero-mean projection, then Pi (p + q)
// refills the records for the next step.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <new>
#include <vector>

#include "../../include/mg_internal.h"
#include "../../include/ns.h"
#include "common.h"

using namespace mgb;

namespace nsk {

constexpr int kCta = 128;  // 4 warps
constexpr int kWarps = kCta / 32;

struct Sell {
  const int64_t *slice_ptr;
  const int32_t *perm;
  const int32_t *col;
  const double *val;  // chunked: element 2j, 2j+1 of entry e at (e - lane) * vpe + 64 j + 2 lane
  int64_t n_slices;
};

__device__ __forceinline__ double2 ldcs2(const double *p) { return __ldcs(reinterpret_cast<const double2 *>(p)); }
__device__ __forceinline__ double2 ldg2(const double *p) { return __ldg(reinterpret_cast<const double2 *>(p)); }

// Step 1.  Lane = velocity node, warp = slice of 32 nodes.
// Per entry (i, j): s = C_x u_{j,1} + C_y u_{j,2} + C_z u_{j,3} is the row of
// sum_d C_d v^d (v^d_{j,c} = u_{j,d} u_{j,c}) before the factor u_{j,c}:
//   acc_c += (s - nu K) u_{j,c} + C_c p_hat_j.
// dtm[i] = dt / m_u[i], or -(k + 1) for the k-th Dirichlet node (value g[k]).
__global__ void __launch_bounds__(kCta) k_ns_momentum(Sell A, const double *__restrict__ U, double *__restrict__ Un,
                                                      const double *__restrict__ dtm, const double *__restrict__ g,
                                                      const double *__restrict__ F, double nu) {
  const int lane = threadIdx.x & 31;
  const int64_t s = int64_t(blockIdx.x) * kWarps + (threadIdx.x >> 5);
  if (s >= A.n_slices) return;
  const int row = A.perm[s * 32 + lane];
  const int64_t e0 = A.slice_ptr[s], e1 = A.slice_ptr[s + 1];
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  int cn = e0 < e1 ? __ldcs(A.col + e0 + lane) : 0;
  int64_t e = e0;
  constexpr int UB = 2;  // two entries' loads in flight per lane (summed in order)
  for (; e + 32 * (UB - 1) < e1; e += 32 * UB) {
    int cc[UB];
    cc[0] = cn;
#pragma unroll
    for (int u = 1; u < UB; ++u) cc[u] = __ldcs(A.col + e + 32 * u + lane);
    if (e + 32 * UB < e1) cn = __ldcs(A.col + e + 32 * UB + lane);
    double2 kc[UB], cz[UB], uv[UB], wp[UB];
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      const double *v = A.val + (e + 32 * u) * 4;
      kc[u] = ldcs2(v + 2 * lane);       // (K, C_x)
      cz[u] = ldcs2(v + 64 + 2 * lane);  // (C_y, C_z)
      uv[u] = ldg2(U + 4 * int64_t(cc[u]));      // (u_1, u_2)
      wp[u] = ldg2(U + 4 * int64_t(cc[u]) + 2);  // (u_3, p_hat)
    }
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      const double sd = fma(cz[u].y, wp[u].x, fma(cz[u].x, uv[u].y, kc[u].y * uv[u].x));
      const double w = fma(-nu, kc[u].x, sd);
      a0 = fma(kc[u].y, wp[u].y, fma(w, uv[u].x, a0));
      a1 = fma(cz[u].x, wp[u].y, fma(w, uv[u].y, a1));
      a2 = fma(cz[u].y, wp[u].y, fma(w, wp[u].x, a2));
    }
  }
  for (; e < e1; e += 32) {
    const int c = cn;
    const double *v = A.val + e * 4;
    const double2 kc = ldcs2(v + 2 * lane), cz = ldcs2(v + 64 + 2 * lane);
    const double2 uv = ldg2(U + 4 * int64_t(c)), wp = ldg2(U + 4 * int64_t(c) + 2);
    const double sd = fma(cz.y, wp.x, fma(cz.x, uv.y, kc.y * uv.x));
    const double w = fma(-nu, kc.x, sd);
    a0 = fma(kc.y, wp.y, fma(w, uv.x, a0));
    a1 = fma(cz.x, wp.y, fma(w, uv.y, a1));
    a2 = fma(cz.y, wp.y, fma(w, wp.x, a2));
  }
  if (row < 0) return;
  const double t = dtm[row];
  double o0, o1, o2;
  if (t >= 0.0) {
    const double2 su = ldg2(U + 4 * int64_t(row));
    const double s3 = __ldg(U + 4 * int64_t(row) + 2);
    if (F) {
      a0 += F[3 * int64_t(row)];
      a1 += F[3 * int64_t(row) + 1];
      a2 += F[3 * int64_t(row) + 2];
    }
    o0 = fma(t, a0, su.x);
    o1 = fma(t, a1, su.y);
    o2 = fma(t, a2, s3);
  } else {
    const int64_t k = int64_t(-t) - 1;
    o0 = g[3 * k], o1 = g[3 * k + 1], o2 = g[3 * k + 2];
  }
  reinterpret_cast<double2 *>(Un + 4 * int64_t(row))[0] = make_double2(o0, o1);
  Un[4 * int64_t(row) + 2] = o2;
}

// Step 2: d_j = sum_c (G_c^T u_c)_j, rhs_j = -d_j / dt.  Warp per pressure row
// (about 125 entries of 3 values), lanes stride the row, shuffle reduction.
__global__ void __launch_bounds__(256) k_ns_div(int64_t n_p, const int64_t *__restrict__ rp,
                                                const int32_t *__restrict__ col, const double *__restrict__ bv,
                                                const double *__restrict__ U, double *__restrict__ d,
                                                double *__restrict__ rhs, double dt) {
  const int lane = threadIdx.x & 31;
  const int64_t j = (int64_t(blockIdx.x) * 256 + threadIdx.x) >> 5;
  if (j >= n_p) return;
  double acc = 0.0;
  const int64_t e1 = rp[j + 1];
  int64_t e = rp[j] + lane;
  constexpr int UB = 4;  // a row holds ~125 entries: all four strides' loads in flight at once
  for (; e < e1; e += 32 * UB) {
    int64_t c[UB];
    double b0[UB], b1[UB], b2[UB];
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      const bool ok = e + 32 * u < e1;
      const int64_t eu = ok ? e + 32 * u : e;  // clamped: every load stays inside the row
      c[u] = __ldcs(col + eu);
      const double z = ok ? 1.0 : 0.0;
      b0[u] = z * __ldcs(bv + 3 * eu);
      b1[u] = z * __ldcs(bv + 3 * eu + 1);
      b2[u] = z * __ldcs(bv + 3 * eu + 2);
    }
    double2 uv[UB];
    double u3[UB];
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      uv[u] = ldg2(U + 4 * c[u]);
      u3[u] = __ldg(U + 4 * c[u] + 2);
    }
#pragma unroll
    for (int u = 0; u < UB; ++u) acc = fma(b2[u], u3[u], fma(b1[u], uv[u].y, fma(b0[u], uv[u].x, acc)));
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) {
    d[j] = acc;
    rhs[j] = -acc / dt;
  }
}

// Step 3: p <- (p + q) - nu d / m_p
__global__ void k_ns_pupdate(int64_t n, double *__restrict__ p, const double *__restrict__ q,
                             const double *__restrict__ d, const double *__restrict__ mp, double nu) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    p[i] = (p[i] + q[i]) - nu * d[i] / mp[i];
}

// p_hat_i = sum_j Pi_ij (p_j + q_j) into slot 3 of the records.  Lane per row.
__global__ void __launch_bounds__(kCta) k_ns_phat(Sell Pi, const double *__restrict__ p, const double *__restrict__ q,
                                                  double *__restrict__ U) {
  const int lane = threadIdx.x & 31;
  const int64_t s = int64_t(blockIdx.x) * kWarps + (threadIdx.x >> 5);
  if (s >= Pi.n_slices) return;
  const int row = Pi.perm[s * 32 + lane];
  double acc = 0.0;
  for (int64_t e = Pi.slice_ptr[s]; e < Pi.slice_ptr[s + 1]; e += 32) {
    const int c = __ldg(Pi.col + e + lane);
    acc = fma(__ldg(Pi.val + e + lane), __ldg(p + c) + __ldg(q + c), acc);
  }
  if (row >= 0) U[4 * int64_t(row) + 3] = acc;
}

__global__ void k_ns_pack(int64_t n, const double *__restrict__ u, double *__restrict__ U) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    U[4 * i] = u[3 * i];
    U[4 * i + 1] = u[3 * i + 1];
    U[4 * i + 2] = u[3 * i + 2];
  }
}

__global__ void k_ns_unpack(int64_t n, const double *__restrict__ U, double *__restrict__ u) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    u[3 * i] = U[4 * i];
    u[3 * i + 1] = U[4 * i + 1];
    u[3 * i + 2] = U[4 * i + 2];
  }
}

}  // namespace nsk

struct ns_ctx_s {
  mg_ctx pres = nullptr;
  cudaStream_t stream = nullptr;
  int device = 0, n_sm = 148, pres_levels = 0;
  int64_t n_u = 0, n_p = 0;
  // Step-1 operator (SELL-32, 4 values per entry) and Pi (SELL-32, 1 value)
  DevArray<int64_t> a_sp, pi_sp;
  DevArray<int32_t> a_perm, a_col, pi_perm, pi_col;
  DevArray<double> a_val, pi_val;
  int64_t a_ns = 0, pi_ns = 0;
  // divergence G^T: CSR n_p x n_u, 3 values per entry
  DevArray<int64_t> b_rp;
  DevArray<int32_t> b_col;
  DevArray<double> b_val;
  // masses, Dirichlet, load
  std::vector<double> m_u_host;
  DevArray<double> dtm, m_p, g, F;
  std::vector<int64_t> dir_rows;
  std::vector<double> dir_vals;
  bool have_F = false;
  // state
  DevArray<double> U[2], p, q, d, rhs, tmp;
  int cur = 0;
  bool state_set = false, have_d = false;
  double nu = 1e-3, dt = 1e-4, rtol = 1e-6;
  int restart = 30, max_iter = 200, timing = 0;
  bool dtm_dirty = true;
  int64_t launches = 0;
  cudaEvent_t ev[5] = {};
  ~ns_ctx_s() {
    for (auto &e : ev)
      if (e) cudaEventDestroy(e);
  }
};

namespace {

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur;
    if (prev >= 0 && cudaGetDevice(&cur) == cudaSuccess && cur != prev) cudaSetDevice(prev);
  }
};

template <class T>
mg_status fetch(std::vector<T> &dst, const T *src, size_t count, int mem) {
  dst.resize(count);
  if (count == 0) return MG_OK;
  if (!src) return fail(MG_ERR_INVALID_ARG, "NULL input array");
  if (mem == MG_MEM_DEVICE) CU(cudaMemcpy(dst.data(), src, count * sizeof(T), cudaMemcpyDeviceToHost));
  else if (mem == MG_MEM_HOST) std::memcpy(dst.data(), src, count * sizeof(T));
  else return fail(MG_ERR_INVALID_ARG, "mem must be MG_MEM_HOST or MG_MEM_DEVICE");
  return MG_OK;
}

mg_status check_ctx(ns_ctx c) {
  if (!c) return fail(MG_ERR_INVALID_ARG, "NULL ns context");
  return MG_OK;
}

mg_status check_launch(const char *what) {
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(MG_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return MG_OK;
}

unsigned ew_grid(const ns_ctx_s *c, int64_t n) {
  return unsigned(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 8 * c->n_sm)));
}

// SELL-32-sigma layout of a CSR matrix (host.cpp), uploaded
mg_status upload_sell(int64_t n, const std::vector<int64_t> &rp, const std::vector<int64_t> &col,
                      const std::vector<double> &val, int vpe, DevArray<int64_t> &sp_d, DevArray<int32_t> &perm_d,
                      DevArray<int32_t> &col_d, DevArray<double> &val_d, int64_t &n_slices) {
  int64_t ns = 0, ne = 0;
  int st = mgi_sell_size(n, rp.data(), kSigma, &ns, &ne);
  if (st) return fail(mg_status(st), "sell layout: invalid input");
  std::vector<int64_t> sp(ns + 1);
  std::vector<int32_t> perm(ns * 32), c(ne);
  std::vector<double> v(size_t(ne) * vpe);
  st = mgi_sell_fill(n, rp.data(), col.data(), val.data(), vpe, kSigma, sp.data(), perm.data(), c.data(), v.data());
  if (st) return fail(mg_status(st), "sell layout: fill failed");
  TRY(sp_d.upload(sp.data(), sp.size()));
  TRY(perm_d.upload(perm.data(), perm.size()));
  TRY(col_d.upload(c.data(), c.size()));
  TRY(val_d.upload(v.data(), v.size()));
  n_slices = ns;
  return MG_OK;
}

mg_status fetch_csr(int64_t n, int64_t n_cols, const int64_t *rp, const int64_t *col, const double *val, int64_t nnz,
                    int vpe, int mem, std::vector<int64_t> &hrp, std::vector<int64_t> &hcol, std::vector<double> &hval,
                    const char *what) {
  if (!rp || (nnz > 0 && (!col || !val))) return fail(MG_ERR_INVALID_ARG, "%s: NULL array", what);
  TRY(fetch(hrp, rp, size_t(n + 1), mem));
  if (hrp[n] != nnz) return fail(MG_ERR_STRUCTURE, "%s: row_ptr[n] != nnz", what);
  TRY(fetch(hcol, col, size_t(nnz), mem));
  TRY(fetch(hval, val, size_t(nnz) * vpe, mem));
  const int st = mgi_validate_csr(n, n_cols, hrp.data(), hcol.data(), hval.data(), vpe, 0, 0);
  if (st) return fail(mg_status(st), "%s: invalid CSR (structure or non-finite values)", what);
  return MG_OK;
}

// dt / m_u, with -(k + 1) at the k-th Dirichlet node
mg_status refresh_dtm(ns_ctx_s *c) {
  if (!c->dtm_dirty) return MG_OK;
  if (c->m_u_host.empty()) return fail(MG_ERR_STATE, "no lumped masses (ns_set_mass)");
  std::vector<double> t(c->n_u);
  for (int64_t i = 0; i < c->n_u; ++i) t[i] = c->dt / c->m_u_host[i];
  for (size_t k = 0; k < c->dir_rows.size(); ++k) t[c->dir_rows[k]] = -double(k + 1);
  TRY(c->dtm.upload(t.data(), t.size()));
  c->dtm_dirty = false;
  return MG_OK;
}

mg_status ready(ns_ctx_s *c) {
  if (!c->a_sp.p) return fail(MG_ERR_STATE, "no momentum operator (ns_set_momentum)");
  if (!c->pi_sp.p || !c->b_rp.p) return fail(MG_ERR_STATE, "no coupling (ns_set_coupling)");
  if (!c->m_p.p) return fail(MG_ERR_STATE, "no lumped masses (ns_set_mass)");
  if (!c->state_set) return fail(MG_ERR_STATE, "no state (ns_set_state)");
  return refresh_dtm(c);
}

mg_status launch_phat(ns_ctx_s *c, double *U) {
  nsk::Sell Pi{c->pi_sp.p, c->pi_perm.p, c->pi_col.p, c->pi_val.p, c->pi_ns};
  const unsigned gp = unsigned(std::max<int64_t>(1, (c->pi_ns + nsk::kWarps - 1) / nsk::kWarps));
  ++g_tally, nsk::k_ns_phat<<<gp, nsk::kCta, 0, c->stream>>>(Pi, c->p.p, c->q.p, U);
  return check_launch("ns p_hat");
}

mg_status launch_momentum(ns_ctx_s *c) {
  nsk::Sell A{c->a_sp.p, c->a_perm.p, c->a_col.p, c->a_val.p, c->a_ns};
  const unsigned ga = unsigned(std::max<int64_t>(1, (c->a_ns + nsk::kWarps - 1) / nsk::kWarps));
  ++g_tally, nsk::k_ns_momentum<<<ga, nsk::kCta, 0, c->stream>>>(A, c->U[c->cur].p, c->U[c->cur ^ 1].p, c->dtm.p,
                                                                  c->g.p, c->have_F ? c->F.p : nullptr, c->nu);
  return check_launch("ns momentum");
}

struct Count {
  ns_ctx_s *c;
  int64_t t0;
  explicit Count(ns_ctx_s *ctx) : c(ctx), t0(g_tally) {}
  ~Count() { c->launches += g_tally - t0; }
};

}  // namespace

extern "C" {

mg_status ns_create(ns_ctx *out, mg_ctx pressure, int64_t n_u, int64_t n_p) {
  if (!out || !pressure || n_u <= 0 || n_p <= 0) return fail(MG_ERR_INVALID_ARG, "ns_create: bad arguments");
  *out = nullptr;
  void *st = nullptr;
  int dev = 0, nl = 0;
  int64_t nf = 0;
  if (mgi_stream_info(pressure, &st, &dev, &nl, &nf)) return fail(MG_ERR_INVALID_ARG, "bad pressure context");
  if (nf != n_p) return fail(MG_ERR_DIMENSION, "pressure context has %lld fine rows, n_p = %lld", (long long)nf,
                             (long long)n_p);
  auto *c = new (std::nothrow) ns_ctx_s();
  if (!c) return fail(MG_ERR_OOM, "ns_create");
  c->pres = pressure;
  c->stream = static_cast<cudaStream_t>(st);
  c->device = dev;
  c->pres_levels = nl;
  c->n_u = n_u;
  c->n_p = n_p;
  DeviceGuard dg(dev);
  cudaDeviceGetAttribute(&c->n_sm, cudaDevAttrMultiProcessorCount, dev);
  mg_status s = MG_OK;
  for (auto &e : c->ev)
    if (cudaEventCreate(&e) != cudaSuccess) s = fail(MG_ERR_CUDA, "event create");
  if (s == MG_OK) s = c->U[0].alloc(size_t(4 * n_u));
  if (s == MG_OK) s = c->U[1].alloc(size_t(4 * n_u));
  if (s == MG_OK) s = c->p.alloc(n_p);
  if (s == MG_OK) s = c->q.alloc(n_p);
  if (s == MG_OK) s = c->d.alloc(n_p);
  if (s == MG_OK) s = c->rhs.alloc(n_p);
  if (s == MG_OK) s = c->g.alloc(3);
  if (s != MG_OK) {
    delete c;
    return s;
  }
  cudaMemset(c->U[0].p, 0, 32 * n_u);
  cudaMemset(c->U[1].p, 0, 32 * n_u);
  *out = c;
  return MG_OK;
}

mg_status ns_destroy(ns_ctx c) {
  if (!c) return MG_OK;
  DeviceGuard dg(c->device);
  cudaStreamSynchronize(c->stream);
  delete c;
  return MG_OK;
}

mg_status ns_set_momentum(ns_ctx c, const int64_t *rp, const int64_t *col, const double *vals, int64_t nnz, int mem) {
  TRY(check_ctx(c));
  DeviceGuard dg(c->device);
  std::vector<int64_t> hrp, hcol;
  std::vector<double> hv;
  TRY(fetch_csr(c->n_u, c->n_u, rp, col, vals, nnz, 4, mem, hrp, hcol, hv, "momentum operator"));
  return upload_sell(c->n_u, hrp, hcol, hv, 4, c->a_sp, c->a_perm, c->a_col, c->a_val, c->a_ns);
}

mg_status ns_set_coupling(ns_ctx c, const int64_t *pi_rp, const int64_t *pi_col, const double *pi_w, int64_t pi_nnz,
                          const int64_t *g_rp, const int64_t *g_col, const double *g_vals, int64_t g_nnz, int mem) {
  TRY(check_ctx(c));
  DeviceGuard dg(c->device);
  std::vector<int64_t> hrp, hcol;
  std::vector<double> hv;
  TRY(fetch_csr(c->n_u, c->n_p, pi_rp, pi_col, pi_w, pi_nnz, 1, mem, hrp, hcol, hv, "Pi"));
  TRY(upload_sell(c->n_u, hrp, hcol, hv, 1, c->pi_sp, c->pi_perm, c->pi_col, c->pi_val, c->pi_ns));
  TRY(fetch_csr(c->n_u, c->n_p, g_rp, g_col, g_vals, g_nnz, 3, mem, hrp, hcol, hv, "G"));
  std::vector<int64_t> trp(c->n_p + 1), tcol(g_nnz);
  std::vector<double> tv(size_t(g_nnz) * 3);
  if (mgi_csr_transpose(c->n_u, c->n_p, hrp.data(), hcol.data(), hv.data(), 3, trp.data(), tcol.data(), tv.data()))
    return fail(MG_ERR_STRUCTURE, "G^T failed");
  std::vector<int32_t> tc32(tcol.begin(), tcol.end());
  TRY(c->b_rp.upload(trp.data(), trp.size()));
  TRY(c->b_col.upload(tc32.data(), tc32.size()));
  TRY(c->b_val.upload(tv.data(), tv.size()));
  return MG_OK;
}

mg_status ns_set_mass(ns_ctx c, const double *m_u, const double *m_p, int mem) {
  TRY(check_ctx(c));
  DeviceGuard dg(c->device);
  std::vector<double> hu, hp;
  TRY(fetch(hu, m_u, size_t(c->n_u), mem));
  TRY(fetch(hp, m_p, size_t(c->n_p), mem));
  for (double v : hu)
    if (!(v > 0.0) || !std::isfinite(v)) return fail(MG_ERR_INVALID_ARG, "m_u must be positive and finite");
  for (double v : hp)
    if (!(v > 0.0) || !std::isfinite(v)) return fail(MG_ERR_INVALID_ARG, "m_p must be positive and finite");
  c->m_u_host = hu;
  TRY(c->m_p.upload(hp.data(), hp.size()));
  c->dtm_dirty = true;
  return MG_OK;
}

mg_status ns_set_dirichlet(ns_ctx c, const int64_t *rows, const double *vals, int64_t n, int mem) {
  TRY(check_ctx(c));
  if (n < 0) return fail(MG_ERR_INVALID_ARG, "n < 0");
  DeviceGuard dg(c->device);
  std::vector<int64_t> r;
  std::vector<double> v;
  TRY(fetch(r, rows, size_t(n), mem));
  TRY(fetch(v, vals, size_t(3 * n), mem));
  for (int64_t k = 0; k < n; ++k) {
    if (r[k] < 0 || r[k] >= c->n_u || (k > 0 && r[k] <= r[k - 1]))
      return fail(MG_ERR_INVALID_ARG, "Dirichlet rows must be ascending, distinct, in [0, n_u)");
  }
  for (double x : v)
    if (!std::isfinite(x)) return fail(MG_ERR_NONFINITE, "non-finite Dirichlet value");
  c->dir_rows = r;
  c->dir_vals = v;
  TRY(c->g.upload(v.data(), std::max<size_t>(3, v.size())));
  c->dtm_dirty = true;
  return MG_OK;
}

mg_status ns_set_force(ns_ctx c, const double *F, int mem) {
  TRY(check_ctx(c));
  DeviceGuard dg(c->device);
  if (!F) {
    c->have_F = false;
    return MG_OK;
  }
  std::vector<double> h;
  TRY(fetch(h, F, size_t(3 * c->n_u), mem));
  TRY(c->F.upload(h.data(), h.size()));
  c->have_F = true;
  return MG_OK;
}

mg_status ns_set_params(ns_ctx c, double nu, double dt, double rtol, int restart, int max_iter, int timing) {
  TRY(check_ctx(c));
  if (!(nu >= 0.0) || !(dt > 0.0) || !(rtol >= 0.0) || !std::isfinite(nu) || !std::isfinite(dt) || max_iter < 0)
    return fail(MG_ERR_INVALID_ARG, "bad NS parameters");
  if (dt != c->dt) c->dtm_dirty = true;
  c->nu = nu;
  c->dt = dt;
  c->rtol = rtol;
  c->restart = restart;
  c->max_iter = max_iter;
  c->timing = timing;
  return MG_OK;
}

mg_status ns_set_state(ns_ctx c, const double *u, const double *p, const double *q, int mem) {
  TRY(check_ctx(c));
  if (!u || !p || !q) return fail(MG_ERR_INVALID_ARG, "NULL state vector");
  if (!c->pi_sp.p) return fail(MG_ERR_STATE, "no coupling (ns_set_coupling)");
  DeviceGuard dg(c->device);
  Count cnt(c);
  DevArray<double> ud;
  const double *du = u;
  if (mem == MG_MEM_HOST) {
    TRY(ud.upload(u, size_t(3 * c->n_u)));
    du = ud.p;
    CU(cudaMemcpy(c->p.p, p, c->n_p * sizeof(double), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(c->q.p, q, c->n_p * sizeof(double), cudaMemcpyHostToDevice));
  } else if (mem == MG_MEM_DEVICE) {
    CU(cudaMemcpyAsync(c->p.p, p, c->n_p * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    CU(cudaMemcpyAsync(c->q.p, q, c->n_p * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  } else {
    return fail(MG_ERR_INVALID_ARG, "bad mem");
  }
  ++g_tally, nsk::k_ns_pack<<<ew_grid(c, c->n_u), 256, 0, c->stream>>>(c->n_u, du, c->U[c->cur].p);
  TRY(check_launch("ns pack"));
  TRY(launch_phat(c, c->U[c->cur].p));
  CU(cudaStreamSynchronize(c->stream));
  c->state_set = true;
  c->have_d = false;
  return MG_OK;
}

mg_status ns_get_state(ns_ctx c, double *u, double *p, double *q, int mem) {
  TRY(check_ctx(c));
  if (!c->state_set) return fail(MG_ERR_STATE, "no state");
  if (mem != MG_MEM_HOST && mem != MG_MEM_DEVICE) return fail(MG_ERR_INVALID_ARG, "bad mem");
  DeviceGuard dg(c->device);
  Count cnt(c);
  const cudaMemcpyKind k = mem == MG_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  if (u) {
    if (!c->tmp.p || c->tmp.n < size_t(3 * c->n_u)) TRY(c->tmp.alloc(size_t(3 * c->n_u)));
    ++g_tally, nsk::k_ns_unpack<<<ew_grid(c, c->n_u), 256, 0, c->stream>>>(c->n_u, c->U[c->cur].p, c->tmp.p);
    TRY(check_launch("ns unpack"));
    CU(cudaMemcpyAsync(u, c->tmp.p, 3 * c->n_u * sizeof(double), k, c->stream));
  }
  if (p) CU(cudaMemcpyAsync(p, c->p.p, c->n_p * sizeof(double), k, c->stream));
  if (q) CU(cudaMemcpyAsync(q, c->q.p, c->n_p * sizeof(double), k, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  return MG_OK;
}

mg_status ns_momentum(ns_ctx c, double *u_new, int mem) {
  TRY(check_ctx(c));
  if (!u_new) return fail(MG_ERR_INVALID_ARG, "NULL output");
  if (mem != MG_MEM_HOST && mem != MG_MEM_DEVICE) return fail(MG_ERR_INVALID_ARG, "bad mem");
  DeviceGuard dg(c->device);
  TRY(ready(c));
  Count cnt(c);
  TRY(launch_momentum(c));
  if (!c->tmp.p || c->tmp.n < size_t(3 * c->n_u)) TRY(c->tmp.alloc(size_t(3 * c->n_u)));
  ++g_tally, nsk::k_ns_unpack<<<ew_grid(c, c->n_u), 256, 0, c->stream>>>(c->n_u, c->U[c->cur ^ 1].p, c->tmp.p);
  TRY(check_launch("ns unpack"));
  CU(cudaMemcpyAsync(u_new, c->tmp.p, 3 * c->n_u * sizeof(double),
                     mem == MG_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  return MG_OK;
}

mg_status ns_step(ns_ctx c, ns_step_info *info) {
  TRY(check_ctx(c));
  DeviceGuard dg(c->device);
  TRY(ready(c));
  Count cnt(c);
  const bool tm = c->timing != 0;
  if (tm) CU(cudaEventRecord(c->ev[0], c->stream));
  TRY(launch_momentum(c));  // Step 1: U[cur] -> U[nxt] (u^m)
  const int nxt = c->cur ^ 1;
  if (tm) CU(cudaEventRecord(c->ev[1], c->stream));
  // Step 2: d = G^T u^m, rhs = -d / dt, then K_p q = rhs (x0 = 0)
  const unsigned gd = unsigned((c->n_p * 32 + 255) / 256);
  ++g_tally, nsk::k_ns_div<<<gd, 256, 0, c->stream>>>(c->n_p, c->b_rp.p, c->b_col.p, c->b_val.p, c->U[nxt].p, c->d.p,
                                                      c->rhs.p, c->dt);
  TRY(check_launch("ns divergence"));
  CU(cudaMemsetAsync(c->q.p, 0, c->n_p * sizeof(double), c->stream));
  if (tm) CU(cudaEventRecord(c->ev[2], c->stream));
  mg_solve_opts o{MG_GMRES, c->restart, c->max_iter, c->rtol};
  mg_solve_info si{};
  const mg_status ss = mg_solve(c->pres, c->q.p, c->rhs.p, &o, &si);
  if (ss != MG_OK && ss != MG_NOT_CONVERGED) return ss;
  if (tm) CU(cudaEventRecord(c->ev[3], c->stream));
  // Step 3: p = p + q - nu d / m_p, int p = 0, then p_hat = Pi (p + q) for the next step
  ++g_tally, nsk::k_ns_pupdate<<<ew_grid(c, c->n_p), 256, 0, c->stream>>>(c->n_p, c->p.p, c->q.p, c->d.p, c->m_p.p,
                                                                          c->nu);
  TRY(check_launch("ns pressure update"));
  TRY(mg_project_zero_mean(c->pres, c->pres_levels - 1, c->p.p));
  TRY(launch_phat(c, c->U[nxt].p));
  if (tm) CU(cudaEventRecord(c->ev[4], c->stream));
  CU(cudaStreamSynchronize(c->stream));
  c->cur = nxt;
  c->have_d = true;
  if (info) {
    info->iterations = si.iterations;
    info->rel_residual = si.rel_residual;
    info->converged = si.converged;
    for (int i = 0; i < 4; ++i) {
      float ms = 0.f;
      if (tm) cudaEventElapsedTime(&ms, c->ev[i], c->ev[i + 1]);
      info->ms[i] = ms;
    }
  }
  return ss;
}

mg_status ns_get_divergence(ns_ctx c, double *d, int mem) {
  TRY(check_ctx(c));
  if (!d) return fail(MG_ERR_INVALID_ARG, "NULL output");
  if (!c->have_d) return fail(MG_ERR_STATE, "no step taken since the last ns_set_state");
  if (mem != MG_MEM_HOST && mem != MG_MEM_DEVICE) return fail(MG_ERR_INVALID_ARG, "bad mem");
  DeviceGuard dg(c->device);
  CU(cudaMemcpyAsync(d, c->d.p, c->n_p * sizeof(double),
                     mem == MG_MEM_HOST ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  return MG_OK;
}

int64_t ns_launch_count(ns_ctx c) { return c ? c->launches : -1; }

}  // extern "C"
