// Device kernels of libmgb200.so (sm_100a).  fp64, HBM-bandwidth bound.
//
// Every sparse operator (A_l, P_l, R_l = P_l^T, H) is stored in the
// SELL-32-sigma layout of include/mg_internal.h: one warp per slice of 32
// rows, lane = row, so the k-th entries of the 32 rows of a slice are
// contiguous and a warp reads its matrix values with fully coalesced 16-byte
// loads (2304 contiguous bytes per 3x3-block step), its column indices with
// one 128-byte load, and never needs a cross-lane reduction.  Rows are
// length-sorted inside windows of sigma rows so padding stays < 1%.
//
// Paper references (PAPER.md line numbers): residual SpMV r = b - A x
// (Alg. gmg Step 2), smoother x + omega D^-1 (b - A x),
// prolongation / restriction, coarse solve, GMRES MGS and
// Givens.
#pragma once
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

namespace mgk {

constexpr int kWarpsPerCta = 8;
constexpr int kCta = 32 * kWarpsPerCta;
constexpr int kRedThreads = 256;

struct Sell {
  const int64_t *slice_ptr;  // [n_slices+1] entry offsets (multiples of 32)
  const int32_t *perm;       // [n_slices*32] row of each lane, -1 = padding
  const int32_t *col;        // [n_entries]
  const double *val;         // [n_entries*vpe], chunked (mg_internal.h)
  int64_t n_slices;
  const float *valf;         // fp32 values (mixed-precision V-cycle operators), fp32 chunk layout
};

// ---------------------------------------------------------------------------
// loads.  STREAM: data read once per pass (matrix values / columns of large
// levels) -> evict-first (.cs); otherwise keep in cache (.nc / __ldg).
// ---------------------------------------------------------------------------
template <bool STREAM>
__device__ __forceinline__ double2 ld_val2(const double *p) {
  if constexpr (STREAM) return __ldcs(reinterpret_cast<const double2 *>(p));
  else return __ldg(reinterpret_cast<const double2 *>(p));
}
template <bool STREAM>
__device__ __forceinline__ double ld_val1(const double *p) {
  if constexpr (STREAM) return __ldcs(p);
  else return __ldg(p);
}
template <bool STREAM>
__device__ __forceinline__ int ld_col(const int32_t *p) {
  if constexpr (STREAM) return __ldcs(p);
  else return __ldg(p);
}

// vectors: read-only cache (CG = false) or L2-coherent loads (CG = true: the
// persistent coarse-tail kernel reads vectors written by its earlier phases)
template <bool CG>
__device__ __forceinline__ double ldv(const double *p) {
  if constexpr (CG) return __ldcg(p);
  else return __ldg(p);
}

// values of entry e of lane `lane`; gval = val + (e - lane) * VPE
template <int VPE, bool STREAM>
__device__ __forceinline__ void load_entry(const double *__restrict__ gval, int lane, double (&v)[VPE]) {
#pragma unroll
  for (int j = 0; j < VPE / 2; ++j) {
    const double2 t = ld_val2<STREAM>(gval + 64 * j + 2 * lane);
    v[2 * j] = t.x;
    v[2 * j + 1] = t.y;
  }
  if constexpr (VPE & 1) v[VPE - 1] = ld_val1<STREAM>(gval + 64 * (VPE / 2) + lane);
}

// fp32 values (layout of mgi_sell_fill_f32), converted exactly to fp64;
// gval = valf + (e - lane) * VPE
template <int VPE, bool STREAM>
__device__ __forceinline__ void load_entry(const float *__restrict__ gval, int lane, double (&v)[VPE]) {
#pragma unroll
  for (int j = 0; j < VPE / 4; ++j) {
    const float4 t = STREAM ? __ldcs(reinterpret_cast<const float4 *>(gval + 128 * j + 4 * lane))
                            : __ldg(reinterpret_cast<const float4 *>(gval + 128 * j + 4 * lane));
    v[4 * j] = t.x;
    v[4 * j + 1] = t.y;
    v[4 * j + 2] = t.z;
    v[4 * j + 3] = t.w;
  }
#pragma unroll
  for (int k = 0; k < VPE % 4; ++k) {
    const float *p = gval + 128 * (VPE / 4) + 32 * k + lane;
    v[4 * (VPE / 4) + k] = STREAM ? __ldcs(p) : __ldg(p);
  }
}

// raw fp32 values of one entry (converted at use)
template <int VPE, bool STREAM>
__device__ __forceinline__ void load_entry_raw(const float *__restrict__ gval, int lane, float (&v)[VPE]) {
#pragma unroll
  for (int j = 0; j < VPE / 4; ++j) {
    const float4 t = STREAM ? __ldcs(reinterpret_cast<const float4 *>(gval + 128 * j + 4 * lane))
                            : __ldg(reinterpret_cast<const float4 *>(gval + 128 * j + 4 * lane));
    v[4 * j] = t.x;
    v[4 * j + 1] = t.y;
    v[4 * j + 2] = t.z;
    v[4 * j + 3] = t.w;
  }
#pragma unroll
  for (int k = 0; k < VPE % 4; ++k) {
    const float *p = gval + 128 * (VPE / 4) + 32 * k + lane;
    v[4 * (VPE / 4) + k] = STREAM ? __ldcs(p) : __ldg(p);
  }
}

// ---------------------------------------------------------------------------
// A-pass kernels: y = alpha A x + beta y, r = b - A x, fused block-Jacobi
// sweep out = x + omega D^-1 (b - A x).  Accumulation per output component in
// CSR order (the oracle's order), with FMA.
// ---------------------------------------------------------------------------
enum { OP_SPMV = 0, OP_RESID = 1, OP_SWEEP = 2 };

// Programmatic dependent launch (PDL).  The standalone V-cycle kernels let the
// next kernel launch as soon as all their CTAs are running (trigger at entry),
// and each one loads what does not depend on its predecessor -- slice
// pointers, row permutation, first column indices, D^-1 -- BEFORE waiting for
// the predecessor's results (x, b, r).  On the small levels, whose kernels are
// a few dependent load round trips each, the launch and the structure loads
// overlap the predecessor's tail.  Both instructions are no-ops for a kernel
// launched without the PDL attribute (mg.cu `kl`) and in the tail kernel.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// HALO: columns >= n_own are ghosts (multi-GPU), read from xg[c - n_own].
template <int BS, bool HALO>
__device__ __forceinline__ const double *col_ptr(const double *x, const double *xg, int n_own, int c) {
  if constexpr (HALO) return c < n_own ? x + int64_t(c) * BS : xg + int64_t(c - n_own) * BS;
  else return x + int64_t(c) * BS;
}

// KS warps per slice ("split-k", for levels with few slices): warp `sub` of a
// slice accumulates entries k = sub, sub + KS, ...; the partial sums are added
// in shared memory in sub order.  KS = 1 keeps the CSR summation order.
template <int BS, int KS>
__device__ __forceinline__ bool combine_split(double (&acc)[BS], int wid, int sub, int lane) {
  if constexpr (KS > 1) {
    __shared__ double part[kWarpsPerCta][BS][32];
    if (sub) {
#pragma unroll
      for (int r = 0; r < BS; ++r) part[wid][r][lane] = acc[r];
    }
    __syncthreads();
    if (!sub) {
#pragma unroll
      for (int k = 1; k < KS; ++k)
#pragma unroll
        for (int r = 0; r < BS; ++r) acc[r] += part[wid + k][r][lane];
    }
    __syncthreads();  // partials are reused by the CTA's next task (persistent kernels)
    return !sub;
  }
  return true;
}

// One CTA-task of an A-pass: slice s = task * (8 / KS) + warp / KS.  All warps
// of the CTA must call it (the split-k combine synchronises the CTA).
template <int BS, int OP, bool STREAM, bool HALO, int KS, bool F32, bool CG, bool WAIT = false>
__device__ __forceinline__ void sell_apply_task(const Sell &A, int64_t task, const double *__restrict__ x,
                                                const double *__restrict__ xg, int n_own,
                                                const double *__restrict__ b, const double *__restrict__ dinv,
                                                double *__restrict__ out, double alpha, double beta) {
  constexpr int V = BS * BS;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int sub = KS == 1 ? 0 : wid % KS;
  const int64_t s = task * (kWarpsPerCta / KS) + wid / KS;
  const bool live = s < A.n_slices;
  if (KS == 1 && !live) return;
  double acc[BS];
#pragma unroll
  for (int r = 0; r < BS; ++r) acc[r] = 0.0;
  int row = -1;
  if (live) {
    const int64_t e0 = A.slice_ptr[s], e1 = A.slice_ptr[s + 1];
    row = A.perm[s * 32 + lane];
    int64_t g = e0 + 32 * sub;
    int cn = g < e1 ? ld_col<STREAM>(A.col + g + lane) : 0;  // column of the next entry (prefetched)
    if constexpr (WAIT) pdl_wait();  // x, b are the predecessor's results
    // Few bytes per entry (fp32 values, or bs <= 2): issue the loads of UB
    // entries before the first use so enough bytes are in flight per warp.
    // Entries are still accumulated in order (bit-identical to UB = 1).
    // Rows are processed in batches of UB entries whose loads are all issued
    // before their (in-order) FMAs; the last, partial batch of a slice is a
    // batch of exactly the remaining count (a warp-uniform switch over
    // compile-time sizes), so short rows -- 9 entries of a 2D Q1 row, 4-5 per
    // warp under split-k 2 -- are one batch of independent loads instead of a
    // dependent column -> x chain per entry.  Summation order unchanged.
    constexpr int UB = F32 ? 4 : (V == 1 ? 8 : (V == 4 ? 4 : 1));
    if constexpr (UB > 1) {
      constexpr int step = 32 * KS;
      auto batch = [&](auto NC) {
        constexpr int N = decltype(NC)::value;
        int cc[N];
        cc[0] = cn;
#pragma unroll
        for (int u = 1; u < N; ++u) cc[u] = ld_col<STREAM>(A.col + g + u * step + lane);
        if (g + N * step < e1) cn = ld_col<STREAM>(A.col + g + N * step + lane);
        double vd[N][V];
        if constexpr (F32) {
          float vf[N][V];
#pragma unroll
          for (int u = 0; u < N; ++u) load_entry_raw<V, STREAM>(A.valf + (g + u * step) * V, lane, vf[u]);
#pragma unroll
          for (int u = 0; u < N; ++u)
#pragma unroll
            for (int j = 0; j < V; ++j) vd[u][j] = double(vf[u][j]);
        } else {
#pragma unroll
          for (int u = 0; u < N; ++u) load_entry<V, STREAM>(A.val + (g + u * step) * V, lane, vd[u]);
        }
        double xv[N][BS];
#pragma unroll
        for (int u = 0; u < N; ++u) {
          const double *xc = col_ptr<BS, HALO>(x, xg, n_own, cc[u]);
#pragma unroll
          for (int q = 0; q < BS; ++q) xv[u][q] = ldv<CG>(xc + q);
        }
#pragma unroll
        for (int u = 0; u < N; ++u)
#pragma unroll
          for (int r = 0; r < BS; ++r)
#pragma unroll
            for (int q = 0; q < BS; ++q) acc[r] = fma(vd[u][r * BS + q], xv[u][q], acc[r]);
        g += N * step;
      };
      while (g + (UB - 1) * step < e1) batch(std::integral_constant<int, UB>{});
      switch (int((e1 - g + step - 1) / step)) {  // 0 .. UB-1 entries left
        case 1: batch(std::integral_constant<int, 1>{}); break;
        case 2: batch(std::integral_constant<int, 2>{}); break;
        case 3: batch(std::integral_constant<int, 3>{}); break;
        case 4: if constexpr (UB > 4) batch(std::integral_constant<int, (UB > 4 ? 4 : 1)>{}); break;
        case 5: if constexpr (UB > 5) batch(std::integral_constant<int, (UB > 5 ? 5 : 1)>{}); break;
        case 6: if constexpr (UB > 6) batch(std::integral_constant<int, (UB > 6 ? 6 : 1)>{}); break;
        case 7: if constexpr (UB > 7) batch(std::integral_constant<int, (UB > 7 ? 7 : 1)>{}); break;
        default: break;
      }
    }
#pragma unroll 4
    for (; g < e1; g += 32 * KS) {
      const int c = cn;
      if (g + 32 * KS < e1) cn = ld_col<STREAM>(A.col + g + 32 * KS + lane);
      double v[V];
      if constexpr (F32) load_entry<V, STREAM>(A.valf + g * V, lane, v);
      else load_entry<V, STREAM>(A.val + g * V, lane, v);
      const double *xc = col_ptr<BS, HALO>(x, xg, n_own, c);
      double xv[BS];
#pragma unroll
      for (int q = 0; q < BS; ++q) xv[q] = ldv<CG>(xc + q);
#pragma unroll
      for (int r = 0; r < BS; ++r)
#pragma unroll
        for (int q = 0; q < BS; ++q) acc[r] = fma(v[r * BS + q], xv[q], acc[r]);
    }
  }
  if constexpr (WAIT) pdl_wait();  // warps without entries (they skipped the loop)
  if (!combine_split<BS, KS>(acc, wid, sub, lane)) return;
  if (!live || row < 0) return;
  const int64_t o = int64_t(row) * BS;
  if constexpr (OP == OP_SPMV) {
#pragma unroll
    for (int r = 0; r < BS; ++r) out[o + r] = (beta == 0.0) ? alpha * acc[r] : alpha * acc[r] + beta * out[o + r];
  } else if constexpr (OP == OP_RESID) {
#pragma unroll
    for (int r = 0; r < BS; ++r) out[o + r] = ldv<CG>(b + o + r) - acc[r];
  } else {
    double t[BS];
#pragma unroll
    for (int r = 0; r < BS; ++r) t[r] = ldv<CG>(b + o + r) - acc[r];
    double d[V];
    load_entry<V, STREAM>(dinv + s * 32 * V, lane, d);
#pragma unroll
    for (int r = 0; r < BS; ++r) {
      double u = 0.0;
#pragma unroll
      for (int q = 0; q < BS; ++q) u = fma(d[r * BS + q], t[q], u);
      out[o + r] = fma(alpha, u, ldv<CG>(x + o + r));
    }
  }
}

// MGB200_KS_MINB (compile-time experiment): minimum CTAs per SM for the split-k
// variants.  6 caps them at 40 registers (no spills) so more of a one-wave grid is
// resident; measured on the same box it LOSES (C3 148.8 -> 146.5 V-cycles/s, C2
// 2194 -> 1964: the lost registers were the batched loads in flight), so 0 = none.
#ifndef MGB200_KS_MINB
#define MGB200_KS_MINB 0
#endif
template <int BS, int OP, bool STREAM, bool HALO, int KS, bool F32 = false>
__global__ void __launch_bounds__(kCta, (KS > 1 && BS <= 3) ? MGB200_KS_MINB : 0) k_sell_apply(Sell A, const double *__restrict__ x,
                                                     const double *__restrict__ xg, int n_own,
                                                     const double *__restrict__ b,
                                                     const double *__restrict__ dinv,
                                                     double *__restrict__ out, double alpha, double beta) {
  pdl_trigger();
  sell_apply_task<BS, OP, STREAM, HALO, KS, F32, false, true>(A, blockIdx.x, x, xg, n_own, b, dinv, out, alpha,
                                                               beta);
}

// First smoothing step from the zero guess: x = omega D^-1 b, A-free.
template <int BS, bool CG, bool WAIT = false>
__device__ __forceinline__ void sweep0_task(int64_t n_slices, int64_t task, const int32_t *__restrict__ perm,
                                            const double *__restrict__ dinv, const double *__restrict__ b,
                                            double *__restrict__ x, double omega) {
  constexpr int V = BS * BS;
  const int lane = threadIdx.x & 31;
  const int64_t s = task * kWarpsPerCta + (threadIdx.x >> 5);
  if (s >= n_slices) return;
  const int row = perm[s * 32 + lane];
  double d[V];
  load_entry<V, true>(dinv + s * 32 * V, lane, d);
  if constexpr (WAIT) pdl_wait();
  if (row < 0) return;
  const int64_t o = int64_t(row) * BS;
  double t[BS];
#pragma unroll
  for (int q = 0; q < BS; ++q) t[q] = ldv<CG>(b + o + q);
#pragma unroll
  for (int r = 0; r < BS; ++r) {
    double u = 0.0;
#pragma unroll
    for (int q = 0; q < BS; ++q) u = fma(d[r * BS + q], t[q], u);
    x[o + r] = omega * u;
  }
}

template <int BS>
__global__ void __launch_bounds__(kCta) k_sweep0(int64_t n_slices, const int32_t *__restrict__ perm,
                                                 const double *__restrict__ dinv, const double *__restrict__ b,
                                                 double *__restrict__ x, double omega) {
  pdl_trigger();
  sweep0_task<BS, false, true>(n_slices, blockIdx.x, perm, dinv, b, x, omega);
}

// Transfer y = T x (ACCUM = 0) or y += T x (ACCUM = 1) with scalar weights
// (WPE = 1) or per-component weights (WPE = BS): restriction R r (P:131,
// P:337), prolongation x + P y, hanging interpolation H x.
template <int BS, int WPE, bool ACCUM, bool STREAM, bool HALO, int KS, bool CG, bool WAIT = false>
__device__ __forceinline__ void transfer_task(const Sell &T, int64_t task, const double *__restrict__ in,
                                              const double *__restrict__ ing, int n_own, double *__restrict__ out) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int sub = KS == 1 ? 0 : wid % KS;
  const int64_t s = task * (kWarpsPerCta / KS) + wid / KS;
  const bool live = s < T.n_slices;
  if (KS == 1 && !live) return;
  double acc[BS];
#pragma unroll
  for (int q = 0; q < BS; ++q) acc[q] = 0.0;
  int row = -1;
  if (live) {
    const int64_t e0 = T.slice_ptr[s], e1 = T.slice_ptr[s + 1];
    row = T.perm[s * 32 + lane];
    int64_t g = e0 + 32 * sub;
    int cn = g < e1 ? ld_col<STREAM>(T.col + g + lane) : 0;
    if constexpr (WAIT) pdl_wait();
    // batches of UB entries' loads in flight (summed in order); the last batch
    // of exactly the remaining count, as in sell_apply_task, so a 1-8-entry
    // prolongation row is one batch
    constexpr int UB = 4;
    constexpr int step = 32 * KS;
    auto batch = [&](auto NC) {
      constexpr int N = decltype(NC)::value;
      int cc[N];
      cc[0] = cn;
#pragma unroll
      for (int u = 1; u < N; ++u) cc[u] = ld_col<STREAM>(T.col + g + u * step + lane);
      if (g + N * step < e1) cn = ld_col<STREAM>(T.col + g + N * step + lane);
      double w[N][WPE], xv[N][BS];
#pragma unroll
      for (int u = 0; u < N; ++u) load_entry<WPE, STREAM>(T.val + (g + u * step) * WPE, lane, w[u]);
#pragma unroll
      for (int u = 0; u < N; ++u) {
        const double *xc = col_ptr<BS, HALO>(in, ing, n_own, cc[u]);
#pragma unroll
        for (int q = 0; q < BS; ++q) xv[u][q] = ldv<CG>(xc + q);
      }
#pragma unroll
      for (int u = 0; u < N; ++u)
#pragma unroll
        for (int q = 0; q < BS; ++q) acc[q] = fma(w[u][WPE == 1 ? 0 : q], xv[u][q], acc[q]);
      g += N * step;
    };
    while (g + (UB - 1) * step < e1) batch(std::integral_constant<int, UB>{});
    switch (int((e1 - g + step - 1) / step)) {
      case 1: batch(std::integral_constant<int, 1>{}); break;
      case 2: batch(std::integral_constant<int, 2>{}); break;
      case 3: batch(std::integral_constant<int, 3>{}); break;
      default: break;
    }
  }
  if constexpr (WAIT) pdl_wait();
  if (!combine_split<BS, KS>(acc, wid, sub, lane)) return;
  if (!live || row < 0) return;
  const int64_t o = int64_t(row) * BS;
#pragma unroll
  for (int q = 0; q < BS; ++q) out[o + q] = ACCUM ? out[o + q] + acc[q] : acc[q];
}

template <int BS, int WPE, bool ACCUM, bool STREAM, bool HALO, int KS>
__global__ void __launch_bounds__(kCta) k_transfer(Sell T, const double *__restrict__ in,
                                                   const double *__restrict__ ing, int n_own,
                                                   double *__restrict__ out) {
  pdl_trigger();
  transfer_task<BS, WPE, ACCUM, STREAM, HALO, KS, false, true>(T, blockIdx.x, in, ing, n_own, out);
}

// Prolongation-add x += P y on CSR rows in NATURAL order (lane = fine row r,
// a warp = 32 consecutive rows), so x is read and written with coalesced
// 768-byte (bs 3) warp accesses.  On SELL-32-sigma the 1-8-entry rows of P are
// length-sorted inside windows of 4096 rows: a warp's 32 rows were scattered,
// every x access a separate sector (ncu r2: 114 cycles per issued instruction,
// long-scoreboard bound, 0.46 of peak).  Entries {column, fp32-exact dyadic
// weight} (WPE = 1) or columns + per-component fp32 weights (WPE = BS) are read
// per lane from the row's CSR range (the 32 rows' entries are contiguous);
// each row is summed in CSR order with FMA, exactly as k_transfer.
struct PCsr {
  const int32_t *rp;  // [n+1] entry offsets
  const int2 *cw;     // WPE = 1: {col, __float_as_int(w)}
  const int32_t *col; // WPE = BS: columns
  const float *w;     // WPE = BS: [entries*BS]
  int64_t n;
};

template <int BS, int WPE, bool HALO>
__global__ void __launch_bounds__(kCta) k_prolong_csr(PCsr P, const double *__restrict__ in,
                                                      const double *__restrict__ ing, int n_own,
                                                      double *__restrict__ out) {
  constexpr int UB = 8;  // entries per batch (a 3D Q1 row has at most 8 without hanging nodes)
  pdl_trigger();
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const bool live = r < P.n;
  int e0 = 0, len = 0;
  if (live) {
    e0 = P.rp[r];
    len = P.rp[r + 1] - e0;
  }
  // Loads past a row's end re-read its first entry (clamped, unconditional):
  // per-lane predicated loads measured slower (C3 V-cycle 5.080 vs 5.059 ms).
  int c[UB];
  float w[UB][WPE];
  auto fetch = [&](int k0) {
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      const int k = k0 + u < len ? e0 + k0 + u : e0;
      if constexpr (WPE == 1) {
        const int2 t = __ldg(P.cw + (len ? k : 0));
        c[u] = t.x;
        w[u][0] = __int_as_float(t.y);
      } else {
        c[u] = __ldg(P.col + (len ? k : 0));
#pragma unroll
        for (int q = 0; q < BS; ++q) w[u][q] = __ldg(P.w + int64_t(len ? k : 0) * BS + q);
      }
    }
  };
  fetch(0);   // structure only: before the predecessor's result is needed
  pdl_wait();  // y = the coarse correction, x = this level's iterate
  if (!live) return;
  double acc[BS], xo[BS];
  const int64_t o = r * BS;
#pragma unroll
  for (int q = 0; q < BS; ++q) acc[q] = 0.0, xo[q] = out[o + q];
  for (int k0 = 0; k0 < len; k0 += UB) {
    if (k0) fetch(k0);
    double y[UB][BS];
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      const double *yc = col_ptr<BS, HALO>(in, ing, n_own, c[u]);
#pragma unroll
      for (int q = 0; q < BS; ++q) y[u][q] = __ldg(yc + q);
    }
#pragma unroll
    for (int u = 0; u < UB; ++u)
#pragma unroll
      for (int q = 0; q < BS; ++q) {
        const double t = fma(double(w[u][WPE == 1 ? 0 : q]), y[u][q], acc[q]);
        acc[q] = k0 + u < len ? t : acc[q];
      }
  }
#pragma unroll
  for (int q = 0; q < BS; ++q) out[o + q] = xo[q] + acc[q];
}

// Transfer on the SELL-C layout of mgi_tsell_fill (C = 32 / BS rows per
// slice): lane (r, q) = (lane / BS, lane % BS) accumulates component q of the
// slice's row r, so the BS components of a gathered node are ONE warp load
// instruction over adjacent lanes (one L1 wavefront per node instead of BS:
// the SELL-32 transfer was bound by L1 data-pipe wavefronts, ncu r2a).  Column
// and weight of an entry are one 8-byte load (int2 {col, fp32 weight bits}:
// the dyadic weights are exact in fp32) when WPE = 1; per-component weights
// (WPE = BS) are fp32 planes indexed e*BS + q, contiguous over the warp.
// Accumulation order per row and split-k combine as k_transfer: bit-identical.
struct TSell {
  const int64_t *slice_ptr;  // [n_slices+1], multiples of C
  const int32_t *perm;       // [n_slices*C] row of each slice position, -1 = padding
  const int2 *cw;            // WPE = 1: {col, __float_as_int(w)} per entry
  const int32_t *col;        // WPE = BS: columns
  const float *w;            // WPE = BS: [entries*BS]
  int64_t n_slices;
};

// NSL consecutive slices per warp (KS warps per slice group): the loads of
// the NSL slices' entries are issued together, so a warp keeps NSL dependent
// column -> value chains in flight (prolongation rows have 1-8 entries: one
// slice alone leaves the warp waiting on a short chain).
template <int BS, int WPE, bool ACCUM, bool HALO, int KS, int NSL>
__global__ void __launch_bounds__(kCta) k_tsell(TSell T, const double *__restrict__ in,
                                                const double *__restrict__ ing, int n_own,
                                                double *__restrict__ out) {
  constexpr int C = 32 / BS;
  pdl_trigger();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int sub = KS == 1 ? 0 : wid % KS;
  const int64_t s0 = (int64_t(blockIdx.x) * (kWarpsPerCta / KS) + wid / KS) * NSL;
  if (KS == 1 && s0 >= T.n_slices) return;
  const int r = lane / BS, q = lane - r * BS;
  double acc[NSL];
  int row[NSL];
  int64_t eb[NSL], len[NSL];
  int64_t kmax = 0;
#pragma unroll
  for (int u = 0; u < NSL; ++u) {
    acc[u] = 0.0;
    row[u] = -1;
    len[u] = 0;
    eb[u] = 0;
    const int64_t s = s0 + u;
    if (s < T.n_slices && r < C) {
      const int64_t e0 = T.slice_ptr[s];
      len[u] = (T.slice_ptr[s + 1] - e0) / C;
      eb[u] = e0 + r;
      row[u] = T.perm[s * C + r];
      kmax = len[u] > kmax ? len[u] : kmax;
    }
  }
  pdl_wait();  // `in` is the predecessor's result
  auto entry = [&](int64_t e, int &c, double &w) {
    if constexpr (WPE == 1) {
      const int2 t = __ldg(T.cw + e);
      c = t.x;
      w = double(__int_as_float(t.y));
    } else {
      c = __ldg(T.col + e);
      w = double(__ldg(T.w + e * BS + q));
    }
  };
  if constexpr (NSL == 1) {
    // loads of UB entries in flight before their use (summed in order); the last
    // batch of exactly the remaining count (len is uniform over the slice)
    constexpr int UB = 4;
    int64_t k = sub;
    auto batch = [&](auto NC) {
      constexpr int N = decltype(NC)::value;
      int c[N];
      double w[N], v[N];
#pragma unroll
      for (int u = 0; u < N; ++u) entry(eb[0] + (k + u * KS) * C, c[u], w[u]);
#pragma unroll
      for (int u = 0; u < N; ++u) v[u] = __ldg(col_ptr<BS, HALO>(in, ing, n_own, c[u]) + q);
#pragma unroll
      for (int u = 0; u < N; ++u) acc[0] = fma(w[u], v[u], acc[0]);
      k += N * KS;
    };
    while (k + (UB - 1) * KS < len[0]) batch(std::integral_constant<int, UB>{});
    switch (int(k < len[0] ? (len[0] - k + KS - 1) / KS : 0)) {
      case 1: batch(std::integral_constant<int, 1>{}); break;
      case 2: batch(std::integral_constant<int, 2>{}); break;
      case 3: batch(std::integral_constant<int, 3>{}); break;
      default: break;
    }
  } else {
    for (int64_t k = sub; k < kmax; k += KS) {
      int c[NSL];
      double w[NSL], v[NSL];
#pragma unroll
      for (int u = 0; u < NSL; ++u)
        if (k < len[u]) entry(eb[u] + k * C, c[u], w[u]);
#pragma unroll
      for (int u = 0; u < NSL; ++u)
        if (k < len[u]) v[u] = __ldg(col_ptr<BS, HALO>(in, ing, n_own, c[u]) + q);
#pragma unroll
      for (int u = 0; u < NSL; ++u)
        if (k < len[u]) acc[u] = fma(w[u], v[u], acc[u]);
    }
  }
  if (!combine_split<NSL, KS>(acc, wid, sub, lane)) return;
#pragma unroll
  for (int u = 0; u < NSL; ++u) {
    if (row[u] < 0) continue;
    const int64_t o = int64_t(row[u]) * BS + q;
    out[o] = ACCUM ? out[o] + acc[u] : acc[u];
  }
}

// Coarse solve y = A_0^{-1} d with the dense inverse (row stride ld, even,
// zero padded): one warp per row, 16-byte loads, shuffle reduction.
template <bool CG>
__device__ __forceinline__ void gemv_row(int64_t N, int64_t ld, const double *__restrict__ M,
                                         const double *__restrict__ d, double *__restrict__ y, int64_t r) {
  const int lane = threadIdx.x & 31;
  const double *row = M + r * ld;
  double acc = 0.0;
  int64_t c = 2 * lane;
  for (; c + 192 + 1 < N; c += 256) {  // four independent 16-byte loads in flight
    double2 m[4], dv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      m[u] = __ldg(reinterpret_cast<const double2 *>(row + c + 64 * u));
      dv[u] = make_double2(ldv<CG>(d + c + 64 * u), ldv<CG>(d + c + 64 * u + 1));
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      acc = fma(m[u].x, dv[u].x, acc);
      acc = fma(m[u].y, dv[u].y, acc);
    }
  }
  for (; c < N; c += 64) {
    const double2 m = __ldg(reinterpret_cast<const double2 *>(row + c));
    acc = fma(m.x, ldv<CG>(d + c), acc);
    if (c + 1 < N) acc = fma(m.y, ldv<CG>(d + c + 1), acc);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) y[r] = acc;
}

// The same product with RS warps per row (a CTA = 8 / RS rows): each warp sums
// a contiguous quarter (RS = 4) of the row with four 16-byte loads in flight
// per lane, the RS partial sums are added in warp order through shared memory.
// The dense inverse (C3: 3000^2 = 72 MB) is read in one wave of short chains
// instead of 3000 chains of 12 dependent steps.
// Partial sum of row r of M d over the column chunk `sub` of RS (the split
// kernel's per-warp work, then a shuffle reduction): shared by k_dense_gemv_split
// and the persistent tail kernel so both produce bit-identical results.
template <int RS, bool CG>
__device__ __forceinline__ double gemv_chunk(int64_t N, int64_t ld, const double *__restrict__ M,
                                             const double *__restrict__ d, int64_t r, int sub) {
  const int lane = threadIdx.x & 31;
  double acc = 0.0;
  const int64_t chunk = ((N + RS - 1) / RS + 1) & ~int64_t(1);  // even: 16-byte loads stay aligned (ld even)
  const int64_t c0 = sub * chunk, c1 = c0 + chunk < N ? c0 + chunk : N;
  const double *row = M + r * ld;
  int64_t c = c0 + 2 * lane;
  for (; c + 192 + 1 < c1; c += 256) {
    double2 m[4], dv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      m[u] = __ldg(reinterpret_cast<const double2 *>(row + c + 64 * u));
      dv[u] = CG ? __ldcg(reinterpret_cast<const double2 *>(d + c + 64 * u))
                 : __ldg(reinterpret_cast<const double2 *>(d + c + 64 * u));
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      acc = fma(m[u].x, dv[u].x, acc);
      acc = fma(m[u].y, dv[u].y, acc);
    }
  }
  for (; c < c1; c += 64) {
    acc = fma(__ldg(row + c), ldv<CG>(d + c), acc);
    if (c + 1 < c1) acc = fma(__ldg(row + c + 1), ldv<CG>(d + c + 1), acc);
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  return acc;
}

template <int RS>
__global__ void __launch_bounds__(kCta) k_dense_gemv_split(int64_t N, int64_t ld, const double *__restrict__ M,
                                                           const double *__restrict__ d, double *__restrict__ y) {
  __shared__ double part[kWarpsPerCta];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int64_t r = int64_t(blockIdx.x) * (kWarpsPerCta / RS) + wid / RS;
  const int sub = wid % RS;
  pdl_trigger();
  pdl_wait();
  const double acc = r < N ? gemv_chunk<RS, false>(N, ld, M, d, r, sub) : 0.0;
  if (lane == 0) part[wid] = acc;
  __syncthreads();
  if (sub == 0 && lane == 0 && r < N) {
    double s = part[wid];
#pragma unroll
    for (int k = 1; k < RS; ++k) s += part[wid + k];
    y[r] = s;
  }
}

__global__ void __launch_bounds__(kCta) k_dense_gemv(int64_t N, int64_t ld, const double *__restrict__ M,
                                                     const double *__restrict__ d, double *__restrict__ y) {
  const int64_t r = (int64_t(blockIdx.x) * kCta + threadIdx.x) >> 5;
  if (r >= N) return;
  gemv_row<false>(N, ld, M, d, y, r);
}

// ---------------------------------------------------------------------------
// Persistent coarse-tail kernel: the V-cycle below a level T (all levels small:
// split-k 4, not distributed) as ONE cooperative launch.  Each phase is the
// standalone kernel's task function over a grid-stride task loop; phases are
// separated by grid-wide barriers.  Same task functions and split factors as
// the standalone kernels, so results are bit-identical; vectors written by an
// earlier phase are read with L2-coherent loads.
// ---------------------------------------------------------------------------
enum { T_SWEEP0 = 0, T_SWEEP, T_RESID, T_RESTRICT, T_PROLONG, T_GEMV, T_COPY, T_ZERO };

struct TailOp {
  int type;
  int ks;   // split-k of A-passes (4 or 8, as in the standalone kernels)
  int f32;  // A values stored fp32 (mixed precision)
  int wpe;  // transfers: weights per entry
  Sell A;   // operator: A (sweeps / residual), R or P
  const double *x;
  const double *b;
  const double *dinv;  // D^-1 (sweeps) or the dense coarse inverse (GEMV)
  double *out;
  double alpha;
  int64_t n;   // GEMV rows / COPY, ZERO length
  int64_t ld;  // GEMV leading dimension
};

template <int BS, int OP, int KS>
__device__ __forceinline__ void tail_apply_ks(const TailOp &op) {
  constexpr int per = kWarpsPerCta / KS;  // slices per CTA-task
  const int64_t nt = (op.A.n_slices + per - 1) / per;
  for (int64_t t = blockIdx.x; t < nt; t += gridDim.x) {
    if (op.f32)
      sell_apply_task<BS, OP, false, false, KS, true, true>(op.A, t, op.x, nullptr, 0, op.b, op.dinv, op.out,
                                                             op.alpha, 0.0);
    else
      sell_apply_task<BS, OP, false, false, KS, false, true>(op.A, t, op.x, nullptr, 0, op.b, op.dinv, op.out,
                                                              op.alpha, 0.0);
  }
}

template <int BS, int OP>
__device__ __forceinline__ void tail_apply(const TailOp &op) {
  if (op.ks == 8) tail_apply_ks<BS, OP, 8>(op);
  else tail_apply_ks<BS, OP, 4>(op);
}

template <int BS, bool ACC, int KS, bool STREAM>
__device__ __forceinline__ void tail_transfer(const TailOp &op) {
  const int per = kWarpsPerCta / KS;
  const int64_t nt = (op.A.n_slices + per - 1) / per;
  for (int64_t t = blockIdx.x; t < nt; t += gridDim.x) {
    if (op.wpe == 1 || BS == 1)
      transfer_task<BS, 1, ACC, STREAM, false, KS, true>(op.A, t, op.x, nullptr, 0, op.out);
    else
      transfer_task<BS, BS, ACC, STREAM, false, KS, true>(op.A, t, op.x, nullptr, 0, op.out);
  }
}

// CLUSTER: the whole grid is one thread-block cluster (<= 16 CTAs) and phases
// are separated by the hardware cluster barrier instead of a grid barrier.
template <int BS, bool CLUSTER>
__global__ void __launch_bounds__(kCta) k_tail(const TailOp *__restrict__ ops, int nops) {
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nth = int64_t(gridDim.x) * blockDim.x;
  for (int p = 0; p < nops; ++p) {
    const TailOp op = ops[p];
    switch (op.type) {
      case T_SWEEP0: {
        const int64_t nt = (op.A.n_slices + kWarpsPerCta - 1) / kWarpsPerCta;
        for (int64_t t = blockIdx.x; t < nt; t += gridDim.x)
          sweep0_task<BS, true>(op.A.n_slices, t, op.A.perm, op.dinv, op.b, op.out, op.alpha);
        break;
      }
      case T_SWEEP: tail_apply<BS, OP_SWEEP>(op); break;
      case T_RESID: tail_apply<BS, OP_RESID>(op); break;
      case T_RESTRICT:  // split factor of the standalone restriction (bit-identical sums)
        if (op.ks == 1) tail_transfer<BS, false, 1, true>(op);
        else if (op.ks == 2) tail_transfer<BS, false, 2, true>(op);
        else tail_transfer<BS, false, 4, true>(op);
        break;
      case T_PROLONG: tail_transfer<BS, true, 1, false>(op); break;
      case T_GEMV:  // the split kernel's four column chunks, summed in the same order
        for (int64_t r = tid >> 5; r < op.n; r += nth >> 5) {
          if (op.ks == 4) {
            double s4 = gemv_chunk<4, true>(op.n, op.ld, op.dinv, op.b, r, 0);
            for (int q = 1; q < 4; ++q) s4 += gemv_chunk<4, true>(op.n, op.ld, op.dinv, op.b, r, q);
            if ((threadIdx.x & 31) == 0) op.out[r] = s4;
          } else {
            gemv_row<true>(op.n, op.ld, op.dinv, op.b, op.out, r);
          }
        }
        break;
      case T_COPY:
        for (int64_t i = tid; i < op.n; i += nth) op.out[i] = __ldcg(op.x + i);
        break;
      default:
        for (int64_t i = tid; i < op.n; i += nth) op.out[i] = 0.0;
        break;
    }
    if constexpr (CLUSTER) cooperative_groups::this_cluster().sync();
    else cooperative_groups::this_grid().sync();
  }
}

// ---------------------------------------------------------------------------
// Reductions: deterministic single-pass grid reduction.  Each CTA reduces its
// grid-stride share (warp shuffles + shared memory) to part[blockIdx.x]; the
// last CTA to arrive (ticket) sums the partials in CTA order and writes the
// result, so the value depends only on n and the fixed grid size.
// ---------------------------------------------------------------------------
__device__ __forceinline__ double block_sum(double v, double *sh) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  if (w == 0) {
    t = lane < int(blockDim.x >> 5) ? sh[lane] : 0.0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
  }
  return t;  // valid in thread 0
}

// finish: last CTA sums part[0..gridDim) in order; result -> *res (sqrt if
// SQRT); also copies to *res2 if non-null.
template <bool SQRT>
__device__ __forceinline__ void grid_finish(double blocksum, double *part, unsigned *ticket, double *res,
                                            double *res2, double *sh) {
  __shared__ bool last;
  if (threadIdx.x == 0) {
    part[blockIdx.x] = blocksum;
    __threadfence();
    last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double v = 0.0;
  for (int i = threadIdx.x; i < int(gridDim.x); i += blockDim.x) v += __ldcg(part + i);
  // ordered: each thread's strided sum, then a fixed tree
  v = block_sum(v, sh);
  if (threadIdx.x == 0) {
    const double r = SQRT ? sqrt(v) : v;
    *res = r;
    if (res2) *res2 = r;
    *ticket = 0u;
  }
}

// MODE 0: res = (a, b).  MODE 1 (MGS step): a -= (*h) * c; res = (a_new, b)
// (b == nullptr => res = ||a_new||_2 with SQRT).  VEC: all pointers 16-byte
// aligned -> double2 loads/stores over the even part, the odd tail in thread 0.
// REV (VEC only): the grid sweeps the vectors from the high end down, so a
// pass that follows a forward pass (or vice versa) starts on the lines the
// previous pass touched last, which are still in L2 (126 MB vs 83 MB vectors
// on C3): the MGS passes of one Arnoldi step alternate direction.
template <int MODE, bool SQRT, bool VEC, bool REV = false>
__global__ void __launch_bounds__(kRedThreads) k_reduce(int64_t n, double *__restrict__ a, const double *__restrict__ b,
                                                        const double *__restrict__ c, const double *__restrict__ h,
                                                        double *part, unsigned *ticket, double *res, double *res2) {
  __shared__ double sh[32];
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  double s = 0.0, s2 = 0.0;
  const double hv = MODE == 1 ? *h : 0.0;
  int64_t i0 = 0;
  if constexpr (VEC) {
    constexpr int U = 4;  // independent 16-byte loads in flight per thread and vector
    const int64_t n2 = n / 2;
    double2 *a2 = reinterpret_cast<double2 *>(a);
    const double2 *b2 = reinterpret_cast<const double2 *>(b);
    const double2 *c2 = reinterpret_cast<const double2 *>(c);
    if constexpr (REV) {  // index j <-> n2 - 1 - j (pointers to the last element, negative strides)
      a2 += n2 - 1;
      b2 += n2 - 1;
      c2 += n2 - 1;
    }
    constexpr int64_t D = REV ? -1 : 1;
    int64_t i = tid;
    for (; i + (U - 1) * stride < n2; i += U * stride) {
      double2 x[U], y[U], v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t j = D * (i + u * stride);
        if constexpr (MODE == 0) {
          x[u] = __ldg(a2 + j);
        } else {
          x[u] = a2[j];
          v[u] = __ldg(c2 + j);
        }
        if (b) y[u] = __ldg(b2 + j);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if constexpr (MODE == 1) {
          x[u].x = fma(-hv, v[u].x, x[u].x);
          x[u].y = fma(-hv, v[u].y, x[u].y);
          a2[D * (i + u * stride)] = x[u];
        }
        const double2 yy = b ? y[u] : x[u];
        s = fma(x[u].x, yy.x, s);
        s2 = fma(x[u].y, yy.y, s2);
      }
    }
    for (; i < n2; i += stride) {
      const int64_t j = D * i;
      double2 x = MODE == 0 ? __ldg(a2 + j) : a2[j];
      if constexpr (MODE == 1) {
        const double2 v = __ldg(c2 + j);
        x.x = fma(-hv, v.x, x.x);
        x.y = fma(-hv, v.y, x.y);
        a2[j] = x;
      }
      const double2 yy = b ? __ldg(b2 + j) : x;
      s = fma(x.x, yy.x, s);
      s2 = fma(x.y, yy.y, s2);
    }
    i0 = 2 * n2;
    s += s2;
    if (tid != 0) i0 = n;  // the odd tail element (if any) goes to thread 0
  }
  for (int64_t i = i0 + (VEC ? 0 : tid); i < n; i += (VEC ? 1 : stride)) {
    if constexpr (MODE == 0) {
      s = fma(__ldg(a + i), __ldg(b + i), s);
    } else {
      const double v = fma(-hv, __ldg(c + i), a[i]);
      a[i] = v;
      s = fma(v, b ? __ldg(b + i) : v, s);
    }
  }
  const double bsum = block_sum(s, sh);
  grid_finish<SQRT>(bsum, part, ticket, res, res2, sh);
}

// ---------------------------------------------------------------------------
// GMRES helpers (right preconditioning, MGS, Givens, reading O8).
// H column-major with leading dimension m+1.
// ---------------------------------------------------------------------------
struct GmresDev {
  double *H;      // (m+1) x m
  double *cs, *sn, *g, *y;
  double *hn;     // [m] ||w|| before normalisation
  double *beta;   // current restart residual norm
  double *beta0;  // initial residual norm
  double *out;    // [4]: est = |g_{j+1}|/beta0, flag, ...
  int m;
  // delayed-CGS2 orthogonalisation (MG_GMRES_DCGS2, reading Z29)
  double *Hraw;   // (m+1) x m unrotated Hessenberg columns (final, last one tentative)
  double *R;      // m x m upper triangular, U = Q R
  double *gpre;   // [m+1] g_j before rotation j
  double *dots;   // [2m+2] a, bb, nu, mu of the step's reduction
  double *coef;   // [2m+2] a, c, 1/beta
  double *nu1;    // ||u_{j+1}||^2
  double *dead;   // 1: breakdown found at the start of a step (u_j in span Q)
  double *y2;     // [m] R^{-1} y
};

// v0 = r / beta; g = (beta, 0, ...)
__global__ void k_gmres_start(GmresDev st) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    for (int i = 0; i <= st.m; ++i) st.g[i] = 0.0;
    st.g[0] = *st.beta;
  }
}

// out = in * (1 / *den) (in-place allowed; a reciprocal multiply: fp64
// division is a long instruction sequence and halves this kernel's bandwidth);
// 16-byte aligned pointers, odd tail in thread 0
__global__ void k_scale_div(int64_t n, const double *in, const double *den, double *out) {
  const double d = *den;
  if (d == 0.0) return;
  const double r = 1.0 / d;
  const int64_t n2 = n / 2;
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  for (int64_t i = tid; i < n2; i += int64_t(gridDim.x) * blockDim.x) {
    double2 v = reinterpret_cast<const double2 *>(in)[i];
    v.x *= r;
    v.y *= r;
    reinterpret_cast<double2 *>(out)[i] = v;
  }
  if (tid == 0 && (n & 1)) out[n - 1] = in[n - 1] * r;
}

// Apply the previous rotations to column j, form the new one, update g and
// the convergence flag (|g_{j+1}| <= rtol * beta0, or breakdown h_{j+1,j} = 0).
// Device-side loop control (mg_solve's conditional-graph restart cycle): with
// `cond`, the step also sets the switch handle to j + 1 (the next Arnoldi step)
// and the while handle to "continue" = no stop yet and j + 1 < mm, so one graph
// launch runs the whole cycle without a host round trip (P:346-347 did the
// Givens part on the CPU).  out[3] = k = j + 1, the steps done so far.
__global__ void k_givens(GmresDev st, int j, double rtol, int mm, cudaGraphConditionalHandle hw,
                         cudaGraphConditionalHandle hs, int cond) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int ld = st.m + 1;
  double *h = st.H + int64_t(j) * ld;
  const double hn = h[j + 1];
  st.hn[j] = hn;
  for (int i = 0; i < j; ++i) {
    const double t = st.cs[i] * h[i] + st.sn[i] * h[i + 1];
    h[i + 1] = -st.sn[i] * h[i] + st.cs[i] * h[i + 1];
    h[i] = t;
  }
  const double rho = hypot(h[j], h[j + 1]);
  st.cs[j] = h[j] / rho;
  st.sn[j] = h[j + 1] / rho;
  h[j] = rho;
  h[j + 1] = 0.0;
  st.g[j + 1] = -st.sn[j] * st.g[j];
  st.g[j] = st.cs[j] * st.g[j];
  const double b0 = *st.beta0;
  st.out[0] = fabs(st.g[j + 1]) / b0;
  const bool stop = fabs(st.g[j + 1]) <= rtol * b0 || hn == 0.0;
  st.out[1] = stop ? 1.0 : 0.0;
  st.out[2] = hn;
  st.out[3] = double(j + 1);
  if (cond) {
    cudaGraphSetConditional(hs, unsigned(j + 1));
    cudaGraphSetConditional(hw, (!stop && j + 1 < mm) ? 1u : 0u);
  }
}

// Back substitution H(0:k,0:k) y = g(0:k).
__global__ void k_backsolve(GmresDev st, int k, const double *kdev) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (kdev) k = int(*kdev);  // steps done, set on the device (conditional-graph cycle)
  const int ld = st.m + 1;
  for (int i = k - 1; i >= 0; --i) {
    double s = 0.0;
    for (int l = i + 1; l < k; ++l) s += st.H[int64_t(l) * ld + i] * st.y[l];
    st.y[i] = (st.g[i] - s) / st.H[int64_t(i) * ld + i];
  }
}

// x += sum_{t<k} y_t Z_t  (Z: k vectors of length n at stride ldz).
__global__ void k_update_x(int64_t n, int k, const double *__restrict__ y, const double *__restrict__ Z, int64_t ldz,
                           double *__restrict__ x, const double *kdev = nullptr) {
  __shared__ double ys[64];
  if (kdev) k = int(*kdev);
  if (threadIdx.x < k) ys[threadIdx.x] = y[threadIdx.x];
  __syncthreads();
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    double v = x[i];
    for (int t = 0; t < k; ++t) v = fma(ys[t], __ldg(Z + int64_t(t) * ldz + i), v);
    x[i] = v;
  }
}

// ---------------------------------------------------------------------------
// GMRES with delayed classical Gram-Schmidt reorthogonalisation (DCGS2,
// MG_GMRES_DCGS2; reading Z29, oracle.gmres_dcgs2): per Arnoldi step ONE
// multi-dot pass (k_dcgs_dots: Q_{j-1}^T u_j, Q_{j-1}^T w^, u_j^T u_j,
// u_j^T w^) and ONE update pass (k_dcgs_update: q_j and u_{j+1}, fused
// ||u_{j+1}||^2) -- 2j + 6 vector passes and 2 all-reduces per step, against
// 4j + 7 passes and j + 2 all-reduces of the paper's MGS.  Q slots at
// stride ldq; slot j holds u_j until the update turns it into q_j; w^ = A z_j
// is written into slot j + 1, where the update leaves u_{j+1}.
// ---------------------------------------------------------------------------
// Block + grid reduction of NO values per thread (deterministic: warp shuffles,
// warps in order, CTAs in order by the last CTA).
// Block + grid reduction of NO per-thread values to nout outputs, value o going
// to output map(o) (< 0: dropped).  Deterministic: warp shuffles, warps in
// order, CTAs in order by the last CTA to arrive.
template <int NO, class Map>
__device__ __forceinline__ void grid_reduce_many(const double (&v)[NO], int nout, Map map, double *part,
                                                 unsigned *ticket, double *out) {
  __shared__ double sh[kRedThreads / 32][NO];
  __shared__ bool last;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 0; o < NO; ++o) {
    const int d = map(o);
    if (d < 0) continue;
    double t = v[o];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) t += __shfl_xor_sync(0xffffffffu, t, off);
    if (lane == 0) sh[w][d] = t;
  }
  __syncthreads();
  for (int o = threadIdx.x; o < nout; o += blockDim.x) {
    double t = 0.0;
    for (int ww = 0; ww < int(blockDim.x >> 5); ++ww) t += sh[ww][o];
    part[int64_t(blockIdx.x) * nout + o] = t;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int o = threadIdx.x; o < nout; o += blockDim.x) {
    double t = 0.0;
    for (int b = 0; b < int(gridDim.x); ++b) t += __ldcg(part + int64_t(b) * nout + o);
    out[o] = t;
  }
  if (threadIdx.x == 0) *ticket = 0u;
}

// out = [a (j) | bb (j) | nu | mu]; JB >= j (template bucket: accumulators in registers)
template <int JB>
__global__ void __launch_bounds__(kRedThreads) k_dcgs_dots(int64_t n, int j, const double *__restrict__ Q,
                                                           int64_t ldq, double *part, unsigned *ticket,
                                                           double *out) {
  double acc[2 * JB + 2];
#pragma unroll
  for (int o = 0; o < 2 * JB + 2; ++o) acc[o] = 0.0;
  const double *u = Q + int64_t(j) * ldq, *wh = Q + int64_t(j + 1) * ldq;
  const int64_t n2 = n / 2;
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  auto body = [&](double2 uu, double2 ww, auto ldq_i) {
    double2 q[JB];
#pragma unroll
    for (int i = 0; i < JB; ++i)
      if (i < j) q[i] = ldq_i(i);
#pragma unroll
    for (int i = 0; i < JB; ++i)
      if (i < j) {
        acc[i] = fma(q[i].y, uu.y, fma(q[i].x, uu.x, acc[i]));
        acc[JB + i] = fma(q[i].y, ww.y, fma(q[i].x, ww.x, acc[JB + i]));
      }
    acc[2 * JB] = fma(uu.y, uu.y, fma(uu.x, uu.x, acc[2 * JB]));
    acc[2 * JB + 1] = fma(uu.y, ww.y, fma(uu.x, ww.x, acc[2 * JB + 1]));
  };
  for (int64_t e = tid; e < n2; e += stride)
    body(__ldcs(reinterpret_cast<const double2 *>(u) + e), __ldcs(reinterpret_cast<const double2 *>(wh) + e),
         [&](int i) { return __ldg(reinterpret_cast<const double2 *>(Q + int64_t(i) * ldq) + e); });
  if ((n & 1) && tid == 0)  // the odd last element (zero second half)
    body(make_double2(u[n - 1], 0.0), make_double2(wh[n - 1], 0.0),
         [&](int i) { return make_double2(Q[int64_t(i) * ldq + n - 1], 0.0); });
  auto map = [j](int o) {
    if (o < JB) return o < j ? o : -1;
    if (o < 2 * JB) return o - JB < j ? j + o - JB : -1;
    return 2 * j + (o - 2 * JB);
  };
  grid_reduce_many<2 * JB + 2>(acc, 2 * j + 2, map, part, ticket, out);
}

// --- warp-split DCGS2 passes (default) -------------------------------------
// Warp w of a CTA owns the basis vectors i = w, w + 8, ... (< j): VPW = ceil(j/8)
// of them, so a thread holds 2 VPW accumulators and (2 + VPW) x U 16-byte loads
// in flight instead of 2j + 2 accumulators (the per-thread version needed 220
// registers at j = 16: one CTA per SM, 4.2-4.6 TB/s).  A CTA walks tiles of
// 32 x U double2; every warp of the CTA walks every tile of the CTA for its own
// vectors (u and w^ are re-read by the 8 warps from L1/L2, DRAM once).
constexpr int kDcgsU = 4;

// out = [a (j) | bb (j) | nu | mu]; the last warp also sums nu and mu
template <int VPW>
__global__ void __launch_bounds__(kRedThreads) k_dcgs_dots_ws(int64_t n, int j, const double *__restrict__ Q,
                                                              int64_t ldq, double *part, unsigned *ticket,
                                                              double *out) {
  constexpr int U = kDcgsU;
  __shared__ double sh[2 * 8 * VPW + 2];
  __shared__ bool last;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nout = 2 * j + 2;
  const double2 *u2 = reinterpret_cast<const double2 *>(Q + int64_t(j) * ldq);
  const double2 *w2 = reinterpret_cast<const double2 *>(Q + int64_t(j + 1) * ldq);
  const bool nm = w == kWarpsPerCta - 1;  // this warp also sums nu, mu
  double aa[VPW], ab[VPW], nu = 0.0, mu = 0.0;
#pragma unroll
  for (int k = 0; k < VPW; ++k) aa[k] = ab[k] = 0.0;
  const int64_t n2 = n / 2, ntiles = (n2 + 32 * U - 1) / (32 * U);
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t e0 = t * 32 * U + lane;
    double2 uu[U], ww[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int64_t e = e0 + 32 * q;
      uu[q] = e < n2 ? __ldg(u2 + e) : make_double2(0.0, 0.0);
      ww[q] = e < n2 ? __ldg(w2 + e) : make_double2(0.0, 0.0);
    }
    double2 qv[VPW][U];
#pragma unroll
    for (int k = 0; k < VPW; ++k) {
      const int i = w + 8 * k;
      if (i < j) {
        const double2 *q2 = reinterpret_cast<const double2 *>(Q + int64_t(i) * ldq);
#pragma unroll
        for (int q = 0; q < U; ++q) {
          const int64_t e = e0 + 32 * q;
          qv[k][q] = e < n2 ? __ldg(q2 + e) : make_double2(0.0, 0.0);
        }
      }
    }
#pragma unroll
    for (int k = 0; k < VPW; ++k)
      if (w + 8 * k < j)
#pragma unroll
        for (int q = 0; q < U; ++q) {
          aa[k] = fma(qv[k][q].y, uu[q].y, fma(qv[k][q].x, uu[q].x, aa[k]));
          ab[k] = fma(qv[k][q].y, ww[q].y, fma(qv[k][q].x, ww[q].x, ab[k]));
        }
    if (nm)
#pragma unroll
      for (int q = 0; q < U; ++q) {
        nu = fma(uu[q].y, uu[q].y, fma(uu[q].x, uu[q].x, nu));
        mu = fma(uu[q].y, ww[q].y, fma(uu[q].x, ww[q].x, mu));
      }
  }
  if ((n & 1) && blockIdx.x == 0 && nm && lane == 0) {  // the odd last element
    const double ul = Q[int64_t(j) * ldq + n - 1], wl = Q[int64_t(j + 1) * ldq + n - 1];
    nu = fma(ul, ul, nu);
    mu = fma(ul, wl, mu);
  }
  if ((n & 1) && blockIdx.x == 0 && lane == 0) {
    const double ul = Q[int64_t(j) * ldq + n - 1], wl = Q[int64_t(j + 1) * ldq + n - 1];
#pragma unroll
    for (int k = 0; k < VPW; ++k) {
      const int i = w + 8 * k;
      if (i < j) {
        const double ql = Q[int64_t(i) * ldq + n - 1];
        aa[k] = fma(ql, ul, aa[k]);
        ab[k] = fma(ql, wl, ab[k]);
      }
    }
  }
  // warp sums -> sh[output] (each output has one owner warp) -> CTA partials -> last CTA
#pragma unroll
  for (int k = 0; k < VPW; ++k) {
    double ta = aa[k], tb = ab[k];
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      ta += __shfl_xor_sync(0xffffffffu, ta, off);
      tb += __shfl_xor_sync(0xffffffffu, tb, off);
    }
    const int i = w + 8 * k;
    if (lane == 0 && i < j) sh[i] = ta, sh[j + i] = tb;
  }
  if (nm) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      nu += __shfl_xor_sync(0xffffffffu, nu, off);
      mu += __shfl_xor_sync(0xffffffffu, mu, off);
    }
    if (lane == 0) sh[2 * j] = nu, sh[2 * j + 1] = mu;
  }
  __syncthreads();
  for (int o = threadIdx.x; o < nout; o += blockDim.x) part[int64_t(blockIdx.x) * nout + o] = sh[o];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = (atomicAdd(ticket, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (int o = threadIdx.x; o < nout; o += blockDim.x) {
    double t = 0.0;
    for (int b = 0; b < int(gridDim.x); ++b) t += __ldcg(part + int64_t(b) * nout + o);
    out[o] = t;
  }
  if (threadIdx.x == 0) *ticket = 0u;
}

// q_j = (u_j - Q_{j-1} a) / beta ; u_{j+1} = w^/beta - Q_{j-1} c_{0:j} - c_j q_j ;
// nu1 = ||u_{j+1}||^2.  Per tile each warp forms the partial sums of its own
// vectors, the CTA adds the 8 warps' partials in warp order through shared memory.
template <int VPW>
__global__ void __launch_bounds__(kRedThreads) k_dcgs_update_ws(int64_t n, int j, double *__restrict__ Q,
                                                                int64_t ldq, const double *__restrict__ coef,
                                                                const double *dead, double *part, unsigned *ticket,
                                                                double *nu1) {
  constexpr int U = kDcgsU;
  constexpr int TE = 32 * U;  // double2 per tile
  __shared__ double2 pa[kWarpsPerCta][TE], pc[kWarpsPerCta][TE];
  __shared__ double cf[2 * 8 * VPW + 2];
  for (int i = threadIdx.x; i < 2 * j + 2; i += blockDim.x) cf[i] = coef[i];
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double s = 0.0;
  if (*dead == 0.0) {
    double2 *u2 = reinterpret_cast<double2 *>(Q + int64_t(j) * ldq);
    double2 *w2 = reinterpret_cast<double2 *>(Q + int64_t(j + 1) * ldq);
    const double ib = cf[2 * j + 1], cj = cf[2 * j];
    const int64_t n2 = n / 2, ntiles = (n2 + TE - 1) / TE;
    static_assert(TE <= kRedThreads, "one combining thread per tile element");
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int64_t e0 = t * TE;
      // the combining thread's u, w^ are loaded up front, with the basis loads
      const int64_t ec = e0 + threadIdx.x;
      const bool comb = threadIdx.x < TE && ec < n2;
      double2 uu = make_double2(0.0, 0.0), wv = make_double2(0.0, 0.0);
      if (comb) uu = u2[ec], wv = w2[ec];
      double2 sa[U], sc[U];
#pragma unroll
      for (int q = 0; q < U; ++q) sa[q] = sc[q] = make_double2(0.0, 0.0);
      double2 qv[VPW][U];
#pragma unroll
      for (int k = 0; k < VPW; ++k) {
        const int i = w + 8 * k;
        if (i < j) {
          const double2 *q2 = reinterpret_cast<const double2 *>(Q + int64_t(i) * ldq);
#pragma unroll
          for (int q = 0; q < U; ++q) {
            const int64_t e = e0 + lane + 32 * q;
            qv[k][q] = e < n2 ? __ldg(q2 + e) : make_double2(0.0, 0.0);
          }
        }
      }
#pragma unroll
      for (int k = 0; k < VPW; ++k) {
        const int i = w + 8 * k;
        if (i < j) {
          const double a = cf[i], c = cf[j + i];
#pragma unroll
          for (int q = 0; q < U; ++q) {
            sa[q].x = fma(a, qv[k][q].x, sa[q].x);
            sa[q].y = fma(a, qv[k][q].y, sa[q].y);
            sc[q].x = fma(c, qv[k][q].x, sc[q].x);
            sc[q].y = fma(c, qv[k][q].y, sc[q].y);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < U; ++q) pa[w][lane + 32 * q] = sa[q], pc[w][lane + 32 * q] = sc[q];
      __syncthreads();
      if (comb) {
        const int el = threadIdx.x;
        const int64_t e = ec;
        {
          double2 ta = pa[0][el], tc = pc[0][el];
#pragma unroll
          for (int ww = 1; ww < kWarpsPerCta; ++ww) {
            ta.x += pa[ww][el].x, ta.y += pa[ww][el].y;
            tc.x += pc[ww][el].x, tc.y += pc[ww][el].y;
          }
          double2 qj, un;
          qj.x = (uu.x - ta.x) * ib;
          qj.y = (uu.y - ta.y) * ib;
          un.x = fma(-cj, qj.x, fma(wv.x, ib, -tc.x));
          un.y = fma(-cj, qj.y, fma(wv.y, ib, -tc.y));
          u2[e] = qj;
          w2[e] = un;
          s = fma(un.y, un.y, fma(un.x, un.x, s));
        }
      }
      __syncthreads();
    }
    if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {  // the odd last element
      double ta = 0.0, tc = 0.0;
      for (int i = 0; i < j; ++i) {
        const double ql = Q[int64_t(i) * ldq + n - 1];
        ta = fma(cf[i], ql, ta);
        tc = fma(cf[j + i], ql, tc);
      }
      double *ul = Q + int64_t(j) * ldq + n - 1, *wl = Q + int64_t(j + 1) * ldq + n - 1;
      const double qj = (*ul - ta) * ib;
      const double un = fma(-cj, qj, fma(*wl, ib, -tc));
      *ul = qj;
      *wl = un;
      s = fma(un, un, s);
    }
  }
  const double v[1] = {s};
  grid_reduce_many<1>(v, 1, [](int o) { return o; }, part, ticket, nu1);
}

// --- bulk-copy (TMA engine) staging of vector tiles ------------------------
// cp.async.bulk moves a contiguous tile global -> shared without registers;
// completion is counted in bytes on an mbarrier.  The Krylov passes stream
// j + 2 vectors at once: staging their tiles through a ring of shared-memory
// stages keeps ~100-200 KB in flight per SM with 256 threads, where register
// staging (one 16-byte load per vector and thread) ran out of registers and
// warps (k_dcgs_*_reg: 220 registers, 8 warps per SM, 4.2-4.5 TB/s).
__device__ __forceinline__ unsigned smem_u32(const void *p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, uint64_t *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// generic-proxy reads of a stage are ordered before the async proxy refills it
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Ring of NST stages, each holding the tiles [e0, e0 + T) of NV strided vectors
// (base + v * ld, v < NV).  Tiles are dealt to CTAs round-robin (tile = b, b +
// grid, ...), so which CTA sums which elements is fixed by (n, T, grid).
struct TileRing {
  double *buf;     // [NST][NV][T]
  uint64_t *full;  // [NST]
  int nst, nv, T;
  const double *base;
  int64_t ld, n;
  __device__ double *stage(int s) const { return buf + int64_t(s) * nv * T; }
  // thread 0: arm stage s with the tile's bytes and issue the NV copies
  __device__ void issue(int64_t tile, int s) const {
    const int64_t e0 = tile * T;
    const int64_t len = n - e0 < T ? n - e0 : T;
    const unsigned bytes = unsigned((len * 8 + 15) & ~int64_t(15));  // may read <= 8 bytes past n (inside the slot)
    mbar_expect_tx(full + s, bytes * unsigned(nv));
    for (int v = 0; v < nv; ++v) bulk_g2s(stage(s) + int64_t(v) * T, base + v * ld + e0, bytes, full + s);
  }
};

// smem layout for the ring: nst * nv * T doubles, then nst mbarriers
__device__ __forceinline__ TileRing make_ring(unsigned char *sm, int nst, int nv, int T, const double *base,
                                              int64_t ld, int64_t n) {
  TileRing r;
  r.buf = reinterpret_cast<double *>(sm);
  r.full = reinterpret_cast<uint64_t *>(sm + size_t(nst) * nv * T * sizeof(double));
  r.nst = nst, r.nv = nv, r.T = T, r.base = base, r.ld = ld, r.n = n;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) mbar_init(r.full + s, 1);
    mbar_fence_init();
  }
  __syncthreads();
  return r;
}

// Runs body(stage_ptr, e0, len) over this CTA's tiles with NST tiles in flight.
template <class Body>
__device__ __forceinline__ void ring_stream(const TileRing &r, Body &&body) {
  const int64_t ntiles = (r.n + r.T - 1) / r.T;
  const int64_t grid = gridDim.x;
  if (threadIdx.x == 0)
    for (int s = 0; s < r.nst; ++s)
      if (blockIdx.x + s * grid < ntiles) r.issue(blockIdx.x + s * grid, s);
  int s = 0;
  unsigned phase = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += grid) {
    mbar_wait(r.full + s, phase);
    const int64_t e0 = tile * r.T;
    body(r.stage(s), e0, int(r.n - e0 < r.T ? r.n - e0 : r.T));
    __syncthreads();  // every thread is done with stage s
    if (threadIdx.x == 0 && tile + int64_t(r.nst) * grid < ntiles) {
      fence_proxy_async();
      r.issue(tile + int64_t(r.nst) * grid, s);
    }
    if (++s == r.nst) s = 0, phase ^= 1u;
  }
}

// k_dcgs_dots with the j + 2 vectors (slots 0..j+1 of Q) staged by bulk copies
template <int JB>
__global__ void __launch_bounds__(kRedThreads) k_dcgs_dots_tma(int64_t n, int j, const double *__restrict__ Q,
                                                               int64_t ldq, int nst, int T, double *part,
                                                               unsigned *ticket, double *out) {
  extern __shared__ __align__(128) unsigned char sm_ring[];
  const TileRing ring = make_ring(sm_ring, nst, j + 2, T, Q, ldq, n);
  double acc[2 * JB + 2];
#pragma unroll
  for (int o = 0; o < 2 * JB + 2; ++o) acc[o] = 0.0;
  ring_stream(ring, [&](const double *st, int64_t, int len) {
    const double *u = st + int64_t(j) * T, *wh = st + int64_t(j + 1) * T;
    for (int e = threadIdx.x; e < len; e += blockDim.x) {
      const double uu = u[e], ww = wh[e];
#pragma unroll
      for (int i = 0; i < JB; ++i)
        if (i < j) {
          const double q = st[int64_t(i) * T + e];
          acc[i] = fma(q, uu, acc[i]);
          acc[JB + i] = fma(q, ww, acc[JB + i]);
        }
      acc[2 * JB] = fma(uu, uu, acc[2 * JB]);
      acc[2 * JB + 1] = fma(uu, ww, acc[2 * JB + 1]);
    }
  });
  auto map = [j](int o) {
    if (o < JB) return o < j ? o : -1;
    if (o < 2 * JB) return o - JB < j ? j + o - JB : -1;
    return 2 * j + (o - 2 * JB);
  };
  grid_reduce_many<2 * JB + 2>(acc, 2 * j + 2, map, part, ticket, out);
}

// k_dcgs_update with the j + 2 vectors staged by bulk copies; q_j and u_{j+1}
// are stored straight to global memory (coalesced)
template <int JB>
__global__ void __launch_bounds__(kRedThreads) k_dcgs_update_tma(int64_t n, int j, double *__restrict__ Q,
                                                                 int64_t ldq, int nst, int T,
                                                                 const double *__restrict__ coef,
                                                                 const double *dead, double *part, unsigned *ticket,
                                                                 double *nu1) {
  extern __shared__ __align__(128) unsigned char sm_ring[];
  __shared__ double cf[2 * JB + 2];
  for (int i = threadIdx.x; i < 2 * j + 2; i += blockDim.x) cf[i] = coef[i];
  const TileRing ring = make_ring(sm_ring, nst, j + 2, T, Q, ldq, n);  // (its __syncthreads covers cf)
  double s = 0.0;
  if (*dead == 0.0) {
    const double ib = cf[2 * j + 1], cj = cf[2 * j];
    double *u = Q + int64_t(j) * ldq, *wh = Q + int64_t(j + 1) * ldq;
    ring_stream(ring, [&](const double *st, int64_t e0, int len) {
      const double *us = st + int64_t(j) * T, *ws = st + int64_t(j + 1) * T;
      for (int e = threadIdx.x; e < len; e += blockDim.x) {
        double qj = us[e], un = ws[e] * ib;
#pragma unroll
        for (int i = 0; i < JB; ++i)
          if (i < j) qj = fma(-cf[i], st[int64_t(i) * T + e], qj);
        qj *= ib;
#pragma unroll
        for (int i = 0; i < JB; ++i)
          if (i < j) un = fma(-cf[j + i], st[int64_t(i) * T + e], un);
        un = fma(-cj, qj, un);
        u[e0 + e] = qj;
        wh[e0 + e] = un;
        s = fma(un, un, s);
      }
    });
  }
  const double v[1] = {s};
  grid_reduce_many<1>(v, 1, [](int o) { return o; }, part, ticket, nu1);
}

// rotations 0..jj-1 applied to raw column jj, rotation jj formed, rotated column
// stored in H, g updated from gpre[jj]
__device__ __forceinline__ void dcgs_rotate(GmresDev &st, int jj) {
  const int ld = st.m + 1;
  const double *raw = st.Hraw + int64_t(jj) * ld;
  double *h = st.H + int64_t(jj) * ld;
  for (int i = 0; i <= jj + 1; ++i) h[i] = raw[i];
  for (int i = 0; i < jj; ++i) {
    const double t = st.cs[i] * h[i] + st.sn[i] * h[i + 1];
    h[i + 1] = -st.sn[i] * h[i] + st.cs[i] * h[i + 1];
    h[i] = t;
  }
  const double rho = hypot(h[jj], h[jj + 1]);
  st.cs[jj] = h[jj] / rho;
  st.sn[jj] = h[jj + 1] / rho;
  h[jj] = rho;
  h[jj + 1] = 0.0;
  st.g[jj + 1] = -st.sn[jj] * st.gpre[jj];
  st.g[jj] = st.cs[jj] * st.gpre[jj];
}

__global__ void k_dcgs_start(GmresDev st) {
  for (int i = threadIdx.x; i < (st.m + 1) * st.m; i += blockDim.x) st.Hraw[i] = 0.0;
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    for (int i = 0; i <= st.m; ++i) st.g[i] = st.gpre[i] = 0.0;
    *st.dead = 0.0;
  }
}

// After the step's reduction: beta, column j of R, column j-1 made final (its
// rotation redone), the coefficients of the update pass.  A breakdown (u_j in
// span Q_{j-1}) ends the cycle with k = j steps.
__global__ void k_dcgs_coef(GmresDev st, int j, int mm, cudaGraphConditionalHandle hw, int cond) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  const int ld = st.m + 1;
  const double *a = st.dots, *bb = st.dots + j;
  const double nu = st.dots[2 * j], mu = st.dots[2 * j + 1];
  double aa = 0.0, ab = 0.0;
  for (int i = 0; i < j; ++i) aa += a[i] * a[i], ab += a[i] * bb[i];
  const double beta = sqrt(fmax(j ? nu - aa : nu, 0.0));
  double *Rc = st.R + int64_t(j) * st.m;
  for (int i = 0; i < j; ++i) Rc[i] = a[i];
  Rc[j] = beta;
  if (j == 0) {
    st.g[0] = beta;
  } else {
    double *raw = st.Hraw + int64_t(j - 1) * ld;
    for (int i = 0; i < j; ++i) raw[i] += a[i];
    raw[j] = beta;
    dcgs_rotate(st, j - 1);
  }
  double *cf = st.coef;
  if (!(beta > 0.0) || !isfinite(beta)) {  // breakdown: the cycle ends after j steps
    *st.dead = 1.0;
    st.out[0] = j ? fabs(st.g[j]) / *st.beta0 : 0.0;
    st.out[1] = 1.0;
    st.out[2] = 0.0;
    st.out[3] = double(j);
    st.out[4] = double(j + 1);
    for (int i = 0; i < 2 * j + 2; ++i) cf[i] = 0.0;
    if (cond) cudaGraphSetConditional(hw, 0u);
    return;
  }
  const double ib = 1.0 / beta;
  double *sraw = st.Hraw + int64_t(j) * ld;
  for (int i = 0; i <= j; ++i) {
    double t = 0.0;  // t = Hbar_{j-1} a
    for (int l = 0; l < j; ++l) t += st.Hraw[int64_t(l) * ld + i] * a[l];
    const double s = i < j ? (bb[i] - t) / beta : ((mu - ab) / beta - t) / beta;
    sraw[i] = s;
    cf[j + i] = t / beta + s;
  }
  for (int i = 0; i < j; ++i) cf[i] = a[i];
  cf[2 * j + 1] = ib;
}

// q_j = (u_j - Q_{j-1} a) / beta ; u_{j+1} = w^/beta - Q_{j-1} c_{0:j} - c_j q_j ;
// nu1 = ||u_{j+1}||^2.  coef = [a (j) | c (j+1) | 1/beta].
template <int JB>
__global__ void __launch_bounds__(kRedThreads) k_dcgs_update(int64_t n, int j, double *__restrict__ Q, int64_t ldq,
                                                             const double *__restrict__ coef, const double *dead,
                                                             double *part, unsigned *ticket, double *nu1) {
  __shared__ double cf[2 * JB + 2];
  for (int i = threadIdx.x; i < 2 * j + 2; i += blockDim.x) cf[i] = coef[i];
  __syncthreads();
  double s = 0.0;
  if (*dead == 0.0) {
    double *u = Q + int64_t(j) * ldq, *wh = Q + int64_t(j + 1) * ldq;
    const double ib = cf[2 * j + 1], cj = cf[2 * j];
    const int64_t n2 = n / 2;
    const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t stride = int64_t(gridDim.x) * blockDim.x;
    auto body = [&](double2 uu, double2 ww, auto ldq_i) {
      double2 q[JB];
#pragma unroll
      for (int i = 0; i < JB; ++i)
        if (i < j) q[i] = ldq_i(i);
      double2 qj = uu, un = make_double2(ww.x * ib, ww.y * ib);
#pragma unroll
      for (int i = 0; i < JB; ++i)
        if (i < j) {
          qj.x = fma(-cf[i], q[i].x, qj.x);
          qj.y = fma(-cf[i], q[i].y, qj.y);
        }
      qj.x *= ib;
      qj.y *= ib;
#pragma unroll
      for (int i = 0; i < JB; ++i)
        if (i < j) {
          un.x = fma(-cf[j + i], q[i].x, un.x);
          un.y = fma(-cf[j + i], q[i].y, un.y);
        }
      un.x = fma(-cj, qj.x, un.x);
      un.y = fma(-cj, qj.y, un.y);
      return make_double4(qj.x, qj.y, un.x, un.y);
    };
    for (int64_t e = tid; e < n2; e += stride) {
      const double4 r = body(reinterpret_cast<const double2 *>(u)[e], reinterpret_cast<const double2 *>(wh)[e],
                             [&](int i) { return __ldg(reinterpret_cast<const double2 *>(Q + int64_t(i) * ldq) + e); });
      reinterpret_cast<double2 *>(u)[e] = make_double2(r.x, r.y);
      reinterpret_cast<double2 *>(wh)[e] = make_double2(r.z, r.w);
      s = fma(r.w, r.w, fma(r.z, r.z, s));
    }
    if ((n & 1) && tid == 0) {  // the odd last element
      const double4 r = body(make_double2(u[n - 1], 0.0), make_double2(wh[n - 1], 0.0),
                             [&](int i) { return make_double2(Q[int64_t(i) * ldq + n - 1], 0.0); });
      u[n - 1] = r.x;
      wh[n - 1] = r.z;
      s = fma(r.z, r.z, s);
    }
  }
  const double v[1] = {s};
  grid_reduce_many<1>(v, 1, [](int o) { return o; }, part, ticket, nu1);
}

// Tentative column j = [s_j ; ||u_{j+1}||] -> rotation j, estimate |g_{j+1}|,
// loop control as k_givens (stop on the estimate or on ||u_{j+1}|| = 0).
__global__ void k_dcgs_givens(GmresDev st, int j, double rtol, int mm, cudaGraphConditionalHandle hw,
                              cudaGraphConditionalHandle hs, int cond) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (*st.dead != 0.0) return;  // k_dcgs_coef ended the cycle
  const int ld = st.m + 1;
  const double hn = sqrt(*st.nu1);
  st.Hraw[int64_t(j) * ld + j + 1] = hn;
  st.hn[j] = hn;
  st.gpre[j] = st.g[j];
  dcgs_rotate(st, j);
  const double b0 = *st.beta0;
  st.out[0] = fabs(st.g[j + 1]) / b0;
  const bool stop = fabs(st.g[j + 1]) <= rtol * b0 || hn == 0.0;
  st.out[1] = stop ? 1.0 : 0.0;
  st.out[2] = hn;
  st.out[3] = double(j + 1);
  st.out[4] = double(j + 1);
  if (cond) {
    cudaGraphSetConditional(hs, unsigned(j + 1));
    cudaGraphSetConditional(hw, (!stop && j + 1 < mm) ? 1u : 0u);
  }
}

// H(0:k,0:k) y = g(0:k), then R y2 = y (z_j = B u_j and U = Q R)
__global__ void k_dcgs_backsolve(GmresDev st, int k, const double *kdev) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  if (kdev) k = int(*kdev);
  const int ld = st.m + 1;
  for (int i = k - 1; i >= 0; --i) {
    double s = 0.0;
    for (int l = i + 1; l < k; ++l) s += st.H[int64_t(l) * ld + i] * st.y[l];
    st.y[i] = (st.g[i] - s) / st.H[int64_t(i) * ld + i];
  }
  for (int i = k - 1; i >= 0; --i) {
    double s = 0.0;
    for (int l = i + 1; l < k; ++l) s += st.R[int64_t(l) * st.m + i] * st.y2[l];
    st.y2[i] = (st.y[i] - s) / st.R[int64_t(i) * st.m + i];
  }
}

// *flag = 1 if any x[i] != 0 (the caller zeroes it first).  Used to take the
// initial residual of a zero guess as b itself: b - A*0 == b exactly for the
// finite operators mg_set_matrix accepts (every product a*0 is +-0, the row
// sums are +0, b - (+0) = b), so the A-pass is skipped, not approximated.
__global__ void k_nonzero_flag(int64_t n, const double *__restrict__ x, int vec, double *flag) {
  const int64_t tid = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  bool nz = false;
  if (vec) {
    const int64_t n2 = n / 2;
    for (int64_t i = tid; i < n2; i += stride) {
      const double2 v = __ldg(reinterpret_cast<const double2 *>(x) + i);
      nz |= (v.x != 0.0) | (v.y != 0.0);
    }
    if (tid == 0 && (n & 1)) nz |= x[n - 1] != 0.0;
  } else {
    for (int64_t i = tid; i < n; i += stride) nz |= __ldg(x + i) != 0.0;
  }
  if (__any_sync(0xffffffffu, nz) && (threadIdx.x & 31) == 0) *flag = 1.0;
}

// Halo pack: out[i] = v[idx[i]] (bs values per item).
template <int BS>
__global__ void k_pack(int64_t n, const int32_t *__restrict__ idx, const double *__restrict__ v,
                       double *__restrict__ out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t s = int64_t(idx[i]) * BS;
#pragma unroll
    for (int q = 0; q < BS; ++q) out[i * BS + q] = v[s + q];
  }
}

__global__ void k_sqrt_copy(double *p, double *copy) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    const double r = sqrt(*p);
    *p = r;
    if (copy) *copy = r;
  }
}

// ---------------------------------------------------------------------------
// Value-only matrix update (mg_update_matrix): same structure, new values.
// ---------------------------------------------------------------------------
// element j of SELL entry e (chunked fp64 layout / fp32 layout)
__device__ __forceinline__ int64_t sell_off64(int64_t e, int V, int j) {
  const int lane = int(e & 31);
  const int64_t base = (e - lane) * V;
  return j < 2 * (V / 2) ? base + 64 * (j / 2) + 2 * lane + (j % 2) : base + 64 * (V / 2) + lane;
}
__device__ __forceinline__ int64_t sell_off32(int64_t e, int V, int j) {
  const int lane = int(e & 31);
  const int64_t base = (e - lane) * V;
  const int q = V / 4;
  return j < 4 * q ? base + 128 * (j / 4) + 4 * lane + (j % 4) : base + 128 * q + 32 * (j - 4 * q) + lane;
}

// original BSR entry k (V = bs*bs row-major values) -> SELL entry map[k],
// chunked fp64 layout (out64) or fp32 layout (out32, rounded to nearest)
// (src: the level entry of part entry k, or nullptr for the identity)
__global__ void k_scatter_values(int64_t nnz, int V, const int64_t *__restrict__ map, const int64_t *__restrict__ src,
                                 const double *__restrict__ vals, double *__restrict__ out64, float *__restrict__ out32,
                                 int *flag) {
  for (int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; k < nnz; k += int64_t(gridDim.x) * blockDim.x) {
    const int64_t e = map[k];
    const int64_t ks = src ? src[k] : k;
    for (int j = 0; j < V; ++j) {
      const double v = vals[ks * V + j];
      if (!isfinite(v)) atomicOr(flag, 1);
      if (out32) out32[sell_off32(e, V, j)] = float(v);
      else out64[sell_off64(e, V, j)] = v;
    }
  }
}

// D^-1 of the diagonal blocks (read from the SELL operator at entries diag_e)
// by Gauss-Jordan with partial pivoting (max |a|, ties -> lowest row), the
// operation sequence of the host mgi_block_diag_inverse with explicit
// round-to-nearest intrinsics (no FMA contraction).  Written to the sliced
// D^-1 layout at row_pos.  flag |= 2 on a singular block.
template <int BS>
__global__ void k_block_inverse(int64_t n, const int64_t *__restrict__ diag_e, const double *__restrict__ val64,
                                const float *__restrict__ val32, const int32_t *__restrict__ row_pos,
                                double *__restrict__ dinv, int *flag) {
  constexpr int V = BS * BS;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    double a[V], inv[V];
    const int64_t e = diag_e[i];
#pragma unroll
    for (int j = 0; j < V; ++j) {
      a[j] = val32 ? double(val32[sell_off32(e, V, j)]) : val64[sell_off64(e, V, j)];
      inv[j] = 0.0;
    }
#pragma unroll
    for (int r = 0; r < BS; ++r) inv[r * BS + r] = 1.0;
    bool ok = true;
#pragma unroll
    for (int k = 0; k < BS; ++k) {
      int p = k;
      double best = fabs(a[k * BS + k]);
#pragma unroll
      for (int r = k + 1; r < BS; ++r) {
        const double v = fabs(a[r * BS + k]);
        if (v > best) best = v, p = r;
      }
      if (!(best > 0.0)) ok = false;
      if (!ok) continue;
      if (p != k) {
#pragma unroll
        for (int c = 0; c < BS; ++c) {
          double t = a[k * BS + c];
          a[k * BS + c] = a[p * BS + c];
          a[p * BS + c] = t;
          t = inv[k * BS + c];
          inv[k * BS + c] = inv[p * BS + c];
          inv[p * BS + c] = t;
        }
      }
      const double d = a[k * BS + k];
#pragma unroll
      for (int c = 0; c < BS; ++c) {
        a[k * BS + c] = __ddiv_rn(a[k * BS + c], d);
        inv[k * BS + c] = __ddiv_rn(inv[k * BS + c], d);
      }
#pragma unroll
      for (int r = 0; r < BS; ++r) {
        if (r == k) continue;
        const double f = a[r * BS + k];
        if (f == 0.0) continue;
#pragma unroll
        for (int c = 0; c < BS; ++c) {
          a[r * BS + c] = __dsub_rn(a[r * BS + c], __dmul_rn(f, a[k * BS + c]));
          inv[r * BS + c] = __dsub_rn(inv[r * BS + c], __dmul_rn(f, inv[k * BS + c]));
        }
      }
    }
#pragma unroll
    for (int j = 0; j < V; ++j)
      if (!isfinite(inv[j])) ok = false;
    if (!ok) atomicOr(flag, 2);
    const int pos = row_pos[i];
    const int lane = pos & 31;
    double *base = dinv + int64_t(pos >> 5) * 32 * V;
#pragma unroll
    for (int j = 0; j < 2 * (V / 2); ++j) base[64 * (j / 2) + 2 * lane + (j % 2)] = ok ? inv[j] : 0.0;
    if (V & 1) base[64 * (V / 2) + lane] = ok ? inv[V - 1] : 0.0;
  }
}

// dense (row-major, leading dimension ld) coarse matrix from BSR entries
__global__ void k_dense_scatter(int64_t nnzb, int bs, const int32_t *__restrict__ brow, const int32_t *__restrict__ bcol,
                                const double *__restrict__ vals, int round32, int64_t ld, double *__restrict__ dense) {
  const int V = bs * bs;
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < nnzb * V; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t k = t / V;
    const int j = int(t % V), r = j / bs, c = j % bs;
    const double v = vals[t];
    dense[(int64_t(brow[k]) * bs + r) * ld + int64_t(bcol[k]) * bs + c] = round32 ? double(float(v)) : v;
  }
}

// x += z
// y += alpha x (mg_axpy: the Newton update w + d).
__global__ void k_axpy(int64_t n, double alpha, const double *__restrict__ x, double *__restrict__ y) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    y[i] = fma(alpha, x[i], y[i]);
}

__global__ void k_axpy1(int64_t n, const double *__restrict__ z, double *__restrict__ x) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    x[i] += z[i];
}

// Finite check of a vector (any NaN/Inf -> *flag = 1).
__global__ void k_nonfinite(int64_t n, const double *__restrict__ a, int *flag) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    if (!isfinite(a[i])) *flag = 1;
}

// ---------------------------------------------------------------------------
// Global constraint w^T x = 0 on a level (int p = 0): the projections
// x -= (a^T x / denom) k with the dot a^T x already reduced into *s.
// ---------------------------------------------------------------------------
__global__ void k_sub_mean(int64_t n, double *__restrict__ x, const double *__restrict__ k,
                           const double *__restrict__ s, double denom) {
  const double coef = *s / denom;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    x[i] = x[i] - coef * k[i];
}

// Small vectors (one CTA): x -= ((d^T x) / denom) k in a single launch -- the
// global constraint's projection on coarse levels, where the two-kernel
// path (grid reduction + update) is pure launch latency.  Fixed summation order.
__global__ void __launch_bounds__(1024) k_mean_project_small(int64_t n, double *__restrict__ x,
                                                            const double *__restrict__ d,
                                                            const double *__restrict__ k, double denom) {
  __shared__ double sh[32];
  double s = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s = fma(d[i], x[i], s);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_down_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_down_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) sh[0] = t;
  }
  __syncthreads();
  const double coef = sh[0] / denom;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) x[i] = x[i] - coef * k[i];
}

// Coarse regularisation A_0 + alpha w w^T, alpha = max_i |a_ii| / w_max^2 (reading
// Z25): one block finds the largest diagonal magnitude, then the rank-1 update.
__global__ void k_diag_absmax(int64_t N, int64_t ld, const double *__restrict__ a, double *out) {
  __shared__ double sh[1024];
  double m = 0.0;
  for (int64_t i = threadIdx.x; i < N; i += blockDim.x) m = fmax(m, fabs(a[i * ld + i]));
  sh[threadIdx.x] = m;
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + st]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sh[0];
}

__global__ void k_rank1_reg(int64_t N, int64_t ld, double *__restrict__ a, const double *__restrict__ w,
                            const double *__restrict__ dmax, double wmax) {
  const double alpha = *dmax / (wmax * wmax);
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < N * N; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = t / N, j = t % N;
    a[i * ld + j] = a[i * ld + j] + alpha * (w[i] * w[j]);
  }
}


// ---------------------------------------------------------------------------
// Vanka-type patch smoother:
//   x <- x + omega sum_p R_p^T W_p A_pp^{-1} R_p (b - A x),
// patches of nl nodes (e.g. the 2^d nodes of a mesh cell), m = nl*BS <= 32
// unknowns, W = diag(1/multiplicity).  Deterministic: a patch pass writes
// c_p = A_pp^{-1} r_p per patch, a node pass gathers sum_p c_p through the
// node -> (patch, corner) list in a fixed order (no atomics).
// ---------------------------------------------------------------------------
constexpr int kVankaWarps = 2;  // warps per CTA of the build kernel (2 x 16.9 KB shared)

// ent[(p*nl + a)*nl + b] = SELL entry of block (node_a, node_b) of patch p, -1 if absent.
__global__ void k_vanka_find(int64_t np, int nl, const int32_t *__restrict__ nodes,
                             const int64_t *__restrict__ slice_ptr, const int32_t *__restrict__ col,
                             const int32_t *__restrict__ row_pos, int64_t *__restrict__ ent) {
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < np * nl; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t p = t / nl;
    int64_t *out = ent + t * nl;
    for (int b = 0; b < nl; ++b) out[b] = -1;
    const int i = nodes[t];
    const int pos = row_pos[i];
    const int s = pos >> 5, lane = pos & 31;
    const int64_t e0 = slice_ptr[s], len = (slice_ptr[s + 1] - e0) >> 5;
    for (int64_t k = 0; k < len; ++k) {
      const int64_t e = e0 + 32 * k + lane;
      const int cj = col[e];
      for (int b = 0; b < nl; ++b)  // first match: padding repeats the last real column
        if (out[b] < 0 && nodes[p * nl + b] == cj) out[b] = e;
    }
  }
}

// Inverse layout: patches in groups of ppw = 32 / m (the patches one warp of
// k_vanka_patch serves); column c of the group's patches is contiguous, so the
// warp reads ppw*m consecutive doubles per column:
//   element (r, c) of patch p at ((p / ppw) * m + c) * (ppw * m) + (p % ppw) * m + r.
__device__ __forceinline__ int64_t vk_off(int64_t p, int m, int ppw, int r, int c) {
  return ((p / ppw) * m + c) * int64_t(ppw * m) + (p % ppw) * m + r;
}

// Dense inverse of every patch matrix A_pp (Gauss-Jordan, partial pivoting,
// ties -> lowest row), in the vk_off layout.  Warp per patch, lane = row.
// flag |= 2 on a singular patch.
template <int BS>
__global__ void __launch_bounds__(32 * kVankaWarps) k_vanka_build(int64_t np, int nl, const int64_t *__restrict__ ent,
                                                                 const double *__restrict__ val64,
                                                                 const float *__restrict__ val32, int ppw,
                                                                 double *__restrict__ inv, int *flag) {
  __shared__ double sA[kVankaWarps][32][33], sI[kVankaWarps][32][33];
  const int w = threadIdx.x >> 5, r = threadIdx.x & 31;
  const int64_t p = int64_t(blockIdx.x) * kVankaWarps + w;
  if (p >= np) return;
  const int m = nl * BS;
  constexpr int V = BS * BS;
  double(*A)[33] = sA[w];
  double(*I)[33] = sI[w];
  if (r < m) {
    const int a = r / BS, rr = r % BS;
    for (int c = 0; c < m; ++c) {
      const int64_t e = ent[(p * nl + a) * nl + c / BS];
      const int j = rr * BS + c % BS;
      A[r][c] = e < 0 ? 0.0 : (val32 ? double(val32[sell_off32(e, V, j)]) : val64[sell_off64(e, V, j)]);
      I[r][c] = r == c ? 1.0 : 0.0;
    }
  }
  __syncwarp();
  bool ok = true;
  for (int k = 0; k < m; ++k) {
    int piv = k;
    double best = fabs(A[k][k]);
    for (int q = k + 1; q < m; ++q) {
      const double v = fabs(A[q][k]);
      if (v > best) best = v, piv = q;
    }
    if (!(best > 0.0)) {
      ok = false;
      break;
    }
    if (piv != k && r < m) {  // lane r swaps column r of rows k and piv
      double t = A[k][r];
      A[k][r] = A[piv][r];
      A[piv][r] = t;
      t = I[k][r];
      I[k][r] = I[piv][r];
      I[piv][r] = t;
    }
    __syncwarp();
    const double d = A[k][k];
    __syncwarp();
    if (r < m) {
      A[k][r] = __ddiv_rn(A[k][r], d);
      I[k][r] = __ddiv_rn(I[k][r], d);
    }
    __syncwarp();
    if (r < m && r != k) {
      const double f = A[r][k];
      for (int c = 0; c < m; ++c) {
        A[r][c] = A[r][c] - f * A[k][c];
        I[r][c] = I[r][c] - f * I[k][c];
      }
    }
    __syncwarp();
  }
  if (!ok) {
    if (r == 0) atomicOr(flag, 2);
    return;
  }
  if (r < m)
    for (int c = 0; c < m; ++c) inv[vk_off(p, m, ppw, r, c)] = I[r][c];
}

// Predicated evict-first load: lanes with !pred issue no access at all (volatile
// asm with an explicit predicate: the compiler cannot if-convert it into an
// unconditional load) and return 0.
__device__ __forceinline__ double ldcs_if(const double *p, bool pred) {
  double v = 0.0;
  asm volatile("{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %2, 0;\n\t@q ld.global.cs.f64 %0, [%1];\n\t}"
               : "+d"(v)
               : "l"(p), "r"(int(pred)));
  return v;
}

// c_p = A_pp^{-1} r_p (r = b - A x, or b itself for a zero start).  ppw =
// 32 / m patches per warp (lane = sub * m + row), columns read as ppw*m
// contiguous doubles.  NL > 0: patch size known at compile time -> all m
// column loads of a lane in flight before the first use (the kernel is
// latency bound otherwise); NL = 0: runtime nl, four columns at a time.
template <int BS, int NL>
__global__ void __launch_bounds__(kCta) k_vanka_patch(int64_t np, int nl_rt, int ppw, const int32_t *__restrict__ nodes,
                                                     const double *__restrict__ inv, const double *__restrict__ r,
                                                     double *__restrict__ cbuf) {
  const int lane = threadIdx.x & 31;
  const int nl = NL > 0 ? NL : nl_rt;
  const int m = nl * BS;
  const int sub = lane / m, row = lane - sub * m;
  const int64_t p0 = (int64_t(blockIdx.x) * kWarpsPerCta + (threadIdx.x >> 5)) * ppw;
  const int64_t p = p0 + sub;
  const bool act = sub < ppw && p < np;
  if (p0 >= np) return;
  // Inactive lanes use the warp's first patch / row 0 for their (never issued)
  // addresses; their loads are predicated off.
  const int64_t pc = act ? p : p0;
  const int rc = act ? row : 0;
  const double *ip = inv + vk_off(pc, m, ppw, rc, 0);
  const int64_t cs = int64_t(ppw) * m;  // column stride
  double acc = 0.0;
  if constexpr (NL > 0) {
    constexpr int M = NL * BS;
    double a[M];
#pragma unroll
    for (int j = 0; j < M; ++j) a[j] = ldcs_if(ip + j * cs, act);
    const double rl = act ? __ldg(r + int64_t(nodes[pc * NL + rc / BS]) * BS + rc % BS) : 0.0;
    const int base = sub * M;
#pragma unroll
    for (int j = 0; j < M; ++j) acc = fma(a[j], __shfl_sync(0xffffffffu, rl, (base + j) & 31), acc);
  } else {
    const double rl = act ? __ldg(r + int64_t(nodes[pc * nl + rc / BS]) * BS + rc % BS) : 0.0;
    const int base = sub * m;
    int j = 0;
    for (; j + 4 <= m; j += 4) {  // four columns' loads in flight per lane
      double a[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) a[u] = ldcs_if(ip + (j + u) * cs, act);
#pragma unroll
      for (int u = 0; u < 4; ++u) acc = fma(a[u], __shfl_sync(0xffffffffu, rl, (base + j + u) & 31), acc);
    }
    for (; j < m; ++j) acc = fma(ldcs_if(ip + j * cs, act), __shfl_sync(0xffffffffu, rl, (base + j) & 31), acc);
  }
  if (act) cbuf[p * m + row] = acc;
}

// x_i = (assign ? 0 : x_i) + omega w_i sum_{(p, a) in list(i)} c_p[a*BS + comp]; thread per DOF.
__global__ void k_vanka_update(int64_t n, int bs, int m, const int64_t *__restrict__ nptr,
                               const int64_t *__restrict__ nlist, const double *__restrict__ wgt,
                               const double *__restrict__ cbuf, double omega, int assign, double *__restrict__ x) {
  for (int64_t t = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; t < n * bs; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = t / bs;
    const int comp = int(t % bs);
    double s = 0.0;
    for (int64_t q = nptr[i]; q < nptr[i + 1]; ++q) s += __ldg(cbuf + nlist[q] + comp);
    const double upd = omega * (wgt[i] * s);
    x[t] = assign ? upd : x[t] + upd;
  }
  (void)m;
}

}  // namespace mgk
