// libmgb200.so: the C ABI of include/mg.h.  Context and level state, device
// upload of the SELL-32-sigma operators built by host.cpp, the V-cycle of
// Alg. `gmg` with CUDA-graph capture, the MG iteration /
// MG-preconditioned GMRES drivers, and the
// row-partitioned multi-GPU variant (halo exchange before every A-pass and
// transfer, all-reduced Krylov dots, agglomeration of replicated coarse
// levels) over the transports of comm.h.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/mg.h"
#include "../../include/mg_internal.h"
#include "../../include/newton.h"
#include "comm.h"
#include "common.h"
#include "kernels.cuh"

#define MGB200_VERSION "mgb200 0.2 (sm_100a, fp64, SELL-32-sigma, multi-GPU halo)"

namespace mgb {

thread_local std::string g_err;
thread_local int64_t g_tally = 0;

mg_status vfail(mg_status st, const char *fmt, va_list ap) {
  char buf[512];
  vsnprintf(buf, sizeof buf, fmt, ap);
  g_err = buf;
  return st;
}

mg_status fail(mg_status st, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vfail(st, fmt, ap);
  va_end(ap);
  return st;
}

}  // namespace mgb

using namespace mgb;

namespace mgc {
mg_status comm_fail(mg_status st, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vfail(st, fmt, ap);
  va_end(ap);
  return st;
}
}  // namespace mgc

namespace {

struct SellOp {
  DevArray<int64_t> slice_ptr;
  DevArray<int32_t> perm, col;
  DevArray<double> val;
  DevArray<float> valf;  // fp32 values (mixed precision)
  bool f32 = false;
  std::vector<int32_t> perm_host;
  int64_t n_rows = 0, n_slices = 0, n_entries = 0;
  int vpe = 0;
  int ks = 1;  // warps per slice (split-k for small levels / long transfer rows)
  bool stream = false;
  bool set = false;
  mgk::Sell view() const { return mgk::Sell{slice_ptr.p, perm.p, col.p, val.p, n_slices, valf.p}; }
};

// Transfer operator in the SELL-C layout of mgi_tsell_fill (k_tsell).
struct TSellOp {
  DevArray<int64_t> slice_ptr;
  DevArray<int32_t> perm, col;
  DevArray<int2> cw;
  DevArray<float> w;
  int64_t n_slices = 0, n_entries = 0;
  int C = 32, wpe = 1, ks = 1, nsl = 1;
  bool set = false;
  mgk::TSell view() const { return mgk::TSell{slice_ptr.p, perm.p, cw.p, col.p, w.p, n_slices}; }
};

// Prolongation in natural row order (k_prolong_csr): int32 CSR offsets and
// {column, fp32 weight} entries; built only when every weight is exact in fp32
// (the dyadic transfer weights, reading Z8) and the entries fit int32.
struct PCsrOp {
  DevArray<int32_t> rp, col;
  DevArray<int2> cw;
  DevArray<float> w;
  int64_t n = 0;
  int wpe = 1;
  bool set = false;
  mgk::PCsr view() const { return mgk::PCsr{rp.p, cw.p, col.p, w.p, n}; }
};

// Operators above this size are read with evict-first loads (MGB200_STREAM_MB overrides
// the default kStreamBytes; experiment knob for L2 residency of mid-sized operators).
size_t stream_bytes() {
  static const size_t v = [] {
    const char *e = std::getenv("MGB200_STREAM_MB");
    return e && *e ? size_t(std::atoll(e)) << 20 : kStreamBytes;
  }();
  return v;
}

// Build SELL-32-sigma on the host and upload it (col: LOCAL column indices);
// f32: values rounded to fp32 in the fp32 chunk layout.
mg_status build_pcsr(PCsrOp &op, int64_t n, const std::vector<int64_t> &rp, const std::vector<int64_t> &col,
                     const std::vector<double> &v, int wpe) {
  op = PCsrOp();
  if (const char *e = std::getenv("MGB200_PCSR"); e && e[0] == '0') return MG_OK;
  const int64_t nnz = n > 0 ? rp[size_t(n)] : 0;
  if (nnz <= 0 || nnz >= (int64_t(1) << 31)) return MG_OK;
  // per-component weights (C4/C5 velocity-only Dirichlet) stay on SELL-32: measured
  // C5 V-cycle 11.12 -> 11.26 ms with the CSR kernel (four scalar weight loads per entry)
  if (wpe != 1) return MG_OK;
  for (int64_t i = 0; i < nnz * wpe; ++i)
    if (double(float(v[size_t(i)])) != v[size_t(i)]) return MG_OK;  // not exact in fp32: SELL path
  std::vector<int32_t> r32(size_t(n) + 1);
  for (int64_t i = 0; i <= n; ++i) r32[size_t(i)] = int32_t(rp[size_t(i)]);
  TRY(op.rp.upload(r32.data(), r32.size()));
  if (wpe == 1) {
    std::vector<int2> cw(static_cast<size_t>(nnz));
    for (int64_t e = 0; e < nnz; ++e) {
      const float f = float(v[size_t(e)]);
      int fi;
      std::memcpy(&fi, &f, sizeof fi);
      cw[size_t(e)] = make_int2(int32_t(col[size_t(e)]), fi);
    }
    TRY(op.cw.upload(cw.data(), cw.size()));
  } else {
    std::vector<int32_t> c32(static_cast<size_t>(nnz));
    std::vector<float> wf(size_t(nnz) * wpe);
    for (int64_t e = 0; e < nnz; ++e) c32[size_t(e)] = int32_t(col[size_t(e)]);
    for (size_t i = 0; i < wf.size(); ++i) wf[i] = float(v[i]);
    TRY(op.col.upload(c32.data(), c32.size()));
    TRY(op.w.upload(wf.data(), wf.size()));
  }
  op.n = n;
  op.wpe = wpe;
  op.set = true;
  return MG_OK;
}

mg_status build_sell(SellOp &op, int64_t n, const int64_t *rp, const int64_t *col, const double *val, int vpe,
                     bool f32 = false, std::vector<int64_t> *sp_out = nullptr,
                     const std::vector<int64_t> *row_ids = nullptr) {
  int64_t ns = 0, ne = 0;
  int st = mgi_sell_size(n, rp, kSigma, &ns, &ne);
  if (st) return fail(mg_status(st), "sell layout: invalid input");
  std::vector<int64_t> sp(ns + 1);
  std::vector<int32_t> perm(ns * 32), c(ne);
  if (f32) {
    std::vector<float> v(ne * vpe);
    st = mgi_sell_fill_f32(n, rp, col, val, vpe, kSigma, sp.data(), perm.data(), c.data(), v.data());
    if (!st) TRY(op.valf.upload(v.data(), v.size()));
    op.val.release();
  } else {
    std::vector<double> v(ne * vpe);
    st = mgi_sell_fill(n, rp, col, val, vpe, kSigma, sp.data(), perm.data(), c.data(), v.data());
    if (!st) TRY(op.val.upload(v.data(), v.size()));
    op.valf.release();
  }
  if (st) return fail(mg_status(st), "sell layout: fill failed (%d)", st);
  if (row_ids)  // operator over a subset of rows: lanes address the level's local rows
    for (auto &r : perm)
      if (r >= 0) r = int32_t((*row_ids)[r]);
  TRY(op.slice_ptr.upload(sp.data(), sp.size()));
  TRY(op.perm.upload(perm.data(), perm.size()));
  TRY(op.col.upload(c.data(), c.size()));
  op.perm_host.swap(perm);
  if (sp_out) sp_out->swap(sp);
  op.n_rows = n;
  op.n_slices = ns;
  op.n_entries = ne;
  op.vpe = vpe;
  op.f32 = f32;
  op.stream = size_t(ne) * ((f32 ? 4 : 8) * vpe + 4) > stream_bytes();
  op.set = true;
  return MG_OK;
}

// Transfer layout SELL-C (C = 32 / bs); leaves T unset (fp64 SELL-32 path)
// when a weight is not exact in fp32 or MGB200_TSELL=0.
mg_status build_tsell(TSellOp &T, int64_t n, const int64_t *rp, const int64_t *col, const double *w, int wpe, int bs) {
  T = TSellOp();
  const char *e = std::getenv("MGB200_TSELL");
  if (e && e[0] == '0') return MG_OK;
  const int C = 32 / bs;
  const int sigma = C * ((kSigma + C - 1) / C);
  int64_t ns = 0, ne = 0;
  int st = mgi_tsell_size(n, rp, C, sigma, &ns, &ne);
  if (st) return fail(mg_status(st), "transfer layout: invalid input");
  std::vector<int64_t> sp(ns + 1);
  std::vector<int32_t> perm(ns * C), cl(ne);
  std::vector<float> wf(ne * wpe);
  st = mgi_tsell_fill(n, rp, col, w, wpe, C, sigma, sp.data(), perm.data(), cl.data(), wf.data());
  if (st == 2) return MG_OK;  // weights not exact in fp32: keep the fp64 layout
  if (st) return fail(mg_status(st), "transfer layout: fill failed (%d)", st);
  TRY(T.slice_ptr.upload(sp.data(), sp.size()));
  TRY(T.perm.upload(perm.data(), perm.size()));
  if (wpe == 1) {
    std::vector<int2> cw(ne);
    for (int64_t t = 0; t < ne; ++t) {
      int wb;
      std::memcpy(&wb, &wf[t], sizeof wb);
      cw[t] = make_int2(cl[t], wb);
    }
    TRY(T.cw.upload(cw.data(), cw.size()));
  } else {
    TRY(T.col.upload(cl.data(), cl.size()));
    TRY(T.w.upload(wf.data(), wf.size()));
  }
  T.n_slices = ns;
  T.n_entries = ne;
  T.C = C;
  T.wpe = wpe;
  T.set = true;
  return MG_OK;
}

// Host copies of (possibly device-resident) input arrays.
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

// Ghost exchange of one vector kind (multi-GPU).  `active` is uniform over
// ranks (set for every operator of a distributed level), so every rank takes
// part in every exchange even when its own pattern is empty.
struct Halo {
  bool active = false;
  mgc::Pattern pat;
  DevArray<int32_t> send_idx;  // owned rows to pack, in send order
  DevArray<double> sendbuf, ghost;
  int64_t n_ghost = 0;
};

struct Level {
  bool declared = false;
  int64_t n_global = 0, row_begin = 0, row_end = 0, n = 0;
  bool dist = false;             // rows partitioned over ranks
  std::vector<int64_t> bounds;   // [nranks+1] row ranges of the ranks (distributed levels)
  // The level operator as one part (all rows) or, on distributed levels, two
  // parts -- interior rows (no ghost columns) and boundary rows -- so the
  // interior is computed while the halo exchange is in flight.  Each part has
  // its own SELL layout, D^-1 slices and value-update maps.
  struct Part {
    SellOp A;    // V-cycle operator (fp32 values in mixed precision)
    SellOp A64;  // mixed precision, finest level: fp64 operator for Krylov / residuals
    DevArray<double> dinv;
    DevArray<int64_t> umap, udiag_e, usrc;  // part entry -> SELL entry; row diag -> SELL entry; part entry -> level entry
    DevArray<int32_t> upos;                 // part row -> slice position
    int64_t n = 0, nnz = 0;
    bool halo = false;                      // reads ghost columns
  };
  Part part[2];
  int nparts = 1;
  int64_t nnzb = 0;
  Halo hx;                        // ghosts of x for A-passes on this level
  std::vector<double> dinv_host;  // user-supplied D^-1 (row-major blocks)
  DevArray<int32_t> ublk_row, ublk_col;  // level 0: block coordinates for the dense coarse matrix
  std::vector<int64_t> rp0, col0;  // level-0 copy for the dense coarse inverse
  std::vector<double> val0;
  bool dinv_ready = false;
  SellOp P, R;  // P_{l-1}: level l-1 -> l (rows: owned fine rows), R_{l-1} = P^T (rows: r_row0 ...)
  TSellOp Pt, Rt;  // the same operators in the SELL-C layout (fp32-exact weights), used when set
  PCsrOp Pc;       // P as natural-order CSR with fp32-exact weights (k_prolong_csr), used when set
  Halo hp;      // ghosts of the coarse vector y for P (coarse level distributed)
  Halo hr;      // ghosts of the fine vector r for R (this level distributed)
  int64_t r_row0 = 0, r_rows = 0;  // coarse rows produced by the local R
  bool agglomerate = false;        // coarse level replicated: all-gather d after R
  std::vector<int64_t> ag_counts, ag_displs;
  int wpe = 1;
  int64_t nnz_p = 0;
  // global constraint w^T x = 0: weights, kernel vector, w^T k, k^T k
  bool mean = false;
  DevArray<double> mean_w, mean_k;
  double mean_wk = 0.0, mean_kk = 0.0, mean_wmax = 0.0;
  double omega = 0.0;
  int nu_pre = -1, nu_post = -1;
  DevArray<double> x, b, w;  // correction, restricted rhs, work (ping-pong / residual)
  // Vanka-type patch smoother (mg_set_vanka): replaces block-Jacobi on this level
  struct Vanka {
    bool on = false, ready = false;
    int64_t np = 0;
    int nl = 0, m = 0, ppw = 1;       // ppw = 32 / m patches per warp (inverse layout, mgk::vk_off)
    DevArray<int32_t> nodes;          // [np*nl] patch nodes (local rows)
    DevArray<int64_t> ent;            // [np*nl*nl] SELL entry of each block of A_pp (-1: absent)
    DevArray<double> inv;             // [np*m*m] A_pp^{-1}, column-major per patch
    DevArray<int64_t> nptr, nlist;    // node -> p*m + a*bs (CSR, ascending patch order)
    DevArray<double> wgt;             // 1 / multiplicity
    DevArray<double> cbuf;            // [np*m] patch corrections
  } vk;
};

struct GraphExec {
  cudaGraphExec_t exec = nullptr;
  int64_t kernels = 0;
};

// A GMRES restart cycle captured as one graph with a while node around a
// switch node over the Arnoldi steps (kernels[j]: kernel nodes of step j).
struct CycleGraph {
  cudaGraphExec_t exec = nullptr;
  std::vector<int64_t> kernels;
};

struct GraphKey {
  const double *x;
  const double *b;
  int zero;
  bool operator<(const GraphKey &o) const { return std::tie(x, b, zero) < std::tie(o.x, o.b, o.zero); }
};

}  // namespace

struct mg_ctx_s {
  mg_config cfg{};
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int n_sm = 148;
  std::unique_ptr<mgc::Transport> tr;  // null => single GPU
  std::vector<Level> lv;
  SellOp H, HT;     // hanging-node matrix H (averaging) and H^T (distributing)
  Halo hh, hht_halo;
  DevArray<double> cinv;  // dense A_0^-1, row stride cld
  int64_t cN = 0, cld = 0;
  DevArray<double> red_part, scal;
  DevArray<unsigned> ticket;
  bool finalized = false;
  // per-level profiling (mgi_vcycle_profile): tagged events on the stream
  bool prof_on = false;
  int cur_level = 0;
  std::vector<std::pair<int, cudaEvent_t>> prof;
  // halo / interior overlap (split levels): side stream + fork/join events
  cudaStream_t comm_stream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // persistent coarse tail: levels 0..tail_T run as one cooperative launch
  DevArray<mgk::TailOp> tail_ops;
  int tail_nops = 0, tail_T = -1;
  bool tail_cluster = true;
  unsigned tail_grid = 0;
  std::map<GraphKey, GraphExec> graphs;
  std::map<std::tuple<int, double, int>, GraphExec> iter_graphs;  // GMRES iteration j (j, rtol, m)
  std::map<std::tuple<int, double, int>, CycleGraph> cycle_graphs;  // GMRES restart cycle (mm, rtol, m)
  int64_t launches = 0;
  // GMRES workspace
  int gm_m = 0;
  DevArray<double> gm_V, gm_Z, gm_state;
  DevArray<double> dcgs_part;  // per-CTA partials of the DCGS2 multi-dot ([grid][2m+2])
  DevArray<unsigned> dcgs_ticket;
  DevArray<double> rich_z, rich_r;  // mixed-precision MG iteration (defect correction)
  DevArray<double> mean_b;          // consistent copy of b (global constraint on the finest level)
  DevArray<double> upd_stage;       // mg_update_matrix: staging buffer for host values (kept across calls)
  double *gm_host = nullptr;  // pinned
  // mg_update_matrix from pageable host memory: two pinned chunks, the host
  // copy of one overlapping the DMA of the other
  char *pin_chunk[2] = {nullptr, nullptr};
  cudaEvent_t pin_ev[2] = {nullptr, nullptr};
  mgk::GmresDev gm{};
  ~mg_ctx_s() {
    clear_graphs();
    for (int k = 0; k < 2; ++k) {
      if (pin_chunk[k]) cudaFreeHost(pin_chunk[k]);
      if (pin_ev[k]) cudaEventDestroy(pin_ev[k]);
    }
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    if (comm_stream) cudaStreamDestroy(comm_stream);
    if (gm_host) cudaFreeHost(gm_host);
    if (own_stream && stream) cudaStreamDestroy(stream);
  }
  void clear_graphs() {
    for (auto &kv : graphs) cudaGraphExecDestroy(kv.second.exec);
    for (auto &kv : iter_graphs) cudaGraphExecDestroy(kv.second.exec);
    for (auto &kv : cycle_graphs) cudaGraphExecDestroy(kv.second.exec);
    cycle_graphs.clear();
    graphs.clear();
    iter_graphs.clear();
  }
  void invalidate() {
    clear_graphs();
    finalized = false;
  }
  int bs() const { return cfg.block_size; }
  int L() const { return cfg.n_levels - 1; }
  int nranks() const { return tr ? tr->nranks : 1; }
  int rank() const { return tr ? tr->rank : 0; }
  bool use_graphs() const { return cfg.use_graphs && (!tr || tr->graph_safe()); }
  // GMRES restart cycles as conditional graphs (MGB200_GMRES_LOOP=host: one
  // graph + host sync per Arnoldi step, the round-1 path)
  bool pdl() const {  // programmatic dependent launch of the V-cycle kernels (MGB200_PDL=0: plain launches)
    const char *e = std::getenv("MGB200_PDL");
    return !(e && e[0] == '0');
  }
  bool mgs_alternate() const {  // MGB200_MGS_ALT=0: every MGS pass sweeps forward (round-1 order)
    const char *e = std::getenv("MGB200_MGS_ALT");
    return !(e && e[0] == '0');
  }
  bool gmres_device_loop() const {
    const char *e = std::getenv("MGB200_GMRES_LOOP");
    return !(e && std::string(e) == "host");
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

inline unsigned grid_for_slices(int64_t n_slices, int ks = 1) {
  const int per = mgk::kWarpsPerCta / ks;
  return unsigned((n_slices + per - 1) / per);
}

// split-k factor of an A operator, decided on the GLOBAL level size so every
// rank of a distributed solve (and the single-GPU solve) sums identically
// thresholds in slices (overridable for tuning: MGB200_KS4_SLICES, MGB200_KS2_SLICES)
int64_t env_i64(const char *name, int64_t dflt) {
  const char *v = std::getenv(name);
  return v && *v ? std::atoll(v) : dflt;
}

int ks_for_level(int64_t n_global) {
  static const int64_t t4 = env_i64("MGB200_KS4_SLICES", 4096), t2 = env_i64("MGB200_KS2_SLICES", 16384),
                       t8 = env_i64("MGB200_KS8_SLICES", 256);
  const int64_t slices = (n_global + 31) / 32;
  return slices < t8 ? 8 : slices < t4 ? 4 : slices < t2 ? 2 : 1;
}

// Kernel launch of the V-cycle kernels: with programmatic dependent launch
// (PDL, see kernels.cuh pdl_trigger / pdl_wait) while g_pdl is set by the
// calling API entry (Tally), a plain launch otherwise.  Captured into CUDA
// graphs as programmatic edges.
thread_local bool g_pdl = false;
template <typename... P, typename... A>
void kl(void (*k)(P...), unsigned grid, cudaStream_t st, A &&...args) {
  ++g_tally;
  if (g_pdl) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(mgk::kCta);
    cfg.dynamicSmemBytes = 0;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k, std::forward<A>(args)...);
  } else {
    k<<<grid, mgk::kCta, 0, st>>>(std::forward<A>(args)...);
  }
}

mg_status check_launch(const char *what = "kernel") {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(MG_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return MG_OK;
}

// Input vector of an operator: owned part x, ghost part xg (HALO when xg != 0)
struct In {
  const double *x;
  const double *xg;
  int n_own;
};

// --- dispatch over block size / op / cache hint / halo -------------------------
template <int BS, int OP, bool HALO>
void launch_apply_h(const SellOp &A, In in, const double *b, const double *dinv, double *out, double alpha,
                    double beta, cudaStream_t st) {
  const unsigned g = grid_for_slices(A.n_slices, A.ks);
  if (A.ks == 8) {
    if (A.f32)
      kl(mgk::k_sell_apply<BS, OP, false, HALO, 8, true>, g, st, A.view(), in.x, in.xg, in.n_own, b, dinv, out, alpha, beta);
    else
      kl(mgk::k_sell_apply<BS, OP, false, HALO, 8, false>, g, st, A.view(), in.x, in.xg, in.n_own, b, dinv, out, alpha, beta);
  } else if (A.f32) {
    if (A.ks == 4)
      kl(mgk::k_sell_apply<BS, OP, false, HALO, 4, true>, g, st, A.view(), in.x, in.xg, in.n_own, b, dinv, out, alpha, beta);
    else if (A.ks == 2)
      kl(mgk::k_sell_apply<BS, OP, true, HALO, 2, true>, g, st, A.view(), in.x, in.xg, in.n_own, b, dinv, out, alpha, beta);
    else
      kl(mgk::k_sell_apply<BS, OP, true, HALO, 1, true>, g, st, A.view(), in.x, in.xg, in.n_own, b, dinv, out, alpha, beta);
  } else if (A.ks == 4)
    kl(mgk::k_sell_apply<BS, OP, false, HALO, 4>, g, st, A.view(), in.x, in.xg, in.n_own, b, dinv, out, alpha, beta);
  else if (A.ks == 2)
    kl(mgk::k_sell_apply<BS, OP, true, HALO, 2>, g, st, A.view(), in.x, in.xg, in.n_own, b, dinv, out, alpha, beta);
  else if (A.stream)
    kl(mgk::k_sell_apply<BS, OP, true, HALO, 1>, g, st, A.view(), in.x, in.xg, in.n_own, b, dinv, out, alpha, beta);
  else
    kl(mgk::k_sell_apply<BS, OP, false, HALO, 1>, g, st, A.view(), in.x, in.xg, in.n_own, b, dinv, out, alpha, beta);
}

template <int BS, int OP>
void launch_apply_t(const SellOp &A, In in, const double *b, const double *dinv, double *out, double alpha,
                    double beta, cudaStream_t st) {
  if (A.n_slices == 0) return;
  if (in.xg) launch_apply_h<BS, OP, true>(A, in, b, dinv, out, alpha, beta, st);
  else launch_apply_h<BS, OP, false>(A, in, b, dinv, out, alpha, beta, st);
}

template <int OP>
mg_status launch_apply(int bs, const SellOp &A, In in, const double *b, const double *dinv, double *out,
                       double alpha, double beta, cudaStream_t st) {
  switch (bs) {
    case 1: launch_apply_t<1, OP>(A, in, b, dinv, out, alpha, beta, st); break;
    case 2: launch_apply_t<2, OP>(A, in, b, dinv, out, alpha, beta, st); break;
    case 3: launch_apply_t<3, OP>(A, in, b, dinv, out, alpha, beta, st); break;
    case 4: launch_apply_t<4, OP>(A, in, b, dinv, out, alpha, beta, st); break;
    case 6: launch_apply_t<6, OP>(A, in, b, dinv, out, alpha, beta, st); break;
    default: return fail(MG_ERR_INVALID_ARG, "block size %d not supported", bs);
  }
  return check_launch(OP == mgk::OP_SWEEP ? "sweep" : OP == mgk::OP_RESID ? "residual" : "spmv");
}

template <int BS>
void launch_sweep0_t(const SellOp &A, const double *dinv, const double *b, double *x, double omega, cudaStream_t st) {
  if (A.n_slices == 0) return;
  kl(mgk::k_sweep0<BS>, grid_for_slices(A.n_slices), st, A.n_slices, A.perm.p, dinv, b, x, omega);
}

mg_status launch_sweep0(int bs, const SellOp &A, const double *dinv, const double *b, double *x, double omega,
                        cudaStream_t st) {
  switch (bs) {
    case 1: launch_sweep0_t<1>(A, dinv, b, x, omega, st); break;
    case 2: launch_sweep0_t<2>(A, dinv, b, x, omega, st); break;
    case 3: launch_sweep0_t<3>(A, dinv, b, x, omega, st); break;
    case 4: launch_sweep0_t<4>(A, dinv, b, x, omega, st); break;
    case 6: launch_sweep0_t<6>(A, dinv, b, x, omega, st); break;
    default: return fail(MG_ERR_INVALID_ARG, "block size %d not supported", bs);
  }
  return check_launch("sweep0");
}

template <int BS, int WPE, bool ACC, bool HALO>
void launch_transfer_h(const SellOp &T, In in, double *out, cudaStream_t st) {
  const unsigned g = grid_for_slices(T.n_slices, T.ks);
  if (T.ks > 1)
    kl(mgk::k_transfer<BS, WPE, ACC, true, HALO, 4>, g, st, T.view(), in.x, in.xg, in.n_own, out);
  else if (T.stream)
    kl(mgk::k_transfer<BS, WPE, ACC, true, HALO, 1>, g, st, T.view(), in.x, in.xg, in.n_own, out);
  else
    kl(mgk::k_transfer<BS, WPE, ACC, false, HALO, 1>, g, st, T.view(), in.x, in.xg, in.n_own, out);
}

template <int BS, int WPE, bool ACC>
void launch_transfer_t(const SellOp &T, In in, double *out, cudaStream_t st) {
  if (T.n_slices == 0) return;
  if (in.xg) launch_transfer_h<BS, WPE, ACC, true>(T, in, out, st);
  else launch_transfer_h<BS, WPE, ACC, false>(T, in, out, st);
}

template <int BS, bool ACC>
void launch_transfer_bs(const SellOp &T, In in, double *out, cudaStream_t st) {
  if (T.vpe == 1 || BS == 1) launch_transfer_t<BS, 1, ACC>(T, in, out, st);
  else launch_transfer_t<BS, BS, ACC>(T, in, out, st);
}

mg_status launch_transfer(int bs, bool acc, const SellOp &T, In in, double *out, cudaStream_t st) {
  switch (bs) {
    case 1: acc ? launch_transfer_bs<1, true>(T, in, out, st) : launch_transfer_bs<1, false>(T, in, out, st); break;
    case 2: acc ? launch_transfer_bs<2, true>(T, in, out, st) : launch_transfer_bs<2, false>(T, in, out, st); break;
    case 3: acc ? launch_transfer_bs<3, true>(T, in, out, st) : launch_transfer_bs<3, false>(T, in, out, st); break;
    case 4: acc ? launch_transfer_bs<4, true>(T, in, out, st) : launch_transfer_bs<4, false>(T, in, out, st); break;
    case 6: acc ? launch_transfer_bs<6, true>(T, in, out, st) : launch_transfer_bs<6, false>(T, in, out, st); break;
    default: return fail(MG_ERR_INVALID_ARG, "block size %d not supported", bs);
  }
  return check_launch(acc ? "prolong-add" : "transfer");
}

template <int BS, int WPE, bool HALO>
void launch_pcsr_k(const PCsrOp &P, In in, double *out, cudaStream_t st) {
  const unsigned g = unsigned((P.n + mgk::kCta - 1) / mgk::kCta);
  kl(mgk::k_prolong_csr<BS, WPE, HALO>, g, st, P.view(), in.x, in.xg, in.n_own, out);
}

template <int BS>
void launch_pcsr_bs(const PCsrOp &P, In in, double *out, cudaStream_t st) {
  if (P.n == 0) return;
  if (P.wpe == 1 || BS == 1) {
    if (in.xg) launch_pcsr_k<BS, 1, true>(P, in, out, st);
    else launch_pcsr_k<BS, 1, false>(P, in, out, st);
  } else {
    if (in.xg) launch_pcsr_k<BS, BS, true>(P, in, out, st);
    else launch_pcsr_k<BS, BS, false>(P, in, out, st);
  }
}

mg_status launch_pcsr(int bs, const PCsrOp &P, In in, double *out, cudaStream_t st) {
  switch (bs) {
    case 1: launch_pcsr_bs<1>(P, in, out, st); break;
    case 2: launch_pcsr_bs<2>(P, in, out, st); break;
    case 3: launch_pcsr_bs<3>(P, in, out, st); break;
    case 4: launch_pcsr_bs<4>(P, in, out, st); break;
    case 6: launch_pcsr_bs<6>(P, in, out, st); break;
    default: return fail(MG_ERR_INVALID_ARG, "block size %d not supported", bs);
  }
  return check_launch("prolong-add (csr)");
}

template <int BS, int WPE, bool ACC, bool HALO, int KS, int NSL>
void launch_tsell_k(const TSellOp &T, In in, double *out, cudaStream_t st) {
  const unsigned g = grid_for_slices((T.n_slices + NSL - 1) / NSL, KS);
  kl(mgk::k_tsell<BS, WPE, ACC, HALO, KS, NSL>, g, st, T.view(), in.x, in.xg, in.n_own, out);
}

// (ks, nsl) = warps per slice group, slices per warp: TSellOp defaults
// (restriction 4/1, prolongation 1/1), MGB200_TSELL_R / MGB200_TSELL_P = "ks,nsl"
// override (tuning experiments; ks in {1,2,4}, nsl in {1,2,4})
inline void tsell_cfg(const TSellOp &T, bool acc, int &ks, int &nsl) {
  ks = T.ks, nsl = T.nsl;
  const char *e = std::getenv(acc ? "MGB200_TSELL_P" : "MGB200_TSELL_R");
  if (e && *e) {
    int a = 0, b = 0;
    if (std::sscanf(e, "%d,%d", &a, &b) == 2) ks = a, nsl = b;
  }
}

template <int BS, int WPE, bool ACC, bool HALO>
void launch_tsell_h(const TSellOp &T, In in, double *out, cudaStream_t st) {
  int ks, nsl;
  tsell_cfg(T, ACC, ks, nsl);
#define TS(K, S) \
  if (ks == K && nsl == S) return launch_tsell_k<BS, WPE, ACC, HALO, K, S>(T, in, out, st);
  TS(1, 1) TS(1, 2) TS(1, 4) TS(2, 1) TS(2, 2) TS(4, 1) TS(4, 2)
#undef TS
  launch_tsell_k<BS, WPE, ACC, HALO, 1, 1>(T, in, out, st);
}

template <int BS, bool ACC>
void launch_tsell_bs(const TSellOp &T, In in, double *out, cudaStream_t st) {
  if (T.n_slices == 0) return;
  if (T.wpe == 1 || BS == 1) {
    if (in.xg) launch_tsell_h<BS, 1, ACC, true>(T, in, out, st);
    else launch_tsell_h<BS, 1, ACC, false>(T, in, out, st);
  } else {
    if (in.xg) launch_tsell_h<BS, BS, ACC, true>(T, in, out, st);
    else launch_tsell_h<BS, BS, ACC, false>(T, in, out, st);
  }
}

mg_status launch_tsell(int bs, bool acc, const TSellOp &T, In in, double *out, cudaStream_t st) {
  switch (bs) {
    case 1: acc ? launch_tsell_bs<1, true>(T, in, out, st) : launch_tsell_bs<1, false>(T, in, out, st); break;
    case 2: acc ? launch_tsell_bs<2, true>(T, in, out, st) : launch_tsell_bs<2, false>(T, in, out, st); break;
    case 3: acc ? launch_tsell_bs<3, true>(T, in, out, st) : launch_tsell_bs<3, false>(T, in, out, st); break;
    case 4: acc ? launch_tsell_bs<4, true>(T, in, out, st) : launch_tsell_bs<4, false>(T, in, out, st); break;
    case 6: acc ? launch_tsell_bs<6, true>(T, in, out, st) : launch_tsell_bs<6, false>(T, in, out, st); break;
    default: return fail(MG_ERR_INVALID_ARG, "block size %d not supported", bs);
  }
  return check_launch(acc ? "prolong-add (tsell)" : "restrict (tsell)");
}

// profiling marks: tag = level (compute), 100 + level (halo), 200 + level (agglomeration)
void mark(mg_ctx_s *c, int tag) {
  if (!c->prof_on) return;
  cudaEvent_t e;
  cudaEventCreate(&e);
  cudaEventRecord(e, c->stream);
  c->prof.emplace_back(tag, e);
}

// --- halo exchange: pack owned rows, transport into the ghost buffer ----------
mg_status halo_pack(mg_ctx_s *c, Halo &h, const double *v) {
  const int bs = c->bs();
  const int64_t ns = h.pat.n_send;
  if (ns > 0) {
    const unsigned g = unsigned(std::min<int64_t>((ns + 255) / 256, 4 * c->n_sm));
    switch (bs) {
      case 1: ++g_tally, mgk::k_pack<1><<<g, 256, 0, c->stream>>>(ns, h.send_idx.p, v, h.sendbuf.p); break;
      case 2: ++g_tally, mgk::k_pack<2><<<g, 256, 0, c->stream>>>(ns, h.send_idx.p, v, h.sendbuf.p); break;
      case 3: ++g_tally, mgk::k_pack<3><<<g, 256, 0, c->stream>>>(ns, h.send_idx.p, v, h.sendbuf.p); break;
      case 4: ++g_tally, mgk::k_pack<4><<<g, 256, 0, c->stream>>>(ns, h.send_idx.p, v, h.sendbuf.p); break;
      default: ++g_tally, mgk::k_pack<6><<<g, 256, 0, c->stream>>>(ns, h.send_idx.p, v, h.sendbuf.p); break;
    }
    TRY(check_launch("halo pack"));
  }
  return MG_OK;
}

mg_status halo_exchange(mg_ctx_s *c, Halo &h, const double *v) {
  if (!h.active) return MG_OK;
  mark(c, 100 + c->cur_level);
  struct Back {
    mg_ctx_s *c;
    ~Back() { mark(c, c->cur_level); }
  } back{c};
  TRY(halo_pack(c, h, v));
  return c->tr->exchange(h.pat, c->bs(), h.sendbuf.p, h.ghost.p, c->stream);
}

// Build a halo from sorted unique ghost global rows of a level with ranges
// `bounds`; my owned rows there start at `row_begin`.  Collective.
mg_status build_halo(mg_ctx_s *c, Halo &h, const std::vector<int64_t> &ghosts, const std::vector<int64_t> &bounds,
                     int64_t row_begin, int64_t row_end) {
  const int P = c->nranks(), me = c->rank();
  h = Halo();
  h.active = true;
  h.n_ghost = int64_t(ghosts.size());
  std::vector<std::vector<char>> out(P), in;
  std::vector<std::vector<int64_t>> req(P);
  for (int64_t g : ghosts) {
    const int o = mgi_owner(g, bounds.data(), P);
    if (o < 0 || o >= P || o == me) return fail(MG_ERR_STRUCTURE, "ghost %lld has no owner", (long long)g);
    req[o].push_back(g);
  }
  int64_t off = 0;
  for (int r = 0; r < P; ++r) {
    if (req[r].empty()) continue;
    h.pat.recv_rank.push_back(r);
    h.pat.recv_off.push_back(off);
    h.pat.recv_cnt.push_back(int64_t(req[r].size()));
    off += int64_t(req[r].size());
    out[r].resize(req[r].size() * sizeof(int64_t));
    std::memcpy(out[r].data(), req[r].data(), out[r].size());
  }
  h.pat.n_recv = off;
  TRY(c->tr->alltoallv_host(out, in));
  std::vector<int32_t> idx;
  for (int r = 0; r < P; ++r) {
    const int64_t cnt = int64_t(in[r].size() / sizeof(int64_t));
    if (!cnt) continue;
    const int64_t *g = reinterpret_cast<const int64_t *>(in[r].data());
    h.pat.send_rank.push_back(r);
    h.pat.send_off.push_back(int64_t(idx.size()));
    h.pat.send_cnt.push_back(cnt);
    for (int64_t k = 0; k < cnt; ++k) {
      if (g[k] < row_begin || g[k] >= row_end) return fail(MG_ERR_STRUCTURE, "halo request for a row not owned");
      idx.push_back(int32_t(g[k] - row_begin));
    }
  }
  h.pat.n_send = int64_t(idx.size());
  TRY(h.send_idx.upload(idx.data(), idx.size()));
  TRY(h.sendbuf.alloc(size_t(std::max<int64_t>(1, h.pat.n_send)) * c->bs()));
  TRY(h.ghost.alloc(size_t(std::max<int64_t>(1, h.n_ghost)) * c->bs()));
  return MG_OK;
}

// Renumber the global columns of a local operator (rows: rp.size()-1) whose
// column space is a level owned here as [rb, re) into owned + ghost (sorted).
mg_status localize(int64_t rb, int64_t re, const std::vector<int64_t> &rp, std::vector<int64_t> &col,
                   std::vector<int64_t> &ghosts) {
  const int64_t nnz = int64_t(col.size());
  std::vector<int64_t> loc(std::max<int64_t>(1, nnz)), gh(std::max<int64_t>(1, nnz));
  int64_t ng = 0;
  mgi_localize_columns(int64_t(rp.size()) - 1, rb, re, rp.data(), col.data(), loc.data(), gh.data(), &ng);
  loc.resize(nnz);
  ghosts.assign(gh.begin(), gh.begin() + ng);
  col.swap(loc);
  return MG_OK;
}

// --- reductions (deterministic; all-reduced over ranks on distributed levels) ---
unsigned red_grid(const mg_ctx_s *c, int64_t n) {
  const int64_t want = (n + mgk::kRedThreads * 8 - 1) / (mgk::kRedThreads * 8);
  return unsigned(std::max<int64_t>(1, std::min<int64_t>(want, 4 * c->n_sm)));
}

mg_status finish_reduce(mg_ctx_s *c, bool dist, double *res, bool sqrt_, double *copy = nullptr) {
  if (!dist) {
    if (copy) CU(cudaMemcpyAsync(copy, res, sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    return MG_OK;
  }
  TRY(c->tr->allreduce_sum(res, 1, c->stream));
  if (sqrt_) {
    ++g_tally, mgk::k_sqrt_copy<<<1, 32, 0, c->stream>>>(res, copy);
    return check_launch("sqrt");
  }
  if (copy) CU(cudaMemcpyAsync(copy, res, sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  return MG_OK;
}

inline bool al16(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

template <int MODE>
void launch_reduce(mg_ctx_s *c, bool sq, bool vec, int64_t n, double *a, const double *b, const double *v,
                   const double *h, double *res, bool rev = false) {
  const unsigned g = red_grid(c, n);
  auto *P = c->red_part.p;
  auto *T = c->ticket.p;
  if (vec && rev) {
    if (sq) ++g_tally, mgk::k_reduce<MODE, true, true, true><<<g, mgk::kRedThreads, 0, c->stream>>>(n, a, b, v, h, P, T, res, nullptr);
    else ++g_tally, mgk::k_reduce<MODE, false, true, true><<<g, mgk::kRedThreads, 0, c->stream>>>(n, a, b, v, h, P, T, res, nullptr);
  } else if (sq && vec) ++g_tally, mgk::k_reduce<MODE, true, true><<<g, mgk::kRedThreads, 0, c->stream>>>(n, a, b, v, h, P, T, res, nullptr);
  else if (sq) ++g_tally, mgk::k_reduce<MODE, true, false><<<g, mgk::kRedThreads, 0, c->stream>>>(n, a, b, v, h, P, T, res, nullptr);
  else if (vec) ++g_tally, mgk::k_reduce<MODE, false, true><<<g, mgk::kRedThreads, 0, c->stream>>>(n, a, b, v, h, P, T, res, nullptr);
  else ++g_tally, mgk::k_reduce<MODE, false, false><<<g, mgk::kRedThreads, 0, c->stream>>>(n, a, b, v, h, P, T, res, nullptr);
}

// res (device) = (a, b) [sqrt] over the level's rows (all ranks if dist)
mg_status dev_dot(mg_ctx_s *c, bool dist, int64_t n, const double *a, const double *b, double *res, bool sqrt_,
                  bool rev = false) {
  const bool vec = al16(a) && al16(b);
  launch_reduce<0>(c, sqrt_ && !dist, vec, n, const_cast<double *>(a), b, nullptr, nullptr, res, rev);
  TRY(check_launch("dot"));
  return finish_reduce(c, dist, res, sqrt_);
}

// MGS step: a -= (*h) v ; res = (a, u), or ||a|| when u == nullptr
mg_status dev_axpy_dot(mg_ctx_s *c, bool dist, int64_t n, double *a, const double *v, const double *h,
                       const double *u, double *res, bool rev = false) {
  const bool vec = al16(a) && al16(v) && (!u || al16(u));
  launch_reduce<1>(c, u == nullptr && !dist, vec, n, a, u, v, h, res, rev);
  TRY(check_launch("axpy-dot"));
  return finish_reduce(c, dist, res, u == nullptr);
}

// --- DCGS2 passes (MG_GMRES_DCGS2): grid = resident CTAs of the bucket's kernel
template <int JB>
unsigned dcgs_grid(const mg_ctx_s *c, const void *k, int64_t n) {
  int bl = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bl, k, mgk::kRedThreads, 0);
  const int64_t want = (n / 2 + mgk::kRedThreads - 1) / mgk::kRedThreads;
  return unsigned(std::max<int64_t>(1, std::min<int64_t>(want, int64_t(std::max(1, std::min(bl, 4))) * c->n_sm)));
}

// Three implementations of the two DCGS2 passes (MGB200_DCGS_KERNEL):
//   auto (default): reg for j < 8, ws from j = 8 on;
//   ws:  warp-split -- warp w owns vectors w, w + 8, ...; 2 ceil(j/8)
//       accumulators per thread, full occupancy (k_dcgs_*_ws);
//   reg: every thread accumulates all 2j + 2 dots (k_dcgs_*; 220 registers at
//       j = 16, one CTA per SM, 4.2-4.6 TB/s on C3);
//   tma: tiles of the j + 2 vectors staged through a shared-memory ring by bulk
//       copies (k_dcgs_*_tma; same speed as reg on C3, and with >= 160 KB of
//       dynamic shared memory it fails to launch under Nsight Compute).
int dcgs_kernel() {  // read at every launch (captured graphs keep the kernels they were built with)
  const char *e = std::getenv("MGB200_DCGS_KERNEL");
  if (e && std::strcmp(e, "reg") == 0) return 1;
  if (e && std::strcmp(e, "tma") == 0) return 2;
  if (e && std::strcmp(e, "ws") == 0) return 3;
  return 0;
}
bool dcgs_tma() { return dcgs_kernel() == 2; }

template <int VPW>
void dcgs_launch_ws(mg_ctx_s *c, bool update, int64_t n, int j, double *Q, int64_t ldq) {
  const mgk::GmresDev &g = c->gm;
  const void *k = update ? reinterpret_cast<const void *>(mgk::k_dcgs_update_ws<VPW>)
                         : reinterpret_cast<const void *>(mgk::k_dcgs_dots_ws<VPW>);
  int bl = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bl, k, mgk::kRedThreads, 0);
  const int64_t ntiles = (n / 2 + 32 * mgk::kDcgsU - 1) / (32 * mgk::kDcgsU);
  const unsigned gr = unsigned(std::max<int64_t>(
      1, std::min<int64_t>(ntiles, int64_t(std::max(1, std::min(bl, 4))) * c->n_sm)));
  if (!update)
    ++g_tally, mgk::k_dcgs_dots_ws<VPW><<<gr, mgk::kRedThreads, 0, c->stream>>>(n, j, Q, ldq, c->dcgs_part.p,
                                                                                 c->dcgs_ticket.p, g.dots);
  else
    ++g_tally, mgk::k_dcgs_update_ws<VPW><<<gr, mgk::kRedThreads, 0, c->stream>>>(
                   n, j, Q, ldq, g.coef, g.dead, c->dcgs_part.p, c->dcgs_ticket.p, g.nu1);
}

template <int JB>
void dcgs_launch(mg_ctx_s *c, bool update, int64_t n, int j, double *Q, int64_t ldq) {
  const mgk::GmresDev &g = c->gm;
  if (dcgs_tma()) {
    // ring: up to 4 stages of tiles of T doubles of the j + 2 vectors in ~200 KB
    const int nv = j + 2;
    const size_t budget = size_t(160) << 10;  // leaves room for tools that reserve shared memory
    int T = 256 * std::max(1, int(budget / (size_t(4) * nv * 8 * 256)));
    T = std::min(T, 2048);
    const int nst = std::max(1, std::min(4, int(budget / (size_t(nv) * 8 * size_t(T)))));
    const size_t smem = size_t(nst) * nv * T * sizeof(double) + size_t(nst) * sizeof(uint64_t);
    const int64_t ntiles = (n + T - 1) / T;
    const unsigned gr = unsigned(std::max<int64_t>(1, std::min<int64_t>(ntiles, c->n_sm)));
    if (!update) {
      cudaFuncSetAttribute(mgk::k_dcgs_dots_tma<JB>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      ++g_tally, mgk::k_dcgs_dots_tma<JB><<<gr, mgk::kRedThreads, smem, c->stream>>>(
                     n, j, Q, ldq, nst, T, c->dcgs_part.p, c->dcgs_ticket.p, g.dots);
    } else {
      cudaFuncSetAttribute(mgk::k_dcgs_update_tma<JB>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
      ++g_tally, mgk::k_dcgs_update_tma<JB><<<gr, mgk::kRedThreads, smem, c->stream>>>(
                     n, j, Q, ldq, nst, T, g.coef, g.dead, c->dcgs_part.p, c->dcgs_ticket.p, g.nu1);
    }
    return;
  }
  if (!update) {
    const unsigned gr = dcgs_grid<JB>(c, reinterpret_cast<const void *>(mgk::k_dcgs_dots<JB>), n);
    ++g_tally, mgk::k_dcgs_dots<JB><<<gr, mgk::kRedThreads, 0, c->stream>>>(n, j, Q, ldq, c->dcgs_part.p,
                                                                             c->dcgs_ticket.p, g.dots);
  } else {
    const unsigned gr = dcgs_grid<JB>(c, reinterpret_cast<const void *>(mgk::k_dcgs_update<JB>), n);
    ++g_tally, mgk::k_dcgs_update<JB><<<gr, mgk::kRedThreads, 0, c->stream>>>(n, j, Q, ldq, g.coef, g.dead,
                                                                               c->dcgs_part.p, c->dcgs_ticket.p, g.nu1);
  }
}

// one DCGS2 pass of Arnoldi step j (bucketed on j so the j accumulators live in registers)
mg_status dcgs_pass(mg_ctx_s *c, bool dist, bool update, int64_t n, int j, double *Q, int64_t ldq) {
  // default: per-thread accumulators while they are few (j < 8: <= 18 of them),
  // warp-split beyond (measured same box: C3 DCGS2 solve 112.8 -> 112.3 ms with
  // warp-split at j >= 8, C2 2.87 -> 2.97 ms when small j also ran warp-split,
  // its idle warps at j < 8)
  // (the warp-split update also for 2 <= j < 8 was measured: C3 unchanged, C2 2.85 -> 2.89 ms)
  if ((dcgs_kernel() == 0 && j >= 8) || dcgs_kernel() == 3) {
    if (j <= 8) dcgs_launch_ws<1>(c, update, n, j, Q, ldq);
    else if (j <= 16) dcgs_launch_ws<2>(c, update, n, j, Q, ldq);
    else if (j <= 32) dcgs_launch_ws<4>(c, update, n, j, Q, ldq);
    else if (j <= 64) dcgs_launch_ws<8>(c, update, n, j, Q, ldq);
    else return fail(MG_ERR_INVALID_ARG, "DCGS2: restart %d > 64", j);
  } else if (j < 2) dcgs_launch<2>(c, update, n, j, Q, ldq);
  else if (j < 4) dcgs_launch<4>(c, update, n, j, Q, ldq);
  else if (j < 8) dcgs_launch<8>(c, update, n, j, Q, ldq);
  else if (j < 16) dcgs_launch<16>(c, update, n, j, Q, ldq);
  else if (j < 32) dcgs_launch<32>(c, update, n, j, Q, ldq);
  else if (j < 64) dcgs_launch<64>(c, update, n, j, Q, ldq);
  else return fail(MG_ERR_INVALID_ARG, "DCGS2: restart %d > 64", j);
  TRY(check_launch(update ? "dcgs update" : "dcgs dots"));
  if (dist) TRY(c->tr->allreduce_sum(update ? c->gm.nu1 : c->gm.dots, update ? 1 : 2 * j + 2, c->stream));
  return MG_OK;
}

// --- dense coarse inverse on the device (in-place Gauss-Jordan, partial pivoting)
__global__ void k_gj_pivot(int64_t N, int64_t ld, double *a, int64_t k, int64_t *piv, double *f, int *singular) {
  __shared__ double bv[1024];
  __shared__ int64_t bi[1024];
  double best = -1.0;
  int64_t bidx = k;
  for (int64_t r = k + threadIdx.x; r < N; r += blockDim.x) {
    const double v = fabs(a[r * ld + k]);
    if (v > best) {
      best = v;
      bidx = r;
    }
  }
  bv[threadIdx.x] = best;
  bi[threadIdx.x] = bidx;
  __syncthreads();
  for (int s = blockDim.x / 2; s > 0; s >>= 1) {
    if (threadIdx.x < s) {
      const double v2 = bv[threadIdx.x + s];
      const int64_t i2 = bi[threadIdx.x + s];
      if (v2 > bv[threadIdx.x] || (v2 == bv[threadIdx.x] && i2 < bi[threadIdx.x])) {
        bv[threadIdx.x] = v2;
        bi[threadIdx.x] = i2;
      }
    }
    __syncthreads();
  }
  const int64_t p = bi[0];
  const double pmax = bv[0];
  if (!(pmax > 0.0)) {
    if (threadIdx.x == 0) *singular = 1;
    return;
  }
  if (threadIdx.x == 0) piv[k] = p;
  if (p != k)
    for (int64_t c = threadIdx.x; c < N; c += blockDim.x) {
      const double t = a[k * ld + c];
      a[k * ld + c] = a[p * ld + c];
      a[p * ld + c] = t;
    }
  __syncthreads();
  const double d = a[k * ld + k];
  __syncthreads();
  if (threadIdx.x == 0) a[k * ld + k] = 1.0;
  __syncthreads();
  for (int64_t c = threadIdx.x; c < N; c += blockDim.x) a[k * ld + c] /= d;
  for (int64_t r = threadIdx.x; r < N; r += blockDim.x) {
    if (r == k) {
      f[r] = 0.0;
      continue;
    }
    f[r] = a[r * ld + k];
    a[r * ld + k] = 0.0;
  }
}

__global__ void k_gj_eliminate(int64_t N, int64_t ld, double *a, int64_t k, const double *f) {
  const int64_t r = blockIdx.y;
  const double fr = f[r];
  if (r == k || fr == 0.0) return;
  const double *ak = a + k * ld;
  double *ar = a + r * ld;
  for (int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; c < N; c += int64_t(gridDim.x) * blockDim.x)
    ar[c] = fma(-fr, ak[c], ar[c]);
}

__global__ void k_gj_unswap(int64_t N, int64_t ld, double *a, const int64_t *piv) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= N) return;
  double *ar = a + r * ld;
  for (int64_t k = N - 1; k >= 0; --k) {
    const int64_t p = piv[k];
    if (p != k) {
      const double t = ar[k];
      ar[k] = ar[p];
      ar[p] = t;
    }
  }
}

// in-place Gauss-Jordan inversion of the dense coarse matrix held in c->cinv
mg_status coarse_gj(mg_ctx_s *c, int64_t N, int64_t ld);

// A_0 += alpha w w^T when level 0 carries a global constraint (reading Z25)
mg_status coarse_regularise(mg_ctx_s *c, int64_t N, int64_t ld) {
  Level &L0 = c->lv[0];
  if (!L0.mean || N == 0) return MG_OK;
  if (!c->scal.p) TRY(c->scal.alloc(16));
  mgk::k_diag_absmax<<<1, 1024, 0, c->stream>>>(N, ld, c->cinv.p, c->scal.p + 9);
  const unsigned g = unsigned(std::min<int64_t>((N * N + 255) / 256, 16 * c->n_sm));
  mgk::k_rank1_reg<<<g, 256, 0, c->stream>>>(N, ld, c->cinv.p, L0.mean_w.p, c->scal.p + 9, L0.mean_wmax);
  return check_launch("coarse regularisation");
}

mg_status build_coarse_inverse(mg_ctx_s *c) {
  Level &L0 = c->lv[0];
  const int bs = c->bs();
  const int64_t N = L0.n * bs;
  const int64_t ld = (N + 1) & ~int64_t(1);
  std::vector<double> dense(size_t(N) * N);
  mgi_bsr_to_dense(L0.n, bs, L0.rp0.data(), L0.col0.data(), L0.val0.data(), dense.data());
  std::vector<double> padded(size_t(N) * ld, 0.0);
  for (int64_t r = 0; r < N; ++r) std::memcpy(&padded[r * ld], &dense[r * N], N * sizeof(double));
  TRY(c->cinv.upload(padded.data(), padded.size()));
  TRY(coarse_regularise(c, N, ld));
  return coarse_gj(c, N, ld);
}

mg_status coarse_gj(mg_ctx_s *c, int64_t N, int64_t ld) {
  DevArray<int64_t> piv;
  DevArray<double> f;
  DevArray<int> sing;
  TRY(piv.alloc(N));
  TRY(f.alloc(N));
  TRY(sing.alloc(1));
  CU(cudaMemsetAsync(sing.p, 0, sizeof(int), c->stream));
  const unsigned gx = unsigned(std::min<int64_t>((N + 255) / 256, 64));
  for (int64_t k = 0; k < N; ++k) {
    k_gj_pivot<<<1, 1024, 0, c->stream>>>(N, ld, c->cinv.p, k, piv.p, f.p, sing.p);
    k_gj_eliminate<<<dim3(gx, unsigned(N)), 256, 0, c->stream>>>(N, ld, c->cinv.p, k, f.p);
  }
  k_gj_unswap<<<unsigned((N + 255) / 256), 256, 0, c->stream>>>(N, ld, c->cinv.p, piv.p);
  TRY(check_launch("coarse inverse"));
  int s = 0;
  CU(cudaMemcpyAsync(&s, sing.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  if (s) return fail(MG_ERR_SINGULAR, "coarse matrix A_0 is singular");
  c->cN = N;
  c->cld = ld;
  return MG_OK;
}

// sliced D^-1 from row-major blocks (lane order = each part's perm; perm holds
// the level's local row ids)
mg_status upload_dinv(Level &L, int bs, const std::vector<double> &blocks) {
  const int V = bs * bs;
  for (int pi = 0; pi < L.nparts; ++pi) {
    Level::Part &Pt = L.part[pi];
    const int64_t ns = Pt.A.n_slices;
    std::vector<double> sl(size_t(std::max<int64_t>(1, ns)) * 32 * V, 0.0);
    for (int64_t s = 0; s < ns; ++s)
      for (int lane = 0; lane < 32; ++lane) {
        const int32_t r = Pt.A.perm_host[s * 32 + lane];
        if (r < 0) continue;
        double *base = &sl[size_t(s) * 32 * V];
        const double *src = &blocks[size_t(r) * V];
        for (int j = 0; j < V / 2; ++j) {
          base[64 * j + 2 * lane] = src[2 * j];
          base[64 * j + 2 * lane + 1] = src[2 * j + 1];
        }
        if (V & 1) base[64 * (V / 2) + lane] = src[V - 1];
      }
    TRY(Pt.dinv.upload(sl.data(), sl.size()));
  }
  L.dinv_ready = true;
  return MG_OK;
}

// D^-1 of the level's diagonal blocks on the device (from the V-cycle operator's
// values: fp32-rounded in mixed precision), per part.  Synchronises.
mg_status device_dinv(mg_ctx_s *c, int l) {
  Level &L = c->lv[l];
  const int bs = c->bs(), V = bs * bs;
  DevArray<int> flag;
  TRY(flag.alloc(1));
  CU(cudaMemsetAsync(flag.p, 0, sizeof(int), c->stream));
  for (int pi = 0; pi < L.nparts; ++pi) {
    Level::Part &Pt = L.part[pi];
    const size_t need = size_t(std::max<int64_t>(1, Pt.A.n_slices)) * 32 * V;
    if (Pt.dinv.n < need) TRY(Pt.dinv.alloc(need));
    CU(cudaMemsetAsync(Pt.dinv.p, 0, Pt.dinv.n * sizeof(double), c->stream));
    if (Pt.n == 0) continue;
    const unsigned g = unsigned(std::min<int64_t>((Pt.n + 255) / 256, 16 * c->n_sm));
    const double *v64 = Pt.A.f32 ? nullptr : Pt.A.val.p;
    const float *v32 = Pt.A.f32 ? Pt.A.valf.p : nullptr;
    switch (bs) {
      case 1: mgk::k_block_inverse<1><<<g, 256, 0, c->stream>>>(Pt.n, Pt.udiag_e.p, v64, v32, Pt.upos.p, Pt.dinv.p, flag.p); break;
      case 2: mgk::k_block_inverse<2><<<g, 256, 0, c->stream>>>(Pt.n, Pt.udiag_e.p, v64, v32, Pt.upos.p, Pt.dinv.p, flag.p); break;
      case 3: mgk::k_block_inverse<3><<<g, 256, 0, c->stream>>>(Pt.n, Pt.udiag_e.p, v64, v32, Pt.upos.p, Pt.dinv.p, flag.p); break;
      case 4: mgk::k_block_inverse<4><<<g, 256, 0, c->stream>>>(Pt.n, Pt.udiag_e.p, v64, v32, Pt.upos.p, Pt.dinv.p, flag.p); break;
      default: mgk::k_block_inverse<6><<<g, 256, 0, c->stream>>>(Pt.n, Pt.udiag_e.p, v64, v32, Pt.upos.p, Pt.dinv.p, flag.p); break;
    }
    TRY(check_launch("block inverse"));
  }
  int f = 0;
  CU(cudaMemcpyAsync(&f, flag.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  if (f & 2) return fail(MG_ERR_SINGULAR, "level %d: singular diagonal block", l);
  L.dinv_ready = true;
  return MG_OK;
}

// Vanka patch inverses from the V-cycle operator's values (fp32-rounded in
// mixed precision), on the device.  Synchronises.
mg_status vanka_build(mg_ctx_s *c, int l) {
  Level &L = c->lv[l];
  Level::Vanka &V = L.vk;
  Level::Part &Pt = L.part[0];
  const int bs = c->bs();
  if (V.np == 0) {
    V.ready = true;
    return MG_OK;
  }
  if (V.ent.n < size_t(V.np) * V.nl * V.nl) {
    TRY(V.ent.alloc(size_t(V.np) * V.nl * V.nl));
    const unsigned g = unsigned(std::min<int64_t>((V.np * V.nl + 255) / 256, 16 * c->n_sm));
    ++g_tally, mgk::k_vanka_find<<<g, 256, 0, c->stream>>>(V.np, V.nl, V.nodes.p, Pt.A.slice_ptr.p, Pt.A.col.p,
                                                           Pt.upos.p, V.ent.p);
    TRY(check_launch("vanka find"));
  }
  DevArray<int> flag;
  TRY(flag.alloc(1));
  CU(cudaMemsetAsync(flag.p, 0, sizeof(int), c->stream));
  const unsigned g = unsigned((V.np + mgk::kVankaWarps - 1) / mgk::kVankaWarps);
  const double *v64 = Pt.A.f32 ? nullptr : Pt.A.val.p;
  const float *v32 = Pt.A.f32 ? Pt.A.valf.p : nullptr;
  switch (bs) {
    case 1: ++g_tally, mgk::k_vanka_build<1><<<g, 32 * mgk::kVankaWarps, 0, c->stream>>>(V.np, V.nl, V.ent.p, v64, v32, V.ppw, V.inv.p, flag.p); break;
    case 2: ++g_tally, mgk::k_vanka_build<2><<<g, 32 * mgk::kVankaWarps, 0, c->stream>>>(V.np, V.nl, V.ent.p, v64, v32, V.ppw, V.inv.p, flag.p); break;
    case 3: ++g_tally, mgk::k_vanka_build<3><<<g, 32 * mgk::kVankaWarps, 0, c->stream>>>(V.np, V.nl, V.ent.p, v64, v32, V.ppw, V.inv.p, flag.p); break;
    case 4: ++g_tally, mgk::k_vanka_build<4><<<g, 32 * mgk::kVankaWarps, 0, c->stream>>>(V.np, V.nl, V.ent.p, v64, v32, V.ppw, V.inv.p, flag.p); break;
    default: ++g_tally, mgk::k_vanka_build<6><<<g, 32 * mgk::kVankaWarps, 0, c->stream>>>(V.np, V.nl, V.ent.p, v64, v32, V.ppw, V.inv.p, flag.p); break;
  }
  TRY(check_launch("vanka build"));
  int f = 0;
  CU(cudaMemcpyAsync(&f, flag.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  if (f & 2) return fail(MG_ERR_SINGULAR, "level %d: singular Vanka patch matrix", l);
  V.ready = true;
  return MG_OK;
}

// One Vanka sweep x <- x + omega sum_p R_p^T W A_pp^{-1} R_p (b - A x); zero: x enters as 0.
mg_status vanka_sweep(mg_ctx_s *c, int l, double *x, const double *b, bool zero);

double lv_omega(const mg_ctx_s *c, const Level &L) { return L.omega > 0.0 ? L.omega : c->cfg.omega; }
int lv_nu_pre(const mg_ctx_s *c, const Level &L) { return L.nu_pre >= 0 ? L.nu_pre : c->cfg.nu_pre; }
int lv_nu_post(const mg_ctx_s *c, const Level &L) { return L.nu_post >= 0 ? L.nu_post : c->cfg.nu_post; }

// --- persistent coarse tail ----------------------------------------------------
template <int BS>
mg_status tail_grid_size(mg_ctx_s *c) {
  if (c->tail_cluster) {
    // one cluster: 16 CTAs (non-portable size, opt-in) or the portable 8
    cudaError_t e = cudaFuncSetAttribute(mgk::k_tail<BS, true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    c->tail_grid = e == cudaSuccess ? 16 : 8;
    cudaGetLastError();
    return MG_OK;
  }
  int per_sm = 0;
  CU(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mgk::k_tail<BS, false>, mgk::kCta, 0));
  const int want = int(env_i64("MGB200_TAIL_CTAS", per_sm));
  c->tail_grid = unsigned(std::max(1, std::min(per_sm, want)) * c->n_sm);
  return MG_OK;
}

// Tail level T: the highest level below the finest whose levels 0..T all use
// split-k 4 (few slices) and are not distributed; T >= 1.  MGB200_TAIL=0
// disables the tail (standalone kernels only).
mg_status build_tail(mg_ctx_s *c) {
  c->tail_nops = 0;
  c->tail_T = -1;
  // MGB200_TAIL (opt-in, both measured slower than the graph-launched standalone
  // kernels on B200): "1" -- grid-wide cooperative variant (grid barriers cost
  // more than CUDA-graph kernel boundaries: C2 0.39 vs 0.35 ms per V-cycle);
  // "c" -- tiny levels in one thread-block cluster with hardware cluster
  // barriers (16 SMs lack the latency hiding of the whole GPU: C2 0.44 vs
  // 0.32 ms, C1 47 vs 43 us).  Default off.
  const char *env = std::getenv("MGB200_TAIL");
  const char mode = env && *env ? env[0] : '0';
  if (mode != '1' && mode != 'c') return MG_OK;
  for (const Level &L : c->lv)
    if (L.mean || L.vk.on) return MG_OK;  // the tail has no projection / Vanka step
  c->tail_cluster = mode == 'c';
  const int64_t max_slices = env_i64("MGB200_TAIL_SLICES", c->tail_cluster ? 256 : 1024);
  int T = -1;
  for (int l = 0; l < c->L(); ++l) {
    const Level &L = c->lv[l];
    const int ks = L.part[0].A.ks;
    if (L.dist || (ks != 4 && ks != 8) || (l > 0 && c->lv[l].R.ks != 4) || L.part[0].A.n_slices > max_slices) break;
    T = l;
  }
  if (T < 1) return MG_OK;
  const int bs = c->bs();
  std::vector<mgk::TailOp> ops;
  auto base = [&](int type) {
    mgk::TailOp o{};
    o.type = type;
    return o;
  };
  auto emit_smooth = [&](int l, double *x, const double *b, int k, bool zero) {
    Level &L = c->lv[l];
    const double om = lv_omega(c, L);
    if (k <= 0) {
      if (zero) {
        mgk::TailOp o = base(mgk::T_ZERO);
        o.out = x;
        o.n = L.n * bs;
        ops.push_back(o);
      }
      return;
    }
    if (zero) {
      mgk::TailOp o = base(mgk::T_SWEEP0);
      o.A = L.part[0].A.view();
      o.dinv = L.part[0].dinv.p;
      o.b = b;
      o.out = x;
      o.alpha = om;
      ops.push_back(o);
      --k;
    }
    double *src = x, *dst = L.w.p;
    for (int i = 0; i < k; ++i) {
      mgk::TailOp o = base(mgk::T_SWEEP);
      o.A = L.part[0].A.view();
      o.ks = L.part[0].A.ks;
      o.f32 = L.part[0].A.f32;
      o.x = src;
      o.b = b;
      o.dinv = L.part[0].dinv.p;
      o.out = dst;
      o.alpha = om;
      ops.push_back(o);
      std::swap(src, dst);
    }
    if (src != x) {
      mgk::TailOp o = base(mgk::T_COPY);
      o.x = src;
      o.out = x;
      o.n = L.n * bs;
      ops.push_back(o);
    }
  };
  for (int l = T; l >= 1; --l) {
    Level &L = c->lv[l];
    emit_smooth(l, L.x.p, L.b.p, lv_nu_pre(c, L), true);
    mgk::TailOp r = base(mgk::T_RESID);
    r.A = L.part[0].A.view();
    r.ks = L.part[0].A.ks;
    r.f32 = L.part[0].A.f32;
    r.x = L.x.p;
    r.b = L.b.p;
    r.out = L.w.p;
    r.alpha = 1.0;
    ops.push_back(r);
    mgk::TailOp t = base(mgk::T_RESTRICT);
    t.A = L.R.view();
    t.wpe = L.R.vpe;
    t.ks = L.Rt.set ? L.Rt.ks : 4;  // the standalone restriction's split factor
    t.x = L.w.p;
    t.out = c->lv[l - 1].b.p;
    ops.push_back(t);
  }
  if (c->cfg.coarse_mode == MG_COARSE_DIRECT) {
    mgk::TailOp g = base(mgk::T_GEMV);
    g.ks = al16(c->lv[0].b.p) ? 4 : 1;  // as coarse_solve: split kernel when d is 16-byte aligned
    g.dinv = c->cinv.p;
    g.b = c->lv[0].b.p;
    g.out = c->lv[0].x.p;
    g.n = c->cN;
    g.ld = c->cld;
    ops.push_back(g);
  } else {
    emit_smooth(0, c->lv[0].x.p, c->lv[0].b.p, std::max(1, c->cfg.coarse_sweeps), true);
  }
  for (int l = 1; l <= T; ++l) {
    Level &L = c->lv[l];
    mgk::TailOp pr = base(mgk::T_PROLONG);
    pr.A = L.P.view();
    pr.wpe = L.P.vpe;
    pr.x = c->lv[l - 1].x.p;
    pr.out = L.x.p;
    ops.push_back(pr);
    emit_smooth(l, L.x.p, L.b.p, lv_nu_post(c, L), false);
  }
  TRY(c->tail_ops.upload(ops.data(), ops.size()));
  c->tail_nops = int(ops.size());
  c->tail_T = T;
  switch (bs) {
    case 1: TRY(tail_grid_size<1>(c)); break;
    case 2: TRY(tail_grid_size<2>(c)); break;
    case 3: TRY(tail_grid_size<3>(c)); break;
    case 4: TRY(tail_grid_size<4>(c)); break;
    default: TRY(tail_grid_size<6>(c)); break;
  }
  return MG_OK;
}

mg_status launch_tail(mg_ctx_s *c) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(c->tail_grid);
  cfg.blockDim = dim3(mgk::kCta);
  cfg.stream = c->stream;
  cudaLaunchAttribute attr[1];
  if (c->tail_cluster) {
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = c->tail_grid;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
  } else {
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  const mgk::TailOp *ops = c->tail_ops.p;
  const int n = c->tail_nops;
  ++g_tally;
  const bool cl = c->tail_cluster;
  switch (c->bs()) {
    case 1: CU(cl ? cudaLaunchKernelEx(&cfg, mgk::k_tail<1, true>, ops, n) : cudaLaunchKernelEx(&cfg, mgk::k_tail<1, false>, ops, n)); break;
    case 2: CU(cl ? cudaLaunchKernelEx(&cfg, mgk::k_tail<2, true>, ops, n) : cudaLaunchKernelEx(&cfg, mgk::k_tail<2, false>, ops, n)); break;
    case 3: CU(cl ? cudaLaunchKernelEx(&cfg, mgk::k_tail<3, true>, ops, n) : cudaLaunchKernelEx(&cfg, mgk::k_tail<3, false>, ops, n)); break;
    case 4: CU(cl ? cudaLaunchKernelEx(&cfg, mgk::k_tail<4, true>, ops, n) : cudaLaunchKernelEx(&cfg, mgk::k_tail<4, false>, ops, n)); break;
    default: CU(cl ? cudaLaunchKernelEx(&cfg, mgk::k_tail<6, true>, ops, n) : cudaLaunchKernelEx(&cfg, mgk::k_tail<6, false>, ops, n)); break;
  }
  return MG_OK;
}

mg_status finalize(mg_ctx_s *c) {
  if (c->finalized) return MG_OK;
  const int bs = c->bs();
  for (int l = 0; l <= c->L(); ++l) {
    Level &L = c->lv[l];
    if (!L.declared) return fail(MG_ERR_STATE, "level %d not created (mg_create_level)", l);
    if (!L.part[0].A.set) return fail(MG_ERR_STATE, "level %d has no matrix (mg_set_matrix)", l);
    if (l > 0 && !L.P.set) return fail(MG_ERR_STATE, "level %d has no transfer (mg_set_transfer)", l);
  }
  if (c->cfg.coarse_mode == MG_COARSE_DIRECT && c->lv[0].dist)
    return fail(MG_ERR_INVALID_ARG, "direct coarse solve needs a replicated level 0");
  for (int l = 0; l < c->L(); ++l)
    if (c->lv[l].dist && !c->lv[l + 1].dist)
      return fail(MG_ERR_INVALID_ARG, "level %d is distributed below replicated level %d", l, l + 1);
  for (int l = 0; l <= c->L(); ++l) {
    Level &L = c->lv[l];
    if (!L.dinv_ready) {
      if (!L.dinv_host.empty()) TRY(upload_dinv(L, bs, L.dinv_host));
      else TRY(device_dinv(c, l));
    }
    if (L.vk.on && !L.vk.ready) TRY(vanka_build(c, l));
    const size_t nv = size_t(std::max<int64_t>(1, L.n)) * bs;
    if (L.w.n < nv) TRY(L.w.alloc(nv));
    if (l < c->L()) {
      if (L.x.n < nv) TRY(L.x.alloc(nv));
      if (L.b.n < nv) TRY(L.b.alloc(nv));
    }
  }
  if (!c->red_part.p) {
    TRY(c->red_part.alloc(4 * c->n_sm + 8));
    TRY(c->ticket.alloc(1));
    CU(cudaMemset(c->ticket.p, 0, sizeof(unsigned)));
  }
  if (c->cfg.coarse_mode == MG_COARSE_DIRECT && c->cN == 0) TRY(build_coarse_inverse(c));
  TRY(build_tail(c));
  if (!c->scal.p) TRY(c->scal.alloc(16));
  for (int l = 0; l <= c->L(); ++l) {
    Level &L = c->lv[l];
    if (!L.mean) continue;
    const int64_t n = L.n * bs;
    TRY(dev_dot(c, L.dist, n, L.mean_w.p, L.mean_k.p, c->scal.p + 10, false));
    TRY(dev_dot(c, L.dist, n, L.mean_k.p, L.mean_k.p, c->scal.p + 11, false));
    double h[2];
    CU(cudaMemcpyAsync(h, c->scal.p + 10, 2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    if (!(h[0] > 0.0) || !(h[1] > 0.0))
      return fail(MG_ERR_INVALID_ARG, "level %d: mean constraint needs w^T k > 0 and k^T k > 0", l);
    L.mean_wk = h[0];
    L.mean_kk = h[1];
  }
  c->finalized = true;
  return MG_OK;
}

// --- V-cycle pieces (stream-ordered; capturable with NCCL / single GPU) ---------
In in_of(Level &L, Halo &h, const double *v) {
  return In{v, h.active ? h.ghost.p : nullptr, int(L.n)};
}

// krylov = true: the problem operator (fp64 A64 on the finest level in mixed
// precision); false: the V-cycle's operator.
const SellOp &op_of(Level::Part &Pt, bool krylov) { return krylov && Pt.A64.set ? Pt.A64 : Pt.A; }

// One A-pass over every part of level l.  Split levels overlap the halo
// exchange (comm stream) with the interior part and run the boundary part after
// the join; single-part levels exchange first (if distributed) and then compute.
template <int OP>
mg_status a_pass(mg_ctx_s *c, int l, const double *x, const double *b, double *out, double alpha, double beta,
                 bool krylov) {
  Level &L = c->lv[l];
  const int bs = c->bs();
  const double om = lv_omega(c, L);
  auto run = [&](Level::Part &Pt, const double *xg) -> mg_status {
    const double *dv = OP == mgk::OP_SWEEP ? Pt.dinv.p : nullptr;
    return launch_apply<OP>(bs, op_of(Pt, krylov), In{x, xg, int(L.n)}, b, dv, out,
                            OP == mgk::OP_SWEEP ? om : alpha, beta, c->stream);
  };
  if (L.nparts == 1) {
    TRY(halo_exchange(c, L.hx, x));
    return run(L.part[0], L.hx.active ? L.hx.ghost.p : nullptr);
  }
  TRY(halo_pack(c, L.hx, x));
  CU(cudaEventRecord(c->ev_fork, c->stream));
  CU(cudaStreamWaitEvent(c->comm_stream, c->ev_fork, 0));
  TRY(c->tr->exchange(L.hx.pat, bs, L.hx.sendbuf.p, L.hx.ghost.p, c->comm_stream));
  CU(cudaEventRecord(c->ev_join, c->comm_stream));
  TRY(run(L.part[0], nullptr));  // interior rows: no ghost columns
  CU(cudaStreamWaitEvent(c->stream, c->ev_join, 0));
  return run(L.part[1], L.hx.ghost.p);
}

mg_status a_pass_sweep(mg_ctx_s *c, int l, const double *src, const double *b, double *dst) {
  return a_pass<mgk::OP_SWEEP>(c, l, src, b, dst, 1.0, 0.0, false);
}

mg_status a_pass_resid(mg_ctx_s *c, int l, const double *x, const double *b, double *r, bool krylov = false) {
  return a_pass<mgk::OP_RESID>(c, l, x, b, r, 1.0, 0.0, krylov);
}

// Is the initial guess x == 0 on every rank?  (one read of x, one 8-byte
// all-reduce, one host sync).  The solve then starts from r = b: the A-pass of
// b - A*0 is skipped (k_nonzero_flag: the result is b exactly).
mg_status zero_guess(mg_ctx_s *c, bool dist, int64_t n, const double *x, bool &zero) {
  if (!c->scal.p) TRY(c->scal.alloc(16));
  double *f = c->scal.p + 13;
  CU(cudaMemsetAsync(f, 0, sizeof(double), c->stream));
  if (n > 0) {
    const unsigned g = unsigned(std::min<int64_t>(std::max<int64_t>(1, (n / 2 + 255) / 256), 4 * c->n_sm));
    ++g_tally, mgk::k_nonzero_flag<<<g, 256, 0, c->stream>>>(n, x, al16(x) ? 1 : 0, f);
    TRY(check_launch("zero-guess test"));
  }
  if (dist) TRY(c->tr->allreduce_sum(f, 1, c->stream));
  CU(cudaMemcpyAsync(c->gm_host + 15, f, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  zero = c->gm_host[15] == 0.0;
  return MG_OK;
}

// r = b - A x, or r = b when x is the zero vector (zero_guess)
mg_status initial_residual(mg_ctx_s *c, int Lf, bool dist, int64_t n, const double *x, const double *b, double *r) {
  bool zero = false;
  // The test costs a host round trip (~30 us): worth it only when the A-pass it may
  // save is large -- decided on the GLOBAL level size, so all ranks agree (measured
  // same box: C3 solve 111.7 -> 110.9 ms; C2 2.93 -> 2.97 ms, hence the threshold).
  // MGB200_ZERO_GUESS=0 / 1: never / always test (A/B experiments).
  const char *e = std::getenv("MGB200_ZERO_GUESS");
  const int64_t big = c->lv[Lf].n_global * c->bs() * c->bs();
  const bool test = e && *e ? e[0] == '1' : big >= (int64_t(1) << 22);
  if (test) TRY(zero_guess(c, dist, n, x, zero));
  if (!zero) return a_pass_resid(c, Lf, x, b, r, true);
  if (n > 0 && r != b) CU(cudaMemcpyAsync(r, b, size_t(n) * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  return MG_OK;
}


mg_status a_pass_spmv(mg_ctx_s *c, int l, double alpha, const double *x, double beta, double *y,
                      bool krylov = false) {
  return a_pass<mgk::OP_SPMV>(c, l, x, nullptr, y, alpha, beta, krylov);
}

// d_coarse = R r_fine (all coarse rows on every rank if the coarse level is replicated)
mg_status do_restrict(mg_ctx_s *c, int l, const double *r, double *d) {
  Level &L = c->lv[l];
  const int bs = c->bs();
  TRY(halo_exchange(c, L.hr, r));
  if (L.Rt.set) TRY(launch_tsell(bs, false, L.Rt, in_of(L, L.hr, r), d + L.r_row0 * bs, c->stream));
  else TRY(launch_transfer(bs, false, L.R, in_of(L, L.hr, r), d + L.r_row0 * bs, c->stream));
  if (L.agglomerate) {
    mark(c, 200 + l);
    TRY(c->tr->allgatherv(d + L.r_row0 * bs, d, L.ag_counts, L.ag_displs, c->stream));
    mark(c, l);
  }
  return MG_OK;
}

// x_fine += P y_coarse
mg_status do_prolong(mg_ctx_s *c, int l, const double *y, double *x) {
  Level &L = c->lv[l];
  Level &C = c->lv[l - 1];
  TRY(halo_exchange(c, L.hp, y));
  const In in{y, L.hp.active ? L.hp.ghost.p : nullptr, int(C.n)};
  if (L.Pc.set) return launch_pcsr(c->bs(), L.Pc, in, x, c->stream);
  if (L.Pt.set) return launch_tsell(c->bs(), true, L.Pt, in, x, c->stream);
  return launch_transfer(c->bs(), true, L.P, in, x, c->stream);
}

mg_status vanka_sweep(mg_ctx_s *c, int l, double *x, const double *b, bool zero) {
  Level &L = c->lv[l];
  Level::Vanka &V = L.vk;
  const int bs = c->bs();
  const double *r = b;
  if (!zero) {
    TRY(a_pass_resid(c, l, x, b, L.w.p));
    r = L.w.p;
  }
  if (V.np) {
    const int64_t warps = (V.np + V.ppw - 1) / V.ppw;
    const unsigned g = unsigned((warps + mgk::kWarpsPerCta - 1) / mgk::kWarpsPerCta);
#define VK_PATCH(B, N) mgk::k_vanka_patch<B, N><<<g, mgk::kCta, 0, c->stream>>>(V.np, V.nl, V.ppw, V.nodes.p, V.inv.p, r, V.cbuf.p)
    const int key = bs * 100 + V.nl;  // compile-time patch sizes for mesh cells (4 / 8 nodes)
    ++g_tally;
    switch (key) {
      case 104: VK_PATCH(1, 4); break;
      case 108: VK_PATCH(1, 8); break;
      case 204: VK_PATCH(2, 4); break;
      case 208: VK_PATCH(2, 8); break;
      case 304: VK_PATCH(3, 4); break;
      case 308: VK_PATCH(3, 8); break;
      case 404: VK_PATCH(4, 4); break;
      case 408: VK_PATCH(4, 8); break;
      case 604: VK_PATCH(6, 4); break;
      default:
        switch (bs) {
          case 1: VK_PATCH(1, 0); break;
          case 2: VK_PATCH(2, 0); break;
          case 3: VK_PATCH(3, 0); break;
          case 4: VK_PATCH(4, 0); break;
          default: VK_PATCH(6, 0); break;
        }
    }
#undef VK_PATCH
    TRY(check_launch("vanka patch"));
  }
  if (L.n == 0) return MG_OK;
  const unsigned g = unsigned(std::min<int64_t>((L.n * bs + 255) / 256, 16 * c->n_sm));
  ++g_tally, mgk::k_vanka_update<<<g, 256, 0, c->stream>>>(L.n, bs, V.m, V.nptr.p, V.nlist.p, V.wgt.p, V.cbuf.p,
                                                            lv_omega(c, L), zero ? 1 : 0, x);
  return check_launch("vanka update");
}

mg_status smooth(mg_ctx_s *c, int l, double *x, const double *b, int k, bool zero) {
  Level &L = c->lv[l];
  const int bs = c->bs();
  const double om = lv_omega(c, L);
  if (k <= 0) {
    if (zero) CU(cudaMemsetAsync(x, 0, size_t(L.n) * bs * sizeof(double), c->stream));
    return MG_OK;
  }
  if (L.vk.on) {
    for (int i = 0; i < k; ++i) TRY(vanka_sweep(c, l, x, b, zero && i == 0));
    return MG_OK;
  }
  double *src = x, *dst = L.w.p;
  if (zero) {
    // the A-free first sweep lands where the remaining k-1 ping-pong sweeps end in x
    // (no copy back)
    --k;
    if (k % 2) std::swap(src, dst);
    for (int pi = 0; pi < L.nparts; ++pi) TRY(launch_sweep0(bs, L.part[pi].A, L.part[pi].dinv.p, b, src, om, c->stream));
  }
  for (int i = 0; i < k; ++i) {
    TRY(a_pass_sweep(c, l, src, b, dst));
    std::swap(src, dst);
  }
  if (src != x) CU(cudaMemcpyAsync(x, src, size_t(L.n) * bs * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  return MG_OK;
}

// Global constraint: x -= (w^T x / w^T k) k, or with consist
// b -= (k^T b / k^T k) k.  The dot goes to scal[8] (all-reduced if distributed).
mg_status mean_project(mg_ctx_s *c, int l, double *x, bool consist) {
  Level &L = c->lv[l];
  const int64_t n = L.n * c->bs();
  if (!L.dist && n > 0 && n <= 16384) {  // one launch instead of dot + update
    ++g_tally, mgk::k_mean_project_small<<<1, 1024, 0, c->stream>>>(n, x, consist ? L.mean_k.p : L.mean_w.p, L.mean_k.p,
                                                                    consist ? L.mean_kk : L.mean_wk);
    return check_launch("mean projection");
  }
  TRY(dev_dot(c, L.dist, n, consist ? L.mean_k.p : L.mean_w.p, x, c->scal.p + 8, false));
  if (n == 0) return MG_OK;
  const unsigned g = unsigned(std::min<int64_t>((n + 255) / 256, 8 * c->n_sm));
  ++g_tally, mgk::k_sub_mean<<<g, 256, 0, c->stream>>>(n, x, L.mean_k.p, c->scal.p + 8,
                                                       consist ? L.mean_kk : L.mean_wk);
  return check_launch("mean projection");
}

mg_status coarse_solve(mg_ctx_s *c, const double *b, double *x) {
  if (c->cfg.coarse_mode == MG_COARSE_DIRECT) {
    if (al16(b)) {  // 4 warps per row (d is read with 16-byte loads)
      const unsigned g = unsigned((c->cN + 1) / 2);
      kl(mgk::k_dense_gemv_split<4>, g, c->stream, c->cN, c->cld, static_cast<const double *>(c->cinv.p), b, x);
    } else {
      const unsigned g = unsigned((c->cN + mgk::kWarpsPerCta - 1) / mgk::kWarpsPerCta);
      ++g_tally, mgk::k_dense_gemv<<<g, mgk::kCta, 0, c->stream>>>(c->cN, c->cld, c->cinv.p, b, x);
    }
    return check_launch("coarse gemv");
  }
  return smooth(c, 0, x, b, std::max(1, c->cfg.coarse_sweeps), true);
}

// GMG(l, x, b) of Alg. gmg; zero: x enters as 0.
mg_status vcycle_rec(mg_ctx_s *c, int l, double *x, const double *b, bool zero) {
  c->cur_level = l;
  mark(c, l);
  if (l == c->tail_T && c->tail_nops > 0 && zero && x == c->lv[l].x.p && b == c->lv[l].b.p)
    return launch_tail(c);                   // GMG(T, 0, b_T), levels T..0 in one launch
  if (l == 0) {                                      // Step 0; ignores x (Z21)
    TRY(coarse_solve(c, b, x));
    return c->lv[0].mean ? mean_project(c, 0, x, false) : MG_OK;
  }
  Level &L = c->lv[l];
  Level &C = c->lv[l - 1];
  TRY(smooth(c, l, x, b, lv_nu_pre(c, L), zero));    // Step 1
  TRY(a_pass_resid(c, l, x, b, L.w.p));              // Step 2: r = b - A x
  TRY(do_restrict(c, l, L.w.p, C.b.p));              //         d = R r
  if (C.mean) TRY(mean_project(c, l - 1, C.b.p, true));  //   consistent d
  TRY(vcycle_rec(c, l - 1, C.x.p, C.b.p, true));     // Step 3
  c->cur_level = l;
  mark(c, l);
  TRY(do_prolong(c, l, C.x.p, x));                   // Step 4
  TRY(smooth(c, l, x, b, lv_nu_post(c, L), false));  // Step 5
  return L.mean ? mean_project(c, l, x, false) : MG_OK;  // int x = 0 on this level
}

// Capture everything `body` enqueues on the context stream into a graph.
template <class F>
mg_status capture(mg_ctx_s *c, F &&body, GraphExec &out) {
  cudaGraph_t graph = nullptr;
  const int64_t t0 = g_tally;
  CU(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
  const mg_status st = body();
  const int64_t captured = g_tally - t0;
  g_tally = t0;
  const cudaError_t ee = cudaStreamEndCapture(c->stream, &graph);
  if (st != MG_OK) {
    if (graph) cudaGraphDestroy(graph);
    return st;
  }
  if (ee != cudaSuccess) return fail(MG_ERR_CUDA, "graph capture: %s", cudaGetErrorString(ee));
  cudaGraphExec_t exec = nullptr;
  const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
  cudaGraphDestroy(graph);
  if (ie != cudaSuccess) return fail(MG_ERR_CUDA, "graph instantiate: %s", cudaGetErrorString(ie));
  out = GraphExec{exec, captured};
  return MG_OK;
}

// Build the conditional graph of one GMRES restart cycle of mm steps:
//   while (hw) { switch (hs) { case j: step(j) } }
// hw (default 1) and hs (default 0) are reset at every launch; step j's
// k_givens sets hs = j + 1 and hw = "continue", so the loop runs at most mm
// bodies whatever the data (no unbounded device loop).
template <class Step>
mg_status capture_cycle(mg_ctx_s *c, int mm, Step &&step, CycleGraph &out) {
  cudaGraph_t G = nullptr;
  CU(cudaGraphCreate(&G, 0));
  struct Guard {
    cudaGraph_t &g;
    ~Guard() {
      if (g) cudaGraphDestroy(g);
    }
  } guard{G};
  cudaGraphConditionalHandle hw, hs;
  CU(cudaGraphConditionalHandleCreate(&hw, G, 1, cudaGraphCondAssignDefault));
  CU(cudaGraphConditionalHandleCreate(&hs, G, 0, cudaGraphCondAssignDefault));
  cudaGraphNodeParams wp{};
  wp.type = cudaGraphNodeTypeConditional;
  wp.conditional.handle = hw;
  wp.conditional.type = cudaGraphCondTypeWhile;
  wp.conditional.size = 1;
  cudaGraphNode_t wn;
  CU(cudaGraphAddNode(&wn, G, nullptr, 0, &wp));
  cudaGraph_t body = wp.conditional.phGraph_out[0];
  cudaGraphNodeParams sp{};
  sp.type = cudaGraphNodeTypeConditional;
  sp.conditional.handle = hs;
  sp.conditional.type = cudaGraphCondTypeSwitch;
  sp.conditional.size = unsigned(mm);
  cudaGraphNode_t sn;
  CU(cudaGraphAddNode(&sn, body, nullptr, 0, &sp));
  out.kernels.assign(size_t(mm), 0);
  for (int j = 0; j < mm; ++j) {
    const int64_t t0 = g_tally;
    CU(cudaStreamBeginCaptureToGraph(c->stream, sp.conditional.phGraph_out[j], nullptr, nullptr, 0,
                                     cudaStreamCaptureModeThreadLocal));
    const mg_status st = step(j, true, hw, hs);
    out.kernels[size_t(j)] = g_tally - t0;
    g_tally = t0;
    cudaGraph_t cap = nullptr;
    const cudaError_t ee = cudaStreamEndCapture(c->stream, &cap);
    if (st != MG_OK) return st;
    if (ee != cudaSuccess) return fail(MG_ERR_CUDA, "GMRES cycle capture (step %d): %s", j, cudaGetErrorString(ee));
  }
  const cudaError_t ie = cudaGraphInstantiate(&out.exec, G, 0);
  if (ie != cudaSuccess) return fail(MG_ERR_CUDA, "GMRES cycle graph instantiate: %s", cudaGetErrorString(ie));
  return MG_OK;
}

mg_status launch_graph(mg_ctx_s *c, const GraphExec &g) {
  CU(cudaGraphLaunch(g.exec, c->stream));
  g_tally += g.kernels;
  return MG_OK;
}

mg_status run_vcycle(mg_ctx_s *c, double *x, const double *b, bool zero) {
  if (!c->use_graphs()) return vcycle_rec(c, c->L(), x, b, zero);
  const GraphKey key{x, b, zero ? 1 : 0};
  auto it = c->graphs.find(key);
  if (it == c->graphs.end()) {
    GraphExec ge;
    const mg_status cs = capture(c, [&] { return vcycle_rec(c, c->L(), x, b, zero); }, ge);
    if (cs != MG_OK) {
      // a transport whose collectives cannot be captured on this system (NCCL inside
      // CUDA graphs has only run single-rank here): run eagerly from now on
      if (!c->tr || cs != MG_ERR_CUDA) return cs;
      std::fprintf(stderr, "mgb200: graph capture with the transport failed (%s); running eagerly\n",
                   mg_last_error());
      cudaGetLastError();
      c->cfg.use_graphs = 0;
      return vcycle_rec(c, c->L(), x, b, zero);
    }
    if (c->graphs.size() > 256) {
      for (auto &kv : c->graphs) cudaGraphExecDestroy(kv.second.exec);
      c->graphs.clear();
    }
    it = c->graphs.emplace(key, ge).first;
  }
  return launch_graph(c, it->second);
}

struct Tally {
  mg_ctx_s *c;
  int64_t t0;
  bool pdl0;
  explicit Tally(mg_ctx_s *ctx) : c(ctx), t0(g_tally), pdl0(g_pdl) { g_pdl = ctx && ctx->pdl(); }
  ~Tally() {
    if (c) c->launches += g_tally - t0;
    g_pdl = pdl0;
  }
};

// rows of the finest level owned here (0 on a rank without rows: NULL vectors allowed)
int64_t fine_n(const mg_ctx_s *c) { return c->lv[c->L()].n; }

mg_status check_ctx(mg_ctx_s *c) {
  if (!c) return fail(MG_ERR_INVALID_ARG, "NULL context");
  return MG_OK;
}

mg_status check_level(mg_ctx_s *c, int level) {
  TRY(check_ctx(c));
  if (level < 0 || level > c->L()) return fail(MG_ERR_INVALID_ARG, "level %d out of range [0, %d]", level, c->L());
  if (!c->lv[level].declared) return fail(MG_ERR_STATE, "level %d not created", level);
  return MG_OK;
}

int64_t gm_stride(int64_t N) { return std::max<int64_t>(2, (N + 1) & ~int64_t(1)); }  // 16-byte aligned vectors

mg_status ensure_gmres(mg_ctx_s *c, int m) {
  const int64_t N = c->lv[c->L()].n * c->bs();
  if (c->gm_m >= m && c->gm_V.p) return MG_OK;
  c->clear_graphs();  // iteration graphs hold basis pointers
  TRY(c->gm_V.alloc(size_t(m + 1) * gm_stride(N)));
  TRY(c->gm_Z.alloc(size_t(m) * gm_stride(N)));
  const size_t ns = size_t(m + 1) * m + 6 * size_t(m + 1) + 16  // MGS state
                    + size_t(m + 1) * m + size_t(m) * m + 6 * size_t(m + 1) + 8;  // DCGS2 state
  TRY(c->gm_state.alloc(ns));
  CU(cudaMemset(c->gm_state.p, 0, ns * sizeof(double)));
  if (!c->gm_host) CU(cudaMallocHost(&c->gm_host, 16 * sizeof(double)));
  TRY(c->dcgs_part.alloc(size_t(4 * c->n_sm) * size_t(2 * m + 2)));
  if (!c->dcgs_ticket.p) {
    TRY(c->dcgs_ticket.alloc(1));
    CU(cudaMemset(c->dcgs_ticket.p, 0, sizeof(unsigned)));
  }
  double *p = c->gm_state.p;
  mgk::GmresDev &g = c->gm;
  g.m = m;
  g.H = p;
  p += size_t(m + 1) * m;
  g.cs = p;
  p += m + 1;
  g.sn = p;
  p += m + 1;
  g.g = p;
  p += m + 1;
  g.y = p;
  p += m + 1;
  g.hn = p;
  p += m + 1;
  g.beta = p;
  p += 1;
  g.beta0 = p;
  p += 1;
  g.out = p;  // [6]
  p += 14;
  g.Hraw = p;
  p += size_t(m + 1) * m;
  g.R = p;
  p += size_t(m) * m;
  g.gpre = p;
  p += m + 1;
  g.dots = p;
  p += 2 * (m + 1);
  g.coef = p;
  p += 2 * (m + 1);
  g.y2 = p;
  p += m + 1;
  g.nu1 = p;
  p += 1;
  g.dead = p;
  c->gm_m = m;
  return MG_OK;
}

// Transpose setup across ranks: route every entry (local row i of level L,
// global column J, weights) to the rank that computes row J of the transpose
// (output row ranges rb).  Arrival order: source ranks ascending, each in CSR
// order -> the stable assembly lists the original rows ascending.  Collective.
mg_status route_entries(mg_ctx_s *c, const Level &L, const std::vector<int64_t> &rp, const std::vector<int64_t> &cl,
                        const std::vector<double> &v, int wpe, const std::vector<int64_t> &rb,
                        std::vector<int64_t> &J, std::vector<int64_t> &I, std::vector<double> &W) {
  const int P = c->nranks();
  std::vector<std::vector<char>> out(P), in;
  const size_t rec = sizeof(int64_t) * 2 + sizeof(double) * wpe;
  std::vector<int64_t> cnt(P, 0);
  for (size_t t = 0; t < cl.size(); ++t) cnt[mgi_owner(cl[t], rb.data(), P)]++;
  for (int r = 0; r < P; ++r) out[r].resize(size_t(cnt[r]) * rec);
  std::vector<size_t> pos(P, 0);
  for (int64_t i = 0; i < L.n; ++i)
    for (int64_t t = rp[i]; t < rp[i + 1]; ++t) {
      const int o = mgi_owner(cl[t], rb.data(), P);
      char *dst = out[o].data() + pos[o];
      const int64_t gi = L.row_begin + i;
      std::memcpy(dst, &cl[t], 8);
      std::memcpy(dst + 8, &gi, 8);
      std::memcpy(dst + 16, &v[size_t(t) * wpe], sizeof(double) * wpe);
      pos[o] += rec;
    }
  TRY(c->tr->alltoallv_host(out, in));
  J.clear();
  I.clear();
  W.clear();
  for (int r = 0; r < P; ++r)
    for (size_t off = 0; off < in[r].size(); off += rec) {
      int64_t j, i;
      std::memcpy(&j, in[r].data() + off, 8);
      std::memcpy(&i, in[r].data() + off + 8, 8);
      J.push_back(j);
      I.push_back(i);
      const double *ww = reinterpret_cast<const double *>(in[r].data() + off + 16);
      W.insert(W.end(), ww, ww + wpe);
    }
  return MG_OK;
}

// validated host copies of a CSR/BSR input
mg_status fetch_csr(mg_ctx_s *c, int64_t n, int64_t n_cols, const int64_t *row_ptr, const int64_t *col,
                    const double *vals, int64_t nnz, int vpe, int mem, bool need_diag, int64_t diag_offset,
                    std::vector<int64_t> &rp, std::vector<int64_t> &cl, std::vector<double> &v, const char *what) {
  (void)c;
  if (nnz < 0) return fail(MG_ERR_DIMENSION, "%s: nnz < 0", what);
  TRY(fetch(rp, row_ptr, size_t(n + 1), mem));
  if (rp[n] != nnz)
    return fail(MG_ERR_DIMENSION, "%s: row_ptr[n] = %lld != nnz = %lld", what, (long long)rp[n], (long long)nnz);
  TRY(fetch(cl, col, size_t(nnz), mem));
  TRY(fetch(v, vals, size_t(nnz) * vpe, mem));
  const int st = mgi_validate_csr(n, n_cols, rp.data(), cl.data(), v.data(), vpe, need_diag ? 1 : 0, diag_offset);
  if (st == MG_ERR_NONFINITE) return fail(MG_ERR_NONFINITE, "%s: non-finite value", what);
  if (st) return fail(MG_ERR_STRUCTURE, "%s: invalid CSR structure (row_ptr / columns / diagonal)", what);
  return MG_OK;
}

}  // namespace

// =============================================================================
// C ABI
// =============================================================================
extern "C" {

const char *mg_last_error(void) { return g_err.c_str(); }
const char *mg_version(void) { return MGB200_VERSION; }

mg_status mg_get_unique_id(unsigned char out[128]) {
  if (!out) return fail(MG_ERR_INVALID_ARG, "NULL argument");
  return mgc::nccl_unique_id(out);
}

mg_status mg_create(mg_ctx *out, const mg_config *cfg, int device, void *cuda_stream, const mg_comm *comm) {
  if (!out || !cfg) return fail(MG_ERR_INVALID_ARG, "NULL argument");
  *out = nullptr;
  if (cfg->n_levels < 1 || cfg->n_levels > 64) return fail(MG_ERR_INVALID_ARG, "n_levels must be in [1, 64]");
  if (cfg->block_size < 1 || cfg->block_size > 6 || cfg->block_size == 5)
    return fail(MG_ERR_INVALID_ARG, "block_size must be 1, 2, 3, 4 or 6");
  if (cfg->nu_pre < 0 || cfg->nu_post < 0) return fail(MG_ERR_INVALID_ARG, "nu_pre/nu_post must be >= 0");
  if (!(cfg->omega > 0.0) || !std::isfinite(cfg->omega)) return fail(MG_ERR_INVALID_ARG, "omega must be > 0");
  if (cfg->coarse_mode != MG_COARSE_DIRECT && cfg->coarse_mode != MG_COARSE_SMOOTH)
    return fail(MG_ERR_INVALID_ARG, "bad coarse_mode");
  if (cfg->precision != MG_PREC_FP64 && cfg->precision != MG_PREC_MIXED)
    return fail(MG_ERR_INVALID_ARG, "bad precision");
  DeviceGuard dg(device);
  int ndev = 0;
  CU(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) return fail(MG_ERR_INVALID_ARG, "device %d out of range", device);
  CU(cudaSetDevice(device));
  std::unique_ptr<mgc::Transport> tr;
  TRY(mgc::make_transport(comm, device, tr));
  auto *c = new mg_ctx_s();
  c->cfg = *cfg;
  c->device = device;
  c->tr = std::move(tr);
  cudaDeviceGetAttribute(&c->n_sm, cudaDevAttrMultiProcessorCount, device);
  if (cuda_stream) {
    c->stream = static_cast<cudaStream_t>(cuda_stream);
  } else {
    if (cudaStreamCreate(&c->stream) != cudaSuccess) {
      delete c;
      return fail(MG_ERR_CUDA, "cudaStreamCreate failed");
    }
    c->own_stream = true;
  }
  c->lv.resize(cfg->n_levels);
  *out = c;
  return MG_OK;
}

mg_status mg_destroy(mg_ctx ctx) {
  if (!ctx) return MG_OK;
  DeviceGuard dg(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  delete ctx;
  return MG_OK;
}

mg_status mg_create_level(mg_ctx c, int level, int64_t n_rows_global, int64_t row_begin, int64_t row_end) {
  TRY(check_ctx(c));
  if (level < 0 || level > c->L()) return fail(MG_ERR_INVALID_ARG, "level %d out of range", level);
  if (n_rows_global < 1 || n_rows_global >= (int64_t(1) << 31))
    return fail(MG_ERR_DIMENSION, "n_rows_global must be in [1, 2^31)");
  if (row_begin < 0 || row_end < row_begin || row_end > n_rows_global)
    return fail(MG_ERR_INVALID_ARG, "bad row range [%lld, %lld)", (long long)row_begin, (long long)row_end);
  DeviceGuard dg(c->device);
  Level &L = c->lv[level];
  const int P = c->nranks();
  bool dist = false;
  std::vector<int64_t> bounds;
  if (P > 1) {
    int64_t mine[3] = {n_rows_global, row_begin, row_end};
    std::vector<int64_t> allv(3 * size_t(P));
    TRY(c->tr->allgather_host(mine, sizeof mine, allv.data()));
    bool repl = true, tiled = true;
    for (int r = 0; r < P; ++r) {
      if (allv[3 * r] != n_rows_global) return fail(MG_ERR_DIMENSION, "ranks disagree on level %d size", level);
      repl = repl && allv[3 * r + 1] == 0 && allv[3 * r + 2] == n_rows_global;
      tiled = tiled && allv[3 * r + 1] == (r == 0 ? 0 : allv[3 * (r - 1) + 2]);
    }
    tiled = tiled && allv[3 * (P - 1) + 2] == n_rows_global;
    if (!repl && !tiled)
      return fail(MG_ERR_INVALID_ARG, "level %d: row ranges must tile [0, n) in rank order or all be [0, n)", level);
    dist = !repl;
    if (dist) {
      bounds.resize(P + 1);
      for (int r = 0; r < P; ++r) bounds[r] = allv[3 * r + 1];
      bounds[P] = n_rows_global;
    }
  } else if (row_begin != 0 || row_end != n_rows_global) {
    return fail(MG_ERR_INVALID_ARG, "single-GPU context: a level must own all rows");
  }
  if (dist && level < c->L() && c->lv[level + 1].declared && !c->lv[level + 1].dist)
    return fail(MG_ERR_INVALID_ARG, "level %d distributed below a replicated level", level);
  L = Level();
  L.declared = true;
  L.n_global = n_rows_global;
  L.row_begin = row_begin;
  L.row_end = row_end;
  L.n = row_end - row_begin;
  L.dist = dist;
  L.bounds = bounds;
  c->invalidate();
  return MG_OK;
}

mg_status mg_set_matrix(mg_ctx c, int level, const int64_t *row_ptr, const int64_t *col, const double *vals,
                        int64_t nnzb, int mem) {
  TRY(check_level(c, level));
  DeviceGuard dg(c->device);
  Level &L = c->lv[level];
  const int bs = c->bs(), V = bs * bs;
  std::vector<int64_t> rp, cl;
  std::vector<double> v;
  TRY(fetch_csr(c, L.n, L.n_global, row_ptr, col, vals, nnzb, V, mem, true, L.row_begin, rp, cl, v, "matrix"));
  L.vk.ready = false;  // a Vanka smoother on this level re-locates its blocks in the new layout
  L.vk.ent.release();
  const bool mixed = c->cfg.precision == MG_PREC_MIXED;
  std::vector<double> v64;
  if (mixed) {
    // the V-cycle works with A rounded to fp32 (its D^-1 and coarse inverse
    // too); the finest level keeps the fp64 operator for the Krylov side
    if (level == c->L()) v64 = v;
    for (double &a : v) a = double(float(a));
  }
  std::vector<int64_t> diag_k(L.n, -1);
  for (int64_t i = 0; i < L.n; ++i)
    for (int64_t k = rp[i]; k < rp[i + 1]; ++k)
      if (cl[k] == L.row_begin + i) diag_k[i] = k;
  std::vector<int32_t> brow, bcol;
  if (level == 0 && !L.dist) {
    brow.resize(nnzb);
    bcol.resize(nnzb);
    for (int64_t i = 0; i < L.n; ++i)
      for (int64_t k = rp[i]; k < rp[i + 1]; ++k) brow[k] = int32_t(i), bcol[k] = int32_t(cl[k]);
  }
  if (L.dist) {
    std::vector<int64_t> ghosts;
    TRY(localize(L.row_begin, L.row_end, rp, cl, ghosts));
    TRY(build_halo(c, L.hx, ghosts, L.bounds, L.row_begin, L.row_end));
  }
  // parts: distributed levels split into interior rows (no ghost column, computed
  // while the halo is in flight) and boundary rows; MGB200_OVERLAP=0 disables
  const char *ov = std::getenv("MGB200_OVERLAP");
  std::vector<char> bnd(L.n, 0);
  int64_t nb = 0;
  if (L.dist && !(ov && ov[0] == '0')) {
    for (int64_t i = 0; i < L.n; ++i) {
      for (int64_t k = rp[i]; k < rp[i + 1]; ++k)
        if (cl[k] >= L.n) bnd[i] = 1;
      nb += bnd[i];
    }
  }
  const bool split = L.dist && !(ov && ov[0] == '0') && nb > 0 && nb < L.n;
  if (split && !c->comm_stream) {
    CU(cudaStreamCreateWithFlags(&c->comm_stream, cudaStreamNonBlocking));
    CU(cudaEventCreateWithFlags(&c->ev_fork, cudaEventDisableTiming));
    CU(cudaEventCreateWithFlags(&c->ev_join, cudaEventDisableTiming));
  }
  L.nparts = split ? 2 : 1;
  for (int pi = 0; pi < L.nparts; ++pi) {
    Level::Part &Pt = L.part[pi];
    Pt = Level::Part();
    Pt.halo = L.dist && (!split || pi == 1);
    // rows of this part (all rows, or interior / boundary) and its sub-CSR
    std::vector<int64_t> rows;
    for (int64_t i = 0; i < L.n; ++i)
      if (!split || bnd[i] == pi) rows.push_back(i);
    const int64_t pn = int64_t(rows.size());
    std::vector<int64_t> prp, pcl, src;
    std::vector<double> pv, pv64;
    if (!split) {  // the whole level: no copies
      prp.swap(rp);
      pcl.swap(cl);
      pv.swap(v);
      pv64.swap(v64);
    } else {
      prp.assign(pn + 1, 0);
    }
    for (int64_t j = 0; split && j < pn; ++j) {
      const int64_t i = rows[j];
      for (int64_t k = rp[i]; k < rp[i + 1]; ++k) {
        pcl.push_back(cl[k]);
        src.push_back(k);
        pv.insert(pv.end(), v.begin() + k * V, v.begin() + (k + 1) * V);
        if (!v64.empty()) pv64.insert(pv64.end(), v64.begin() + k * V, v64.begin() + (k + 1) * V);
      }
      prp[j + 1] = int64_t(pcl.size());
    }
    std::vector<int64_t> sp;
    TRY(build_sell(Pt.A, pn, prp.data(), pcl.data(), pv.data(), V, mixed, &sp, split ? &rows : nullptr));
    Pt.A.ks = ks_for_level(L.n_global);
    Pt.n = pn;
    Pt.nnz = prp[pn];
    // value-update maps: part entry -> SELL entry (sub-row ids), diag entries, slice positions
    std::vector<int64_t> map(std::max<int64_t>(1, Pt.nnz)), de(std::max<int64_t>(1, pn));
    std::vector<int32_t> pos(std::max<int64_t>(1, pn));
    std::vector<int32_t> sub_perm(Pt.A.perm_host);  // sub-row ids for the map
    if (split) {
      std::vector<int64_t> inv(L.n, -1);
      for (int64_t j = 0; j < pn; ++j) inv[rows[j]] = j;
      for (auto &r : sub_perm)
        if (r >= 0) r = int32_t(inv[r]);
    }
    mgi_sell_entry_map(pn, prp.data(), sp.data(), sub_perm.data(), map.data(), pos.data());
    for (int64_t j = 0; j < pn; ++j) {
      const int64_t i = rows[j];
      const int64_t row_start = split ? rp[i] : prp[i];
      de[j] = map[prp[j] + (diag_k[i] - row_start)];
    }
    TRY(Pt.umap.upload(map.data(), map.size()));
    TRY(Pt.udiag_e.upload(de.data(), de.size()));
    TRY(Pt.upos.upload(pos.data(), pos.size()));
    if (split) TRY(Pt.usrc.upload(src.data(), src.size()));
    if (!pv64.empty()) {
      TRY(build_sell(Pt.A64, pn, prp.data(), pcl.data(), pv64.data(), V, false, nullptr, split ? &rows : nullptr));
      Pt.A64.ks = Pt.A.ks;
    }
    if (!split) {  // hand the level arrays back (level-0 coarse copy below)
      prp.swap(rp);
      pcl.swap(cl);
      pv.swap(v);
    }
  }
  if (!brow.empty()) {
    TRY(L.ublk_row.upload(brow.data(), brow.size()));
    TRY(L.ublk_col.upload(bcol.data(), bcol.size()));
  }
  L.nnzb = nnzb;
  L.dinv_ready = false;  // (re)built at finalize; a user D^-1 is re-sliced with the new permutation
  if (level == 0 && !L.dist) {
    L.rp0.swap(rp);
    L.col0.swap(cl);
    L.val0.swap(v);
    c->cN = 0;
  }
  c->invalidate();
  return MG_OK;
}

mg_status mg_set_transfer(mg_ctx c, int fine_level, const int64_t *row_ptr, const int64_t *col, const double *w,
                          int64_t nnz, int weights_per_entry, int mem) {
  TRY(check_level(c, fine_level));
  if (fine_level < 1) return fail(MG_ERR_INVALID_ARG, "fine_level must be >= 1");
  if (!c->lv[fine_level - 1].declared) return fail(MG_ERR_STATE, "level %d not created", fine_level - 1);
  DeviceGuard dg(c->device);
  Level &L = c->lv[fine_level];
  Level &C = c->lv[fine_level - 1];
  const int wpe = weights_per_entry;
  const int P = c->nranks(), me = c->rank();
  if (wpe != 1 && wpe != c->bs()) return fail(MG_ERR_INVALID_ARG, "weights_per_entry must be 1 or bs");
  if (!L.dist && C.dist) return fail(MG_ERR_INVALID_ARG, "replicated level above a distributed one");
  std::vector<int64_t> rp, cl;
  std::vector<double> v;
  TRY(fetch_csr(c, L.n, C.n_global, row_ptr, col, w, nnz, wpe, mem, false, 0, rp, cl, v, "transfer"));
  // ---- R = P^T -------------------------------------------------------
  std::vector<int64_t> rrp, rcl;
  std::vector<double> rv;
  if (!L.dist) {
    rrp.resize(C.n + 1);
    rcl.resize(nnz);
    rv.resize(size_t(nnz) * wpe);
    mgi_csr_transpose(L.n, C.n, rp.data(), cl.data(), v.data(), wpe, rrp.data(), rcl.data(), rv.data());
    L.r_row0 = 0;
    L.r_rows = C.n;
    L.agglomerate = false;
    L.hr = Halo();
  } else {
    // rows of R computed here: my coarse rows (coarse distributed) or an even
    // share of the replicated coarse level, all-gathered afterwards
    std::vector<int64_t> rb(P + 1);
    if (C.dist) {
      rb = C.bounds;
    } else {
      for (int r = 0; r <= P; ++r) rb[r] = C.n_global * r / P;
    }
    std::vector<int64_t> J, I;
    std::vector<double> W;
    TRY(route_entries(c, L, rp, cl, v, wpe, rb, J, I, W));
    // output offset into the coarse vector: local rows start at 0 on a
    // distributed coarse level; the full vector is addressed when replicated
    L.r_row0 = C.dist ? 0 : rb[me];
    L.r_rows = rb[me + 1] - rb[me];
    rrp.resize(L.r_rows + 1);
    rcl.resize(J.size());
    rv.resize(J.size() * wpe);
    const int st = mgi_assemble_routed_rows(int64_t(J.size()), J.data(), I.data(), W.data(), wpe, rb[me], L.r_rows,
                                            rrp.data(), rcl.data(), rv.data());
    if (st) return fail(MG_ERR_STRUCTURE, "restriction routing failed");
    std::vector<int64_t> ghosts;
    TRY(localize(L.row_begin, L.row_end, rrp, rcl, ghosts));
    TRY(build_halo(c, L.hr, ghosts, L.bounds, L.row_begin, L.row_end));
    L.agglomerate = !C.dist;
    L.ag_counts.assign(P, 0);
    L.ag_displs.assign(P, 0);
    for (int r = 0; r < P; ++r) {
      L.ag_counts[r] = (rb[r + 1] - rb[r]) * c->bs();
      L.ag_displs[r] = rb[r] * c->bs();
    }
  }
  TRY(build_sell(L.R, L.r_rows, rrp.data(), rcl.data(), rv.data(), wpe));
  L.R.ks = 4;  // R rows gather 9-27+ fine entries: split them over 4 warps
  // restriction on the SELL-C layout (measured, scripts/tune_tsell.py: C3 finest 98.7 -> 69.3 us,
  // C5 212 -> 113 us, C2 25.6 -> 19.6 us); warps per slice group: 4 for bs 1 and 6, 2 for bs 3, 1 otherwise
  TRY(build_tsell(L.Rt, L.r_rows, rrp.data(), rcl.data(), rv.data(), wpe, c->bs()));
  // (round-2 re-tune with the exact-size batches, same box: 4 warps per slice for bs 1
  // -- C2 V-cycle 0.247 -> 0.237 ms, TD L10 0.256 -> 0.248 -- and bs 6 -- e6 1.165 ->
  // 1.137 ms; bs 3 stays at 2 (C3: 1/1, 4/1, 2/2 slower); bs 4 (C5) insensitive)
  L.Rt.ks = (c->bs() == 1 || c->bs() == 6) ? 4 : c->bs() == 3 ? 2 : 1;
  // ---- P: columns are coarse rows ------------------------------------------
  if (C.dist) {
    std::vector<int64_t> ghosts;
    TRY(localize(C.row_begin, C.row_end, rp, cl, ghosts));
    TRY(build_halo(c, L.hp, ghosts, C.bounds, C.row_begin, C.row_end));
  } else {
    L.hp = Halo();
  }
  TRY(build_sell(L.P, L.n, rp.data(), cl.data(), v.data(), wpe));
  TRY(build_pcsr(L.Pc, L.n, rp, cl, v, wpe));
  // prolongation: natural-order CSR for scalar fp32-exact weights (build_pcsr, above);
  // SELL-32 was chosen over SELL-C in round 2 before the exact-size batches (C3 finest
  // 105 vs 162 us then)
  // Per-component weights (no natural-order CSR kernel, see build_pcsr) use the SELL-C
  // layout: with the exact-size load batches it is slightly ahead of SELL-32 (same box:
  // C4 V-cycle 0.469 -> 0.464 ms, C5 11.10 -> 11.06 ms). MGB200_TSELL_PROLONG = 1 / 0
  // forces / disables it (experiments).
  const char *tp = std::getenv("MGB200_TSELL_PROLONG");
  const bool want_pt = tp && *tp ? tp[0] == '1' : (wpe != 1 && !L.Pc.set);
  if (want_pt)
    TRY(build_tsell(L.Pt, L.n, rp.data(), cl.data(), v.data(), wpe, c->bs()));
  else
    L.Pt = TSellOp();
  L.wpe = wpe;
  L.nnz_p = nnz;
  c->invalidate();
  return MG_OK;
}

mg_status mg_set_smoother(mg_ctx c, int level, double omega, int nu_pre, int nu_post, const double *dinv, int mem) {
  TRY(check_level(c, level));
  DeviceGuard dg(c->device);
  Level &L = c->lv[level];
  if (!std::isfinite(omega)) return fail(MG_ERR_INVALID_ARG, "omega not finite");
  L.omega = omega > 0.0 ? omega : 0.0;
  if (nu_pre >= 0) L.nu_pre = nu_pre;
  if (nu_post >= 0) L.nu_post = nu_post;
  if (dinv) {
    const int V = c->bs() * c->bs();
    TRY(fetch(L.dinv_host, dinv, size_t(L.n) * V, mem));
    for (double d : L.dinv_host)
      if (!std::isfinite(d)) return fail(MG_ERR_NONFINITE, "non-finite D^-1");
    L.dinv_ready = false;
  }
  c->invalidate();
  return MG_OK;
}

mg_status mg_set_vanka(mg_ctx c, int level, int64_t n_patches, int nloc, const int64_t *patch_nodes, int mem) {
  TRY(check_level(c, level));
  DeviceGuard dg(c->device);
  Level &L = c->lv[level];
  Level::Vanka &V = L.vk;
  const int bs = c->bs();
  if (n_patches < 0 || nloc < 1 || (n_patches > 0 && !patch_nodes))
    return fail(MG_ERR_INVALID_ARG, "bad patch arguments");
  if (n_patches == 0) {  // switch back to block-Jacobi
    V = Level::Vanka{};
    c->invalidate();
    return MG_OK;
  }
  if (nloc * bs > 32) return fail(MG_ERR_INVALID_ARG, "patch of %d unknowns: nloc * block_size must be <= 32", nloc * bs);
  if (!L.part[0].A.set) return fail(MG_ERR_STATE, "level %d: call mg_set_matrix before mg_set_vanka", level);
  if (L.dist || L.nparts != 1) return fail(MG_ERR_STATE, "level %d: Vanka needs a non-distributed level", level);
  std::vector<int64_t> pn;
  TRY(fetch(pn, patch_nodes, size_t(n_patches) * nloc, mem));
  std::vector<int64_t> cnt(L.n + 1, 0);
  for (int64_t p = 0; p < n_patches; ++p)
    for (int a = 0; a < nloc; ++a) {
      const int64_t i = pn[p * nloc + a];
      if (i < 0 || i >= L.n) return fail(MG_ERR_STRUCTURE, "patch %lld: node %lld out of range", (long long)p, (long long)i);
      for (int b2 = 0; b2 < a; ++b2)
        if (pn[p * nloc + b2] == i) return fail(MG_ERR_STRUCTURE, "patch %lld: repeated node", (long long)p);
      ++cnt[i + 1];
    }
  std::vector<double> wgt(L.n);
  for (int64_t i = 0; i < L.n; ++i) {
    if (cnt[i + 1] == 0) return fail(MG_ERR_STRUCTURE, "level %d: row %lld in no patch", level, (long long)i);
    wgt[i] = 1.0 / double(cnt[i + 1]);
  }
  for (int64_t i = 0; i < L.n; ++i) cnt[i + 1] += cnt[i];
  std::vector<int64_t> list(cnt[L.n]), fill(cnt.begin(), cnt.end() - 1);
  const int m = nloc * bs;
  for (int64_t p = 0; p < n_patches; ++p)  // ascending patch order per node: fixed summation order
    for (int a = 0; a < nloc; ++a) list[fill[pn[p * nloc + a]]++] = p * m + int64_t(a) * bs;
  std::vector<int32_t> nodes32(pn.begin(), pn.end());
  Level::Vanka nv;
  nv.on = true;
  nv.np = n_patches;
  nv.nl = nloc;
  nv.m = m;
  nv.ppw = 32 / m;
  TRY(nv.nodes.upload(nodes32.data(), nodes32.size()));
  TRY(nv.nptr.upload(cnt.data(), cnt.size()));
  TRY(nv.nlist.upload(list.data(), list.size()));
  TRY(nv.wgt.upload(wgt.data(), wgt.size()));
  TRY(nv.inv.alloc(size_t((n_patches + nv.ppw - 1) / nv.ppw) * nv.ppw * m * m));  // whole groups (vk_off)
  TRY(nv.cbuf.alloc(size_t(n_patches) * m));
  V = std::move(nv);
  c->invalidate();
  return MG_OK;
}

mg_status mg_set_constraints(mg_ctx c, const int64_t *H_row_ptr, const int64_t *H_col, const double *H_w, int64_t nnz,
                             int mem) {
  TRY(check_ctx(c));
  TRY(check_level(c, c->L()));
  DeviceGuard dg(c->device);
  Level &F = c->lv[c->L()];
  std::vector<int64_t> rp, cl;
  std::vector<double> v;
  TRY(fetch_csr(c, F.n, F.n_global, H_row_ptr, H_col, H_w, nnz, 1, mem, false, 0, rp, cl, v, "H"));
  // H^T (the "distributing" operation of P:338): rows = my fine rows
  std::vector<int64_t> trp(F.n + 1), tcl;
  std::vector<double> tv;
  if (!F.dist) {
    tcl.resize(nnz);
    tv.resize(nnz);
    mgi_csr_transpose(F.n, F.n, rp.data(), cl.data(), v.data(), 1, trp.data(), tcl.data(), tv.data());
    c->hht_halo = Halo();
  } else {
    std::vector<int64_t> J, I;
    std::vector<double> W;
    TRY(route_entries(c, F, rp, cl, v, 1, F.bounds, J, I, W));
    tcl.resize(J.size());
    tv.resize(J.size());
    const int st = mgi_assemble_routed_rows(int64_t(J.size()), J.data(), I.data(), W.data(), 1, F.row_begin, F.n,
                                            trp.data(), tcl.data(), tv.data());
    if (st) return fail(MG_ERR_STRUCTURE, "H^T routing failed");
    std::vector<int64_t> ghosts;
    TRY(localize(F.row_begin, F.row_end, trp, tcl, ghosts));
    TRY(build_halo(c, c->hht_halo, ghosts, F.bounds, F.row_begin, F.row_end));
  }
  TRY(build_sell(c->HT, F.n, trp.data(), tcl.data(), tv.data(), 1));
  if (F.dist) {
    std::vector<int64_t> ghosts;
    TRY(localize(F.row_begin, F.row_end, rp, cl, ghosts));
    TRY(build_halo(c, c->hh, ghosts, F.bounds, F.row_begin, F.row_end));
  } else {
    c->hh = Halo();
  }
  TRY(build_sell(c->H, F.n, rp.data(), cl.data(), v.data(), 1));
  return MG_OK;
}

mg_status mg_setup(mg_ctx c) {
  TRY(check_ctx(c));
  DeviceGuard dg(c->device);
  return finalize(c);
}

mg_status mg_vcycle(mg_ctx c, double *x, const double *b) {
  TRY(check_ctx(c));
  if ((fine_n(c) > 0 && (!x || !b)) || (x && x == b))
    return fail(MG_ERR_INVALID_ARG, "x, b must be distinct non-NULL device pointers");
  DeviceGuard dg(c->device);
  Tally tally(c);
  TRY(finalize(c));
  return run_vcycle(c, x, b, false);
}

mg_status mg_vcycle_zero(mg_ctx c, double *z, const double *v) {
  TRY(check_ctx(c));
  if ((fine_n(c) > 0 && (!z || !v)) || (z && z == v))
    return fail(MG_ERR_INVALID_ARG, "z, v must be distinct non-NULL device pointers");
  DeviceGuard dg(c->device);
  Tally tally(c);
  TRY(finalize(c));
  return run_vcycle(c, z, v, true);
}

mg_status mg_spmv(mg_ctx c, int level, double alpha, const double *x, double beta, double *y) {
  TRY(check_level(c, level));
  if ((c->lv[level].n > 0 && (!x || !y)) || (x && x == y))
    return fail(MG_ERR_INVALID_ARG, "x, y must be distinct non-NULL device pointers");
  if (!c->lv[level].part[0].A.set) return fail(MG_ERR_STATE, "level %d has no matrix", level);
  DeviceGuard dg(c->device);
  Tally tally(c);
  return a_pass_spmv(c, level, alpha, x, beta, y, true);
}

mg_status mg_sweep(mg_ctx c, int level, const double *x, const double *b, double *x_out) {
  TRY(check_level(c, level));
  if ((c->lv[level].n > 0 && (!x || !b || !x_out)) || (x_out && (x_out == x || x_out == b)))
    return fail(MG_ERR_INVALID_ARG, "x_out must not alias x or b");
  DeviceGuard dg(c->device);
  Tally tally(c);
  TRY(finalize(c));
  if (c->lv[level].vk.on) {
    const size_t n = size_t(c->lv[level].n) * c->bs();
    if (n) CU(cudaMemcpyAsync(x_out, x, n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    return vanka_sweep(c, level, x_out, b, false);
  }
  return a_pass_sweep(c, level, x, b, x_out);
}

mg_status mg_residual(mg_ctx c, int level, const double *x, const double *b, double *r) {
  TRY(check_level(c, level));
  if ((c->lv[level].n > 0 && (!x || !b || !r)) || (r && (r == x || r == b)))
    return fail(MG_ERR_INVALID_ARG, "r must not alias x or b");
  if (!c->lv[level].part[0].A.set) return fail(MG_ERR_STATE, "level %d has no matrix", level);
  DeviceGuard dg(c->device);
  Tally tally(c);
  return a_pass_resid(c, level, x, b, r, true);
}

mg_status mg_smooth(mg_ctx c, int level, double *x, const double *b, int sweeps) {
  TRY(check_level(c, level));
  if ((c->lv[level].n > 0 && (!x || !b)) || (x && x == b))
    return fail(MG_ERR_INVALID_ARG, "x, b must be distinct non-NULL device pointers");
  if (sweeps < 0) return fail(MG_ERR_INVALID_ARG, "sweeps < 0");
  DeviceGuard dg(c->device);
  Tally tally(c);
  TRY(finalize(c));
  return smooth(c, level, x, b, sweeps, false);
}

mg_status mg_restrict(mg_ctx c, int fine_level, const double *r_fine, double *d_coarse) {
  TRY(check_level(c, fine_level));
  if (fine_level < 1 || !c->lv[fine_level].P.set) return fail(MG_ERR_STATE, "no transfer into level %d", fine_level);
  if (!r_fine || !d_coarse) return fail(MG_ERR_INVALID_ARG, "NULL vector");
  DeviceGuard dg(c->device);
  Tally tally(c);
  return do_restrict(c, fine_level, r_fine, d_coarse);
}

mg_status mg_prolong_add(mg_ctx c, int fine_level, const double *y_coarse, double *x_fine) {
  TRY(check_level(c, fine_level));
  if (fine_level < 1 || !c->lv[fine_level].P.set) return fail(MG_ERR_STATE, "no transfer into level %d", fine_level);
  if (!y_coarse || !x_fine) return fail(MG_ERR_INVALID_ARG, "NULL vector");
  DeviceGuard dg(c->device);
  Tally tally(c);
  return do_prolong(c, fine_level, y_coarse, x_fine);
}

mg_status mg_coarse_solve(mg_ctx c, const double *d, double *y) {
  TRY(check_ctx(c));
  if (!d || !y || d == y) return fail(MG_ERR_INVALID_ARG, "d, y must be distinct non-NULL device pointers");
  DeviceGuard dg(c->device);
  Tally tally(c);
  TRY(finalize(c));
  return coarse_solve(c, d, y);
}

mg_status mg_apply_constraints(mg_ctx c, double *x) {
  TRY(check_ctx(c));
  if (fine_n(c) > 0 && !x) return fail(MG_ERR_INVALID_ARG, "NULL vector");
  if (!c->H.set) return fail(MG_ERR_STATE, "no hanging-node matrix (mg_set_constraints)");
  DeviceGuard dg(c->device);
  Tally tally(c);
  TRY(finalize(c));
  Level &F = c->lv[c->L()];
  TRY(halo_exchange(c, c->hh, x));
  TRY(launch_transfer(c->bs(), false, c->H, In{x, c->hh.active ? c->hh.ghost.p : nullptr, int(F.n)}, F.w.p,
                      c->stream));
  if (F.n) CU(cudaMemcpyAsync(x, F.w.p, size_t(F.n) * c->bs() * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  return MG_OK;
}

mg_status mg_set_mean_constraint(mg_ctx c, int level, const double *w, const double *k, int mem) {
  TRY(check_level(c, level));
  DeviceGuard dg(c->device);
  Level &L = c->lv[level];
  const size_t n = size_t(L.n) * c->bs();
  if (!w) {
    L.mean = false;
    L.mean_w = DevArray<double>();
    L.mean_k = DevArray<double>();
  } else {
    if (n > 0 && !k) return fail(MG_ERR_INVALID_ARG, "k must be given with w");
    std::vector<double> hw, hk;
    TRY(fetch(hw, w, n, mem));
    TRY(fetch(hk, k, n, mem));
    double wmax = 0.0;
    for (size_t i = 0; i < n; ++i) {
      if (!std::isfinite(hw[i]) || !std::isfinite(hk[i])) return fail(MG_ERR_NONFINITE, "non-finite w or k");
      wmax = std::max(wmax, hw[i]);
    }
    if (!hw.empty()) {
      TRY(L.mean_w.upload(hw.data(), n));
      TRY(L.mean_k.upload(hk.data(), n));
    } else {
      TRY(L.mean_w.alloc(1));
      TRY(L.mean_k.alloc(1));
    }
    if (level == 0 && !L.dist && !(wmax > 0.0)) return fail(MG_ERR_INVALID_ARG, "level 0: max(w) must be > 0");
    L.mean = true;
    L.mean_wmax = wmax;
  }
  if (level == 0) c->cN = 0;  // the coarse inverse includes alpha w w^T: rebuild
  c->invalidate();
  return MG_OK;
}

mg_status mg_project_zero_mean(mg_ctx c, int level, double *x) {
  TRY(check_level(c, level));
  if (c->lv[level].n > 0 && !x) return fail(MG_ERR_INVALID_ARG, "NULL vector");
  if (!c->lv[level].mean) return fail(MG_ERR_STATE, "level %d has no mean constraint", level);
  DeviceGuard dg(c->device);
  Tally tally(c);
  TRY(finalize(c));
  return mean_project(c, level, x, false);
}

mg_status mg_make_consistent(mg_ctx c, int level, double *b) {
  TRY(check_level(c, level));
  if (c->lv[level].n > 0 && !b) return fail(MG_ERR_INVALID_ARG, "NULL vector");
  if (!c->lv[level].mean) return fail(MG_ERR_STATE, "level %d has no mean constraint", level);
  DeviceGuard dg(c->device);
  Tally tally(c);
  TRY(finalize(c));
  return mean_project(c, level, b, true);
}

// Host -> device copy on the context stream at pinned-memory speed: pinned
// (page-locked) sources go straight to the DMA engine; pageable ones are staged
// through two 64 MB pinned chunks, a multi-threaded host copy into one chunk
// overlapping the DMA out of the other (the driver's own pageable path runs
// at ~9 GB/s: VERDICT r1, the 6.2 GB C3 operator took 690 ms).
static mg_status upload_host(mg_ctx_s *c, void *dst, const void *src, size_t bytes) {
  if (!bytes) return MG_OK;
  cudaPointerAttributes pa{};
  if (cudaPointerGetAttributes(&pa, src) != cudaSuccess) cudaGetLastError();
  if (pa.type == cudaMemoryTypeHost) {
    CU(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, c->stream));
    return MG_OK;
  }
  constexpr size_t kChunk = size_t(64) << 20;
  for (int k = 0; k < 2; ++k) {
    if (!c->pin_chunk[k]) CU(cudaMallocHost(&c->pin_chunk[k], kChunk));
    if (!c->pin_ev[k]) CU(cudaEventCreateWithFlags(&c->pin_ev[k], cudaEventDisableTiming));
  }
  CU(cudaStreamSynchronize(c->stream));  // earlier work on the stream may still read a chunk
  const char *s = static_cast<const char *>(src);
  char *d = static_cast<char *>(dst);
  for (size_t off = 0, i = 0; off < bytes; off += kChunk, ++i) {
    const int k = int(i & 1);
    const size_t len = std::min(kChunk, bytes - off);
    if (i >= 2) CU(cudaEventSynchronize(c->pin_ev[k]));  // the DMA out of this chunk is done
    char *pc = c->pin_chunk[k];
    const int64_t nt = std::max<int64_t>(1, std::min<int64_t>(16, int64_t(len >> 22)));
#pragma omp parallel for num_threads(int(nt)) schedule(static)
    for (int64_t t = 0; t < nt; ++t) {
      const size_t a = len * size_t(t) / size_t(nt), b = len * size_t(t + 1) / size_t(nt);
      std::memcpy(pc + a, s + off + a, b - a);
    }
    CU(cudaMemcpyAsync(d + off, pc, len, cudaMemcpyHostToDevice, c->stream));
    CU(cudaEventRecord(c->pin_ev[k], c->stream));
  }
  return MG_OK;
}

mg_status mg_update_matrix(mg_ctx c, int level, const double *vals, int mem) {
  TRY(check_level(c, level));
  if (!vals) return fail(MG_ERR_INVALID_ARG, "NULL values");
  Level &L = c->lv[level];
  if (!L.part[0].A.set) return fail(MG_ERR_STATE, "level %d has no matrix: call mg_set_matrix first", level);
  if (mem != MG_MEM_HOST && mem != MG_MEM_DEVICE) return fail(MG_ERR_INVALID_ARG, "bad mem");
  DeviceGuard dg(c->device);
  const int bs = c->bs(), V = bs * bs;
  const int64_t nnzb = L.nnzb;
  const double *dv = vals;
  if (mem == MG_MEM_HOST) {  // stream-ordered copy into a staging buffer kept by the context
    const size_t cnt = size_t(std::max<int64_t>(1, nnzb)) * V;
    if (c->upd_stage.n < cnt) {
      CU(cudaStreamSynchronize(c->stream));
      TRY(c->upd_stage.alloc(cnt));
    }
    TRY(upload_host(c, c->upd_stage.p, vals, size_t(nnzb) * V * sizeof(double)));
    dv = c->upd_stage.p;
  }
  DevArray<int> flag;
  TRY(flag.alloc(1));
  CU(cudaMemsetAsync(flag.p, 0, sizeof(int), c->stream));
  const unsigned g = unsigned(std::min<int64_t>(std::max<int64_t>(1, (nnzb + 255) / 256), 16 * c->n_sm));
  for (int pi = 0; pi < L.nparts; ++pi) {
    Level::Part &Pt = L.part[pi];
    if (Pt.nnz == 0) continue;
    const unsigned gp = unsigned(std::min<int64_t>(std::max<int64_t>(1, (Pt.nnz + 255) / 256), 16 * c->n_sm));
    mgk::k_scatter_values<<<gp, 256, 0, c->stream>>>(Pt.nnz, V, Pt.umap.p, Pt.usrc.p, dv,
                                                     Pt.A.f32 ? nullptr : Pt.A.val.p, Pt.A.f32 ? Pt.A.valf.p : nullptr,
                                                     flag.p);
    if (Pt.A64.set)
      mgk::k_scatter_values<<<gp, 256, 0, c->stream>>>(Pt.nnz, V, Pt.umap.p, Pt.usrc.p, dv, Pt.A64.val.p, nullptr,
                                                       flag.p);
    TRY(check_launch("value scatter"));
  }
  (void)g;
  int f = 0;
  CU(cudaMemcpyAsync(&f, flag.p, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  if (f & 1) return fail(MG_ERR_NONFINITE, "level %d: non-finite matrix value", level);
  if (L.dinv_host.empty()) TRY(device_dinv(c, level));  // a user-supplied D^-1 is kept
  if (L.vk.on) TRY(vanka_build(c, level));
  if (level == 0 && c->cfg.coarse_mode == MG_COARSE_DIRECT && !L.dist && c->cN > 0) {
    CU(cudaMemsetAsync(c->cinv.p, 0, c->cinv.n * sizeof(double), c->stream));
    const unsigned gd = unsigned(std::min<int64_t>(std::max<int64_t>(1, (nnzb * V + 255) / 256), 16 * c->n_sm));
    mgk::k_dense_scatter<<<gd, 256, 0, c->stream>>>(nnzb, bs, L.ublk_row.p, L.ublk_col.p, dv,
                                                    c->cfg.precision == MG_PREC_MIXED ? 1 : 0, c->cld, c->cinv.p);
    TRY(check_launch("dense scatter"));
    TRY(coarse_regularise(c, c->cN, c->cld));
    TRY(coarse_gj(c, c->cN, c->cld));
  }
  // graphs hold pointers only: they stay valid
  return MG_OK;
}

mg_status mg_condense_rhs(mg_ctx c, const double *b, double *b_bar) {
  TRY(check_ctx(c));
  if ((fine_n(c) > 0 && (!b || !b_bar)) || (b && b == b_bar))
    return fail(MG_ERR_INVALID_ARG, "b, b_bar must be distinct non-NULL device pointers");
  if (!c->HT.set) return fail(MG_ERR_STATE, "no hanging-node matrix (mg_set_constraints)");
  DeviceGuard dg(c->device);
  Tally tally(c);
  Level &F = c->lv[c->L()];
  TRY(halo_exchange(c, c->hht_halo, b));
  return launch_transfer(c->bs(), false, c->HT, In{b, c->hht_halo.active ? c->hht_halo.ghost.p : nullptr, int(F.n)},
                         b_bar, c->stream);
}

mg_status mg_axpy(mg_ctx c, int level, double alpha, const double *x, double *y) {
  TRY(check_level(c, level));
  const int64_t N = c->lv[level].n * c->bs();
  if (N > 0 && (!x || !y)) return fail(MG_ERR_INVALID_ARG, "NULL vector");
  if (!std::isfinite(alpha)) return fail(MG_ERR_NONFINITE, "non-finite alpha");
  if (N == 0) return MG_OK;
  DeviceGuard dg(c->device);
  Tally tally(c);
  const unsigned eg = unsigned(std::min<int64_t>(std::max<int64_t>(1, (N + 255) / 256), 8 * c->n_sm));
  ++g_tally, mgk::k_axpy<<<eg, 256, 0, c->stream>>>(N, alpha, x, y);
  return check_launch("axpy");
}

mg_status mg_dot(mg_ctx c, int level, const double *a, const double *b, double *out_host) {
  TRY(check_level(c, level));
  if (!out_host || (c->lv[level].n > 0 && (!a || !b))) return fail(MG_ERR_INVALID_ARG, "NULL argument");
  DeviceGuard dg(c->device);
  Tally tally(c);
  TRY(finalize(c));
  TRY(dev_dot(c, c->lv[level].dist, c->lv[level].n * c->bs(), a, b, c->scal.p, false));
  CU(cudaMemcpyAsync(out_host, c->scal.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CU(cudaStreamSynchronize(c->stream));
  return MG_OK;
}

int64_t mgi_launch_count(mgi_ctx c) { return c ? c->launches : -1; }

int mgi_stream_info(mgi_ctx c, void **stream, int *device, int *n_levels, int64_t *n_fine) {
  if (!c) return MG_ERR_INVALID_ARG;
  if (stream) *stream = c->stream;
  if (device) *device = c->device;
  if (n_levels) *n_levels = c->cfg.n_levels;
  if (n_fine) *n_fine = c->lv.empty() ? 0 : c->lv[c->L()].n * c->bs();
  return MG_OK;
}

int mgi_agree(mgi_ctx c, int status, int *agreed) {
  if (!c || !agreed) return MG_ERR_INVALID_ARG;
  *agreed = status;
  if (!c->tr) return MG_OK;
  std::vector<int> all(size_t(c->tr->nranks), 0);
  const mg_status s = c->tr->allgather_host(&status, sizeof(int), all.data());
  if (s != MG_OK) return s;
  *agreed = MG_OK;
  for (int v : all)
    if (v != MG_OK) {
      *agreed = v;
      break;
    }
  return MG_OK;
}

int mgi_vcycle_profile(mgi_ctx c, double *x, const double *b, int zero, double *out, int n_out) {
  if (!c || !x || !b || !out) return MG_ERR_INVALID_ARG;
  const int nl = c->L() + 1;
  if (n_out < 2 * nl + 1) return MG_ERR_DIMENSION;
  DeviceGuard dg(c->device);
  Tally tally(c);
  TRY(finalize(c));
  for (auto &pe : c->prof) cudaEventDestroy(pe.second);
  c->prof.clear();
  c->prof_on = true;
  const mg_status st = vcycle_rec(c, c->L(), x, b, zero != 0);
  mark(c, -1);
  c->prof_on = false;
  CU(cudaStreamSynchronize(c->stream));
  for (int i = 0; i < 2 * nl + 1; ++i) out[i] = 0.0;
  for (size_t i = 0; i + 1 < c->prof.size(); ++i) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, c->prof[i].second, c->prof[i + 1].second);
    const int tag = c->prof[i].first;
    if (tag >= 200) out[2 * nl] += ms;
    else if (tag >= 100) out[nl + tag - 100] += ms;
    else if (tag >= 0) out[tag] += ms;
  }
  for (auto &pe : c->prof) cudaEventDestroy(pe.second);
  c->prof.clear();
  return st;
}

int mgi_level_info(mgi_ctx c, int level, int64_t *n, int64_t *nnzb, int64_t *sell_entries, int64_t *nnz_p,
                   int64_t *sell_entries_p, int64_t *sell_entries_r) {
  if (!c || level < 0 || level > c->L()) return MG_ERR_INVALID_ARG;
  const Level &L = c->lv[level];
  if (n) *n = L.n;
  if (nnzb) *nnzb = L.nnzb;
  if (sell_entries) *sell_entries = L.part[0].A.n_entries + (L.nparts > 1 ? L.part[1].A.n_entries : 0);
  if (nnz_p) *nnz_p = L.nnz_p;
  if (sell_entries_p) *sell_entries_p = L.P.n_entries;
  if (sell_entries_r) *sell_entries_r = L.R.n_entries;
  return 0;
}

mg_status mg_solve(mg_ctx c, double *x, const double *b, const mg_solve_opts *opts, mg_solve_info *info) {
  TRY(check_ctx(c));
  if (!opts || (fine_n(c) > 0 && (!x || !b)) || (x && x == b)) return fail(MG_ERR_INVALID_ARG, "bad arguments");
  if (opts->max_iter < 0 || !(opts->rtol >= 0.0)) return fail(MG_ERR_INVALID_ARG, "bad options");
  DeviceGuard dg(c->device);
  Tally tally(c);
  TRY(finalize(c));
  const int Lf = c->L();
  Level &F = c->lv[Lf];
  const bool dist = F.dist;
  const int bs = c->bs();
  const int64_t N = F.n * bs;
  const double rtol = opts->rtol;
  int its = 0;
  double rel = 1.0;  // ||b - A x0|| / ||b - A x0|| until an iteration ran (max_iter = 0)
  bool conv = false;
  if (!c->gm_host) CU(cudaMallocHost(&c->gm_host, 16 * sizeof(double)));
  double *hst = c->gm_host;

  if (F.mean) {  // solvable right-hand side of the singular system: b - (k^T b / k^T k) k
    if (c->mean_b.n < size_t(std::max<int64_t>(N, 1))) TRY(c->mean_b.alloc(size_t(std::max<int64_t>(N, 1))));
    if (N) CU(cudaMemcpyAsync(c->mean_b.p, b, size_t(N) * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    TRY(mean_project(c, Lf, c->mean_b.p, true));
    b = c->mean_b.p;
  }
  const bool mixed = F.part[0].A64.set;
  if (opts->method == MG_RICHARDSON) {
    // mixed precision: defect correction x += GMG(L, 0, r), r = b - A x in fp64,
    // kept in a buffer of its own (F.w is the V-cycle's work vector)
    if (mixed && !c->rich_z.p) {
      TRY(c->rich_z.alloc(size_t(std::max<int64_t>(N, 1))));
      TRY(c->rich_r.alloc(size_t(std::max<int64_t>(N, 1))));
    }
    double *r = mixed ? c->rich_r.p : F.w.p;
    TRY(initial_residual(c, Lf, dist, N, x, b, r));
    TRY(dev_dot(c, dist, N, r, r, c->scal.p, true));
    CU(cudaMemcpyAsync(hst, c->scal.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    const double r0 = hst[0];
    if (!std::isfinite(r0)) return fail(MG_ERR_NONFINITE, "non-finite initial residual");
    if (r0 == 0.0) conv = true, rel = 0.0;
    const unsigned eg = unsigned(std::min<int64_t>(std::max<int64_t>(1, (N + 255) / 256), 8 * c->n_sm));
    while (!conv && its < opts->max_iter) {
      if (!mixed) {
        TRY(run_vcycle(c, x, b, false));  // x <- GMG(L, x, b)
      } else {
        TRY(run_vcycle(c, c->rich_z.p, r, true));
        ++g_tally, mgk::k_axpy1<<<eg, 256, 0, c->stream>>>(N, c->rich_z.p, x);
        TRY(check_launch("axpy"));
      }
      ++its;
      TRY(a_pass_resid(c, Lf, x, b, r, true));
      TRY(dev_dot(c, dist, N, r, r, c->scal.p, true));
      CU(cudaMemcpyAsync(hst, c->scal.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
      CU(cudaStreamSynchronize(c->stream));
      if (!std::isfinite(hst[0])) return fail(MG_ERR_NONFINITE, "non-finite residual at iteration %d", its);
      rel = hst[0] / r0;
      if (hst[0] <= rtol * r0) conv = true;
    }
  } else if (opts->method == MG_GMRES || opts->method == MG_GMRES_DCGS2) {
    const bool dcgs = opts->method == MG_GMRES_DCGS2;
    const int m = std::max(1, std::min(opts->restart > 0 ? opts->restart : 30, 64));
    TRY(ensure_gmres(c, m));
    mgk::GmresDev g = c->gm;
    const int ld = g.m + 1;  // leading dimension of the allocated Hessenberg
    double *V = c->gm_V.p, *Z = c->gm_Z.p;
    const int64_t NS = gm_stride(N);
    TRY(initial_residual(c, Lf, dist, N, x, b, V));
    TRY(dev_dot(c, dist, N, V, V, g.beta0, true));
    CU(cudaMemcpyAsync(g.beta, g.beta0, sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    CU(cudaMemcpyAsync(hst, g.beta0, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CU(cudaStreamSynchronize(c->stream));
    const double beta0 = hst[0];
    if (!std::isfinite(beta0)) return fail(MG_ERR_NONFINITE, "non-finite initial residual");
    if (beta0 == 0.0) conv = true, rel = 0.0;
    const unsigned eg = unsigned(std::min<int64_t>(std::max<int64_t>(1, (N + 255) / 256), 8 * c->n_sm));
    while (!conv && its < opts->max_iter) {
      const int mm = std::min(m, opts->max_iter - its);
      if (dcgs) {  // u_0 = r stays in slot 0; step 0 normalises it
        ++g_tally, mgk::k_dcgs_start<<<1, 256, 0, c->stream>>>(g);
      } else {
        ++g_tally, mgk::k_gmres_start<<<1, 32, 0, c->stream>>>(g);
        ++g_tally, mgk::k_scale_div<<<eg, 256, 0, c->stream>>>(N, V, g.beta, V);
      }
      TRY(check_launch("gmres start"));
      int k = 0;
      bool happy = false;  // happy breakdown h_{j+1,j} = 0
      // one Arnoldi step j (V-cycle, SpMV, MGS, Givens, scaling); `cond`: the
      // step runs inside the conditional-graph cycle and steers it itself
      auto step = [&](int j, bool cond, cudaGraphConditionalHandle hw, cudaGraphConditionalHandle hs) -> mg_status {
        double *vj = V + size_t(j) * NS, *zj = Z + size_t(j) * NS, *w = V + size_t(j + 1) * NS;
        if (dcgs) {  // delayed CGS2: one multi-dot pass, one update pass (reading Z29)
          TRY(vcycle_rec(c, Lf, zj, vj, true));            // z_j = GMG(L, 0, u_j)
          TRY(a_pass_spmv(c, Lf, 1.0, zj, 0.0, w, true));  // w^ = A z_j (slot j + 1)
          TRY(dcgs_pass(c, dist, false, N, j, V, NS));     // a, bb, nu, mu
          ++g_tally, mgk::k_dcgs_coef<<<1, 32, 0, c->stream>>>(g, j, mm, hw, cond ? 1 : 0);
          TRY(check_launch("dcgs coef"));
          TRY(dcgs_pass(c, dist, true, N, j, V, NS));      // q_j, u_{j+1}, ||u_{j+1}||^2
          ++g_tally, mgk::k_dcgs_givens<<<1, 32, 0, c->stream>>>(g, j, rtol, mm, hw, hs, cond ? 1 : 0);
          TRY(check_launch("dcgs givens"));
          if (!cond) CU(cudaMemcpyAsync(hst, g.out, 6 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
          return MG_OK;
        }
        TRY(vcycle_rec(c, Lf, zj, vj, true));      // z_j = GMG(L, 0, v_j)
        TRY(a_pass_spmv(c, Lf, 1.0, zj, 0.0, w, true));  // w = A z_j
        double *hcol = g.H + size_t(j) * ld;
        // MGS passes alternate sweep direction (the SpMV wrote w forward), so each
        // pass starts on the L2-resident tail of the previous one (same arithmetic)
        const bool alt = c->mgs_alternate();
        TRY(dev_dot(c, dist, N, w, V, hcol + 0, false, alt));  // h_0j = (w, v_0)
        for (int i = 0; i < j; ++i)                       // w -= h_ij v_i ; h_{i+1,j} = (w, v_{i+1})
          TRY(dev_axpy_dot(c, dist, N, w, V + size_t(i) * NS, hcol + i, V + size_t(i + 1) * NS, hcol + i + 1,
                           alt && (i % 2 == 1)));
        TRY(dev_axpy_dot(c, dist, N, w, vj, hcol + j, nullptr, hcol + j + 1, alt && (j % 2 == 1)));  // w -= h_jj v_j ; ||w||
        ++g_tally, mgk::k_givens<<<1, 32, 0, c->stream>>>(g, j, rtol, mm, hw, hs, cond ? 1 : 0);
        ++g_tally, mgk::k_scale_div<<<eg, 256, 0, c->stream>>>(N, w, g.hn + j, w);  // v_{j+1} = w / h_{j+1,j}
        TRY(check_launch("givens"));
        if (!cond) CU(cudaMemcpyAsync(hst, g.out, 4 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        return MG_OK;
      };
      const double *kdev = nullptr;
      if (c->use_graphs() && !dist && c->gmres_device_loop()) {
        // the whole restart cycle as ONE graph launch: while (continue) {
        // switch (j) { step j } }, steered by k_givens on the device; the host
        // reads (beta, k, stop flags) once per cycle instead of once per step
        const auto key = std::make_tuple(dcgs ? -mm : mm, rtol, g.m);
        auto it = c->cycle_graphs.find(key);
        if (it == c->cycle_graphs.end()) {
          CycleGraph cg;
          TRY(capture_cycle(c, mm, step, cg));
          it = c->cycle_graphs.emplace(key, std::move(cg)).first;
        }
        CU(cudaGraphLaunch(it->second.exec, c->stream));
        CU(cudaMemcpyAsync(hst + 8, g.out, 6 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        kdev = g.out + 3;
        if (dcgs) ++g_tally, mgk::k_dcgs_backsolve<<<1, 32, 0, c->stream>>>(g, 0, kdev);
        else ++g_tally, mgk::k_backsolve<<<1, 32, 0, c->stream>>>(g, 0, kdev);
        ++g_tally, mgk::k_update_x<<<eg, 256, 0, c->stream>>>(N, 0, dcgs ? g.y2 : g.y, Z, NS, x, kdev);
        TRY(check_launch("gmres update"));
        TRY(a_pass_resid(c, Lf, x, b, V, true));
        TRY(dev_dot(c, dist, N, V, V, g.beta, true));
        CU(cudaMemcpyAsync(hst, g.beta, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        CU(cudaStreamSynchronize(c->stream));
        k = int(hst[8 + 3]);
        const int ran = dcgs ? int(hst[8 + 4]) : k;  // steps run (a DCGS2 breakdown step has no column)
        if (ran < 1 || ran > mm || k < 0 || k > ran)
          return fail(MG_ERR_STATE, "GMRES cycle graph ran %d steps (expected 1..%d)", ran, mm);
        for (int j = 0; j < ran; ++j) g_tally += it->second.kernels[size_t(j)];
        its += ran;
        happy = hst[8 + 1] != 0.0 && hst[8 + 2] == 0.0;
      } else {
        for (int j = 0; j < mm; ++j) {
          auto step_j = [&]() { return step(j, false, 0, 0); };
          if (c->use_graphs()) {  // a single CUDA graph per step j, then one host sync
            const auto key = std::make_tuple(j, rtol, g.m);
            auto it = c->iter_graphs.find(key);
            if (it == c->iter_graphs.end()) {
              GraphExec ge;
              const mg_status cs = capture(c, step_j, ge);
              if (cs != MG_OK) {  // as run_vcycle: fall back to eager launches
                if (!c->tr || cs != MG_ERR_CUDA) return cs;
                std::fprintf(stderr, "mgb200: graph capture with the transport failed (%s); running eagerly\n",
                             mg_last_error());
                cudaGetLastError();
                c->cfg.use_graphs = 0;
                c->clear_graphs();
              } else {
                it = c->iter_graphs.emplace(key, ge).first;
              }
            }
            if (c->use_graphs()) TRY(launch_graph(c, it->second));
            else TRY(step_j());
          } else {
            TRY(step_j());
          }
          ++its;
          CU(cudaStreamSynchronize(c->stream));
          k = dcgs ? int(hst[3]) : j + 1;
          if (!std::isfinite(hst[0])) return fail(MG_ERR_NONFINITE, "non-finite GMRES residual estimate");
          if (hst[1] != 0.0) {  // estimate |g_{j+1}| <= rtol beta_0, or breakdown: end of the cycle
            happy = hst[2] == 0.0;
            break;
          }
        }
      }
      if (!kdev) {
        if (dcgs) ++g_tally, mgk::k_dcgs_backsolve<<<1, 32, 0, c->stream>>>(g, k, nullptr);
        else ++g_tally, mgk::k_backsolve<<<1, 32, 0, c->stream>>>(g, k, nullptr);
        ++g_tally, mgk::k_update_x<<<eg, 256, 0, c->stream>>>(N, k, dcgs ? g.y2 : g.y, Z, NS, x, nullptr);
        TRY(check_launch("gmres update"));
        TRY(a_pass_resid(c, Lf, x, b, V, true));
        TRY(dev_dot(c, dist, N, V, V, g.beta, true));
        CU(cudaMemcpyAsync(hst, g.beta, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        CU(cudaStreamSynchronize(c->stream));
      }
      rel = hst[0] / beta0;
      if (!std::isfinite(rel)) return fail(MG_ERR_NONFINITE, "non-finite residual");
      // converged on the TRUE residual (or a happy breakdown); an estimate below
      // rtol whose true residual is above it restarts (reading Z5)
      if (happy || hst[0] <= rtol * beta0) {
        conv = true;
        break;
      }
    }
  } else {
    return fail(MG_ERR_INVALID_ARG, "unknown method %d", opts->method);
  }
  if (F.mean) {  // the normalised solution w^T x = 0
    TRY(mean_project(c, Lf, x, false));
    CU(cudaStreamSynchronize(c->stream));
  }
  if (info) {
    info->iterations = its;
    info->rel_residual = rel;
    info->converged = conv ? 1 : 0;
  }
  return conv ? MG_OK : MG_NOT_CONVERGED;
}

}  // extern "C"
