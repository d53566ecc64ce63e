// Newton's method around GMRES + multigrid (include/newton.h): the paper's
// hybrid workflow, Jacobian and residual assembled on the CPU by the caller,
// everything else on the device.
//
// Built only on the public C ABI (mg.h, newton.h) plus two mgi_ queries for
// sizes: the host loop sequences assemble -> ||F|| (device dot) ->
// mg_update_matrix (every level) -> mg_solve -> mg_axpy + mg_apply_constraints.
// The host buffers (w, F, per-level Jacobian values) are pinned so the
// per-step copies run at full PCIe/C2C bandwidth.
#include <cuda_runtime.h>

#include <chrono>
#include <cmath>
#include <vector>

#include "../../include/mg_internal.h"
#include "../../include/newton.h"
#include "common.h"

using namespace mgb;

namespace {

struct Pinned {
  double *p = nullptr;
  ~Pinned() {
    if (p) cudaFreeHost(p);
  }
  mg_status alloc(size_t n) {
    CU(cudaMallocHost(&p, std::max<size_t>(n, 1) * sizeof(double)));
    return MG_OK;
  }
};

struct DevBuf {
  double *p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  mg_status alloc(size_t n) {
    CU(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(double)));
    return MG_OK;
  }
};

double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

}  // namespace

extern "C" {

// Every rank learns whether any rank's assembly callback failed, so all ranks
// leave together instead of the healthy ones blocking in the next collective.
static mg_status agree_assembly(mg_ctx ctx, mg_status as) {
  int all = as;
  const int s = mgi_agree(ctx, as, &all);
  if (s != MG_OK) return mg_status(s);
  if (all == MG_OK) return MG_OK;
  if (as != MG_OK) return as == MG_NOT_CONVERGED ? fail(MG_ERR_INVALID_ARG, "assemble returned %d", as) : as;
  return fail(MG_ERR_STATE, "the assembly callback failed on another rank (status %d)", all);
}

mg_status mg_newton(mg_ctx ctx, double *x, mg_newton_assemble_fn assemble, void *user, const mg_newton_opts *opts,
                    mg_newton_info *info) {
  if (!ctx || !assemble || !opts) return fail(MG_ERR_INVALID_ARG, "NULL ctx, assemble or opts");
  if (opts->max_newton < 0 || opts->max_newton > MG_NEWTON_MAX_HIST || !(opts->ntol >= 0.0) || !(opts->atol >= 0.0))
    return fail(MG_ERR_INVALID_ARG, "bad Newton options (max_newton in [0, %d], tolerances >= 0)", MG_NEWTON_MAX_HIST);
  void *sp = nullptr;
  int device = 0, nl = 0;
  int64_t N = 0;
  if (mgi_stream_info(ctx, &sp, &device, &nl, &N) != 0) return fail(MG_ERR_INVALID_ARG, "bad context");
  if (N > 0 && !x) return fail(MG_ERR_INVALID_ARG, "NULL x");
  int prev = 0;
  CU(cudaGetDevice(&prev));
  CU(cudaSetDevice(device));
  struct Restore {
    int d;
    ~Restore() { cudaSetDevice(d); }
  } restore{prev};
  cudaStream_t st = static_cast<cudaStream_t>(sp);
  const int L = nl - 1;
  int64_t n_f = 0;
  if (mgi_level_info(ctx, L, &n_f, nullptr, nullptr, nullptr, nullptr, nullptr) != 0)
    return fail(MG_ERR_STATE, "context not set up");
  const int bs = n_f > 0 ? int(N / n_f) : 1;
  std::vector<Pinned> vals(nl);
  std::vector<double *> vptr(nl);
  for (int l = 0; l < nl; ++l) {
    int64_t n = 0, nnzb = 0;
    if (mgi_level_info(ctx, l, &n, &nnzb, nullptr, nullptr, nullptr, nullptr) != 0)
      return fail(MG_ERR_STATE, "level %d not set up", l);
    TRY(vals[l].alloc(size_t(nnzb) * bs * bs));
    vptr[l] = vals[l].p;
  }
  Pinned w, Fh;
  TRY(w.alloc(size_t(N)));
  TRY(Fh.alloc(size_t(N)));
  DevBuf f, b, d;
  TRY(f.alloc(size_t(N)));
  TRY(b.alloc(size_t(N)));
  TRY(d.alloc(size_t(N)));
  struct Events {
    cudaEvent_t e[3] = {nullptr, nullptr, nullptr};
    ~Events() {
      for (auto x : e)
        if (x) cudaEventDestroy(x);
    }
  } ev;
  for (auto &x : ev.e) CU(cudaEventCreate(&x));
  mg_newton_info inf{};
  double F0 = -1.0;
  mg_status result = MG_NOT_CONVERGED;
  double Fprev = -1.0;
  for (int k = 0;; ++k) {
    double t0 = now_ms();
    if (N) CU(cudaMemcpyAsync(w.p, x, size_t(N) * sizeof(double), cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
    mg_status as = assemble(user, w.p, Fh.p, nullptr);
    TRY(agree_assembly(ctx, as));
    inf.ms_assemble += now_ms() - t0;
    // f = F, ||F||_2 on the device over all ranks
    if (N) CU(cudaMemcpyAsync(f.p, Fh.p, size_t(N) * sizeof(double), cudaMemcpyHostToDevice, st));
    double nF2 = 0.0;
    TRY(mg_dot(ctx, L, f.p, f.p, &nF2));
    const double nF = std::sqrt(nF2);
    if (!std::isfinite(nF)) return fail(MG_ERR_NONFINITE, "non-finite Newton residual at step %d", k);
    inf.res_norm[k] = nF;
    if (F0 < 0.0) F0 = nF;
    if (nF <= opts->ntol * F0 || nF <= opts->atol) {
      result = MG_OK;
      break;
    }
    if (k == opts->max_newton) break;
    const bool keep = k > 0 && opts->reuse_rate > 0.0 && nF <= opts->reuse_rate * Fprev;
    Fprev = nF;
    CU(cudaEventRecord(ev.e[0], st));
    if (!keep) {
      const double t1 = now_ms();
      as = assemble(user, w.p, nullptr, vptr.data());
      TRY(agree_assembly(ctx, as));
      inf.ms_assemble += now_ms() - t1;
      CU(cudaEventRecord(ev.e[0], st));
      for (int l = 0; l < nl; ++l) TRY(mg_update_matrix(ctx, l, vptr[l], MG_MEM_HOST));
      ++inf.jacobians;
    }
    CU(cudaEventRecord(ev.e[1], st));
    // b = -F, d = 0, solve J d = b, x <- H (x + d)
    if (N) CU(cudaMemsetAsync(b.p, 0, size_t(N) * sizeof(double), st));
    if (N) CU(cudaMemsetAsync(d.p, 0, size_t(N) * sizeof(double), st));
    TRY(mg_axpy(ctx, L, -1.0, f.p, b.p));
    mg_solve_info si{};
    const mg_status ss = mg_solve(ctx, d.p, b.p, &opts->lin, &si);
    if (ss != MG_OK && ss != MG_NOT_CONVERGED) return ss;
    TRY(mg_axpy(ctx, L, 1.0, d.p, x));
    const mg_status hs = mg_apply_constraints(ctx, x);
    if (hs != MG_OK && hs != MG_ERR_STATE) return hs;  // MG_ERR_STATE: no hanging matrix set
    inf.lin_its[k] = si.iterations;
    inf.gmres_its += si.iterations;
    inf.newton_its = k + 1;
    CU(cudaEventRecord(ev.e[2], st));
    CU(cudaStreamSynchronize(st));
    float a = 0.f, b2 = 0.f;
    CU(cudaEventElapsedTime(&a, ev.e[0], ev.e[1]));
    CU(cudaEventElapsedTime(&b2, ev.e[1], ev.e[2]));
    inf.ms_upload += a;
    inf.ms_solve += b2;
  }
  inf.converged = result == MG_OK;
  if (info) *info = inf;
  return result;
}

}  // extern "C"
