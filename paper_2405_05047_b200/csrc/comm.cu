// Transports of libmgb200.so: NCCL (dlopen'd libnccl.so.2) and the in-process
// LOCAL hub (virtual ranks as host threads on one device).  See comm.h.
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "comm.h"

namespace mgc {

mg_status comm_fail(mg_status st, const char *fmt, ...);  // defined in mg.cu (thread-local error text)

#define CUC(x)                                                                          \
  do {                                                                                  \
    cudaError_t e_ = (x);                                                               \
    if (e_ != cudaSuccess) return comm_fail(MG_ERR_CUDA, "%s: %s", #x, cudaGetErrorString(e_)); \
  } while (0)

// =============================================================================
// NCCL (dlopen so the library loads without NCCL; MG_ERR_NCCL if missing)
// =============================================================================
struct NcclApi {
  void *h = nullptr;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
  bool load() {
    if (h) return true;
    for (const char *name : {"libnccl.so.2", "libnccl.so"}) {
      h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) return false;
#define SYM(f) f = reinterpret_cast<decltype(f)>(dlsym(h, "nccl" #f))
    SYM(GetUniqueId);
    SYM(CommInitRank);
    SYM(CommDestroy);
    SYM(Send);
    SYM(Recv);
    SYM(AllReduce);
    SYM(AllGather);
    SYM(GroupStart);
    SYM(GroupEnd);
    SYM(GetErrorString);
#undef SYM
    return GetUniqueId && CommInitRank && Send && Recv && AllReduce && AllGather && GroupStart && GroupEnd;
  }
};
NcclApi &nccl() {
  static NcclApi api;
  return api;
}

#define NCC(x)                                                                                    \
  do {                                                                                            \
    ncclResult_t r_ = (x);                                                                        \
    if (r_ != ncclSuccess)                                                                        \
      return comm_fail(MG_ERR_NCCL, "%s: %s", #x, nccl().GetErrorString ? nccl().GetErrorString(r_) : "?"); \
  } while (0)

mg_status nccl_unique_id(unsigned char out[128]) {
  if (!nccl().load()) return comm_fail(MG_ERR_NCCL, "libnccl.so.2 not found");
  ncclUniqueId id;
  NCC(nccl().GetUniqueId(&id));
  std::memcpy(out, &id, 128);
  return MG_OK;
}

class NcclTransport final : public Transport {
 public:
  ncclComm_t comm = nullptr;
  ~NcclTransport() override {
    if (comm && nccl().CommDestroy) nccl().CommDestroy(comm);
  }
  mg_status init(const mg_comm *c) {
    if (!nccl().load()) return comm_fail(MG_ERR_NCCL, "libnccl.so.2 not found");
    ncclUniqueId id;
    std::memcpy(&id, c->nccl_id, 128);
    NCC(nccl().CommInitRank(&comm, c->nranks, id, c->rank));
    rank = c->rank;
    nranks = c->nranks;
    return MG_OK;
  }
  bool graph_safe() const override { return true; }
  mg_status exchange(const Pattern &p, int width, const double *sendbuf, double *recvbuf, cudaStream_t st) override {
    NCC(nccl().GroupStart());
    for (size_t k = 0; k < p.send_rank.size(); ++k)
      NCC(nccl().Send(sendbuf + p.send_off[k] * width, size_t(p.send_cnt[k]) * width, ncclFloat64, p.send_rank[k],
                      comm, st));
    for (size_t k = 0; k < p.recv_rank.size(); ++k)
      NCC(nccl().Recv(recvbuf + p.recv_off[k] * width, size_t(p.recv_cnt[k]) * width, ncclFloat64, p.recv_rank[k],
                      comm, st));
    NCC(nccl().GroupEnd());
    return MG_OK;
  }
  mg_status allreduce_sum(double *dev, int count, cudaStream_t st) override {
    NCC(nccl().AllReduce(dev, dev, size_t(count), ncclFloat64, ncclSum, comm, st));
    return MG_OK;
  }
  mg_status allgatherv(const double *send, double *recv, const std::vector<int64_t> &counts,
                       const std::vector<int64_t> &displs, cudaStream_t st) override {
    NCC(nccl().GroupStart());
    for (int r = 0; r < nranks; ++r) {
      if (r == rank) continue;
      if (counts[rank]) NCC(nccl().Send(send, size_t(counts[rank]), ncclFloat64, r, comm, st));
      if (counts[r]) NCC(nccl().Recv(recv + displs[r], size_t(counts[r]), ncclFloat64, r, comm, st));
    }
    NCC(nccl().GroupEnd());
    if (send != recv + displs[rank] && counts[rank])
      CUC(cudaMemcpyAsync(recv + displs[rank], send, counts[rank] * sizeof(double), cudaMemcpyDeviceToDevice, st));
    return MG_OK;
  }
  mg_status allgather_host(const void *mine, size_t bytes, void *all) override {
    void *d = nullptr;
    CUC(cudaMalloc(&d, bytes * (nranks + 1)));
    char *dc = static_cast<char *>(d);
    cudaMemcpy(dc + bytes * nranks, mine, bytes, cudaMemcpyHostToDevice);
    ncclResult_t r = nccl().AllGather(dc + bytes * nranks, dc, bytes, ncclChar, comm, 0);
    cudaError_t e = cudaStreamSynchronize(0);
    if (r == ncclSuccess && e == cudaSuccess) e = cudaMemcpy(all, dc, bytes * nranks, cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (r != ncclSuccess) return comm_fail(MG_ERR_NCCL, "allgather_host failed");
    if (e != cudaSuccess) return comm_fail(MG_ERR_CUDA, "allgather_host: %s", cudaGetErrorString(e));
    return MG_OK;
  }
  mg_status alltoallv_host(const std::vector<std::vector<char>> &out, std::vector<std::vector<char>> &in) override {
    std::vector<int64_t> mine(nranks), all(size_t(nranks) * nranks);
    for (int r = 0; r < nranks; ++r) mine[r] = int64_t(out[r].size());
    mg_status s = allgather_host(mine.data(), sizeof(int64_t) * nranks, all.data());
    if (s != MG_OK) return s;
    int64_t tot_out = 0, tot_in = 0;
    std::vector<int64_t> ooff(nranks + 1, 0), ioff(nranks + 1, 0);
    for (int r = 0; r < nranks; ++r) {
      ooff[r + 1] = ooff[r] + mine[r];
      ioff[r + 1] = ioff[r] + all[size_t(r) * nranks + rank];
    }
    tot_out = ooff[nranks];
    tot_in = ioff[nranks];
    char *d = nullptr;
    CUC(cudaMalloc(&d, size_t(tot_out + tot_in + 1)));
    std::vector<char> flat(static_cast<size_t>(tot_out));
    for (int r = 0; r < nranks; ++r)
      if (mine[r]) std::memcpy(flat.data() + ooff[r], out[r].data(), size_t(mine[r]));
    if (tot_out) cudaMemcpy(d, flat.data(), size_t(tot_out), cudaMemcpyHostToDevice);
    ncclResult_t res = nccl().GroupStart();
    for (int r = 0; r < nranks && res == ncclSuccess; ++r) {
      if (mine[r]) res = nccl().Send(d + ooff[r], size_t(mine[r]), ncclChar, r, comm, 0);
      const int64_t ni = ioff[r + 1] - ioff[r];
      if (ni && res == ncclSuccess) res = nccl().Recv(d + tot_out + ioff[r], size_t(ni), ncclChar, r, comm, 0);
    }
    if (res == ncclSuccess) res = nccl().GroupEnd();
    cudaError_t e = cudaStreamSynchronize(0);
    std::vector<char> fin(static_cast<size_t>(tot_in));
    if (res == ncclSuccess && e == cudaSuccess && tot_in)
      e = cudaMemcpy(fin.data(), d + tot_out, size_t(tot_in), cudaMemcpyDeviceToHost);
    cudaFree(d);
    if (res != ncclSuccess) return comm_fail(MG_ERR_NCCL, "alltoallv_host failed");
    if (e != cudaSuccess) return comm_fail(MG_ERR_CUDA, "alltoallv_host: %s", cudaGetErrorString(e));
    in.assign(nranks, {});
    for (int r = 0; r < nranks; ++r) in[r].assign(fin.begin() + ioff[r], fin.begin() + ioff[r + 1]);
    return MG_OK;
  }
};

// =============================================================================
// LOCAL: virtual ranks = host threads of one process on one device
// =============================================================================
constexpr int kMaxLocal = 16;

struct SumPtrs {
  const double *p[kMaxLocal];
};

__global__ void k_sum_ranks(int count, int nranks, SumPtrs ptrs, double *out) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < nranks; ++r) s += ptrs.p[r][i];  // fixed rank order: deterministic
    out[i] = s;
  }
}

struct Hub {
  int P = 0;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  int64_t generation = 0;
  std::vector<const void *> ptr;
  std::vector<const Pattern *> pat;
  std::vector<const std::vector<std::vector<char>> *> outs;
  std::vector<cudaEvent_t> ready, done;
  explicit Hub(int n) : P(n), ptr(n), pat(n), outs(n), ready(n), done(n) {
    for (int r = 0; r < n; ++r) {
      cudaEventCreateWithFlags(&ready[r], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&done[r], cudaEventDisableTiming);
    }
  }
  ~Hub() {
    for (int r = 0; r < P; ++r) {
      cudaEventDestroy(ready[r]);
      cudaEventDestroy(done[r]);
    }
  }
  // false after 300 s without the other ranks (a rank failed): no silent hang
  bool barrier() {
    std::unique_lock<std::mutex> lk(m);
    const int64_t gen = generation;
    if (++arrived == P) {
      arrived = 0;
      ++generation;
      cv.notify_all();
      return true;
    }
    if (!cv.wait_for(lk, std::chrono::seconds(300), [&] { return generation != gen; })) {
      --arrived;
      return false;
    }
    return true;
  }
};

std::mutex g_hub_mu;
std::map<std::string, std::weak_ptr<Hub>> g_hubs;

class LocalTransport final : public Transport {
 public:
  std::shared_ptr<Hub> hub;
  double *tmp = nullptr;
  int tmp_n = 0;
  ~LocalTransport() override {
    if (tmp) cudaFree(tmp);
  }
  mg_status init(const mg_comm *c) {
    if (c->nranks > kMaxLocal) return comm_fail(MG_ERR_INVALID_ARG, "LOCAL transport supports <= %d ranks", kMaxLocal);
    std::string key(reinterpret_cast<const char *>(c->nccl_id), 128);
    std::lock_guard<std::mutex> g(g_hub_mu);
    auto it = g_hubs.find(key);
    if (it != g_hubs.end()) hub = it->second.lock();
    if (!hub) {
      hub = std::make_shared<Hub>(c->nranks);
      g_hubs[key] = hub;
    }
    if (hub->P != c->nranks) return comm_fail(MG_ERR_INVALID_ARG, "LOCAL group size mismatch");
    rank = c->rank;
    nranks = c->nranks;
    return MG_OK;
  }
  bool graph_safe() const override { return false; }
  mg_status exchange(const Pattern &p, int width, const double *sendbuf, double *recvbuf, cudaStream_t st) override {
    Hub &h = *hub;
    h.ptr[rank] = sendbuf;
    h.pat[rank] = &p;
    CUC(cudaEventRecord(h.ready[rank], st));
    if (!h.barrier()) return comm_fail(MG_ERR_STATE, "LOCAL transport: barrier timeout (another rank failed)");
    for (size_t k = 0; k < p.recv_rank.size(); ++k) {
      const int src = p.recv_rank[k];
      const Pattern &sp = *h.pat[src];
      int64_t off = -1, cnt = 0;
      for (size_t q = 0; q < sp.send_rank.size(); ++q)
        if (sp.send_rank[q] == rank) off = sp.send_off[q], cnt = sp.send_cnt[q];
      if (off < 0 || cnt != p.recv_cnt[k]) return comm_fail(MG_ERR_STATE, "LOCAL exchange: inconsistent patterns");
      CUC(cudaStreamWaitEvent(st, h.ready[src], 0));
      CUC(cudaMemcpyAsync(recvbuf + p.recv_off[k] * width, static_cast<const double *>(h.ptr[src]) + off * width,
                          size_t(cnt) * width * sizeof(double), cudaMemcpyDeviceToDevice, st));
    }
    CUC(cudaEventRecord(h.done[rank], st));
    if (!h.barrier()) return comm_fail(MG_ERR_STATE, "LOCAL transport: barrier timeout (another rank failed)");
    for (int dst : p.send_rank) CUC(cudaStreamWaitEvent(st, h.done[dst], 0));
    return MG_OK;
  }
  mg_status allreduce_sum(double *dev, int count, cudaStream_t st) override {
    Hub &h = *hub;
    if (tmp_n < count) {
      if (tmp) cudaFree(tmp);
      CUC(cudaMalloc(&tmp, sizeof(double) * count));
      tmp_n = count;
    }
    h.ptr[rank] = dev;
    CUC(cudaEventRecord(h.ready[rank], st));
    if (!h.barrier()) return comm_fail(MG_ERR_STATE, "LOCAL transport: barrier timeout (another rank failed)");
    SumPtrs sp{};
    for (int r = 0; r < nranks; ++r) {
      sp.p[r] = static_cast<const double *>(h.ptr[r]);
      CUC(cudaStreamWaitEvent(st, h.ready[r], 0));
    }
    k_sum_ranks<<<1, 256, 0, st>>>(count, nranks, sp, tmp);
    CUC(cudaGetLastError());
    CUC(cudaEventRecord(h.done[rank], st));
    if (!h.barrier()) return comm_fail(MG_ERR_STATE, "LOCAL transport: barrier timeout (another rank failed)");
    for (int r = 0; r < nranks; ++r) CUC(cudaStreamWaitEvent(st, h.done[r], 0));
    CUC(cudaMemcpyAsync(dev, tmp, sizeof(double) * count, cudaMemcpyDeviceToDevice, st));
    return MG_OK;
  }
  mg_status allgatherv(const double *send, double *recv, const std::vector<int64_t> &counts,
                       const std::vector<int64_t> &displs, cudaStream_t st) override {
    Hub &h = *hub;
    h.ptr[rank] = send;
    CUC(cudaEventRecord(h.ready[rank], st));
    if (!h.barrier()) return comm_fail(MG_ERR_STATE, "LOCAL transport: barrier timeout (another rank failed)");
    for (int r = 0; r < nranks; ++r) {
      if (!counts[r]) continue;
      const double *src = static_cast<const double *>(h.ptr[r]);
      if (r == rank && src == recv + displs[r]) continue;
      CUC(cudaStreamWaitEvent(st, h.ready[r], 0));
      CUC(cudaMemcpyAsync(recv + displs[r], src, counts[r] * sizeof(double), cudaMemcpyDeviceToDevice, st));
    }
    CUC(cudaEventRecord(h.done[rank], st));
    if (!h.barrier()) return comm_fail(MG_ERR_STATE, "LOCAL transport: barrier timeout (another rank failed)");
    for (int r = 0; r < nranks; ++r) CUC(cudaStreamWaitEvent(st, h.done[r], 0));
    return MG_OK;
  }
  mg_status alltoallv_host(const std::vector<std::vector<char>> &out, std::vector<std::vector<char>> &in) override {
    Hub &h = *hub;
    h.outs[rank] = &out;
    if (!h.barrier()) return comm_fail(MG_ERR_STATE, "LOCAL transport: barrier timeout (another rank failed)");
    in.assign(nranks, {});
    for (int r = 0; r < nranks; ++r) in[r] = (*h.outs[r])[rank];
    if (!h.barrier()) return comm_fail(MG_ERR_STATE, "LOCAL transport: barrier timeout (another rank failed)");
    return MG_OK;
  }
  mg_status allgather_host(const void *mine, size_t bytes, void *all) override {
    Hub &h = *hub;
    h.ptr[rank] = mine;
    if (!h.barrier()) return comm_fail(MG_ERR_STATE, "LOCAL transport: barrier timeout (another rank failed)");
    for (int r = 0; r < nranks; ++r) std::memcpy(static_cast<char *>(all) + bytes * r, h.ptr[r], bytes);
    if (!h.barrier()) return comm_fail(MG_ERR_STATE, "LOCAL transport: barrier timeout (another rank failed)");
    return MG_OK;
  }
};

mg_status make_transport(const mg_comm *c, int device, std::unique_ptr<Transport> &out) {
  out.reset();
  if (!c || c->nranks <= 1) return MG_OK;
  if (c->rank < 0 || c->rank >= c->nranks) return comm_fail(MG_ERR_INVALID_ARG, "rank out of range");
  if (c->transport == MG_TRANSPORT_NCCL) {
    auto t = std::make_unique<NcclTransport>();
    mg_status s = t->init(c);
    if (s != MG_OK) return s;
    out = std::move(t);
  } else if (c->transport == MG_TRANSPORT_LOCAL) {
    auto t = std::make_unique<LocalTransport>();
    mg_status s = t->init(c);
    if (s != MG_OK) return s;
    out = std::move(t);
  } else {
    return comm_fail(MG_ERR_INVALID_ARG, "unknown transport %d", c->transport);
  }
  (void)device;
  return MG_OK;
}

}  // namespace mgc
