// Transports of libmgb200.so: NCCL (dlopen'd libnccl.so.2) and the in-process
// LOCAL hub (virtual ranks as host threads on one device).  See comm.h.
#include <dlfcn.h>
#include <fcntl.h>
#include <nccl.h>
#include <sys/mman.h>
#include <sys/stat.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <condition_variable>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <thread>

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
  // ncclGroupStart ... ncclGroupEnd with the group always closed, also when a
  // call inside it fails (an open group would swallow the next NCCL call)
  template <class F>
  mg_status grouped(const char *what, F &&body) {
    NCC(nccl().GroupStart());
    ncclResult_t r = body();
    const ncclResult_t e = nccl().GroupEnd();
    if (r == ncclSuccess) r = e;
    if (r != ncclSuccess)
      return comm_fail(MG_ERR_NCCL, "%s: %s", what, nccl().GetErrorString ? nccl().GetErrorString(r) : "?");
    return MG_OK;
  }
  mg_status exchange(const Pattern &p, int width, const double *sendbuf, double *recvbuf, cudaStream_t st) override {
    return grouped("halo exchange", [&]() -> ncclResult_t {
      for (size_t k = 0; k < p.send_rank.size(); ++k) {
        ncclResult_t r = nccl().Send(sendbuf + p.send_off[k] * width, size_t(p.send_cnt[k]) * width, ncclFloat64,
                                     p.send_rank[k], comm, st);
        if (r != ncclSuccess) return r;
      }
      for (size_t k = 0; k < p.recv_rank.size(); ++k) {
        ncclResult_t r = nccl().Recv(recvbuf + p.recv_off[k] * width, size_t(p.recv_cnt[k]) * width, ncclFloat64,
                                     p.recv_rank[k], comm, st);
        if (r != ncclSuccess) return r;
      }
      return ncclSuccess;
    });
  }
  mg_status allreduce_sum(double *dev, int count, cudaStream_t st) override {
    NCC(nccl().AllReduce(dev, dev, size_t(count), ncclFloat64, ncclSum, comm, st));
    return MG_OK;
  }
  mg_status allgatherv(const double *send, double *recv, const std::vector<int64_t> &counts,
                       const std::vector<int64_t> &displs, cudaStream_t st) override {
    mg_status s = grouped("allgatherv", [&]() -> ncclResult_t {
      for (int r = 0; r < nranks; ++r) {
        if (r == rank) continue;
        ncclResult_t e = ncclSuccess;
        if (counts[rank]) e = nccl().Send(send, size_t(counts[rank]), ncclFloat64, r, comm, st);
        if (e == ncclSuccess && counts[r]) e = nccl().Recv(recv + displs[r], size_t(counts[r]), ncclFloat64, r, comm, st);
        if (e != ncclSuccess) return e;
      }
      return ncclSuccess;
    });
    if (s != MG_OK) return s;
    if (send != recv + displs[rank] && counts[rank])
      CUC(cudaMemcpyAsync(recv + displs[rank], send, counts[rank] * sizeof(double), cudaMemcpyDeviceToDevice, st));
    return MG_OK;
  }
  mg_status allgather_host(const void *mine, size_t bytes, void *all) override {
    void *d = nullptr;
    CUC(cudaMalloc(&d, bytes * (nranks + 1)));
    char *dc = static_cast<char *>(d);
    cudaError_t e = cudaMemcpy(dc + bytes * nranks, mine, bytes, cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      cudaFree(d);
      return comm_fail(MG_ERR_CUDA, "allgather_host: %s", cudaGetErrorString(e));
    }
    ncclResult_t r = nccl().AllGather(dc + bytes * nranks, dc, bytes, ncclChar, comm, 0);
    e = cudaStreamSynchronize(0);
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
    cudaError_t e = tot_out ? cudaMemcpy(d, flat.data(), size_t(tot_out), cudaMemcpyHostToDevice) : cudaSuccess;
    if (e != cudaSuccess) {
      cudaFree(d);
      return comm_fail(MG_ERR_CUDA, "alltoallv_host: %s", cudaGetErrorString(e));
    }
    ncclResult_t res = nccl().GroupStart();
    if (res == ncclSuccess) {
      for (int r = 0; r < nranks && res == ncclSuccess; ++r) {
        if (mine[r]) res = nccl().Send(d + ooff[r], size_t(mine[r]), ncclChar, r, comm, 0);
        const int64_t ni = ioff[r + 1] - ioff[r];
        if (ni && res == ncclSuccess) res = nccl().Recv(d + tot_out + ioff[r], size_t(ni), ncclChar, r, comm, 0);
      }
      const ncclResult_t ge = nccl().GroupEnd();  // always close the group
      if (res == ncclSuccess) res = ge;
    }
    e = cudaStreamSynchronize(0);
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


// =============================================================================
// IPC: one PROCESS per rank on one node; ranks may share a device (NCCL
// refuses that) or sit on different GPUs (peer loads over NVLink).  Device
// data moves through one mailbox buffer per rank, exported once with a CUDA
// IPC memory handle; order between processes comes from inter-process CUDA
// events plus a host barrier in a POSIX shared-memory control block.  Every
// collective is:  stage into my mailbox, record ready[me];  barrier;  wait on
// the peers' ready events and copy out of their mailboxes, record done[me];
// barrier;  wait on the done events of the peers that read my mailbox (before
// it may be overwritten).  Host barriers => not graph-capturable.
// =============================================================================
constexpr int kMaxIpc = 16;
constexpr int64_t kIpcMagic = 0x6d67623230304950ll;  // "mgb200IP"

struct IpcCtl {  // lives in POSIX shared memory
  std::atomic<int64_t> magic;
  std::atomic<int> opened;
  std::atomic<int> bar_count;
  std::atomic<int64_t> bar_gen;
  std::atomic<int> failed;
  int nranks;
  struct Rank {
    cudaIpcMemHandle_t mem;
    std::atomic<int64_t> mem_gen;
    cudaIpcEventHandle_t ready, done;
    int64_t seg_off[kMaxIpc], seg_cnt[kMaxIpc];  // current exchange: my data for rank q (doubles)
    int64_t host_bytes;                          // current host blob
  } r[kMaxIpc];
};

class IpcTransport final : public Transport {
 public:
  std::string base;  // shm name prefix
  IpcCtl *ctl = nullptr;
  int device = 0;
  double *mb = nullptr;  // my mailbox
  int64_t mb_cap = 0;    // doubles
  std::vector<double *> old_mb;  // superseded mailboxes (peers may still map them; freed at destruction)
  double *tmp = nullptr;
  int64_t tmp_n = 0;
  cudaEvent_t ready = nullptr, done = nullptr;
  struct Peer {
    void *ptr = nullptr;
    int64_t gen = -1;
    std::vector<void *> old;
    cudaEvent_t ready = nullptr, done = nullptr;
  };
  std::vector<Peer> peer;
  int64_t host_seq = 0;

  ~IpcTransport() override {
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(device);
    cudaDeviceSynchronize();
    for (auto &q : peer) {
      if (q.ptr) cudaIpcCloseMemHandle(q.ptr);
      for (void *o : q.old) cudaIpcCloseMemHandle(o);
      if (q.ready) cudaEventDestroy(q.ready);
      if (q.done) cudaEventDestroy(q.done);
    }
    if (mb) cudaFree(mb);
    for (double *o : old_mb) cudaFree(o);
    if (tmp) cudaFree(tmp);
    if (ready) cudaEventDestroy(ready);
    if (done) cudaEventDestroy(done);
    if (ctl) munmap(ctl, sizeof(IpcCtl));
    cudaSetDevice(cur);
  }

  static bool timed_out(std::chrono::steady_clock::time_point t0) {
    return std::chrono::steady_clock::now() - t0 > std::chrono::seconds(300);
  }

  // sense-free generation barrier over the ranks' processes; false after 300 s
  // (or once any rank gave up): callers turn it into MG_ERR_STATE, not a hang
  bool barrier() {
    const int64_t gen = ctl->bar_gen.load(std::memory_order_acquire);
    if (ctl->bar_count.fetch_add(1, std::memory_order_acq_rel) == nranks - 1) {
      ctl->bar_count.store(0, std::memory_order_relaxed);
      ctl->bar_gen.fetch_add(1, std::memory_order_acq_rel);
      return true;
    }
    const auto t0 = std::chrono::steady_clock::now();
    for (int spin = 0; ctl->bar_gen.load(std::memory_order_acquire) == gen; ++spin) {
      if (ctl->failed.load(std::memory_order_acquire)) return false;
      if (spin > 2000) {
        std::this_thread::sleep_for(std::chrono::microseconds(20));
        if (timed_out(t0)) {
          ctl->failed.store(1, std::memory_order_release);
          return false;
        }
      }
    }
    return true;
  }
#define IPC_BARRIER()                                                                                  \
  do {                                                                                                 \
    if (!barrier()) return comm_fail(MG_ERR_STATE, "IPC transport: barrier timeout (another rank failed)"); \
  } while (0)

  mg_status init(const mg_comm *c, int dev) {
    if (c->nranks > kMaxIpc) return comm_fail(MG_ERR_INVALID_ARG, "IPC transport supports <= %d ranks", kMaxIpc);
    rank = c->rank;
    nranks = c->nranks;
    device = dev;
    static const char *hex = "0123456789abcdef";
    base = "/mgb200_";
    for (int i = 0; i < 16; ++i) base += hex[c->nccl_id[i] >> 4], base += hex[c->nccl_id[i] & 15];
    const std::string name = base + "_ctl";
    const auto t0 = std::chrono::steady_clock::now();
    int fd = -1;
    if (rank == 0) {
      fd = shm_open(name.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
      if (fd < 0 && errno == EEXIST) {  // stale segment of a crashed run with the same key
        shm_unlink(name.c_str());
        fd = shm_open(name.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
      }
      if (fd < 0) return comm_fail(MG_ERR_STATE, "IPC transport: shm_open(%s) failed (errno %d)", name.c_str(), errno);
      if (ftruncate(fd, sizeof(IpcCtl)) != 0) {
        close(fd);
        return comm_fail(MG_ERR_STATE, "IPC transport: ftruncate failed (errno %d)", errno);
      }
    } else {
      while ((fd = shm_open(name.c_str(), O_RDWR, 0600)) < 0) {
        if (timed_out(t0)) return comm_fail(MG_ERR_STATE, "IPC transport: rank 0's segment %s never appeared", name.c_str());
        std::this_thread::sleep_for(std::chrono::milliseconds(2));
      }
      struct stat sb;
      while (fstat(fd, &sb) == 0 && size_t(sb.st_size) < sizeof(IpcCtl)) {
        if (timed_out(t0)) {
          close(fd);
          return comm_fail(MG_ERR_STATE, "IPC transport: segment %s not sized", name.c_str());
        }
        std::this_thread::sleep_for(std::chrono::milliseconds(2));
      }
    }
    void *m = mmap(nullptr, sizeof(IpcCtl), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
    close(fd);
    if (m == MAP_FAILED) return comm_fail(MG_ERR_STATE, "IPC transport: mmap failed (errno %d)", errno);
    ctl = static_cast<IpcCtl *>(m);
    if (rank == 0) {
      new (ctl) IpcCtl();  // zero-initialised atomics
      ctl->nranks = nranks;
      for (int r = 0; r < kMaxIpc; ++r) ctl->r[r].mem_gen.store(-1);
      ctl->magic.store(kIpcMagic, std::memory_order_release);
    } else {
      while (ctl->magic.load(std::memory_order_acquire) != kIpcMagic) {
        if (timed_out(t0)) return comm_fail(MG_ERR_STATE, "IPC transport: segment %s not initialised", name.c_str());
        std::this_thread::sleep_for(std::chrono::milliseconds(1));
      }
      if (ctl->nranks != nranks) return comm_fail(MG_ERR_INVALID_ARG, "IPC transport: group size mismatch");
    }
    int cur = 0;
    CUC(cudaGetDevice(&cur));
    CUC(cudaSetDevice(device));
    CUC(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming | cudaEventInterprocess));
    CUC(cudaEventCreateWithFlags(&done, cudaEventDisableTiming | cudaEventInterprocess));
    CUC(cudaIpcGetEventHandle(&ctl->r[rank].ready, ready));
    CUC(cudaIpcGetEventHandle(&ctl->r[rank].done, done));
    mg_status s = grow(1024, nullptr);
    if (s != MG_OK) return s;
    ctl->opened.fetch_add(1);
    IPC_BARRIER();
    peer.assign(nranks, Peer());
    for (int r = 0; r < nranks; ++r) {
      if (r == rank) continue;
      CUC(cudaIpcOpenEventHandle(&peer[r].ready, ctl->r[r].ready));
      CUC(cudaIpcOpenEventHandle(&peer[r].done, ctl->r[r].done));
    }
    IPC_BARRIER();
    if (rank == 0) shm_unlink(name.c_str());  // every rank has it mapped: nothing left behind
    CUC(cudaSetDevice(cur));
    return MG_OK;
  }
  bool graph_safe() const override { return false; }

  // make my mailbox hold `need` doubles (before the barrier of a collective:
  // peers pick up the new handle after it)
  mg_status grow(int64_t need, cudaStream_t st) {
    if (need <= mb_cap) return MG_OK;
    const int64_t cap = std::max<int64_t>(need, 2 * mb_cap);
    if (st) CUC(cudaStreamSynchronize(st));
    if (mb) old_mb.push_back(mb);  // a peer may still map it: freed at destruction
    mb = nullptr;
    CUC(cudaMalloc(&mb, size_t(cap) * sizeof(double)));
    mb_cap = cap;
    CUC(cudaIpcGetMemHandle(&ctl->r[rank].mem, mb));
    ctl->r[rank].mem_gen.fetch_add(1, std::memory_order_release);
    return MG_OK;
  }
  // the peer's current mailbox (after a barrier)
  mg_status peer_mb(int r, const double **out) {
    if (r == rank) {
      *out = mb;
      return MG_OK;
    }
    Peer &q = peer[r];
    const int64_t gen = ctl->r[r].mem_gen.load(std::memory_order_acquire);
    if (gen != q.gen) {
      if (q.ptr) q.old.push_back(q.ptr);
      q.ptr = nullptr;
      CUC(cudaIpcOpenMemHandle(&q.ptr, ctl->r[r].mem, cudaIpcMemLazyEnablePeerAccess));
      q.gen = gen;
    }
    *out = static_cast<const double *>(q.ptr);
    return MG_OK;
  }

  mg_status exchange(const Pattern &p, int width, const double *sendbuf, double *recvbuf, cudaStream_t st) override {
    const int64_t ns = p.n_send * width;
    mg_status s = grow(std::max<int64_t>(ns, 1), st);
    if (s != MG_OK) return s;
    if (ns) CUC(cudaMemcpyAsync(mb, sendbuf, size_t(ns) * sizeof(double), cudaMemcpyDeviceToDevice, st));
    IpcCtl::Rank &me = ctl->r[rank];
    for (int q = 0; q < kMaxIpc; ++q) me.seg_off[q] = 0, me.seg_cnt[q] = 0;
    for (size_t k = 0; k < p.send_rank.size(); ++k) {
      me.seg_off[p.send_rank[k]] = p.send_off[k] * width;
      me.seg_cnt[p.send_rank[k]] = p.send_cnt[k] * width;
    }
    CUC(cudaEventRecord(ready, st));
    IPC_BARRIER();
    for (size_t k = 0; k < p.recv_rank.size(); ++k) {
      const int src = p.recv_rank[k];
      if (ctl->r[src].seg_cnt[rank] != p.recv_cnt[k] * width)
        return comm_fail(MG_ERR_STATE, "IPC exchange: rank %d sends %lld doubles, rank %d expects %lld", src,
                         (long long)ctl->r[src].seg_cnt[rank], rank, (long long)(p.recv_cnt[k] * width));
      const double *src_mb = nullptr;
      if ((s = peer_mb(src, &src_mb)) != MG_OK) return s;
      CUC(cudaStreamWaitEvent(st, peer[src].ready, 0));
      CUC(cudaMemcpyAsync(recvbuf + p.recv_off[k] * width, src_mb + ctl->r[src].seg_off[rank],
                          size_t(p.recv_cnt[k]) * width * sizeof(double), cudaMemcpyDeviceToDevice, st));
    }
    CUC(cudaEventRecord(done, st));
    IPC_BARRIER();
    for (int dst : p.send_rank) CUC(cudaStreamWaitEvent(st, peer[dst].done, 0));
    return MG_OK;
  }
  mg_status allreduce_sum(double *dev, int count, cudaStream_t st) override {
    mg_status s = grow(std::max(count, 1), st);
    if (s != MG_OK) return s;
    if (tmp_n < count) {
      if (tmp) cudaFree(tmp);
      tmp = nullptr;
      CUC(cudaMalloc(&tmp, sizeof(double) * count));
      tmp_n = count;
    }
    CUC(cudaMemcpyAsync(mb, dev, sizeof(double) * count, cudaMemcpyDeviceToDevice, st));
    CUC(cudaEventRecord(ready, st));
    IPC_BARRIER();
    SumPtrs sp{};
    for (int r = 0; r < nranks; ++r) {
      if ((s = peer_mb(r, &sp.p[r])) != MG_OK) return s;
      if (r != rank) CUC(cudaStreamWaitEvent(st, peer[r].ready, 0));
    }
    k_sum_ranks<<<1, 256, 0, st>>>(count, nranks, sp, tmp);  // fixed rank order, as LOCAL: deterministic
    CUC(cudaGetLastError());
    CUC(cudaEventRecord(done, st));
    IPC_BARRIER();
    for (int r = 0; r < nranks; ++r)
      if (r != rank) CUC(cudaStreamWaitEvent(st, peer[r].done, 0));
    CUC(cudaMemcpyAsync(dev, tmp, sizeof(double) * count, cudaMemcpyDeviceToDevice, st));
    return MG_OK;
  }
  mg_status allgatherv(const double *send, double *recv, const std::vector<int64_t> &counts,
                       const std::vector<int64_t> &displs, cudaStream_t st) override {
    mg_status s = grow(std::max<int64_t>(counts[rank], 1), st);
    if (s != MG_OK) return s;
    if (counts[rank]) CUC(cudaMemcpyAsync(mb, send, size_t(counts[rank]) * sizeof(double), cudaMemcpyDeviceToDevice, st));
    CUC(cudaEventRecord(ready, st));
    IPC_BARRIER();
    for (int r = 0; r < nranks; ++r) {
      if (!counts[r]) continue;
      if (r == rank) {
        if (send != recv + displs[r])
          CUC(cudaMemcpyAsync(recv + displs[r], send, size_t(counts[r]) * sizeof(double), cudaMemcpyDeviceToDevice, st));
        continue;
      }
      const double *src = nullptr;
      if ((s = peer_mb(r, &src)) != MG_OK) return s;
      CUC(cudaStreamWaitEvent(st, peer[r].ready, 0));
      CUC(cudaMemcpyAsync(recv + displs[r], src, size_t(counts[r]) * sizeof(double), cudaMemcpyDeviceToDevice, st));
    }
    CUC(cudaEventRecord(done, st));
    IPC_BARRIER();
    for (int r = 0; r < nranks; ++r)
      if (r != rank) CUC(cudaStreamWaitEvent(st, peer[r].done, 0));
    return MG_OK;
  }

  // host collectives (setup only): every rank publishes one blob in a
  // shared-memory segment of its own; after a barrier every rank reads what
  // it needs from the others' blobs; after a second barrier the blobs go.
  template <class Reader>
  mg_status host_blobs(const char *data, size_t bytes, Reader &&read) {
    const std::string mine = base + "_h" + std::to_string(host_seq) + "_" + std::to_string(rank);
    ++host_seq;
    int fd = shm_open(mine.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
    if (fd < 0 && errno == EEXIST) {
      shm_unlink(mine.c_str());
      fd = shm_open(mine.c_str(), O_CREAT | O_EXCL | O_RDWR, 0600);
    }
    if (fd < 0) return comm_fail(MG_ERR_STATE, "IPC transport: shm_open(%s) failed (errno %d)", mine.c_str(), errno);
    const size_t sz = std::max<size_t>(bytes, 1);
    if (ftruncate(fd, off_t(sz)) != 0) {
      close(fd);
      shm_unlink(mine.c_str());
      return comm_fail(MG_ERR_STATE, "IPC transport: ftruncate failed (errno %d)", errno);
    }
    if (bytes) {
      void *m = mmap(nullptr, sz, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
      if (m == MAP_FAILED) {
        close(fd);
        shm_unlink(mine.c_str());
        return comm_fail(MG_ERR_STATE, "IPC transport: mmap failed (errno %d)", errno);
      }
      std::memcpy(m, data, bytes);
      munmap(m, sz);
    }
    close(fd);
    ctl->r[rank].host_bytes = int64_t(bytes);
    bool ok = barrier();
    for (int r = 0; ok && r < nranks; ++r) {
      if (r == rank) {
        read(r, data, bytes);
        continue;
      }
      const size_t nb = size_t(ctl->r[r].host_bytes);
      if (!nb) {
        read(r, nullptr, 0);
        continue;
      }
      const std::string theirs = base + "_h" + std::to_string(host_seq - 1) + "_" + std::to_string(r);
      const int f = shm_open(theirs.c_str(), O_RDONLY, 0600);
      if (f < 0) {
        ok = false;
        break;
      }
      void *m = mmap(nullptr, nb, PROT_READ, MAP_SHARED, f, 0);
      close(f);
      if (m == MAP_FAILED) {
        ok = false;
        break;
      }
      read(r, static_cast<const char *>(m), nb);
      munmap(m, nb);
    }
    if (!ok) ctl->failed.store(1, std::memory_order_release);
    const bool ok2 = barrier();
    shm_unlink(mine.c_str());
    if (!ok || !ok2) return comm_fail(MG_ERR_STATE, "IPC transport: host collective failed");
    return MG_OK;
  }
  mg_status allgather_host(const void *mine, size_t bytes, void *all) override {
    return host_blobs(static_cast<const char *>(mine), bytes, [&](int r, const char *p, size_t n) {
      if (n == bytes && n) std::memcpy(static_cast<char *>(all) + bytes * r, p, bytes);
    });
  }
  mg_status alltoallv_host(const std::vector<std::vector<char>> &out, std::vector<std::vector<char>> &in) override {
    std::vector<int64_t> off(nranks + 1, 0);
    for (int r = 0; r < nranks; ++r) off[r + 1] = off[r] + int64_t(out[r].size());
    const size_t hdr = sizeof(int64_t) * (nranks + 1);
    std::vector<char> blob(hdr + size_t(off[nranks]));
    std::memcpy(blob.data(), off.data(), hdr);
    for (int r = 0; r < nranks; ++r)
      if (!out[r].empty()) std::memcpy(blob.data() + hdr + off[r], out[r].data(), out[r].size());
    in.assign(nranks, {});
    return host_blobs(blob.data(), blob.size(), [&](int r, const char *p, size_t n) {
      if (n < hdr) return;
      int64_t o[2];
      std::memcpy(o, p + sizeof(int64_t) * rank, sizeof(o));
      in[r].assign(p + hdr + o[0], p + hdr + o[1]);
    });
  }
#undef IPC_BARRIER
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
  } else if (c->transport == MG_TRANSPORT_IPC) {
    auto t = std::make_unique<IpcTransport>();
    mg_status s = t->init(c, device);
    if (s != MG_OK) return s;
    out = std::move(t);
  } else {
    return comm_fail(MG_ERR_INVALID_ARG, "unknown transport %d", c->transport);
  }
  return MG_OK;
}

}  // namespace mgc
