// Transport layer of libmgb200.so for row-partitioned multi-GPU solves
// (the paper is single-GPU, multi-GPU is its future work,
// P:800-802).  One rank per GPU.  Two implementations:
//   NCCL  -- ncclSend/ncclRecv halos, ncclAllReduce dots, ncclAllGather for
//            agglomeration, over NVLink / NVSwitch (libnccl.so.2 dlopen'd);
//   LOCAL -- all ranks are host threads of one process sharing one device;
//            stream-ordered device copies + events through an in-process hub.
//            Exists so the complete distributed algorithm runs (and is
//            parity-tested) on a single GPU.  Not graph-capturable.
// All calls are collective over the ranks, in the same order on every rank.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <memory>
#include <vector>

#include "../../include/mg.h"

namespace mgc {

// A neighbour exchange pattern: this rank sends send_cnt[k] items to
// send_rank[k] (from sendbuf offset send_off[k]) and receives recv_cnt[k]
// items from recv_rank[k] (into recvbuf offset recv_off[k]); an item is
// `width` doubles.
struct Pattern {
  std::vector<int> send_rank, recv_rank;
  std::vector<int64_t> send_off, send_cnt, recv_off, recv_cnt;
  int64_t n_send = 0, n_recv = 0;
};

class Transport {
 public:
  virtual ~Transport() = default;
  int rank = 0, nranks = 1;
  virtual bool graph_safe() const = 0;
  // stream-ordered device exchange of doubles
  virtual mg_status exchange(const Pattern &p, int width, const double *sendbuf, double *recvbuf,
                             cudaStream_t st) = 0;
  // in-place sum over ranks of `count` doubles in device memory (summed in rank
  // order for LOCAL; NCCL's order otherwise)
  virtual mg_status allreduce_sum(double *dev, int count, cudaStream_t st) = 0;
  // device allgather-v: rank r contributes counts[r] doubles at displs[r]
  virtual mg_status allgatherv(const double *send, double *recv, const std::vector<int64_t> &counts,
                               const std::vector<int64_t> &displs, cudaStream_t st) = 0;
  // host-memory all-to-all-v of bytes (setup only; synchronous)
  virtual mg_status alltoallv_host(const std::vector<std::vector<char>> &out,
                                   std::vector<std::vector<char>> &in) = 0;
  // host-memory allgather of a fixed-size record (setup only)
  virtual mg_status allgather_host(const void *mine, size_t bytes, void *all) = 0;
};

// Create a transport for mg_comm (NULL or nranks == 1 -> nullptr, single GPU).
mg_status make_transport(const mg_comm *comm, int device, std::unique_ptr<Transport> &out);
mg_status nccl_unique_id(unsigned char out[128]);

}  // namespace mgc
