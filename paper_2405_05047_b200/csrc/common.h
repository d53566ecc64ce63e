// Shared internals of libmgb200.so (mg.cu, ns.cu): error reporting, launch
// accounting, the CU/TRY status macros and the owning device array.
#pragma once
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstddef>
#include <cstdint>
#include <string>

#include "../../include/mg.h"

namespace mgb {

extern thread_local std::string g_err;
extern thread_local int64_t g_tally;  // kernel launches issued by this thread (bench accounting)

mg_status vfail(mg_status st, const char *fmt, va_list ap);
mg_status fail(mg_status st, const char *fmt, ...);

#define CU(x)                                                                                \
  do {                                                                                       \
    cudaError_t e_ = (x);                                                                    \
    if (e_ != cudaSuccess) {                                                                 \
      if (e_ == cudaErrorMemoryAllocation) return fail(MG_ERR_OOM, "%s: out of memory", #x); \
      return fail(MG_ERR_CUDA, "%s: %s", #x, cudaGetErrorString(e_));                        \
    }                                                                                        \
  } while (0)
#define TRY(x)                  \
  do {                          \
    mg_status s_ = (x);         \
    if (s_ != MG_OK) return s_; \
  } while (0)

constexpr int kSigma = 4096;                       // sorting window of SELL-32-sigma
constexpr size_t kStreamBytes = size_t(32) << 20;  // operators larger than this use evict-first loads

template <class T>
struct DevArray {
  T *p = nullptr;
  size_t n = 0;
  DevArray() = default;
  DevArray(const DevArray &) = delete;
  DevArray &operator=(const DevArray &) = delete;
  DevArray(DevArray &&o) noexcept : p(o.p), n(o.n) { o.p = nullptr, o.n = 0; }
  DevArray &operator=(DevArray &&o) noexcept {
    if (this != &o) {
      release();
      p = o.p, n = o.n;
      o.p = nullptr, o.n = 0;
    }
    return *this;
  }
  ~DevArray() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  mg_status alloc(size_t count) {
    release();
    if (count == 0) count = 1;
    CU(cudaMalloc(&p, count * sizeof(T)));
    n = count;
    return MG_OK;
  }
  mg_status upload(const T *h, size_t count) {
    TRY(alloc(count));
    if (h && count) CU(cudaMemcpy(p, h, count * sizeof(T), cudaMemcpyHostToDevice));
    return MG_OK;
  }
};

}  // namespace mgb
