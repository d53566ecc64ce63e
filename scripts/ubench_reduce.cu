// Scratch microbenchmark: fused MGS axpy+dot and scaling kernels at C3 size
// (N = 10,329,843 doubles), grid / block / unroll variants.  nvcc -arch=sm_100a.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int U>
__global__ void k_axpy_dot(long n2, double2 *a, const double2 *b, const double2 *c, const double *h, double *part) {
  __shared__ double sh[32];
  const double hv = *h;
  long tid = long(blockIdx.x) * blockDim.x + threadIdx.x, st = long(gridDim.x) * blockDim.x;
  double s0 = 0, s1 = 0;
  long i = tid;
  for (; i + (U - 1) * st < n2; i += U * st) {
    double2 x[U], v[U], y[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { x[u] = a[i + u * st]; v[u] = __ldg(c + i + u * st); y[u] = __ldg(b + i + u * st); }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      x[u].x = fma(-hv, v[u].x, x[u].x); x[u].y = fma(-hv, v[u].y, x[u].y);
      a[i + u * st] = x[u];
      s0 = fma(x[u].x, y[u].x, s0); s1 = fma(x[u].y, y[u].y, s1);
    }
  }
  for (; i < n2; i += st) {
    double2 x = a[i], v = __ldg(c + i), y = __ldg(b + i);
    x.x = fma(-hv, v.x, x.x); x.y = fma(-hv, v.y, x.y); a[i] = x;
    s0 = fma(x.x, y.x, s0); s1 = fma(x.y, y.y, s1);
  }
  double s = warp_sum(s0 + s1);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double t = threadIdx.x < blockDim.x / 32 ? sh[threadIdx.x] : 0.0;
    t = warp_sum(t);
    if (threadIdx.x == 0) part[blockIdx.x] = t;
  }
}

template <int U>
__global__ void k_scale(long n2, const double2 *in, const double *den, double2 *out, int recip) {
  const double d = *den, r = 1.0 / d;
  long tid = long(blockIdx.x) * blockDim.x + threadIdx.x, st = long(gridDim.x) * blockDim.x;
  for (long i = tid; i < n2; i += st) {
    double2 v = in[i];
    if (recip) { v.x *= r; v.y *= r; } else { v.x /= d; v.y /= d; }
    out[i] = v;
  }
}

int main() {
  const long N = 10329843 + 1, n2 = N / 2;
  double2 *a, *b, *c;
  double *h, *part;
  cudaMalloc(&a, n2 * 16); cudaMalloc(&b, n2 * 16); cudaMalloc(&c, n2 * 16);
  cudaMalloc(&h, 8); cudaMalloc(&part, 8 * 65536);
  cudaMemset(a, 0, n2 * 16); cudaMemset(b, 0, n2 * 16); cudaMemset(c, 0, n2 * 16); cudaMemset(h, 0, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  auto timeit = [&](auto launch, const char *name, double bytes) {
    for (int w = 0; w < 3; ++w) launch();
    cudaEventRecord(e0);
    for (int r = 0; r < 20; ++r) launch();
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1); ms /= 20;
    printf("%-40s %8.1f us  %7.0f GB/s\n", name, ms * 1e3, bytes / (ms * 1e-3) / 1e9);
  };
  const double mgs_bytes = 4.0 * N * 8, sc_bytes = 2.0 * N * 8;
  char nm[128];
  for (int tpb : {256, 512}) for (int mult : {2, 4, 8, 16}) {
    int g = sms * mult;
    snprintf(nm, 128, "axpy_dot U1 tpb %d grid %dx", tpb, mult);
    timeit([&] { k_axpy_dot<1><<<g, tpb>>>(n2, a, b, c, h, part); }, nm, mgs_bytes);
    snprintf(nm, 128, "axpy_dot U2 tpb %d grid %dx", tpb, mult);
    timeit([&] { k_axpy_dot<2><<<g, tpb>>>(n2, a, b, c, h, part); }, nm, mgs_bytes);
    snprintf(nm, 128, "axpy_dot U4 tpb %d grid %dx", tpb, mult);
    timeit([&] { k_axpy_dot<4><<<g, tpb>>>(n2, a, b, c, h, part); }, nm, mgs_bytes);
  }
  for (int mult : {4, 8, 16, 32}) for (int rc : {0, 1}) {
    int g = sms * mult;
    snprintf(nm, 128, "scale %s grid %dx", rc ? "recip" : "div", mult);
    cudaMemcpy(h, &sc_bytes, 8, cudaMemcpyHostToDevice);
    timeit([&] { k_scale<1><<<g, 256>>>(n2, a, h, a, rc); }, nm, sc_bytes);
  }
  return 0;
}
