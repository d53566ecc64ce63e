// Micro-benchmark: per-kernel cost of a chain of dependent small kernels in a CUDA
// graph, plain vs Programmatic Dependent Launch (griddepcontrol.wait at the top).
#include <cstdio>
#include <cuda_runtime.h>

template <bool PDL>
__global__ void k_step(double *x, int n) {
  if constexpr (PDL) cudaGridDependencySynchronize();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) x[i] = x[i] * 0.5 + 1.0;
  if constexpr (PDL) cudaTriggerProgrammaticLaunchCompletion();
}

template <bool PDL>
float run(double *x, int n, int grid, int chain, cudaStream_t st) {
  cudaGraph_t g;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
  for (int i = 0; i < chain; ++i) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(256);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = PDL ? 1 : 0;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_step<PDL>, x, n);
  }
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  for (int w = 0; w < 3; ++w) cudaGraphLaunch(ge, st);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a, st);
  const int reps = 10;
  for (int r = 0; r < reps; ++r) cudaGraphLaunch(ge, st);
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(g);
  return 1000.f * ms / (reps * chain);
}

int main() {
  cudaStream_t st;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  double *x;
  cudaMalloc(&x, sizeof(double) * (1 << 22));
  cudaMemset(x, 0, sizeof(double) * (1 << 22));
  const int chain = 400;
  for (int n : {256, 4096, 65536, 1 << 20}) {
    for (int grid : {1, 16, 148, 1184}) {
      if (grid * 256 > 4 * n && grid > 1) continue;
      const float p = run<false>(x, n, grid, chain, st);
      const float q = run<true>(x, n, grid, chain, st);
      printf("n %8d grid %5d: plain %.2f us/kernel, PDL %.2f us/kernel\n", n, grid, p, q);
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
