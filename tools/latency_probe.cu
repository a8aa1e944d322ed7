// Latency floor of dependent kernel chains on B200 (graph-launched, with/without PDL): what a V-cycle phase costs
// before any arithmetic.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lp tools/latency_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_noop(double* y) { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
__global__ void k_ldst(const double* x, double* y, int n) {   // each thread: 1 dependent load + store
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = x[i] + 1.0;
}
__global__ void k_ld36(const double* x, double* y, int n) {   // 36 independent loads per thread, then a store
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double v[36];
#pragma unroll
  for (int j = 0; j < 36; ++j) v[j] = __ldg(x + (i * 37 + j * 101) % (1 << 20));
  double s = 0;
#pragma unroll
  for (int j = 0; j < 36; ++j) s += v[j];
  y[i] = s;
}
__global__ void k_chain4(const double* x, double* y, int n) {   // 4 dependent loads (pointer-chase-like)
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = x[i];
  for (int j = 0; j < 4; ++j) s = x[((int)s + i * 7 + j) & ((1 << 20) - 1)];
  y[i] = s;
}

template <typename F>
float timed(F launch, cudaStream_t st, int reps) {
  cudaGraph_t g; cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  for (int i = 0; i < reps; ++i) launch();
  cudaStreamEndCapture(st, &g);
  cudaGraphInstantiate(&ge, g, 0);
  cudaGraphLaunch(ge, st);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a, st);
  for (int k = 0; k < 5; ++k) cudaGraphLaunch(ge, st);
  cudaEventRecord(b, st);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms * 1e3f / (5 * reps);
}

template <typename... KArgs, typename... Args>
void lk(bool pdl, void (*k)(KArgs...), int grid, int block, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t c = {}; c.gridDim = grid; c.blockDim = block; c.stream = s;
  cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  c.attrs = at; c.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&c, k, static_cast<KArgs>(args)...);
}

int main() {
  double *x, *y;
  cudaMalloc(&x, sizeof(double) << 20); cudaMalloc(&y, sizeof(double) << 20);
  cudaMemset(x, 0, sizeof(double) << 20);
  cudaStream_t s; cudaStreamCreate(&s);
  const int reps = 200;
  for (int pdl = 0; pdl < 2; ++pdl) {
    printf("pdl=%d\n", pdl);
    printf("  noop 1 block          %.2f us\n", timed([&] { lk(pdl, k_noop, 1, 128, s, y); }, s, reps));
    printf("  noop 148 blocks       %.2f us\n", timed([&] { lk(pdl, k_noop, 148, 128, s, y); }, s, reps));
    for (int n : {128, 4096, 141578}) {
      printf("  ldst  n=%-7d        %.2f us\n", n, timed([&] { lk(pdl, k_ldst, (n + 127) / 128, 128, s, (const double*)x, y, n); }, s, reps));
      printf("  ld36  n=%-7d        %.2f us\n", n, timed([&] { lk(pdl, k_ld36, (n + 127) / 128, 128, s, (const double*)x, y, n); }, s, reps));
      printf("  chain4 n=%-7d       %.2f us\n", n, timed([&] { lk(pdl, k_chain4, (n + 127) / 128, 128, s, (const double*)x, y, n); }, s, reps));
    }
  }
  return 0;
}
