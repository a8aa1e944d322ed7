// Cost of a software grid barrier in a persistent cooperative kernel on B200 (all CTAs co-resident), versus the
// per-kernel cost of a dependent chain: decides whether the small-level V-cycle tail is worth fusing.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/grid_barrier_probe tools/grid_barrier_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void grid_sync(unsigned* count, volatile unsigned* gen, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(count, 1u) == nblocks - 1) {
      *count = 0;
      __threadfence();
      *gen = g + 1;
    } else {
      while (*gen == g) { }
    }
    __threadfence();
  }
  __syncthreads();
}

__global__ void barrier_loop(unsigned* count, unsigned* gen, int iters, double* x) {
  double v = 0;
  for (int i = 0; i < iters; ++i) {
    v += x[(blockIdx.x * 7 + i) & 1023];   // one dependent L2 load per phase
    grid_sync(count, gen, gridDim.x);
  }
  if (v == 12345.0) x[0] = v;
}

int main() {
  unsigned *count, *gen;
  double* x;
  cudaMalloc(&count, 4); cudaMalloc(&gen, 4); cudaMalloc(&x, 8192 * 8);
  cudaMemset(count, 0, 4); cudaMemset(gen, 0, 4); cudaMemset(x, 0, 8192 * 8);
  for (int bpsm : {1, 2}) {
    for (int threads : {128, 256}) {
      int blocks = 148 * bpsm, iters = 2000;
      void* args[] = {&count, &gen, &iters, &x};
      cudaLaunchCooperativeKernel((void*)barrier_loop, blocks, threads, args, 0, 0);
      cudaDeviceSynchronize();
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)barrier_loop, blocks, threads, args, 0, 0);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("blocks %d threads %d: %.3f us per phase (barrier + 1 load)  err=%s\n", blocks, threads, ms * 1e3 / iters,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
