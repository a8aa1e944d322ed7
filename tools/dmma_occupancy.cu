#include <cstdio>
#include <cuda_runtime.h>
template <int CH>
__global__ void dmma_loop(double* out, int iters) {
  double a = 1e-3 * (threadIdx.x & 7), b = 1e-3 * (threadIdx.x >> 3);
  double c[CH][2];
#pragma unroll
  for (int t = 0; t < CH; ++t) { c[t][0] = 0; c[t][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < CH; ++t)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int t = 0; t < CH; ++t) s += c[t][0] + c[t][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// smem-fed: per k-step load MT A-frags + NT B-frags from smem then MT*NT DMMAs
template <int MT, int NT>
__global__ void dmma_smem(double* out, int iters) {
  __shared__ double As[64][20];
  __shared__ double Bs[32][20];
  for (int i = threadIdx.x; i < 64 * 20; i += blockDim.x) (&As[0][0])[i] = i * 1e-6;
  for (int i = threadIdx.x; i < 32 * 20; i += blockDim.x) (&Bs[0][0])[i] = i * 1e-6;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int ks = 0; ks < 16; ks += 4) {
      double af[MT], bf[NT];
#pragma unroll
      for (int i = 0; i < MT; ++i) af[i] = As[(i * 8 + (lane >> 2)) & 63][ks + (lane & 3)];
#pragma unroll
      for (int j = 0; j < NT; ++j) bf[j] = Bs[(j * 8 + (lane >> 2)) & 31][ks + (lane & 3)];
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j)
          asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n" : "+d"(acc[i][j][0]), "+d"(acc[i][j][1]) : "d"(af[i]), "d"(bf[j]));
    }
    __syncthreads();
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) s += acc[i][j][0] + acc[i][j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int SYNC_dummy;
template <int CH> void run(int warps_per_sm, double* out) {
  int threads = 32 * (warps_per_sm >= 8 ? 8 : warps_per_sm), bps = warps_per_sm * 32 / threads, blocks = 148 * bps, iters = 4000;
  dmma_loop<CH><<<blocks, threads>>>(out, 10);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); dmma_loop<CH><<<blocks, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = 512.0 * CH * iters * (threads / 32) * blocks;
  printf("reg-fed chains=%2d warps/SM=%2d : %.2f TF/s\n", CH, warps_per_sm, fl / ms / 1e9);
}
template <int MT, int NT> void runs(int warps_per_sm, double* out) {
  int threads = 32 * (warps_per_sm >= 8 ? 8 : warps_per_sm), bps = warps_per_sm * 32 / threads, blocks = 148 * bps, iters = 2000;
  dmma_smem<MT, NT><<<blocks, threads>>>(out, 10);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); dmma_smem<MT, NT><<<blocks, threads>>>(out, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double fl = 512.0 * MT * NT * 4 * iters * (threads / 32) * blocks;
  printf("smem-fed MTxNT=%dx%d warps/SM=%2d sync=1: %.2f TF/s\n", MT, NT, warps_per_sm, fl / ms / 1e9);
}
int main() {
  double* out; cudaMalloc(&out, sizeof(double) << 22);
  for (int w : {4, 8, 16, 32}) { run<28>(w, out); run<14>(w, out); run<8>(w, out); run<4>(w, out); }
  for (int w : {8, 16, 32}) { runs<7, 4>(w, out); runs<7, 2>(w, out); runs<2, 1>(w, out); runs<4, 4>(w, out); }
  return 0;
}
