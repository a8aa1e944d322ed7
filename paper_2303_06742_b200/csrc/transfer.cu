// K5 grid transfer and K6 coarse solve (sm_100a, fp64).
//   prolongation by interpolation, restriction by the transpose.  Per (Radau node, field, component)
//   the prolongation is the tensor product of 1D interpolation matrices (coarse Q_r / Q_{r-1} Lagrange basis at
//   the fine nodes), stored as per-axis CSR tables; no temporal coarsening (reading A15).
//   direct solve on T_0 = one GEMV with the equilibrated explicit inverse (readings A16, A18); the same GEMV
//   applies the assembled coarse sub-cycle (api.cu build_fold).
#include "stgmg_internal.cuh"

namespace stgmg {

// Restriction / prolongation kernels live in nodal.cu (node-mapped).

// K6: y = A x, A row-major (n x n, lda); one warp per row, fixed-order lane partials + shuffle tree.
__global__ void gemv_kernel(const double* __restrict__ A, int n, int lda, const double* __restrict__ x,
                            double* __restrict__ y) {
  pdl_trigger();
  pdl_wait();
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const double* a = A + (long long)row * lda;
  double s = 0.0;
#pragma unroll 4
  for (int j = lane; j < n; j += 32) s = fma(a[j], x[j], s);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) y[row] = s;
}

cudaError_t launch_gemv(const double* A, int n, int lda, const double* x, double* y, cudaStream_t s) {
  return launch_pdl(gemv_kernel, dim3((n + 7) / 8), dim3(256), 0, s, A, n, lda, x, y);
}

}  // namespace stgmg
