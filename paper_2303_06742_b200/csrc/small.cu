// Small-level fast path (sm_100a, fp64).  On the coarse levels of the V-cycle every kernel is a latency chain: a few
// thousand DoFs, one warp per SM sub-partition, so a kernel costs (instructions on its critical path) x (their
// latency).  There the operator, the grid transfer and the averaging update are table driven:
//   csr_spmv_kernel : y = beta * base + alpha * M x for an assembled sparse M (CSR, columns ascending) —
//                     the level operator A_l (assembled from the per-cell-type element matrices: the
//                     residual r = b - A_l d of Alg. 1 in ONE kernel instead of element kernel + node gather), the
//                     prolongation P and the restriction P^T;
//   avg_table_kernel: Alg. 1's averaging update d <- d + (omega / p_mu) * sum_{P containing mu} y_P[mu_hat]
//                     (reading A17) with the <= 3^d (patch, local index) offsets of every DoF
//                     precomputed in lexicographic patch order.
// A few lanes per row, strided partial sums combined by a fixed shuffle tree: deterministic, and identical on every
// rank of the x-slab decomposition (the window CSR has the same rows, columns and summation order).
#include "stgmg_internal.cuh"

namespace stgmg {

template <int LPR>
__global__ void __launch_bounds__(256) csr_spmv_kernel(int nrows, const int* __restrict__ rp, const int* __restrict__ ci,
                                                       const double* __restrict__ v, const double* __restrict__ x,
                                                       const double* base, double* y, double alpha, double beta) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int row = t / LPR, sub = t % LPR;
  const bool ok = row < nrows;
  int lo = 0, hi = 0;
  if (ok) {
    lo = __ldg(rp + row);
    hi = __ldg(rp + row + 1);
  }
  pdl_wait();
  double s = 0.0;
  for (int j = lo + sub; j < hi; j += LPR) s = fma(__ldg(v + j), __ldg(x + __ldg(ci + j)), s);
#pragma unroll
  for (int o = LPR / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o, LPR);
  if (ok && sub == 0) y[row] = (base ? beta * base[row] : 0.0) + alpha * s;
}

cudaError_t launch_csr_spmv(int nrows, int lpr, const int* rp, const int* ci, const double* v, const double* x,
                            const double* base, double* y, double alpha, double beta, cudaStream_t s) {
  const int bs = 256;
  const unsigned grid = (unsigned)(((long long)nrows * lpr + bs - 1) / bs);
  switch (lpr) {
    case 4: return launch_pdl(csr_spmv_kernel<4>, dim3(grid), dim3(bs), 0, s, nrows, rp, ci, v, x, base, y, alpha, beta);
    case 8: return launch_pdl(csr_spmv_kernel<8>, dim3(grid), dim3(bs), 0, s, nrows, rp, ci, v, x, base, y, alpha, beta);
    case 16: return launch_pdl(csr_spmv_kernel<16>, dim3(grid), dim3(bs), 0, s, nrows, rp, ci, v, x, base, y, alpha, beta);
    default: return launch_pdl(csr_spmv_kernel<32>, dim3(grid), dim3(bs), 0, s, nrows, rp, ci, v, x, base, y, alpha, beta);
  }
}

// tab[s * N + mu] = offset of y_P[mu_hat] in Y for the s-th patch containing mu (lexicographic), -1 past the last
template <int NS>
__global__ void __launch_bounds__(128) avg_table_kernel(int N, const int* __restrict__ tab, const double* __restrict__ Y,
                                                        double omega, int zero_init, double* __restrict__ dvec,
                                                        int overwrite) {
  const int mu = blockIdx.x * blockDim.x + threadIdx.x;
  if (mu >= N) return;
  int off[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) off[s] = __ldg(tab + (long long)s * N + mu);
  pdl_wait();
  double v[NS];
#pragma unroll
  for (int s = 0; s < NS; ++s) v[s] = __ldg(Y + (off[s] >= 0 ? off[s] : 0));
  const double dold = zero_init ? 0.0 : dvec[mu];
  double z = 0.0;
  int p = 0;
#pragma unroll
  for (int s = 0; s < NS; ++s) {
    if (overwrite) z = off[s] >= 0 ? v[s] : z;   // N2(iii): the last patch's update
    else z += off[s] >= 0 ? v[s] : 0.0;
    p += off[s] >= 0 ? 1 : 0;
  }
  const double upd = z * (overwrite ? omega : omega / (double)p);
  dvec[mu] = zero_init ? upd : dold + upd;
}

cudaError_t launch_avg_table(int d, int N, const int* tab, const double* Y, double omega, int zero_init, double* dvec,
                             cudaStream_t s, int overwrite) {
  const unsigned grid = (unsigned)((N + 127) / 128);
  if (d == 3)
    return launch_pdl(avg_table_kernel<27>, dim3(grid), dim3(128), 0, s, N, tab, Y, omega, zero_init, dvec, overwrite);
  return launch_pdl(avg_table_kernel<9>, dim3(grid), dim3(128), 0, s, N, tab, Y, omega, zero_init, dvec, overwrite);
}

}  // namespace stgmg
