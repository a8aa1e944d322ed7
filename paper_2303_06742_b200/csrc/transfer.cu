// K5 grid transfer and K6 coarse solve (sm_100a, fp64).
//   prolongation by interpolation, restriction by the transpose.  Per (Radau node, field, component)
//   the prolongation is the tensor product of 1D interpolation matrices (coarse Q_r / Q_{r-1} Lagrange basis at
//   the fine nodes), stored as per-axis CSR tables; no temporal coarsening (reading A15).
//   direct solve on T_0 = one GEMV with the equilibrated explicit inverse (readings A16, A18).
#include "stgmg_internal.cuh"

namespace stgmg {

struct Decoded {
  int m, fslot, pres;
  int idx[3];
};

__device__ __forceinline__ Decoded decode(const LevelGeom& g, long long mu) {
  Decoded o;
  const int d = g.d;
  o.m = (int)(mu / g.block);
  long long rem = mu - (long long)o.m * g.block;
  long long node;
  if (rem < 2 * g.R) {
    o.fslot = (int)(rem / g.nq);
    node = rem - (long long)o.fslot * g.nq;
    o.pres = 0;
  } else {
    o.fslot = 2 * d;
    node = rem - 2 * g.R;
    o.pres = 1;
  }
  for (int a = 0; a < 3; ++a) o.idx[a] = 0;
  for (int a = 0; a < d; ++a) {
    const int na = o.pres ? g.pn[a] : g.qn[a];
    o.idx[a] = (int)(node % na);
    node /= na;
  }
  return o;
}

__device__ __forceinline__ long long encode(const LevelGeom& g, int m, int fslot, int pres, const int* idx) {
  long long node = 0;
  for (int a = 0; a < g.d; ++a) node += (long long)idx[a] * (pres ? g.ps[a] : g.qs[a]);
  return (long long)m * g.block + (pres ? 2 * g.R : (long long)fslot * g.nq) + node;
}

// b_c = P^T r_f : one thread per coarse DoF, sum over the fine nodes of its 1D supports.
__global__ void restrict_kernel(LevelGeom f, LevelGeom c, TransferTables t, const double* __restrict__ rf,
                                double* __restrict__ bc) {
  pdl_wait();
  const long long mu = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (mu >= c.N) return;
  const Decoded o = decode(c, mu);
  const Interp1D* T = o.pres ? t.p : t.q;
  const int d = c.d;
  int lo[3] = {0, 0, 0}, hi[3] = {1, 1, 1};
  for (int a = 0; a < d; ++a) {
    lo[a] = T[a].rp_c[o.idx[a]];
    hi[a] = T[a].rp_c[o.idx[a] + 1];
  }
  double s = 0.0;
  int fi[3] = {0, 0, 0};
  for (int e2 = lo[2]; e2 < hi[2]; ++e2) {
    double w2 = 1.0;
    if (d > 2) { fi[2] = T[2].ci_c[e2]; w2 = T[2].v_c[e2]; }
    for (int e1 = lo[1]; e1 < hi[1]; ++e1) {
      double w1 = w2;
      if (d > 1) { fi[1] = T[1].ci_c[e1]; w1 *= T[1].v_c[e1]; }
      for (int e0 = lo[0]; e0 < hi[0]; ++e0) {
        fi[0] = T[0].ci_c[e0];
        s = fma(w1 * T[0].v_c[e0], rf[encode(f, o.m, o.fslot, o.pres, fi)], s);
      }
    }
  }
  bc[mu] = s;
}

// d_f += P d_c : one thread per fine DoF.
__global__ void prolong_kernel(LevelGeom f, LevelGeom c, TransferTables t, const double* __restrict__ dc,
                               double* __restrict__ df) {
  pdl_wait();
  const long long mu = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (mu >= f.N) return;
  const Decoded o = decode(f, mu);
  const Interp1D* T = o.pres ? t.p : t.q;
  const int d = f.d;
  int lo[3] = {0, 0, 0}, hi[3] = {1, 1, 1};
  for (int a = 0; a < d; ++a) {
    lo[a] = T[a].rp_f[o.idx[a]];
    hi[a] = T[a].rp_f[o.idx[a] + 1];
  }
  double s = 0.0;
  int ci[3] = {0, 0, 0};
  for (int e2 = lo[2]; e2 < hi[2]; ++e2) {
    double w2 = 1.0;
    if (d > 2) { ci[2] = T[2].ci_f[e2]; w2 = T[2].v_f[e2]; }
    for (int e1 = lo[1]; e1 < hi[1]; ++e1) {
      double w1 = w2;
      if (d > 1) { ci[1] = T[1].ci_f[e1]; w1 *= T[1].v_f[e1]; }
      for (int e0 = lo[0]; e0 < hi[0]; ++e0) {
        ci[0] = T[0].ci_f[e0];
        s = fma(w1 * T[0].v_f[e0], dc[encode(c, o.m, o.fslot, o.pres, ci)], s);
      }
    }
  }
  df[mu] += s;
}

cudaError_t launch_restrict(const LevelGeom& fine, const LevelGeom& coarse, int, const TransferTables& t,
                            const double* rf, double* bc, cudaStream_t s) {
  const int bs = 256;
  return launch_pdl(restrict_kernel, dim3((unsigned)((coarse.N + bs - 1) / bs)), dim3(bs), 0, s, fine, coarse, t, rf, bc);
}

cudaError_t launch_prolong_add(const LevelGeom& fine, const LevelGeom& coarse, int, const TransferTables& t,
                               const double* dc, double* df, cudaStream_t s) {
  const int bs = 256;
  return launch_pdl(prolong_kernel, dim3((unsigned)((fine.N + bs - 1) / bs)), dim3(bs), 0, s, fine, coarse, t, dc, df);
}

// K6: y = A x, A row-major (n x n, lda); one warp per row, fixed-order lane partials + shuffle tree.
__global__ void gemv_kernel(const double* __restrict__ A, int n, int lda, const double* __restrict__ x,
                            double* __restrict__ y) {
  pdl_wait();
  const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const double* a = A + (long long)row * lda;
  double s = 0.0;
  for (int j = lane; j < n; j += 32) s = fma(a[j], x[j], s);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) y[row] = s;
}

cudaError_t launch_gemv(const double* A, int n, int lda, const double* x, double* y, cudaStream_t s) {
  return launch_pdl(gemv_kernel, dim3((n + 7) / 8), dim3(256), 0, s, A, n, lda, x, y);
}

}  // namespace stgmg
