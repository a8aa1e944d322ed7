// Patch-wise Vanka smoother kernels (sm_100a, fp64): Def:VankaOP and Algorithm 1.
//   K2 vanka_patch_gemm : y_P = A_P^{-1} R_P r for every vertex patch, as a grouped GEMM per patch class
//                         (one shared equilibrated inverse per class) on the FP64 tensor pipe
//                         (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4); the B operand is gathered from r.
//   K3 vanka_average    : d <- d + omega * (sum_{P containing mu} y_P[mu_hat]) / p_mu (pull form, patches in
//                         lexicographic vertex order; reading A17), no atomics.
//   K4 setup            : A_P extraction from the dense operator of a 4^d-cell "mini level" with the same h and
//                         boundary conditions, power-of-2 equilibration and Gauss–Jordan inversion with partial
//                         pivoting (ties -> lowest row) ("inverse ... by LAPACK routines", reading A19).
#include "stgmg_internal.cuh"

namespace stgmg {

// ------------------------------------------------------------------------------------------------ K2 --------
constexpr int GBM = 64, GBN = 32, GBK = 16, GTHREADS = 128;

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(GTHREADS) patch_gemm_kernel(LevelGeom g, int r, int k1,
                                                             const PatchClass* __restrict__ cls,
                                                             const TileDesc* __restrict__ tiles,
                                                             const int* __restrict__ relidx,
                                                             const double* __restrict__ inv, int lda,
                                                             const double* __restrict__ rvec,
                                                             double* __restrict__ Y, int ldy) {
  __shared__ double As[GBK][GBM + 4];
  __shared__ double Bs[GBK][GBN + 4];
  __shared__ long long baseQ[GBN], baseP[GBN], plin[GBN];
  const TileDesc td = tiles[blockIdx.x];
  const PatchClass pc = cls[td.cls];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int d = g.d;
  if (tid < GBN) {
    const int col = td.n0 + tid;
    long long bq = 0, bp = 0, pl = -1;
    if (col < pc.ncols) {
      int rem = col;
      long long vs = 1;
      pl = 0;
      for (int a = 0; a < d; ++a) {
        const int v = pc.vlo[a] + rem % pc.cnt[a];
        rem /= pc.cnt[a];
        const int c0 = v > 0 ? v - 1 : 0;       // lowest patch cell along a
        bq += (long long)(r * c0) * g.qs[a];
        bp += (long long)((r - 1) * c0) * g.ps[a];
        pl += (long long)v * vs;
        vs *= (g.n[a] + 1);
      }
    }
    baseQ[tid] = bq;
    baseP[tid] = bp;
    plin[tid] = pl;
  }
  __syncthreads();
  const double* A = inv + pc.inv_off;
  const int* rel = relidx + pc.rel_off;
  // warp tile: 32 (m) x 16 (n) -> 4 x 2 mma tiles
  const int wm = (warp & 1) * 32, wn = (warp >> 1) * 16;
  double acc[4][2][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int kend = pc.cp;
  for (int k0 = 0; k0 < kend; k0 += GBK) {
    // A chunk: rows m0..m0+63, cols k0..k0+15 (zero padded in memory up to lda)
    for (int i = tid; i < GBM * GBK; i += GTHREADS) {
      const int mm = i / GBK, kk = i % GBK;
      const int row = td.m0 + mm, col = k0 + kk;
      As[kk][mm] = (row < lda && col < lda) ? A[(long long)row * lda + col] : 0.0;
    }
    // B chunk: gathered R_P r
    for (int i = tid; i < GBK * GBN; i += GTHREADS) {
      const int kk = i / GBN, nn = i % GBN;
      const int kr = k0 + kk;
      double v = 0.0;
      if (kr < kend && plin[nn] >= 0) {
        const int code = rel[kr];
        v = rvec[(code >> 1) + ((code & 1) ? baseP[nn] : baseQ[nn])];
      }
      Bs[kk][nn] = v;
    }
    __syncthreads();
#pragma unroll
    for (int ks = 0; ks < GBK; ks += 4) {
      double af[4], bf[2];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = As[ks + (lane & 3)][wm + i * 8 + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < 2; ++j) bf[j] = Bs[ks + (lane & 3)][wn + j * 8 + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 2; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();
  }
  // store: C fragment thread t holds C[t/4][2(t%4) + {0,1}] of each 8x8 tile
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int row = td.m0 + wm + i * 8 + (lane >> 2);
        const int nn = wn + j * 8 + 2 * (lane & 3) + e;
        if (row < pc.cp && plin[nn] >= 0) Y[plin[nn] * ldy + row] = acc[i][j][e];
      }
}

cudaError_t launch_patch_gemm(const LevelGeom& g, int r, int k1, const PatchClass* cls_dev, const TileDesc* tiles,
                              int ntiles, const int* relidx, const double* inv, int lda, const double* rvec,
                              double* Y, int ldy, cudaStream_t s) {
  patch_gemm_kernel<<<ntiles, GTHREADS, 0, s>>>(g, r, k1, cls_dev, tiles, relidx, inv, lda, rvec, Y, ldy);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------------ K3 --------
__global__ void vanka_average_kernel(LevelGeom g, int r, int k1, const double* __restrict__ Y, int ldy, double omega,
                                     int zero_init, double* __restrict__ dvec) {
  const long long mu = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (mu >= g.N) return;
  const int d = g.d;
  const int m = (int)(mu / g.block);
  long long rem = mu - (long long)m * g.block;
  int fslot;   // 0..2d-1 = (f, c) Q_r components, 2d = pressure
  long long node;
  if (rem < 2 * g.R) {
    fslot = (int)(rem / g.nq);
    node = rem - (long long)fslot * g.nq;
  } else {
    fslot = 2 * d;
    node = rem - 2 * g.R;
  }
  const bool pres = (fslot == 2 * d);
  const int deg = pres ? r - 1 : r;
  int idx[3];
  {
    long long t = node;
    for (int a = 0; a < d; ++a) {
      const int na = pres ? g.pn[a] : g.qn[a];
      idx[a] = (int)(t % na);
      t /= na;
    }
  }
  // per-axis candidate patches (vertex indices), ascending
  int pv[3][3], np_[3];
  for (int a = 0; a < d; ++a) {
    const int i = idx[a], n = g.n[a];
    np_[a] = 0;
    if (i % deg == 0) {
      const int v = i / deg;
      if (v >= 1) pv[a][np_[a]++] = v - 1;
      pv[a][np_[a]++] = v;
      if (v <= n - 1) pv[a][np_[a]++] = v + 1;
    } else {
      const int cc = i / deg;
      pv[a][np_[a]++] = cc;
      pv[a][np_[a]++] = cc + 1;
    }
  }
  const int n1 = np_[0], n2 = d > 1 ? np_[1] : 1, n3 = d > 2 ? np_[2] : 1;
  double z = 0.0;
  for (int i3 = 0; i3 < n3; ++i3)
    for (int i2 = 0; i2 < n2; ++i2)
      for (int i1 = 0; i1 < n1; ++i1) {
        const int sel[3] = {i1, i2, i3};
        long long plin = 0, vs = 1;
        int loc = 0, ls = 1;
        long long nQ = 1, nP = 1;
        for (int a = 0; a < d; ++a) {
          const int v = pv[a][sel[a]];
          const int lo = v > 0 ? v - 1 : 0;
          const int ncell = (v > 0 ? 1 : 0) + (v < g.n[a] ? 1 : 0);
          const int boxa = deg * ncell + 1;
          loc += (idx[a] - deg * lo) * ls;
          ls *= boxa;
          nQ *= r * ncell + 1;
          nP *= (r - 1) * ncell + 1;
          plin += (long long)v * vs;
          vs *= (g.n[a] + 1);
        }
        const long long blk = 2 * d * nQ + nP;
        const long long muh = m * blk + (pres ? 2 * d * nQ : fslot * nQ) + loc;
        z += Y[plin * ldy + muh];
      }
  int p = 1;
  for (int a = 0; a < d; ++a) p *= np_[a];
  const double upd = omega * z / (double)p;
  dvec[mu] = zero_init ? upd : dvec[mu] + upd;
}

cudaError_t launch_vanka_average(const LevelGeom& g, int r, int k1, const double* Y, int ldy, double omega,
                                 int zero_init, double* dvec, cudaStream_t s) {
  const int bs = 256;
  vanka_average_kernel<<<(unsigned)((g.N + bs - 1) / bs), bs, 0, s>>>(g, r, k1, Y, ldy, omega, zero_init, dvec);
  return cudaGetLastError();
}

// ------------------------------------------------------------------------------------------------ K4 --------
// inv[c][i][j] = A_mini[dof_c(i)][dof_c(j)], A_mini column-major (column j = A e_j), row-major output, zero pad.
__global__ void extract_kernel(const double* __restrict__ Adense, long long ldA, const int* __restrict__ cps,
                               const long long* __restrict__ offs, const int* __restrict__ dofs, double* inv,
                               int lda) {
  const int c = blockIdx.y;
  const int i = blockIdx.x;
  const int cp = cps[c];
  double* out = inv + (long long)c * lda * lda + (long long)i * lda;
  if (i >= lda) return;
  for (int j = threadIdx.x; j < lda; j += blockDim.x) {
    double v = 0.0;
    if (i < cp && j < cp) v = Adense[(long long)dofs[offs[c] + j] * ldA + dofs[offs[c] + i]];
    else if (i == j) v = 1.0;     // identity padding keeps the padded block invertible
    out[j] = v;
  }
}

cudaError_t launch_extract_patch(const LevelGeom&, int, int, const double* Adense, long long ldA, const int*,
                                 int nclass, const int* cps, const long long* rel_offs, const int* dofs, double* inv,
                                 int lda, cudaStream_t s) {
  extract_kernel<<<dim3(lda, nclass), 256, 0, s>>>(Adense, ldA, cps, rel_offs, dofs, inv, lda);
  return cudaGetLastError();
}

// Power-of-two symmetric equilibration: pre = 1 computes s_i = 2^-round(log2 sqrt|a_ii|) and A <- S A S;
// pre = 0 applies A <- S A S with the stored s (turns (SAS)^{-1} into A^{-1}).
__global__ void gj_equilibrate(double* mats, int lda, const int* n_each, double* scale, int pre, int* status) {
  const int c = blockIdx.x;
  const int n = n_each[c];
  double* A = mats + (long long)c * lda * lda;
  double* s = scale + (long long)c * lda;
  if (pre) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const double a = fabs(A[(long long)i * lda + i]);
      if (a == 0.0) {
        status[c] = -(i + 1);
        s[i] = 1.0;
      } else {
        s[i] = exp2(-rint(0.5 * log2(a)));
      }
    }
    __syncthreads();
  }
  for (long long e = threadIdx.x; e < (long long)n * n; e += blockDim.x) {
    const int i = (int)(e / n), j = (int)(e % n);
    A[(long long)i * lda + j] *= s[i] * s[j];
  }
}

__global__ void gj_pivot(double* mats, int lda, const int* n_each, int k, int* perm, double* colk, int* status) {
  const int c = blockIdx.x;
  const int n = n_each[c];
  if (k >= n || status[c] != 0) return;
  double* A = mats + (long long)c * lda * lda;
  double* ck = colk + (long long)c * lda;
  __shared__ double bv[1024];
  __shared__ int bi[1024];
  double best = -1.0;
  int bidx = n;
  for (int i = k + threadIdx.x; i < n; i += blockDim.x) {
    const double v = fabs(A[(long long)i * lda + k]);
    if (v > best || (v == best && i < bidx)) {
      best = v;
      bidx = i;
    }
  }
  bv[threadIdx.x] = best;
  bi[threadIdx.x] = bidx;
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if (threadIdx.x < st) {
      const double v2 = bv[threadIdx.x + st];
      const int i2 = bi[threadIdx.x + st];
      if (v2 > bv[threadIdx.x] || (v2 == bv[threadIdx.x] && i2 < bi[threadIdx.x])) {
        bv[threadIdx.x] = v2;
        bi[threadIdx.x] = i2;
      }
    }
    __syncthreads();
  }
  const int p = bi[0];
  if (bv[0] <= 0.0) {
    if (threadIdx.x == 0) status[c] = k + 1;
    return;
  }
  if (threadIdx.x == 0) perm[(long long)c * lda + k] = p;
  if (p != k) {
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
      const double t = A[(long long)k * lda + j];
      A[(long long)k * lda + j] = A[(long long)p * lda + j];
      A[(long long)p * lda + j] = t;
    }
  }
  __syncthreads();
  const double piv = A[(long long)k * lda + k];
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    ck[i] = A[(long long)i * lda + k];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x) A[(long long)i * lda + k] = (i == k) ? 1.0 : 0.0;
  __syncthreads();
  const double ip = 1.0 / piv;
  for (int j = threadIdx.x; j < n; j += blockDim.x) A[(long long)k * lda + j] *= ip;
}

__global__ void gj_elim(double* mats, int lda, const int* n_each, int k, const double* colk, const int* status) {
  const int c = blockIdx.y;
  const int n = n_each[c];
  if (k >= n || status[c] != 0) return;
  double* A = mats + (long long)c * lda * lda;
  const double* ck = colk + (long long)c * lda;
  const double* rowk = A + (long long)k * lda;
  const int rows_per_block = 8;
  for (int rr = 0; rr < rows_per_block; ++rr) {
    const int i = blockIdx.x * rows_per_block + rr;
    if (i >= n || i == k) continue;
    const double f = ck[i];
    if (f == 0.0) continue;
    double* Ai = A + (long long)i * lda;
    for (int j = threadIdx.x; j < n; j += blockDim.x) Ai[j] = fma(-f, rowk[j], Ai[j]);
  }
}

__global__ void gj_colperm(double* mats, int lda, const int* n_each, const int* perm) {
  const int c = blockIdx.x;
  const int n = n_each[c];
  double* A = mats + (long long)c * lda * lda;
  const int* pm = perm + (long long)c * lda;
  for (int k = n - 1; k >= 0; --k) {
    const int p = pm[k];
    if (p == k) continue;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const double t = A[(long long)i * lda + k];
      A[(long long)i * lda + k] = A[(long long)i * lda + p];
      A[(long long)i * lda + p] = t;
    }
    __syncthreads();
  }
}

// Batched in-place inverse of nmat matrices (row-major, lda) of sizes n_each (device array).  Returns 0 or the
// negative CUDA error; status[c] != 0 marks a singular matrix (checked by the caller after a sync).
int gauss_jordan_inverse(double* mats, int nmat, int n_max, const int* n_each, int lda, int* perm, double* colk,
                         double* scale, int* status, cudaStream_t s) {
  gj_equilibrate<<<nmat, 256, 0, s>>>(mats, lda, n_each, scale, 1, status);
  for (int k = 0; k < n_max; ++k) {
    gj_pivot<<<nmat, 1024, 0, s>>>(mats, lda, n_each, k, perm, colk, status);
    gj_elim<<<dim3((n_max + 7) / 8, nmat), 256, 0, s>>>(mats, lda, n_each, k, colk, status);
  }
  gj_colperm<<<nmat, 256, 0, s>>>(mats, lda, n_each, perm);
  gj_equilibrate<<<nmat, 256, 0, s>>>(mats, lda, n_each, scale, 0, status);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

}  // namespace stgmg
