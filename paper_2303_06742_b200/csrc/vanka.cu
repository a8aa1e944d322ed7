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
// Grouped GEMM  Y[:, P] = Ainv_class * R_P r.  A CTA computes a BM (patch-local rows mu_hat) x BN (patches of one
// class) tile; K runs in chunks of 16 through a multi-stage cp.async pipeline: the A chunk (rows of the class
// inverse, row-major, L2-resident) and the gathered B chunk (R_P r; zero-filled beyond C_P / past the last patch)
// are copied asynchronously into shared memory while the previous chunk is multiplied on the FP64 tensor pipe
// (mma.sync m8n8k4 -> DMMA.8x8x4).  The class's gather table (C_P ints) is staged in shared memory once per CTA.
// Tile variants (WM x WN warps, each MT x NT m8n8 tiles) are picked per level by the patch count so that small
// levels spread over many SMs (latency) and large levels reuse A across many patches (L2 traffic):
//   big 112 x 32 (2x2 warps of 7x2, split-K 2, two CTAs per SM), medium 56 x 32 (1x2 warps of 7x2, split-K 4),
//   small 32 x 8 (2x1 warps of 2x1, split-K 4), tall 224 x 32 (4x1 warps of 7x4, split-K 2: every patch vector is
//   gathered once when C_P <= 224); split-K partial sums are added in a fixed order (deterministic).
constexpr int K2_BK = 16;
constexpr int K2_MAXCP = 2048;       // largest C_P whose gather table is staged in shared memory

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? 8 : 0;   // src-size 0 -> zero fill
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz));
}

__device__ __forceinline__ void cp_async16(double* smem, const double* gmem, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(gmem), "r"(sz));
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <int WM, int WN, int MT, int NT, int STAGES, int KS>
struct K2Cfg {
  static constexpr int BM = WM * MT * 8, BN = WN * NT * 8, THREADS = 32 * WM * WN * KS, NSTAGE = STAGES;
  static constexpr int ASLD = K2_BK + 4;   // 20 doubles: a half-warp's 16 fragment loads hit distinct banks
  static constexpr int BSLD = K2_BK + 4;   // B staged patch-major [BN][16 + 4] (same conflict-free pattern as A)
  static constexpr size_t PIPE = sizeof(double) * STAGES * (BM * ASLD + BN * BSLD);
  static constexpr size_t RED = sizeof(double) * (KS - 1) * BM * BN;   // split-K partial sums (reuses the pipe)
  static constexpr size_t SMEM = PIPE > RED ? PIPE : RED;
};

template <int WM, int WN, int MT, int NT, int K2_STAGES, int KS>
__global__ void __launch_bounds__(32 * WM * WN * KS, (MT * NT <= 16 ? 2 : 1)) patch_gemm_kernel(LevelGeom g, int r,
                                                                  const PatchClass* __restrict__ cls,
                                                                  const TileDesc* __restrict__ tiles,
                                                                  const int* __restrict__ relidx,
                                                                  const double* __restrict__ inv, int lda,
                                                                  const double* __restrict__ rvec,
                                                                  double* __restrict__ Y, int ldy) {
  using C = K2Cfg<WM, WN, MT, NT, K2_STAGES, KS>;
  constexpr int BM = C::BM, BN = C::BN, NTH = C::THREADS, ASLD = C::ASLD, BSLD = C::BSLD;
  extern __shared__ __align__(16) double k2smem[];
  double(*As)[BM][ASLD] = reinterpret_cast<double(*)[BM][ASLD]>(k2smem);
  double(*Bs)[BN][BSLD] = reinterpret_cast<double(*)[BN][BSLD]>(k2smem + K2_STAGES * BM * ASLD);
  __shared__ int baseQ[BN], baseP[BN], plin[BN];
  __shared__ int srel[K2_MAXCP];
  const TileDesc td = tiles[blockIdx.x];
  const PatchClass pc = cls[td.cls];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int d = g.d;
  for (int t = tid; t < BN; t += NTH) {
    const int col = td.n0 + t;
    int bq = 0, bp = 0, pl = -1;
    if (col < pc.ncols) {
      int rem = col, vs = 1;
      pl = 0;
      for (int a = 0; a < d; ++a) {
        const int v = pc.vlo[a] + rem % pc.cnt[a];
        rem /= pc.cnt[a];
        const int c0 = v > 0 ? v - 1 : 0;   // lowest patch cell along a
        bq += (r * c0) * (int)g.qs[a];
        bp += ((r - 1) * c0) * (int)g.ps[a];
        pl += v * vs;
        vs *= (g.n[a] + 1);
      }
    }
    baseQ[t] = bq;
    baseP[t] = bp;
    plin[t] = pl;
  }
  const double* A = inv + pc.inv_off;
  const int cp = pc.cp;
  for (int i = tid; i < cp; i += NTH) srel[i] = __ldg(relidx + pc.rel_off + i);
  __syncthreads();
  pdl_wait();
  const int nchunks = (cp + K2_BK - 1) / K2_BK;

  auto load_chunk = [&](int ch, int buf) {
    const int k0 = ch * K2_BK;
    for (int e = tid; e < BM * 8; e += NTH) {          // A: BM rows x 16 doubles (8 x 16 B per row)
      const int mm = e >> 3, kk = (e & 7) * 2;
      const int row = td.m0 + mm;
      const bool ok = row < lda;
      cp_async16(&As[buf][mm][kk], ok ? A + (long long)row * lda + k0 + kk : A, ok);
    }
    for (int e = tid; e < K2_BK * BN; e += NTH) {      // B: 16 rows x BN patches, gathered from r
      const int kk = e % K2_BK, nn = e / K2_BK;       // lanes run along mu_hat: x-contiguous node runs in r
      const int kr = k0 + kk;
      const bool ok = (kr < cp) && (plin[nn] >= 0);
      const double* src = rvec;
      if (ok) {
        const int code = srel[kr];
        src = rvec + (code >> 1) + ((code & 1) ? baseP[nn] : baseQ[nn]);
      }
      cp_async8(&Bs[buf][nn][kk], src, ok);
    }
    cp_async_commit();
  };

  const int kslice = warp / (WM * WN);            // split-K: warp group kslice takes k4 steps kslice, kslice+KS, ..
  const int wt = warp % (WM * WN);
  const int wm = (wt % WM) * (MT * 8), wn = (wt / WM) * (NT * 8);
  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

#pragma unroll
  for (int st = 0; st < K2_STAGES - 1; ++st) {
    if (st < nchunks) load_chunk(st, st);
    else cp_async_commit();
  }
  for (int ch = 0; ch < nchunks; ++ch) {
    const int buf = ch % K2_STAGES;
    cp_async_wait<K2_STAGES - 2>();
    __syncthreads();
    {
      const int nx = ch + K2_STAGES - 1;   // refill the stage consumed in iteration ch-1
      if (nx < nchunks) load_chunk(nx, nx % K2_STAGES);
      else cp_async_commit();
    }
#pragma unroll
    for (int ks = kslice * 4; ks < K2_BK; ks += 4 * KS) {
      double af[MT], bf[NT];
#pragma unroll
      for (int i = 0; i < MT; ++i) af[i] = As[buf][wm + i * 8 + (lane >> 2)][ks + (lane & 3)];
#pragma unroll
      for (int j = 0; j < NT; ++j) bf[j] = Bs[buf][wn + j * 8 + (lane >> 2)][ks + (lane & 3)];
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();
  if (KS > 1) {   // deterministic split-K reduction: slices 1..KS-1 park their partial sums, slice 0 adds in order
    __syncthreads();
    double* red = k2smem;
    if (kslice > 0) {
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e)
            red[((kslice - 1) * BM + wm + i * 8 + (lane >> 2)) * BN + wn + j * 8 + 2 * (lane & 3) + e] = acc[i][j][e];
    }
    __syncthreads();
    if (kslice > 0) return;
    for (int sl = 1; sl < KS; ++sl)
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e)
            acc[i][j][e] += red[((sl - 1) * BM + wm + i * 8 + (lane >> 2)) * BN + wn + j * 8 + 2 * (lane & 3) + e];
  }
  // C fragment: thread t holds C[t/4][2(t%4) + e] of each 8x8 tile
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int row = td.m0 + wm + i * 8 + (lane >> 2);
        const int nn = wn + j * 8 + 2 * (lane & 3) + e;
        if (row < cp && plin[nn] >= 0) Y[(long long)plin[nn] * ldy + row] = acc[i][j][e];
      }
}

template <int WM, int WN, int MT, int NT, int ST, int KS>
static cudaError_t launch_k2(const LevelGeom& g, int r, const PatchClass* cls_dev, const TileDesc* tiles, int ntiles,
                             const int* relidx, const double* inv, int lda, const double* rvec, double* Y, int ldy,
                             cudaStream_t s) {
  using C = K2Cfg<WM, WN, MT, NT, ST, KS>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(patch_gemm_kernel<WM, WN, MT, NT, ST, KS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)C::SMEM);
    attr = true;
  }
  return launch_pdl(patch_gemm_kernel<WM, WN, MT, NT, ST, KS>, dim3(ntiles), dim3(C::THREADS), C::SMEM, s, g, r, cls_dev, tiles,
                    relidx, inv, lda, rvec, Y, ldy);
}

using K2Big = K2Cfg<2, 2, 7, 2, 4, 2>;     // 112 x 32, 8 warps (2-way split-K), 2 CTAs / SM
using K2Med = K2Cfg<1, 2, 7, 2, 4, 4>;     // 56 x 32, 8 warps (4-way split-K), 2 CTAs / SM
using K2Small = K2Cfg<2, 1, 2, 1, 4, 4>;   // 32 x 8, 8 warps (4-way split-K)
using K2Tall = K2Cfg<4, 1, 7, 4, 3, 2>;    // 224 x 32, 8 warps (2-way split-K): the whole C_P <= 224 in one tile

void k2_tile_shape(int variant, int* bm, int* bn) {
  if (variant == 3) { *bm = K2Tall::BM; *bn = K2Tall::BN; }
  else if (variant == 2) { *bm = K2Big::BM; *bn = K2Big::BN; }
  else if (variant == 1) { *bm = K2Med::BM; *bn = K2Med::BN; }
  else { *bm = K2Small::BM; *bn = K2Small::BN; }
}

int k2_pick_variant(long long npatch, int maxcp) {
  if (maxcp <= 224 && npatch >= 2000) return 3;
  if (npatch >= 2000) return 2;
  if (npatch >= 1000) return 1;
  return 0;
}

cudaError_t launch_patch_gemm(const LevelGeom& g, int r, int variant, const PatchClass* cls_dev, const TileDesc* tiles,
                              int ntiles, const int* relidx, const double* inv, int lda, const double* rvec,
                              double* Y, int ldy, cudaStream_t s) {
  if (variant == 3) return launch_k2<4, 1, 7, 4, 3, 2>(g, r, cls_dev, tiles, ntiles, relidx, inv, lda, rvec, Y, ldy, s);
  if (variant == 2) return launch_k2<2, 2, 7, 2, 4, 2>(g, r, cls_dev, tiles, ntiles, relidx, inv, lda, rvec, Y, ldy, s);
  if (variant == 1) return launch_k2<1, 2, 7, 2, 4, 4>(g, r, cls_dev, tiles, ntiles, relidx, inv, lda, rvec, Y, ldy, s);
  return launch_k2<2, 1, 2, 1, 4, 4>(g, r, cls_dev, tiles, ntiles, relidx, inv, lda, rvec, Y, ldy, s);
}

// ------------------------------------------------------------------------------------------------ K3 --------
__global__ void vanka_average_kernel(LevelGeom g, int r, int k1, const double* __restrict__ Y, int ldy, double omega,
                                     int zero_init, double* __restrict__ dvec) {
  const int mu = blockIdx.x * blockDim.x + threadIdx.x;
  pdl_wait();
  if (mu >= (int)g.N) return;
  const int gblock = (int)g.block, gnq = (int)g.nq, gR2 = (int)(2 * g.R);
  const int d = g.d;
  const int m = mu / gblock;
  int rem = mu - m * gblock;
  int fslot;   // 0..2d-1 = (f, c) Q_r components, 2d = pressure
  int node;
  if (rem < gR2) {
    fslot = rem / gnq;
    node = rem - fslot * gnq;
  } else {
    fslot = 2 * d;
    node = rem - gR2;
  }
  const bool pres = (fslot == 2 * d);
  const int deg = pres ? r - 1 : r;
  int idx[3];
  {
    int t = node;
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
  for (int a = d; a < 3; ++a) { np_[a] = 1; pv[a][0] = 0; }
  // issue all (<= 27) loads first, then sum in the fixed lexicographic patch order
  double yv[27];
#pragma unroll
  for (int i3 = 0; i3 < 3; ++i3)
#pragma unroll
    for (int i2 = 0; i2 < 3; ++i2)
#pragma unroll
      for (int i1 = 0; i1 < 3; ++i1) {
        const int slot = (i3 * 3 + i2) * 3 + i1;
        yv[slot] = 0.0;
        if (i1 < np_[0] && i2 < np_[1] && i3 < np_[2]) {
          const int sel[3] = {i1, i2, i3};
          int plin = 0, vs = 1, loc = 0, ls = 1, nQ = 1, nP = 1;
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            if (a >= d) break;
            const int v = pv[a][sel[a]];
            const int lo = v > 0 ? v - 1 : 0;
            const int ncell = (v > 0 ? 1 : 0) + (v < g.n[a] ? 1 : 0);
            loc += (idx[a] - deg * lo) * ls;
            ls *= deg * ncell + 1;
            nQ *= r * ncell + 1;
            nP *= (r - 1) * ncell + 1;
            plin += v * vs;
            vs *= (g.n[a] + 1);
          }
          const int blk = 2 * d * nQ + nP;
          const int muh = m * blk + (pres ? 2 * d * nQ : fslot * nQ) + loc;
          yv[slot] = __ldg(Y + (long long)plin * ldy + muh);
        }
      }
  double z = 0.0;
#pragma unroll
  for (int i = 0; i < 27; ++i) z += yv[i];
  int p = 1;
  for (int a = 0; a < d; ++a) p *= np_[a];
  const double upd = omega * z / (double)p;
  dvec[mu] = zero_init ? upd : dvec[mu] + upd;
}

cudaError_t launch_vanka_average(const LevelGeom& g, int r, int k1, const double* Y, int ldy, double omega,
                                 int zero_init, double* dvec, cudaStream_t s) {
  const int bs = 256;
  return launch_pdl(vanka_average_kernel, dim3((unsigned)((g.N + bs - 1) / bs)), dim3(bs), 0, s, g, r, k1, Y, ldy, omega,
                    zero_init, dvec);
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

// Element matrices (3D operator): E[t][e][e'] = Ycb[mdof_t(e') * ycstride + rep_t * ne + e], where Ycb holds the
// element results of the mini level for every unit vector (column j at offset j * ycstride) and rep_t is the
// patch-major slot of the representative cell of type t.
__global__ void extract_elem_kernel(const double* __restrict__ Ycb, long long ycstride, int ne,
                                    const long long* __restrict__ rep, const int* __restrict__ mdofs, double* E,
                                    int lda) {
  const int t = blockIdx.y;
  const int e = blockIdx.x;
  double* out = E + (long long)t * lda * lda + (long long)e * lda;
  for (int j = threadIdx.x; j < lda; j += blockDim.x) {
    double v = (e == j) ? 1.0 : 0.0;   // identity padding
    if (e < ne && j < ne) v = Ycb[(long long)mdofs[(long long)t * ne + j] * ycstride + rep[t] * ne + e];
    out[j] = v;
  }
}

cudaError_t launch_extract_elem(const double* Ycb, long long ycstride, int ne, int ntypes, const long long* rep,
                                const int* mdofs, double* E, int lda, cudaStream_t s) {
  extract_elem_kernel<<<dim3(lda, ntypes), 128, 0, s>>>(Ycb, ycstride, ne, rep, mdofs, E, lda);
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
