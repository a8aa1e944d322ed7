// Patch-wise Vanka smoother kernels (sm_100a, fp64): Def:VankaOP and Algorithm 1.
//   K2 vanka_patch_gemm : y_P = A_P^{-1} R_P r for every vertex patch, as a grouped GEMM per patch class
//                         (one shared equilibrated inverse per class) on the FP64 tensor pipe
//                         (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4); the B operand is gathered from r.
//   K3 vanka_average    : d <- d + omega * (sum_{P containing mu} y_P[mu_hat]) / p_mu (pull form, patches in
//                         lexicographic vertex order; reading A17), no atomics.
//   K4 setup            : A_P extraction from the dense operator of a 4^d-cell "mini level" with the same h and
//                         boundary conditions, power-of-2 equilibration and Gauss–Jordan inversion with partial
//                         pivoting (ties -> lowest row) ("inverse ... by LAPACK routines", reading A19).
#include <algorithm>
#include <cstdlib>

#include "stgmg_internal.cuh"

namespace stgmg {

// ------------------------------------------------------------------------------------------------ K2 --------
// Grouped GEMM  Y[:, P] = Ainv_class * R_P r  on the FP64 tensor pipe (mma.sync m8n8k4 -> SASS DMMA.8x8x4).
// A CTA computes a BM (patch-local rows mu_hat) x BN (patches of one class) tile; K runs in chunks of 16.
//   A operand: the class inverse is stored chunk-major and bank-swizzled (see launch_chunk_swizzle), so the BM x 16
//     slab of a chunk is ONE contiguous run of BM x 128 bytes, fetched by a single bulk async copy (cp.async.bulk,
//     completion counted on the stage's mbarrier).
//   B operand: R_P r gathered element-wise with cp.async (zero fill beyond C_P / for absent columns).
//   S-stage pipeline, one __syncthreads per chunk.  (Multicasting A over thread-block clusters and a
//   warp-specialised variant of THIS gathered-B kernel were measured slower; the dense K2D below,
//   whose B is pre-expanded, is the warp-specialised kernel.)
// Tile variants (WM x WN warps, each MT x NT m8n8 tiles, split-K KS): big 112 x 32, wide 112 x 64, medium 56 x 32,
// small 32 x 8; the dense K2D (pre-expanded B, warp-specialised), the shared-B K2S and the latency variants K2L below
// (k2_pick_variant: which level gets which).  Split-K partial sums are added in a fixed order, every output
// element is computed by exactly one CTA with the same k order whatever the tiling: bitwise reproducible.
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

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* b, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* b, unsigned parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// one chunk (16 k) of a warp's MT x NJ block of m8n8 tiles (NJ <= NT leading column blocks; k4 steps of its slice)
template <int MT, int NT, int NJ, int KS, int BM, int BSLD, int BN>
__device__ __forceinline__ void k2_mma_impl(double (&acc)[MT][NT][2], const double (*A)[16], const double (*B)[BSLD],
                                            int wm, int wn, int kslice, int lane, int swz) {
#pragma unroll
  for (int ks = kslice * 4; ks < 16; ks += 4 * KS) {
    double af[MT], bf[NJ];
#pragma unroll
    for (int i = 0; i < MT; ++i) af[i] = A[wm + i * 8 + (lane >> 2)][(ks + (lane & 3)) ^ swz];
#pragma unroll
    for (int j = 0; j < NJ; ++j) bf[j] = B[wn + j * 8 + (lane >> 2)][ks + (lane & 3)];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < NJ; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
  }
}

template <int WM, int WN, int MT, int NT, int STAGES, int KS>
struct K2Cfg {
  static constexpr int BM = WM * MT * 8, BN = WN * NT * 8, THREADS = 32 * WM * WN * KS, NSTAGE = STAGES;
  static constexpr int BSLD = K2_BK + 4;   // B staged patch-major [BN][16 + 4]: conflict-free fragment loads
  static constexpr size_t ABYTES = sizeof(double) * BM * K2_BK;   // one A chunk (swizzled, unpadded)
  static constexpr size_t PIPE = sizeof(double) * STAGES * (BM * K2_BK + BN * BSLD);
  static constexpr size_t RED = sizeof(double) * (KS - 1) * BM * BN;   // split-K partial sums (reuses the pipe)
  static constexpr size_t BAR_OFF = (PIPE > RED ? PIPE : RED);
  static constexpr size_t SMEM = BAR_OFF + 8 * STAGES;
};

template <int WM, int WN, int MT, int NT, int K2_STAGES, int KS>
__global__ void __launch_bounds__(32 * WM * WN * KS, (MT * NT <= 16 ? 2 : 1)) patch_gemm_kernel(LevelGeom g, int r,
                                                                  const PatchClass* __restrict__ cls,
                                                                  const TileDesc* __restrict__ tiles,
                                                                  const int* __restrict__ relidx,
                                                                  const double* __restrict__ invc, int lda,
                                                                  const double* __restrict__ rvec,
                                                                  double* __restrict__ Y, int ldy) {
  pdl_trigger();
  using C = K2Cfg<WM, WN, MT, NT, K2_STAGES, KS>;
  constexpr int BM = C::BM, BN = C::BN, NTH = C::THREADS, BSLD = C::BSLD, S = K2_STAGES;
  extern __shared__ __align__(128) double k2smem[];
  double(*As)[BM][K2_BK] = reinterpret_cast<double(*)[BM][K2_BK]>(k2smem);
  double(*Bs)[BN][BSLD] = reinterpret_cast<double(*)[BN][BSLD]>(k2smem + S * BM * K2_BK);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(k2smem) + C::BAR_OFF);
  __shared__ int baseQ[BN], baseP[BN], plin[BN];
  __shared__ int srel[K2_MAXCP];
  const TileDesc td = tiles[blockIdx.x];
  const PatchClass pc = cls[td.cls];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cp = pc.cp;
  const int nchunks = (cp + K2_BK - 1) / K2_BK;
  // A chunk ch of this tile: rows [m0, m0 + BM) of chunk ch of the class's chunk-major inverse (lda rows per chunk)
  const double* Ab = invc + pc.inv_off + (long long)td.m0 * K2_BK;
  const long long achunk = (long long)lda * K2_BK;
  auto issue_a = [&](int ch, int buf) {   // thread 0 only
    mbar_expect_tx(&full[buf], (unsigned)C::ABYTES);
    bulk_copy(&As[buf][0][0], Ab + ch * achunk, (unsigned)C::ABYTES, &full[buf]);
  };
  if (tid == 0) {
    for (int st = 0; st < S; ++st) mbar_init(&full[st], 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  // the class inverse is static: its first chunks stream in while the previous kernel drains (PDL)
  if (tid == 0)
    for (int st = 0; st < S - 1; ++st)
      if (st < nchunks) issue_a(st, st);
  const int d = g.d;
  for (int t = tid; t < BN; t += NTH) {
    const int col = td.n0 + t;
    int bq = 0, bp = 0, pl = -1;
    if (t < td.nn && col < pc.ncols) {
      int rem = col, vs = 1;
      pl = 0;
      for (int a = 0; a < d; ++a) {
        const int v = pc.vlo[a] + (rem % pc.cnt[a]) * pc.vst;
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
  for (int i = tid; i < cp; i += NTH) srel[i] = __ldg(relidx + pc.rel_off + i);
  __syncthreads();
  pdl_wait();

  auto load_b = [&](int ch, int buf) {
    const int k0 = ch * K2_BK;
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
  for (int st = 0; st < S - 1; ++st) {
    if (st < nchunks) load_b(st, st);
    cp_async_commit();
  }
  const int swz = ((lane >> 2) & 3) << 2;         // A bank swizzle of this lane's fragment rows (row & 3 == lane>>2 & 3)
  const int nj = td.nn > wn ? min(NT, (td.nn - wn + 7) / 8) : 0;   // non-empty 8-column blocks of this warp
  for (int ch = 0; ch < nchunks; ++ch) {
    const int buf = ch % S;
    mbar_wait(&full[buf], (unsigned)((ch / S) & 1));
    cp_async_wait<S - 2>();
    __syncthreads();
    // warp-uniform branch on the number of non-empty 8-column blocks (predicated-off DMMAs still occupy the pipe)
    if (nj == NT) k2_mma_impl<MT, NT, NT, KS, BM, BSLD, BN>(acc, As[buf], Bs[buf], wm, wn, kslice, lane, swz);
    else if (nj == NT - 1) k2_mma_impl<MT, NT, (NT > 1 ? NT - 1 : 1), KS, BM, BSLD, BN>(acc, As[buf], Bs[buf], wm, wn, kslice, lane, swz);
    else if (nj == NT - 2) k2_mma_impl<MT, NT, (NT > 2 ? NT - 2 : 1), KS, BM, BSLD, BN>(acc, As[buf], Bs[buf], wm, wn, kslice, lane, swz);
    else if (nj == NT - 3) k2_mma_impl<MT, NT, (NT > 3 ? NT - 3 : 1), KS, BM, BSLD, BN>(acc, As[buf], Bs[buf], wm, wn, kslice, lane, swz);
    else if (nj == NT - 4) k2_mma_impl<MT, NT, (NT > 4 ? NT - 4 : 1), KS, BM, BSLD, BN>(acc, As[buf], Bs[buf], wm, wn, kslice, lane, swz);
    const int nx = ch + S - 1;                    // refill the stage consumed in iteration ch - 1
    if (nx < nchunks) {
      if (tid == 0) issue_a(nx, nx % S);
      load_b(nx, nx % S);
    }
    cp_async_commit();
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
static void k2_set_attr() {
  using C = K2Cfg<WM, WN, MT, NT, ST, KS>;
  static PerDeviceOnce attr;
  attr.run([] {
    cudaFuncSetAttribute(patch_gemm_kernel<WM, WN, MT, NT, ST, KS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)C::SMEM);
  });
}

template <int WM, int WN, int MT, int NT, int ST, int KS>
static cudaError_t launch_k2(const LevelGeom& g, int r, const PatchClass* cls_dev, const TileDesc* tiles, int ntiles,
                             const int* relidx, const double* invc, int lda, const double* rvec, double* Y, int ldy,
                             cudaStream_t s) {
  using C = K2Cfg<WM, WN, MT, NT, ST, KS>;
  k2_set_attr<WM, WN, MT, NT, ST, KS>();
  return launch_pdl(patch_gemm_kernel<WM, WN, MT, NT, ST, KS>, dim3(ntiles), dim3(C::THREADS), C::SMEM, s, g, r, cls_dev,
                    tiles, relidx, invc, lda, rvec, Y, ldy);
}

#define K2_BIG 2, 2, 7, 2, 5, 2     // 112 x 32, 8 warps (2-way split-K), 2 CTAs / SM
#define K2_MED 1, 2, 7, 2, 4, 4     // 56 x 32, 8 warps (4-way split-K)
#define K2_SMALL 2, 1, 2, 1, 4, 4   // 32 x 8, 8 warps (4-way split-K)
#define K2_WIDE 2, 4, 7, 2, 3, 1    // 112 x 64, 8 warps (no split-K), 2 CTAs / SM

template <int WM, int WN, int MT, int NT, int ST, int KS>
static int k2_occ() {
  using C = K2Cfg<WM, WN, MT, NT, ST, KS>;
  k2_set_attr<WM, WN, MT, NT, ST, KS>();
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, patch_gemm_kernel<WM, WN, MT, NT, ST, KS>, C::THREADS,
                                                    C::SMEM) != cudaSuccess || nb <= 0) {
    cudaGetLastError();
    nb = 1;
  }
  return nb * 148;
}

// K2D: dense variant of K2 for large levels.  The residual arrives patch-expanded (gather_expand_kernel: class
// chunk-major, bank-swizzled, zero beyond C_P), so BOTH operands of a chunk are single contiguous bulk async copies.
// Warp-specialised: one producer warp (one elected lane issues the two copies per chunk; completion counted on the
// stage's "full" mbarrier by transaction bytes), NCONS consumer warps wait on "full", run the DMMAs and release the
// stage on its "empty" mbarrier.  Same k order and split-K reduction as K2: identical arithmetic.
__device__ __forceinline__ void mbar_arrive(unsigned long long* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(b)) : "memory");
}

template <int MT, int NT, int NJ, int KS>
__device__ __forceinline__ void k2d_mma(double (&acc)[MT][NT][2], const double (*A)[16], const double (*B)[16], int wm,
                                        int wn, int kslice, int lane, int swz) {
#pragma unroll
  for (int ks = kslice * 4; ks < 16; ks += 4 * KS) {
    double af[MT], bf[NJ];
#pragma unroll
    for (int i = 0; i < MT; ++i) af[i] = A[wm + i * 8 + (lane >> 2)][(ks + (lane & 3)) ^ swz];
#pragma unroll
    for (int j = 0; j < NJ; ++j) bf[j] = B[wn + j * 8 + (lane >> 2)][(ks + (lane & 3)) ^ swz];
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < NJ; ++j) dmma884(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
  }
}

template <int WM, int WN, int MT, int NT, int STAGES, int KS>
struct K2DCfg {
  static constexpr int BM = WM * MT * 8, BN = WN * NT * 8, NCONS = WM * WN * KS, THREADS = 32 * (NCONS + 1);
  static constexpr size_t ABYTES = sizeof(double) * BM * K2_BK;
  static constexpr size_t PIPE = sizeof(double) * STAGES * (BM + BN) * K2_BK;
  static constexpr size_t RED = sizeof(double) * (KS - 1) * BM * BN;
  static constexpr size_t BAR_OFF = (PIPE > RED ? PIPE : RED);
  static constexpr size_t SMEM = BAR_OFF + 16 * STAGES;
};

template <int WM, int WN, int MT, int NT, int S, int KS>
__global__ void __launch_bounds__(32 * (WM * WN * KS + 1), 2)
    patch_gemm_dense_kernel(LevelGeom g, const PatchClass* __restrict__ cls, const TileDesc* __restrict__ tiles,
                            const double* __restrict__ invc, int lda, const double* __restrict__ rexp,
                            double* __restrict__ Y, int ldy) {
  using C = K2DCfg<WM, WN, MT, NT, S, KS>;
  constexpr int BM = C::BM, BN = C::BN, NCONS = C::NCONS;
  extern __shared__ __align__(128) double k2dsmem[];
  double(*As)[BM][K2_BK] = reinterpret_cast<double(*)[BM][K2_BK]>(k2dsmem);
  double(*Bs)[BN][K2_BK] = reinterpret_cast<double(*)[BN][K2_BK]>(k2dsmem + S * BM * K2_BK);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(k2dsmem) + C::BAR_OFF);
  unsigned long long* empty = full + S;
  __shared__ int plin[BN];
  const TileDesc td = tiles[blockIdx.x];
  const PatchClass pc = cls[td.cls];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cp = pc.cp;
  const int nchunks = (cp + K2_BK - 1) / K2_BK;
  if (tid == 0) {
    for (int st = 0; st < S; ++st) {
      mbar_init(&full[st], 1);
      mbar_init(&empty[st], NCONS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  for (int t = tid; t < BN; t += C::THREADS) {
    int pl = -1;
    if (t < td.nn && td.n0 + t < pc.ncols) {
      int rem = td.n0 + t, vs = 1;
      pl = 0;
      for (int a = 0; a < g.d; ++a) {
        const int v = pc.vlo[a] + (rem % pc.cnt[a]) * pc.vst;
        rem /= pc.cnt[a];
        pl += v * vs;
        vs *= (g.n[a] + 1);
      }
    }
    plin[t] = pl;
  }
  __syncthreads();
  const int kslice = warp / (WM * WN);
  const int wt = warp % (WM * WN);
  const int wm = (wt % WM) * (MT * 8), wn = (wt / WM) * (NT * 8);
  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  if (warp == NCONS) {
    if (lane == 0) {   // producer: A (static) and B (expanded residual of the previous kernel) per chunk
      const double* Ab = invc + pc.inv_off + (long long)td.m0 * K2_BK;
      const long long achunk = (long long)lda * K2_BK;
      const double* Bb = rexp + pc.rexp_off + (long long)td.n0 * K2_BK;
      const long long bchunk = (long long)pc.ncols * K2_BK;
      const unsigned bbytes = (unsigned)(td.nn * K2_BK * sizeof(double));
      // the class inverse is static: the first S chunks of A stream in while the previous kernel drains (PDL);
      // each stage's barrier expects A + B bytes, so it completes only when B has landed too
      const int pre = nchunks < S ? nchunks : S;
      for (int ch = 0; ch < pre; ++ch) {
        mbar_expect_tx(&full[ch], (unsigned)C::ABYTES + bbytes);
        bulk_copy(&As[ch][0][0], Ab + ch * achunk, (unsigned)C::ABYTES, &full[ch]);
      }
      pdl_wait();
      for (int ch = 0; ch < pre; ++ch) bulk_copy(&Bs[ch][0][0], Bb + ch * bchunk, bbytes, &full[ch]);
      for (int ch = pre; ch < nchunks; ++ch) {
        const int st = ch % S;
        if (ch >= S) mbar_wait(&empty[st], (unsigned)(((ch / S) - 1) & 1));
        mbar_expect_tx(&full[st], (unsigned)C::ABYTES + bbytes);
        bulk_copy(&As[st][0][0], Ab + ch * achunk, (unsigned)C::ABYTES, &full[st]);
        bulk_copy(&Bs[st][0][0], Bb + ch * bchunk, bbytes, &full[st]);
      }
    }
  } else {
    const int swz = ((lane >> 2) & 3) << 2;
    const int nj = td.nn > wn ? min(NT, (td.nn - wn + 7) / 8) : 0;
    for (int ch = 0; ch < nchunks; ++ch) {
      const int st = ch % S;
      mbar_wait(&full[st], (unsigned)((ch / S) & 1));
      if (nj == NT) k2d_mma<MT, NT, NT, KS>(acc, As[st], Bs[st], wm, wn, kslice, lane, swz);
      else if (nj == NT - 1) k2d_mma<MT, NT, (NT > 1 ? NT - 1 : 1), KS>(acc, As[st], Bs[st], wm, wn, kslice, lane, swz);
      else if (nj == NT - 2) k2d_mma<MT, NT, (NT > 2 ? NT - 2 : 1), KS>(acc, As[st], Bs[st], wm, wn, kslice, lane, swz);
      else if (nj == NT - 3) k2d_mma<MT, NT, (NT > 3 ? NT - 3 : 1), KS>(acc, As[st], Bs[st], wm, wn, kslice, lane, swz);
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
    }
  }
  __syncthreads();   // all chunks consumed: the pipe buffer can take the split-K partial sums
  if (warp == NCONS) return;
  if (KS > 1) {
    double* red = k2dsmem;
    if (kslice > 0) {
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j)
#pragma unroll
          for (int e = 0; e < 2; ++e)
            red[((kslice - 1) * BM + wm + i * 8 + (lane >> 2)) * BN + wn + j * 8 + 2 * (lane & 3) + e] = acc[i][j][e];
    }
    asm volatile("bar.sync 1, %0;\n" ::"n"(32 * NCONS) : "memory");
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

#define K2D_BIG 2, 2, 7, 2, 5, 2    // 112 x 32, 8 consumer warps (2-way split-K) + producer
#define K2D_WIDE 2, 4, 7, 2, 4, 1   // 112 x 64, 8 consumer warps + producer

template <int WM, int WN, int MT, int NT, int S, int KS>
static cudaError_t launch_k2d(const LevelGeom& g, const PatchClass* cls_dev, const TileDesc* tiles, int ntiles,
                              const double* invc, int lda, const double* rexp, double* Y, int ldy, cudaStream_t s) {
  using C = K2DCfg<WM, WN, MT, NT, S, KS>;
  static PerDeviceOnce attr;
  attr.run([] {
    cudaFuncSetAttribute(patch_gemm_dense_kernel<WM, WN, MT, NT, S, KS>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)C::SMEM);
  });
  return launch_pdl(patch_gemm_dense_kernel<WM, WN, MT, NT, S, KS>, dim3(ntiles), dim3(C::THREADS), C::SMEM, s, g,
                    cls_dev, tiles, invc, lda, rexp, Y, ldy);
}

// variant 2 (big tiles) or 6 (wide tiles) of the dense K2
cudaError_t launch_patch_gemm_dense(const LevelGeom& g, int variant, const PatchClass* cls_dev, const TileDesc* tiles,
                                    int ntiles, const double* invc, int lda, const double* rexp, double* Y, int ldy,
                                    cudaStream_t s) {
  if (variant == 6) return launch_k2d<K2D_WIDE>(g, cls_dev, tiles, ntiles, invc, lda, rexp, Y, ldy, s);
  return launch_k2d<K2D_BIG>(g, cls_dev, tiles, ntiles, invc, lda, rexp, Y, ldy, s);
}

int k2d_slots(int variant) {
  int nb = 0;
  cudaError_t e;
  if (variant == 6) {
    using C = K2DCfg<K2D_WIDE>;
    cudaFuncSetAttribute(patch_gemm_dense_kernel<K2D_WIDE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, patch_gemm_dense_kernel<K2D_WIDE>, C::THREADS, C::SMEM);
  } else {
    using C = K2DCfg<K2D_BIG>;
    cudaFuncSetAttribute(patch_gemm_dense_kernel<K2D_BIG>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, patch_gemm_dense_kernel<K2D_BIG>, C::THREADS, C::SMEM);
  }
  if (e != cudaSuccess || nb <= 0) {
    cudaGetLastError();
    nb = 1;
  }
  return nb * 148;
}

// K2L: latency variant of K2 for small levels (few patches; the V-cycle there is a chain of latency-bound kernels).
// CTA = 8*MT rows x 8*NT patch columns of one class.  No shared-memory pipeline: warp w takes the 16-wide K chunks
// w, w + nw, ..; every lane loads its m8n8k4 A fragments straight from the chunk-major inverse (L2) and its B
// fragment element from r (through the class gather table).  Within a chunk, lane q of a fragment row takes
// k = 4q + s in the s-th m8n8k4 step (A and B alike), so its four A values are one contiguous, 32-byte aligned block of
// the swizzled row (block q ^ (row mod 4)): ONE 256-bit load per row fragment (LDG.256) instead of four 64-bit loads
// that touch a single sector of each of eight lines — the L1/L2 request rate, not the bytes, bounded the A stream.  The inverse and the gather table are static (setup),
// so the A fragments and gather codes of a warp's first chunk, the codes of its second and the output vertex of
// every column are fetched BEFORE the programmatic-dependent-launch wait, while the previous kernel drains; after
// the wait the critical path is one L2 round trip (the B elements of both chunks and the second A chunk in flight
// together), the DMMAs and the reduction.  The nw partial products are added in warp order (fixed) through shared
// memory.
constexpr int k2l_max_warps(int nt) { return nt == 1 ? 16 : nt == 2 ? 7 : 4; }

template <int MT, int NT>
__global__ void __launch_bounds__(32 * k2l_max_warps(NT), NT == 1 ? 1 : 2) patch_gemm_lat_kernel(LevelGeom g, int r, const PatchClass* __restrict__ cls,
                                                             const TileDesc* __restrict__ tiles,
                                                             const int* __restrict__ relidx,
                                                             const double* __restrict__ invc, int lda,
                                                             const double* __restrict__ rvec, double* __restrict__ Y,
                                                             int ldy) {
  pdl_trigger();
  extern __shared__ double lred[];   // [nw][MT][NT][2][32]
  __shared__ int splin[NT * 8];
  const TileDesc td = tiles[blockIdx.x];
  const PatchClass pc = cls[td.cls];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int cp = pc.cp, nch = (cp + K2_BK - 1) / K2_BK;
  const int d = g.d;
  auto col_base = [&](int col, int& bq, int& bp, int& pl) {   // gather bases / vertex index of patch column col
    int rem = col, vs = 1;
    bq = 0; bp = 0; pl = 0;
    for (int a = 0; a < d; ++a) {
      const int v = pc.vlo[a] + (rem % pc.cnt[a]) * pc.vst;
      rem /= pc.cnt[a];
      const int c0 = v > 0 ? v - 1 : 0;
      bq += (r * c0) * (int)g.qs[a];
      bp += ((r - 1) * c0) * (int)g.ps[a];
      pl += v * vs;
      vs *= (g.n[a] + 1);
    }
  };
  if (threadIdx.x < NT * 8) {
    const int n = threadIdx.x;
    int q, p, pl = -1;
    if (n < td.nn && td.n0 + n < pc.ncols) col_base(td.n0 + n, q, p, pl);
    splin[n] = pl;
  }
  // this lane's B columns j*8 + lane/4 (m8n8k4 .col fragment: k = lane & 3)
  bool cvalid[NT];
  int bq[NT], bp[NT];
#pragma unroll
  for (int j = 0; j < NT; ++j) {
    const int nl = j * 8 + (lane >> 2);
    cvalid[j] = nl < td.nn && td.n0 + nl < pc.ncols;
    int pl = 0;
    bq[j] = bp[j] = 0;
    if (cvalid[j]) col_base(td.n0 + nl, bq[j], bp[j], pl);
  }
  const double* Ab = invc + pc.inv_off + (long long)(td.m0 + (lane >> 2)) * K2_BK;
  const int* rel = relidx + pc.rel_off;
  auto load_codes = [&](int ch, int (&code)[4]) {
#pragma unroll
    for (int st = 0; st < 4; ++st) {
      const int k = ch * K2_BK + (lane & 3) * 4 + st;
      code[st] = (ch < nch && k < cp) ? __ldg(rel + k) : -1;
    }
  };
  auto load_a = [&](int ch, double (&a)[4][MT]) {
    const double* Ac = Ab + (long long)ch * lda * K2_BK + (((lane & 3) ^ ((lane >> 2) & 3)) << 2);
#pragma unroll
    for (int i = 0; i < MT; ++i)
      asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];\n"
                   : "=d"(a[0][i]), "=d"(a[1][i]), "=d"(a[2][i]), "=d"(a[3][i])
                   : "l"(Ac + i * 8 * K2_BK));
  };
  auto load_b = [&](const int (&code)[4], double (&b)[4][NT]) {
#pragma unroll
    for (int st = 0; st < 4; ++st)
#pragma unroll
      for (int j = 0; j < NT; ++j)
        b[st][j] = (cvalid[j] && code[st] >= 0) ? __ldg(rvec + (code[st] >> 1) + ((code[st] & 1) ? bp[j] : bq[j]))
                                                : 0.0;
  };
  double acc[MT][NT][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  auto mma = [&](const double (&a)[4][MT], const double (&b)[4][NT]) {
#pragma unroll
    for (int st = 0; st < 4; ++st)
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < NT; ++j) dmma884(acc[i][j][0], acc[i][j][1], a[st][i], b[st][j]);
  };
  const int c0 = warp, c1 = warp + nw;
  int k0[4], k1[4];
  double a0[4][MT];
  load_codes(c0, k0);
  load_codes(c1, k1);
  if (c0 < nch) load_a(c0, a0);
  pdl_wait();
  if (c0 < nch) {
    double b0[4][NT], b1[4][NT], a1[4][MT];
    load_b(k0, b0);
    if (c1 < nch) {
      load_b(k1, b1);
      load_a(c1, a1);
    }
    mma(a0, b0);
    if (c1 < nch) mma(a1, b1);
    for (int ch = c1 + nw; ch < nch; ch += nw) {   // more than two chunks per warp (large C_P)
      int kc[4];
      double ac[4][MT], bc[4][NT];
      load_codes(ch, kc);
      load_a(ch, ac);
      load_b(kc, bc);
      mma(ac, bc);
    }
  }
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) lred[(((warp * MT + i) * NT + j) * 2 + e) * 32 + lane] = acc[i][j][e];
  __syncthreads();
  for (int t = threadIdx.x; t < MT * NT * 2 * 32; t += blockDim.x) {
    const int ln = t & 31, e = (t >> 5) & 1, j = (t >> 6) % NT, i = (t >> 6) / NT;
    double sum = 0.0;
    for (int w = 0; w < nw; ++w) sum += lred[(((w * MT + i) * NT + j) * 2 + e) * 32 + ln];
    const int row = td.m0 + i * 8 + (ln >> 2);
    const int pl = splin[j * 8 + 2 * (ln & 3) + e];
    if (row < cp && pl >= 0) Y[(long long)pl * ldy + row] = sum;
  }
}

constexpr int K2L_MT = 4;   // 32-row tiles

template <int NT>
static int k2l_warps(int lda) {   // at most k2l_max_warps(NT), the chunks spread evenly (2 per warp on cfg1's level 4)
  const int nch = std::max(1, lda / K2_BK), maxw = k2l_max_warps(NT);
  const int per = (nch + maxw - 1) / maxw;
  return (nch + per - 1) / per;
}

template <int NT>
static size_t k2l_smem(int nw) { return sizeof(double) * nw * K2L_MT * NT * 2 * 32; }

template <int NT>
static cudaError_t launch_k2l(const LevelGeom& g, int r, const PatchClass* cls_dev, const TileDesc* tiles, int ntiles,
                              const int* relidx, const double* invc, int lda, const double* rvec, double* Y, int ldy,
                              cudaStream_t s) {
  const int nw = k2l_warps<NT>(lda);
  return launch_pdl(patch_gemm_lat_kernel<K2L_MT, NT>, dim3(ntiles), dim3(32 * nw), k2l_smem<NT>(nw), s, g, r,
                    cls_dev, tiles, relidx, invc, lda, rvec, Y, ldy);
}

template <int NT>
static int k2l_slots() {
  int nb = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, patch_gemm_lat_kernel<K2L_MT, NT>, 32 * k2l_max_warps(NT),
                                                    k2l_smem<NT>(k2l_max_warps(NT))) != cudaSuccess || nb <= 0) {
    cudaGetLastError();
    nb = 1;
  }
  return nb * 148;
}

// K2S: shared-B variant for the middle levels (C_P <= 256, up to a few thousand patches).  CTA = 8*NW rows x 32
// patch columns, no split-K: warp w owns rows [m0 + 8w, m0 + 8w + 8) over the whole K.  The B tile (32 columns x
// all of K) is gathered from r ONCE per CTA into shared memory (consecutive threads along k: contiguous node runs)
// and read by every warp; each warp streams only its own A rows from L2 with one 256-bit load per chunk (k = 4q + s
// lane mapping as K2L), one chunk ahead.  Against K2L (32 x 16 tiles, every warp re-reading A per column tile) this
// halves the A stream and fits a level in one wave of CTAs.  Static operands (gather codes, column bases, the first
// A chunk) are fetched before the PDL wait.  Summation over k is sequential per output (chunk order, then the
// m8n8k4 steps), bitwise reproducible.
constexpr int K2S_NW = 7;          // 56 rows: C_P = 218 -> 4 row tiles with no empty warp
constexpr int K2S_BN = 32;
constexpr int K2S_MAXLDA = 256;
constexpr int K2S_AD = 6;          // A chunks in flight per warp
constexpr int K2S_GU = 16;         // B gather loads in flight per thread
__host__ __device__ constexpr int k2s_ldb(int lda) { return lda + 2; }   // row shift 16 B: conflict-free LDS.128

template <int NJ>
__device__ __forceinline__ void k2s_chunk(double (&acc)[4][2], const double (&a)[4], const double* bs, int ldb, int k0,
                                          int lane) {
  const double* bl = bs + (lane >> 2) * ldb + k0 + ((lane & 3) << 2);
  double2 b[NJ][2];
#pragma unroll
  for (int j = 0; j < NJ; ++j) {
    b[j][0] = *reinterpret_cast<const double2*>(bl + j * 8 * ldb);
    b[j][1] = *reinterpret_cast<const double2*>(bl + j * 8 * ldb + 2);
  }
#pragma unroll
  for (int j = 0; j < NJ; ++j) dmma884(acc[j][0], acc[j][1], a[0], b[j][0].x);   // s outer, columns inner:
#pragma unroll                                                                    // independent accumulators
  for (int j = 0; j < NJ; ++j) dmma884(acc[j][0], acc[j][1], a[1], b[j][0].y);   // between dependent DMMAs
#pragma unroll
  for (int j = 0; j < NJ; ++j) dmma884(acc[j][0], acc[j][1], a[2], b[j][1].x);
#pragma unroll
  for (int j = 0; j < NJ; ++j) dmma884(acc[j][0], acc[j][1], a[3], b[j][1].y);
}

__global__ void __launch_bounds__(32 * K2S_NW, 2) patch_gemm_smb_kernel(LevelGeom g, int r,
                                                                          const PatchClass* __restrict__ cls,
                                                                          const TileDesc* __restrict__ tiles,
                                                                          const int* __restrict__ relidx,
                                                                          const double* __restrict__ invc, int lda,
                                                                          const double* __restrict__ rvec,
                                                                          double* __restrict__ Y, int ldy) {
  pdl_trigger();
  extern __shared__ __align__(16) double bsm[];   // [K2S_BN][ldb]
  __shared__ int sbq[K2S_BN], sbp[K2S_BN], splin[K2S_BN];
  __shared__ int srel[K2S_MAXLDA];
  constexpr int NTH = 32 * K2S_NW;
  const TileDesc td = tiles[blockIdx.x];
  const PatchClass pc = cls[td.cls];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int cp = pc.cp, nch = (cp + K2_BK - 1) / K2_BK, kp = nch * K2_BK;
  const int ldb = k2s_ldb(lda);
  if (tid < K2S_BN) {
    int bq = 0, bp = 0, pl = -1;
    if (tid < td.nn && td.n0 + tid < pc.ncols) {
      int rem = td.n0 + tid, vs = 1;
      pl = 0;
      for (int a = 0; a < g.d; ++a) {
        const int v = pc.vlo[a] + (rem % pc.cnt[a]) * pc.vst;
        rem /= pc.cnt[a];
        const int c0 = v > 0 ? v - 1 : 0;
        bq += (r * c0) * (int)g.qs[a];
        bp += ((r - 1) * c0) * (int)g.ps[a];
        pl += v * vs;
        vs *= (g.n[a] + 1);
      }
    }
    sbq[tid] = bq;
    sbp[tid] = bp;
    splin[tid] = pl;
  }
  for (int k = tid; k < kp; k += NTH) srel[k] = k < cp ? __ldg(relidx + pc.rel_off + k) : -1;
  const int row0 = td.m0 + 8 * warp;
  const bool wact = row0 < cp;
  const double* Aw = invc + pc.inv_off + (long long)(row0 + (lane >> 2)) * K2_BK + (((lane & 3) ^ ((lane >> 2) & 3)) << 2);
  const long long achunk = (long long)lda * K2_BK;
  // A ring of K2S_AD chunks in registers (static indexing: the chunk loop is unrolled by K2S_AD)
  double a[K2S_AD][4];
#pragma unroll
  for (int u = 0; u < K2S_AD; ++u) {
    a[u][0] = a[u][1] = a[u][2] = a[u][3] = 0.0;
    if (wact && u < nch)
      asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];\n"
                   : "=d"(a[u][0]), "=d"(a[u][1]), "=d"(a[u][2]), "=d"(a[u][3])
                   : "l"(Aw + u * achunk));
  }
  __syncthreads();
  pdl_wait();
  const int ncol = td.nn;
  const int ncz = ((ncol + 7) / 8) * 8;   // columns the DMMAs read (absent ones zero-filled)
  for (int k = tid; k < kp; k += NTH) {   // B tile, thread per k: one gather code, then every column (no division)
    const int code = srel[k];
    const int off = code >> 1;
    const bool isp = (code & 1) != 0;
    for (int c0 = 0; c0 < ncz; c0 += K2S_GU) {
      double v[K2S_GU];
#pragma unroll
      for (int u = 0; u < K2S_GU; ++u) {   // all loads of the batch in flight before the stores
        const int col = c0 + u;
        v[u] = 0.0;
        if (col < ncol && code >= 0 && splin[col] >= 0) v[u] = __ldg(rvec + off + (isp ? sbp[col] : sbq[col]));
      }
#pragma unroll
      for (int u = 0; u < K2S_GU; ++u)
        if (c0 + u < ncz) bsm[(c0 + u) * ldb + k] = v[u];
    }
  }
  __syncthreads();
  if (!wact) return;
  const int nj = (ncol + 7) / 8;
  double acc[4][2];
#pragma unroll
  for (int j = 0; j < 4; ++j) acc[j][0] = acc[j][1] = 0.0;
  for (int c0 = 0; c0 < nch; c0 += K2S_AD) {
#pragma unroll
    for (int u = 0; u < K2S_AD; ++u) {
      const int ch = c0 + u;
      if (ch < nch) {
        if (nj >= 4) k2s_chunk<4>(acc, a[u], bsm, ldb, ch * K2_BK, lane);
        else if (nj == 3) k2s_chunk<3>(acc, a[u], bsm, ldb, ch * K2_BK, lane);
        else if (nj == 2) k2s_chunk<2>(acc, a[u], bsm, ldb, ch * K2_BK, lane);
        else k2s_chunk<1>(acc, a[u], bsm, ldb, ch * K2_BK, lane);
        if (ch + K2S_AD < nch)
          asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];\n"
                       : "=d"(a[u][0]), "=d"(a[u][1]), "=d"(a[u][2]), "=d"(a[u][3])
                       : "l"(Aw + (ch + K2S_AD) * achunk));
      }
    }
  }
  const int row = row0 + (lane >> 2);
  if (row < cp)
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int pl = splin[j * 8 + 2 * (lane & 3) + e];
        if (j < nj && pl >= 0) Y[(long long)pl * ldy + row] = acc[j][e];
      }
}

static size_t k2s_smem(int lda) { return sizeof(double) * K2S_BN * k2s_ldb(lda); }

static cudaError_t launch_k2s(const LevelGeom& g, int r, const PatchClass* cls_dev, const TileDesc* tiles, int ntiles,
                              const int* relidx, const double* invc, int lda, const double* rvec, double* Y, int ldy,
                              cudaStream_t s) {
  if (lda > K2S_MAXLDA) return cudaErrorInvalidValue;
  static PerDeviceOnce attr;
  attr.run([] {
    cudaFuncSetAttribute(patch_gemm_smb_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)k2s_smem(K2S_MAXLDA));
  });
  return launch_pdl(patch_gemm_smb_kernel, dim3(ntiles), dim3(32 * K2S_NW), k2s_smem(lda), s, g, r, cls_dev, tiles,
                    relidx, invc, lda, rvec, Y, ldy);
}

static int k2s_slots() {
  int nb = 0;
  cudaFuncSetAttribute(patch_gemm_smb_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)k2s_smem(K2S_MAXLDA));
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, patch_gemm_smb_kernel, 32 * K2S_NW, k2s_smem(K2S_MAXLDA)) !=
          cudaSuccess || nb <= 0) {
    cudaGetLastError();
    nb = 1;
  }
  return nb * 148;
}

// resident CTA slots of the whole GPU for a tile variant
int k2_slots(int variant) {
  if (variant == 9) return k2s_slots();
  if (variant == 4) return k2l_slots<1>();
  if (variant == 7) return k2l_slots<2>();
  if (variant == 8) return k2l_slots<4>();
  if (variant == 6) return k2_occ<K2_WIDE>();
  if (variant == 2) return k2_occ<K2_BIG>();
  if (variant == 1) return k2_occ<K2_MED>();
  return k2_occ<K2_SMALL>();
}

void k2_tile_shape(int variant, int* bm, int* bn) {
  using B = K2Cfg<K2_BIG>;
  using M = K2Cfg<K2_MED>;
  using Sm = K2Cfg<K2_SMALL>;
  if (variant == 9) { *bm = 8 * K2S_NW; *bn = K2S_BN; }
  else if (variant == 4) { *bm = 8 * K2L_MT; *bn = 8; }
  else if (variant == 7) { *bm = 8 * K2L_MT; *bn = 16; }
  else if (variant == 8) { *bm = 8 * K2L_MT; *bn = 32; }
  else if (variant == 6) { *bm = K2Cfg<K2_WIDE>::BM; *bn = K2Cfg<K2_WIDE>::BN; }
  else if (variant == 2) { *bm = B::BM; *bn = B::BN; }
  else if (variant == 1) { *bm = M::BM; *bn = M::BN; }
  else { *bm = Sm::BM; *bn = Sm::BN; }
}

// Variants: 0 small, 1 medium, 2 big, 6 wide (pipelined, gathered B; 2 / 6 run as the dense K2D where the level has
// the expanded residual), 4 / 7 / 8 K2L with 8 / 16 / 32 columns.  Measured choices on B200 in the comments.
int k2_pick_variant(long long npatch, int maxcp) {
  if (const char* ev = std::getenv("STGMG_K2L_MAX")) { if (npatch < std::atoll(ev)) return 4; }
  else if (npatch < 64 && maxcp <= 700) return 4;   // latency variant 32 x 8 on the smallest 2D levels (25 patches)
  if (npatch >= 500 && npatch < 2000 && maxcp <= 256) return 9;   // K2S shared-B 56 x 32 (cfg1 level 4: 12.6 -> 10.4 us;
                                                                   // slower than K2L below ~500 patches)
  if (npatch < 2000 && maxcp <= 256) return 7;   // K2L 32 x 16 (cfg1 level 4: 16.4 -> 12.7 us, level 3: 8.0 -> 6.4 us,
                                                  // level 2: 5.8 -> 5.4 us; slower on cfg2's C_P = 663)
  if (npatch < 200 && maxcp <= 700) return 4;     // 3D coarse levels stream ~1 GB of inverses: pipelined is faster
  if (npatch >= 20000) return 6;      // wide 112 x 64 (cfg2 fine 25.6 -> 27.6 TF/s, cfg3 fine 27.1 -> 27.3)
  if (npatch >= 2000) return 2;
  if (npatch >= 1000) return maxcp > 256 ? 2 : 1;   // cfg2 level 4 (C_P 663): big 56 us vs medium 90 us
  return 0;
}

cudaError_t launch_patch_gemm(const LevelGeom& g, int r, int variant, const PatchClass* cls_dev, const TileDesc* tiles,
                              int ntiles, const int* relidx, const double* invc, int lda, const double* rvec,
                              double* Y, int ldy, cudaStream_t s) {
  if (variant == 9) return launch_k2s(g, r, cls_dev, tiles, ntiles, relidx, invc, lda, rvec, Y, ldy, s);
  if (variant == 4) return launch_k2l<1>(g, r, cls_dev, tiles, ntiles, relidx, invc, lda, rvec, Y, ldy, s);
  if (variant == 7) return launch_k2l<2>(g, r, cls_dev, tiles, ntiles, relidx, invc, lda, rvec, Y, ldy, s);
  if (variant == 8) return launch_k2l<4>(g, r, cls_dev, tiles, ntiles, relidx, invc, lda, rvec, Y, ldy, s);
  if (variant == 6) return launch_k2<K2_WIDE>(g, r, cls_dev, tiles, ntiles, relidx, invc, lda, rvec, Y, ldy, s);
  if (variant == 2) return launch_k2<K2_BIG>(g, r, cls_dev, tiles, ntiles, relidx, invc, lda, rvec, Y, ldy, s);
  if (variant == 1) return launch_k2<K2_MED>(g, r, cls_dev, tiles, ntiles, relidx, invc, lda, rvec, Y, ldy, s);
  return launch_k2<K2_SMALL>(g, r, cls_dev, tiles, ntiles, relidx, invc, lda, rvec, Y, ldy, s);
}

// Row-major lda x lda matrices -> chunk-major, bank-swizzled layout read by K2:
//   element (i, j) of matrix c at  c*lda*lda + (j/16)*lda*16 + i*16 + ((j%16) ^ (4*(i%4)))
// so that rows [m0, m0+BM) of chunk j/16 are one contiguous block and the m8n8k4 A-fragment loads of a half-warp
// (rows i..i+3, columns k..k+3) hit 16 distinct bank pairs.
__global__ void chunk_swizzle_kernel(const double* __restrict__ src, double* __restrict__ dst, int lda) {
  const int c = blockIdx.y;
  const int i = blockIdx.x;
  const double* a = src + (long long)c * lda * lda + (long long)i * lda;
  double* o = dst + (long long)c * lda * lda;
  for (int j = threadIdx.x; j < lda; j += blockDim.x)
    o[(long long)(j / K2_BK) * lda * K2_BK + (long long)i * K2_BK + ((j % K2_BK) ^ (4 * (i % 4)))] = a[j];
}

cudaError_t launch_chunk_swizzle(const double* src, double* dst, int nmat, int lda, cudaStream_t s) {
  chunk_swizzle_kernel<<<dim3(lda, nmat), 128, 0, s>>>(src, dst, lda);
  return cudaGetLastError();
}

// Expanded residual for the dense K2 (pull form): every element of the class chunk-major, bank-swizzled block
//   Rexp[rexp_off + q * ncols * 16 + col * 16 + pos],  mu_hat = 16 q + (pos XOR 4 (col mod 4)),
// is r at the DoF of patch-local index mu_hat of patch column col (0 past C_P).  Threads run along Rexp, so the
// stores are fully coalesced; the gather code of mu_hat and the column bases are static and fetched before the PDL
// wait.  Replaces the push-form gather_expand (node threads scattering 8-byte stores into <= 3^d patch slots), whose
// store request rate bounded it (cfg2 fine level: expansion 300 us on top of the node gather).
// EXPAND_COLS (stgmg_internal.cuh) patch columns per block: 512 elements, 2 per thread

constexpr int EXP_THREADS = 128, EXP_PER = EXPAND_COLS * 16 / EXP_THREADS;   // 4 elements (loads in flight) per thread

__global__ void __launch_bounds__(EXP_THREADS) expand_pull_kernel(const int4* __restrict__ blocks,
                                                                  const PatchClass* __restrict__ cls,
                                                                  const int* __restrict__ relidx,
                                                                  const int2* __restrict__ colbase,
                                                                  const double* __restrict__ r,
                                                                  double* __restrict__ rexp) {
  pdl_trigger();
  const int4 bd = blocks[blockIdx.x];   // class, chunk, first column, columns in this block
  const PatchClass& pc = cls[bd.x];
  const int cp = pc.cp, ncols = pc.ncols;
  int src[EXP_PER];
  long long dst[EXP_PER];
#pragma unroll
  for (int i = 0; i < EXP_PER; ++i) {
    const int e = threadIdx.x + EXP_THREADS * i;
    const int cl = e >> 4, pos = e & 15, col = bd.z + cl;
    const int mu = bd.y * 16 + (pos ^ ((col & 3) << 2));
    src[i] = -1;
    dst[i] = -1;
    if (cl < bd.w) {
      dst[i] = pc.rexp_off + ((long long)bd.y * ncols + col) * 16 + pos;
      if (mu < cp) {
        const int code = __ldg(relidx + pc.rel_off + mu);
        const int2 cb = __ldg(colbase + pc.col_off + col);
        src[i] = (code >> 1) + ((code & 1) ? cb.y : cb.x);
      }
    }
  }
  pdl_wait();
  double v[EXP_PER];
#pragma unroll
  for (int i = 0; i < EXP_PER; ++i) v[i] = src[i] >= 0 ? __ldg(r + src[i]) : 0.0;
#pragma unroll
  for (int i = 0; i < EXP_PER; ++i)
    if (dst[i] >= 0) rexp[dst[i]] = v[i];
}

cudaError_t launch_expand_pull(const int4* blocks, int nblocks, const PatchClass* cls, const int* relidx,
                               const int2* colbase, const double* r, double* rexp, cudaStream_t s) {
  return launch_pdl(expand_pull_kernel, dim3(nblocks), dim3(EXP_THREADS), 0, s, blocks, cls, relidx, colbase, r, rexp);
}

// K3 (averaging update) lives in nodal.cu (node-mapped).

// Multiplicative colour-ordered Vanka: the update d[Z(P)] += omega y_P of one colour's
// patches; one block per patch, threads over the patch-local DoFs mu_hat.
__global__ void colour_update_kernel(LevelGeom g, int r, const PatchClass* __restrict__ cls, const int2* __restrict__ items,
                                     const int* __restrict__ relidx, const double* __restrict__ Y, int ldy,
                                     double omega, double* __restrict__ dvec) {
  const int2 it = items[blockIdx.x];
  const PatchClass pc = cls[it.x];
  int rem = it.y, vs = 1, bq = 0, bp = 0, pl = 0;
  for (int a = 0; a < g.d; ++a) {
    const int v = pc.vlo[a] + (rem % pc.cnt[a]) * pc.vst;
    rem /= pc.cnt[a];
    const int c0 = v > 0 ? v - 1 : 0;
    bq += (r * c0) * (int)g.qs[a];
    bp += ((r - 1) * c0) * (int)g.ps[a];
    pl += v * vs;
    vs *= (g.n[a] + 1);
  }
  pdl_wait();
  const double* y = Y + (long long)pl * ldy;
  for (int mh = threadIdx.x; mh < pc.cp; mh += blockDim.x) {
    const int code = __ldg(relidx + pc.rel_off + mh);
    const long long dof = (code >> 1) + ((code & 1) ? bp : bq);
    dvec[dof] += omega * y[mh];
  }
}

cudaError_t launch_colour_update(const LevelGeom& g, int r, const PatchClass* cls, const int2* items, int nitems,
                                 const int* relidx, const double* Y, int ldy, double omega, double* dvec,
                                 cudaStream_t s) {
  if (nitems == 0) return cudaSuccess;
  return launch_pdl(colour_update_kernel, dim3(nitems), dim3(128), 0, s, g, r, cls, items, relidx, Y, ldy, omega, dvec);
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

// ---- blocked Gauss–Jordan (K4 on the FP64 tensor pipe) ----
// The same in-place Gauss–Jordan with partial pivoting (max |a|, ties -> lowest row) as gj_pivot / gj_elim, in
// column panels of GJB_NB pivots: the panel kernel runs the NB elimination steps on the panel columns only (L2
// resident) and records the composite row permutation pi; the NB steps act on every other column c as
//   M[:, c] <- M[pi(:), c] + W M[pi(panel rows), c],   W = (panel result) - I[:, panel],
// (the in-place panel column k0 + j ends as the product of the steps' elementary matrices applied to e_{k0+j}), a
// rank-NB update done by gjb_trailing with DMMA out of place (ping-pong buffers).  Memory traffic per pivot drops by
// NB: the unblocked rank-1 updates stream every matrix once per pivot (3D levels: 125 x 1568^2 doubles, 1554 times).
constexpr int GJB_NB = 64, GJB_BM = 64, GJB_BN = 64;
// shared row strides = 4 (mod 16) doubles: the m8n8k4 fragments of a half warp hit 16 distinct 8-byte bank pairs
constexpr int GJB_WS = GJB_NB + 4, GJB_TS = GJB_BN + 4;
constexpr size_t GJB_TSMEM = sizeof(double) * (GJB_BM * GJB_WS + GJB_NB * GJB_TS);

// One CTA per matrix.  Per step: argmax of the pivot column (block reduction), row swap on the panel columns, then ONE
// pass over the n x nbe panel that applies the whole elementary step (column k := e_k, pivot row scaled by 1 / pivot,
// rank-1 elimination of every other row) from the pivot column and the scaled pivot row held in shared memory, with
// GJB_UNR independent loads in flight per thread (the L2-resident panel made every step latency-bound).
constexpr int GJB_PT = 1024, GJB_UNR = 8;

__global__ void __launch_bounds__(GJB_PT) gjb_panel(double* mats, int lda, const int* n_each, int k0, int* perm,
                                                    int* pi, double* colk, int* status) {
  const int c = blockIdx.x;
  const int n = n_each[c];
  if (k0 >= n || status[c] != 0) return;
  double* A = mats + (long long)c * lda * lda;
  int* pm = perm + (long long)c * lda;
  int* pc = pi + (long long)c * lda;
  extern __shared__ double gsm[];
  double* ck = gsm;                  // pivot column (lda)
  double* pr = ck + lda;             // scaled pivot row on the panel columns (GJB_NB)
  __shared__ double bv[GJB_PT / 32];
  __shared__ int bi[GJB_PT / 32];
  const int nbe = min(GJB_NB, n - k0);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = k0 + threadIdx.x; i < n; i += blockDim.x) pc[i] = i;
  __syncthreads();
  for (int j = 0; j < nbe; ++j) {
    const int k = k0 + j;
    double best = -1.0;
    int bidx = n;
    for (int i = k + threadIdx.x; i < n; i += blockDim.x) {
      const double v = fabs(A[(long long)i * lda + k]);
      if (v > best) { best = v; bidx = i; }   // rows ascending per thread: ties keep the lowest row
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double v2 = __shfl_xor_sync(0xffffffffu, best, o);
      const int i2 = __shfl_xor_sync(0xffffffffu, bidx, o);
      if (v2 > best || (v2 == best && i2 < bidx)) { best = v2; bidx = i2; }
    }
    if (lane == 0) { bv[warp] = best; bi[warp] = bidx; }
    __syncthreads();
    if (warp == 0) {
      best = lane < GJB_PT / 32 ? bv[lane] : -1.0;
      bidx = lane < GJB_PT / 32 ? bi[lane] : n;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double v2 = __shfl_xor_sync(0xffffffffu, best, o);
        const int i2 = __shfl_xor_sync(0xffffffffu, bidx, o);
        if (v2 > best || (v2 == best && i2 < bidx)) { best = v2; bidx = i2; }
      }
      if (lane == 0) { bv[0] = best; bi[0] = bidx; }
    }
    __syncthreads();
    const int p = bi[0];
    if (bv[0] <= 0.0) {
      if (threadIdx.x == 0) status[c] = k + 1;
      return;
    }
    if (p != k) {   // swap the panel rows and the permutation entries
      for (int q = threadIdx.x; q < nbe; q += blockDim.x) {
        const double t = A[(long long)k * lda + k0 + q];
        A[(long long)k * lda + k0 + q] = A[(long long)p * lda + k0 + q];
        A[(long long)p * lda + k0 + q] = t;
      }
      if (threadIdx.x == 0) {
        const int t = pc[k];
        pc[k] = pc[p];
        pc[p] = t;
      }
    }
    if (threadIdx.x == 0) pm[k] = p;
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) ck[i] = A[(long long)i * lda + k];
    if (threadIdx.x < nbe) {
      const double ip = 1.0 / A[(long long)k * lda + k];
      pr[threadIdx.x] = (threadIdx.x == j ? 1.0 : A[(long long)k * lda + k0 + threadIdx.x]) * ip;
    }
    __syncthreads();
    // thread = (row group, panel columns lane, lane + 32): rows i = rg, rg + GJB_PT / 32, ... (32-bit index math)
    const int rg = warp;
    for (int q = lane; q < nbe; q += 32) {
      const double prq = pr[q];
      constexpr int RS = GJB_PT / 32;
      for (int i0 = rg; i0 < n; i0 += GJB_UNR * RS) {
        double old[GJB_UNR];
#pragma unroll
        for (int u = 0; u < GJB_UNR; ++u) {
          const int i = i0 + u * RS;
          old[u] = 0.0;
          if (i < n) old[u] = q == j ? (i == k ? 1.0 : 0.0) : A[(size_t)i * lda + k0 + q];
        }
#pragma unroll
        for (int u = 0; u < GJB_UNR; ++u) {
          const int i = i0 + u * RS;
          if (i < n) A[(size_t)i * lda + k0 + q] = i == k ? prq : fma(-ck[i], prq, old[u]);
        }
      }
    }
    __syncthreads();
  }
}

// out[i][c] = in[i][c] on the panel columns, padding and rows / columns >= n; otherwise
// in[pi(i)][c] + sum_j W[i][j] in[pi(k0 + j)][c] with W[i][j] = in[i][k0 + j] - delta_{i, k0+j} (DMMA m8n8k4).
// One CTA per 64 x 64 output tile; 8 warps in a 4 x 2 grid, warp tile 16 x 32 (2 x 4 m8n8k4 DMMA per k-step; a
// 64 x 128 tile with 32 x 32 warp tiles, 2 CTAs per SM, measured 18 % slower).
__device__ __forceinline__ void gjb_cp8(double* dst, const double* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src) : "memory");
}

__global__ void __launch_bounds__(256, 3) gjb_trailing(const double* __restrict__ in, double* __restrict__ out, int lda,
                                                    const int* n_each, int k0, const int* __restrict__ pi,
                                                    const int* status) {
  const int c = blockIdx.z;
  const int n = n_each[c];
  const double* A = in + (long long)c * lda * lda;
  double* O = out + (long long)c * lda * lda;
  const int r0 = blockIdx.y * GJB_BM, c0 = blockIdx.x * GJB_BN;
  const bool active = k0 < n && status[c] == 0;
  const int nbe = active ? min(GJB_NB, n - k0) : 0;
  const int* pc = pi + (long long)c * lda;
  extern __shared__ double sraw[];
  double (*Ws)[GJB_WS] = reinterpret_cast<double (*)[GJB_WS]>(sraw);
  double (*Ts)[GJB_TS] = reinterpret_cast<double (*)[GJB_TS]>(sraw + GJB_BM * GJB_WS);
  __shared__ int prow[GJB_BM];
  // operand tiles by asynchronous 8-byte copies (all of a thread's copies in flight at once); zero padding by stores
  for (int e = threadIdx.x; e < GJB_BM * GJB_NB; e += blockDim.x) {
    const int i = e / GJB_NB, j = e % GJB_NB, row = r0 + i;
    if (j < nbe && row < n) gjb_cp8(&Ws[i][j], A + (long long)row * lda + k0 + j);
    else Ws[i][j] = 0.0;
  }
  for (int e = threadIdx.x; e < GJB_NB * GJB_BN; e += blockDim.x) {
    const int j = e / GJB_BN, q = e % GJB_BN, col = c0 + q;
    if (j < nbe && col < lda) gjb_cp8(&Ts[j][q], A + (long long)pc[k0 + j] * lda + col);
    else Ts[j][q] = 0.0;
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  for (int i = threadIdx.x; i < GJB_BM; i += blockDim.x) {
    const int row = r0 + i;
    prow[i] = (active && row >= k0 && row < n) ? pc[row] : row;
  }
  __syncthreads();   // prow
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = (warp & 3) * 16, wn = (warp >> 2) * 32;
  // the epilogue's base values (row-permuted input, or the unchanged input) loaded while the operands arrive
  double base[2][4][2];
  bool upd[2][4][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int i = wm + 8 * a + (lane >> 2), row = r0 + i;
        const int col = c0 + wn + 8 * b + 2 * (lane & 3) + e;
        upd[a][b][e] = !(!active || row >= n || col >= n || (col >= k0 && col < k0 + nbe));
        base[a][b][e] = (row < lda && col < lda) ? A[(long long)(upd[a][b][e] ? prow[i] : row) * lda + col] : 0.0;
      }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  // W = (panel result) - I on the panel rows
  for (int j = threadIdx.x; j < nbe; j += blockDim.x) {
    const int i = k0 + j - r0;
    if (i >= 0 && i < GJB_BM) Ws[i][j] -= 1.0;
  }
  __syncthreads();
  double acc[2][4][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const int ksn = (nbe + 3) / 4;
#pragma unroll 4
  for (int ks = 0; ks < ksn; ++ks) {
    double af[2], bf[4];
#pragma unroll
    for (int a = 0; a < 2; ++a) af[a] = Ws[wm + 8 * a + (lane >> 2)][4 * ks + (lane & 3)];
#pragma unroll
    for (int b = 0; b < 4; ++b) bf[b] = Ts[4 * ks + (lane & 3)][wn + 8 * b + (lane >> 2)];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(acc[a][b][0]), "+d"(acc[a][b][1])
                     : "d"(af[a]), "d"(bf[b]));
  }
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int row = r0 + wm + 8 * a + (lane >> 2);
        const int col = c0 + wn + 8 * b + 2 * (lane & 3) + e;
        if (row >= lda || col >= lda) continue;
        O[(long long)row * lda + col] = upd[a][b][e] ? base[a][b][e] + acc[a][b][e] : base[a][b][e];
      }
}

// Batched in-place inverse of nmat matrices (row-major, lda) of sizes n_each (device array).  Returns 0 or the
// negative CUDA error; status[c] != 0 marks a singular matrix (checked by the caller after a sync).  Matrices of
// >= 128 rows take the blocked form (STGMG_GJ_UNBLOCKED=1: always the rank-1 form).
int gauss_jordan_inverse(double* mats, int nmat, int n_max, const int* n_each, int lda, int* perm, double* colk,
                         double* scale, int* status, cudaStream_t s, GjScratch* scr) {
  gj_equilibrate<<<nmat, 256, 0, s>>>(mats, lda, n_each, scale, 1, status);
  static const bool unblocked = std::getenv("STGMG_GJ_UNBLOCKED") != nullptr;
  const size_t psmem = sizeof(double) * ((size_t)lda + GJB_NB);   // pivot column + scaled pivot row
  const size_t need_buf = sizeof(double) * (size_t)nmat * lda * lda, need_pi = sizeof(int) * (size_t)nmat * lda;
  GjScratch local;
  GjScratch* sc = scr ? scr : &local;
  bool blocked = !unblocked && n_max >= 128 && psmem <= 200 * 1024;
  if (blocked && (sc->buf_bytes < need_buf || sc->pi_bytes < need_pi)) {   // grow the caller's scratch
    if (sc->buf) cudaFree(sc->buf);
    if (sc->pi) cudaFree(sc->pi);
    sc->buf = nullptr;
    sc->pi = nullptr;
    sc->buf_bytes = sc->pi_bytes = 0;
    if (cudaMalloc(&sc->buf, need_buf) == cudaSuccess && cudaMalloc(&sc->pi, need_pi) == cudaSuccess) {
      sc->buf_bytes = need_buf;
      sc->pi_bytes = need_pi;
    } else {
      cudaGetLastError();
      blocked = false;
    }
  }
  if (blocked) {
    static PerDeviceOnce attr;
    attr.run([] {
      cudaFuncSetAttribute(gjb_panel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      cudaFuncSetAttribute(gjb_trailing, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)GJB_TSMEM);
    });
    double *cur = mats, *nxt = sc->buf;
    int* pi = sc->pi;
    const dim3 tg((lda + GJB_BN - 1) / GJB_BN, (lda + GJB_BM - 1) / GJB_BM, nmat);
    for (int k0 = 0; k0 < n_max; k0 += GJB_NB) {
      gjb_panel<<<nmat, GJB_PT, psmem, s>>>(cur, lda, n_each, k0, perm, pi, colk, status);
      gjb_trailing<<<tg, 256, GJB_TSMEM, s>>>(cur, nxt, lda, n_each, k0, pi, status);
      std::swap(cur, nxt);
    }
    if (cur != mats) cudaMemcpyAsync(mats, cur, sizeof(double) * (size_t)nmat * lda * lda, cudaMemcpyDeviceToDevice, s);
    if (sc == &local) {
      cudaStreamSynchronize(s);
      cudaFree(local.buf);
      cudaFree(local.pi);
    }
  } else {
    for (int k = 0; k < n_max; ++k) {
      gj_pivot<<<nmat, 1024, 0, s>>>(mats, lda, n_each, k, perm, colk, status);
      gj_elim<<<dim3((n_max + 7) / 8, nmat), 256, 0, s>>>(mats, lda, n_each, k, colk, status);
    }
  }
  gj_colperm<<<nmat, 256, 0, s>>>(mats, lda, n_each, perm);
  gj_equilibrate<<<nmat, 256, 0, s>>>(mats, lda, n_each, scale, 0, status);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

}  // namespace stgmg
