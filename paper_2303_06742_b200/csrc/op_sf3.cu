// K1 — the 3D Q2 slab operator by sum factorisation on the FP64 pipe, for the cells without Dirichlet faces
// (volume terms only; the cells of the Nitsche face types stay on the factored element GEMMs of op_fgemm.cu).
//
// Operator (Problem 3.1, Eq:DPQ_A0; block form per SURVEY reading A5 / App. A.1), forms of Def:ACB /
// Def:ab without face terms, per cell K and Radau node b:
//   (A X)_{phi,b} = rho  M (sum_a T_ba U_a - theta_b V_b)                       M  = |K| (M1 x M1 x M1)
//   (A X)_{chi,b} = rho  M (sum_a T_ba V_a) + theta_b (sigma(U_b) - alpha P_b I, grad chi)_K
//   (A X)_{psi,b} = c0 Mp (sum_a T_ba P_a) + theta_b ((alpha div V_b, psi)_K + (K grad P_b, grad psi)_K)
// The mass terms are Kronecker products of the 1D Gauss mass M1[i][j] = sum_g w_g l_i(x_g) l_j(x_g) (3-point Gauss
// rule: exact for Q2 x Q2), applied as three 3x3 passes on the temporally mixed nodal values.  The stiffness terms
// go through the 27 Gauss points: U_b interpolated (B = l_j(x_g) per axis) and differentiated by the collocation
// matrix Dc = Dm B^-1 (exact: the interpolant of a Q2 function at 3 Gauss points per axis is the function); div V_b
// by Dm along its own axis; P_b (Q1) interpolated by Bp and differentiated by Dc; the test side is the transpose.
// Per cell 13.4k FMA (SURVEY §8(d)'s 270 flop per DoF) instead of the factored GEMMs' 28.5k padded DMMA slots.
//
// Execution: CTA = 32 cells of one volume-only cell type (tile {type, first cell, cells} as op_fgemm), 96 threads:
// warp c owns vector component c, lane = cell.  Each thread keeps its 27-point fields in registers (passes fully
// unrolled, matrices in the __grid_constant__ parameter block); the per-point coupling of the components (stress,
// trace, div, K grad p) goes through shared memory laid out [quantity][point][cell] (conflict-free).  Results are
// written cell-fastest Y[element DoF][cell] like op_fgemm, and summed per node by the deterministic gather.
#include <cmath>

#include "op_common.cuh"

namespace stgmg {

template <int K1>
struct Sf3Consts {
  double B[3][3];      // B[g][j]   = l_j(x_g)            (Q2 basis on the GLL nodes at the Gauss points, [0,1])
  double Bt[3][3];     // transpose
  double Dc[3][3];     // Dc = Dm B^-1: derivative at the Gauss points from the values at the Gauss points
  double Dct[3][3];
  double Dm[3][3];     // Dm[g][j]  = l_j'(x_g)
  double Dmt[3][3];
  double M1[3][3];     // 1D Gauss mass of Q2
  double Bp[3][2];     // Q1 basis at the Gauss points
  double Bpt[2][3];
  double Mp1[2][2];    // 1D Gauss mass of Q1
  double wq[27];       // |K| w_x w_y w_z at Gauss point q = x + 3 y + 9 z
  double hinv[3];
  double T[K1][K1];    // T[b][a]
  double th[K1];       // theta_b
  double rho, rho_vol, c0_vol, alpha, lam, mu, K[9];
};

// out = pass of `in` (dims N0 x N1 x N2, x fastest) along axis AX with the NO x NI row-major matrix M.
template <int N0, int N1, int N2, int AX, int NO>
__device__ __forceinline__ void sf_pass(const double* __restrict__ M, const double* in, double* out) {
  constexpr int NI = AX == 0 ? N0 : (AX == 1 ? N1 : N2);
  constexpr int O0 = AX == 0 ? NO : N0, O1 = AX == 1 ? NO : N1, O2 = AX == 2 ? NO : N2;
#pragma unroll
  for (int i2 = 0; i2 < O2; ++i2)
#pragma unroll
    for (int i1 = 0; i1 < O1; ++i1)
#pragma unroll
      for (int i0 = 0; i0 < O0; ++i0) {
        const int io = AX == 0 ? i0 : (AX == 1 ? i1 : i2);
        double s = 0.0;
#pragma unroll
        for (int j = 0; j < NI; ++j) {
          const int s0 = AX == 0 ? j : i0, s1 = AX == 1 ? j : i1, s2 = AX == 2 ? j : i2;
          s = fma(M[io * NI + j], in[s0 + N0 * (s1 + N1 * s2)], s);
        }
        out[i0 + O0 * (i1 + O1 * i2)] = s;
      }
}

// 27-point tensor apply with the same 3x3 matrix on every axis except axis DA, which takes MD.
template <int DA>
__device__ __forceinline__ void sf_apply3(const double* M, const double* MD, const double* in, double* out) {
  double t1[27], t2[27];
  sf_pass<3, 3, 3, 0, 3>(DA == 0 ? MD : M, in, t1);
  sf_pass<3, 3, 3, 1, 3>(DA == 1 ? MD : M, t1, t2);
  sf_pass<3, 3, 3, 2, 3>(DA == 2 ? MD : M, t2, out);
}

template <int K1>
__global__ void __launch_bounds__(96, 2) op_sf3_kernel(LevelGeom g, const int4* __restrict__ tiles,
                                                       const PatchClass* __restrict__ ecls,
                                                       const __grid_constant__ Sf3Consts<K1> p,
                                                       const double* __restrict__ x, double* __restrict__ Y,
                                                       long long ncell) {
  constexpr int NQ = 27, NP = 8, NE1 = 6 * NQ + NP;
  constexpr int NC = 32;
  // shared: G[9][27][NC] (grad U_b, then in place the chi gradient coefficients), dV[3][27][NC] (d_c V_c),
  // Pv[27][NC] (P_b, then the psi value coefficient), gP[3][27][NC] (grad P_b, then the psi gradient coefficients);
  // laid out [quantity][point][cell]: a warp touches 32 consecutive doubles
  extern __shared__ double sm[];
  double* G = sm;
  double* dV = G + 9 * NQ * NC;
  double* Pv = dV + 3 * NQ * NC;
  double* gP = Pv + NQ * NC;
  pdl_trigger();
  const int lane = threadIdx.x & 31, c = threadIdx.x >> 5;
  const int4 td = tiles[blockIdx.x];
  const PatchClass& pc = ecls[td.x];
  const bool act = lane < td.z;
  long long qb = 0, pb = 0, pl = 0;
  {
    int rem = td.y + (act ? lane : 0);
    long long vs = 1;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const int ca = pc.vlo[a] - 1 + rem % pc.cnt[a];
      rem /= pc.cnt[a];
      qb += (long long)(2 * ca) * g.qs[a];
      pb += (long long)ca * g.ps[a];
      pl += (long long)ca * vs;
      vs *= g.n[a];
    }
  }
  const long long qs1 = g.qs[1], qs2 = g.qs[2], ps1 = g.ps[1], ps2 = g.ps[2];
  auto qoff = [&](int j) { return (long long)(j % 3) + (long long)((j / 3) % 3) * qs1 + (long long)(j / 9) * qs2; };
  auto poff = [&](int j) { return (long long)(j & 1) + (long long)((j >> 1) & 1) * ps1 + (long long)(j >> 2) * ps2; };
  const double* xV = x + (long long)c * g.nq + qb;         // V_c of Radau node 0 (+ a * block)
  const double* xU = x + (long long)(3 + c) * g.nq + qb;   // U_c
  const double* xP = x + 2 * g.R + pb;
  double* Yc = Y + pl;
  const int lq0 = 9 * c;   // this thread's Gauss points in the pointwise phase: lq0 .. lq0 + 8
  pdl_wait();

#pragma unroll 1
  for (int b = 0; b < K1; ++b) {
    const long long ob = (long long)b * g.block;
    // ---- forward: grad U_b,c ; d_c V_b,c ; P_b and d_c P_b at the Gauss points ----
    {
      double u[27], uq[27];
#pragma unroll
      for (int j = 0; j < NQ; ++j) u[j] = act ? __ldg(xU + ob + qoff(j)) : 0.0;
      sf_apply3<0>(&p.B[0][0], &p.B[0][0], u, uq);
#pragma unroll
      for (int l = 0; l < 3; ++l) {
        double gq[27];
        if (l == 0) sf_pass<3, 3, 3, 0, 3>(&p.Dc[0][0], uq, gq);
        if (l == 1) sf_pass<3, 3, 3, 1, 3>(&p.Dc[0][0], uq, gq);
        if (l == 2) sf_pass<3, 3, 3, 2, 3>(&p.Dc[0][0], uq, gq);
        const double hl = p.hinv[l];
#pragma unroll
        for (int q = 0; q < NQ; ++q) G[((c * 3 + l) * NQ + q) * NC + lane] = gq[q] * hl;
      }
    }
    {
      double v[27], dq[27];
#pragma unroll
      for (int j = 0; j < NQ; ++j) v[j] = act ? __ldg(xV + ob + qoff(j)) : 0.0;
      if (c == 0) sf_apply3<0>(&p.B[0][0], &p.Dm[0][0], v, dq);
      if (c == 1) sf_apply3<1>(&p.B[0][0], &p.Dm[0][0], v, dq);
      if (c == 2) sf_apply3<2>(&p.B[0][0], &p.Dm[0][0], v, dq);
      const double hc = p.hinv[c];
#pragma unroll
      for (int q = 0; q < NQ; ++q) dV[(c * NQ + q) * NC + lane] = dq[q] * hc;
    }
    {
      double pn[8], t1[12], t2[18], pq[27], gq[27];
#pragma unroll
      for (int j = 0; j < NP; ++j) pn[j] = act ? __ldg(xP + ob + poff(j)) : 0.0;
      sf_pass<2, 2, 2, 0, 3>(&p.Bp[0][0], pn, t1);
      sf_pass<3, 2, 2, 1, 3>(&p.Bp[0][0], t1, t2);
      sf_pass<3, 3, 2, 2, 3>(&p.Bp[0][0], t2, pq);
      if (c == 0) sf_pass<3, 3, 3, 0, 3>(&p.Dc[0][0], pq, gq);
      if (c == 1) sf_pass<3, 3, 3, 1, 3>(&p.Dc[0][0], pq, gq);
      if (c == 2) sf_pass<3, 3, 3, 2, 3>(&p.Dc[0][0], pq, gq);
      const double hc = p.hinv[c];
#pragma unroll
      for (int q = 0; q < NQ; ++q) gP[(c * NQ + q) * NC + lane] = gq[q] * hc;
      if (c == 0) {
#pragma unroll
        for (int q = 0; q < NQ; ++q) Pv[q * NC + lane] = pq[q];
      }
    }
    __syncthreads();
    // ---- pointwise coefficients at Gauss points lq0 .. lq0 + 8 of this thread's cell (in place):
    //      chi gradient: theta w (mu (G + G^T) + (lambda tr G - alpha P) I) h_j^-1 ; psi gradient: theta w (K grad P)_i
    //      h_i^-1 ; psi value (stiffness part): theta w alpha div V ----
    {
      const double th = p.th[b];
#pragma unroll 3
      for (int t = 0; t < 9; ++t) {
        const int q = lq0 + t;
        const double w = p.wq[q];
        double Gm[3][3];
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int j = 0; j < 3; ++j) Gm[i][j] = G[((i * 3 + j) * NQ + q) * NC + lane];
        const double pv = Pv[q * NC + lane];
        const double dv = dV[q * NC + lane] + dV[(NQ + q) * NC + lane] + dV[(2 * NQ + q) * NC + lane];
        const double tr = Gm[0][0] + Gm[1][1] + Gm[2][2];
        const double tw = th * w;
        const double diag = p.lam * tr - p.alpha * pv;
#pragma unroll
        for (int i = 0; i < 3; ++i)
#pragma unroll
          for (int j = 0; j < 3; ++j) {
            const double s = p.mu * (Gm[i][j] + Gm[j][i]) + (i == j ? diag : 0.0);
            G[((i * 3 + j) * NQ + q) * NC + lane] = tw * s * p.hinv[j];
          }
        double gp[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) gp[j] = gP[(j * NQ + q) * NC + lane];
#pragma unroll
        for (int i = 0; i < 3; ++i)
          gP[(i * NQ + q) * NC + lane] =
              tw * (p.K[i * 3] * gp[0] + p.K[i * 3 + 1] * gp[1] + p.K[i * 3 + 2] * gp[2]) * p.hinv[i];
        Pv[q * NC + lane] = tw * p.alpha * dv;
      }
    }
    __syncthreads();
    // ---- backward: chi_b,c = B^T^3 (sum_l Dc_l^T S_cl + rho w B^3 sum_a T_ba V_a,c) and phi_b,c ; psi_b on warp 2
    {
      double z[27], zt[27];
#pragma unroll
      for (int q = 0; q < NQ; ++q) z[q] = 0.0;
#pragma unroll
      for (int l = 0; l < 3; ++l) {
        double s[27];
#pragma unroll
        for (int q = 0; q < NQ; ++q) s[q] = G[((c * 3 + l) * NQ + q) * NC + lane];
        if (l == 0) sf_pass<3, 3, 3, 0, 3>(&p.Dct[0][0], s, zt);
        if (l == 1) sf_pass<3, 3, 3, 1, 3>(&p.Dct[0][0], s, zt);
        if (l == 2) sf_pass<3, 3, 3, 2, 3>(&p.Dct[0][0], s, zt);
#pragma unroll
        for (int q = 0; q < NQ; ++q) z[q] += zt[q];
      }
      {
        double m[27], mq[27];
#pragma unroll
        for (int j = 0; j < NQ; ++j) {
          double s = 0.0;
#pragma unroll
          for (int a = 0; a < K1; ++a) s = fma(p.T[b][a], act ? __ldg(xV + (long long)a * g.block + qoff(j)) : 0.0, s);
          m[j] = s;
        }
        sf_apply3<0>(&p.B[0][0], &p.B[0][0], m, mq);
#pragma unroll
        for (int q = 0; q < NQ; ++q) z[q] = fma(p.rho * p.wq[q], mq[q], z[q]);
      }
      sf_apply3<0>(&p.Bt[0][0], &p.Bt[0][0], z, zt);
      if (act) {
        double* yc = Yc + (long long)(b * NE1 + (3 + c) * NQ) * ncell;
#pragma unroll
        for (int j = 0; j < NQ; ++j) yc[(long long)j * ncell] = zt[j];
      }
      double m[27];
#pragma unroll
      for (int j = 0; j < NQ; ++j) {
        double s = -p.th[b] * (act ? __ldg(xV + ob + qoff(j)) : 0.0);
#pragma unroll
        for (int a = 0; a < K1; ++a) s = fma(p.T[b][a], act ? __ldg(xU + (long long)a * g.block + qoff(j)) : 0.0, s);
        m[j] = s * p.rho_vol;
      }
      sf_apply3<0>(&p.M1[0][0], &p.M1[0][0], m, zt);
      if (act) {
        double* yc = Yc + (long long)(b * NE1 + c * NQ) * ncell;
#pragma unroll
        for (int j = 0; j < NQ; ++j) yc[(long long)j * ncell] = zt[j];
      }
    }
    if (c == 2) {
      double z[27], zt[27];
#pragma unroll
      for (int q = 0; q < NQ; ++q) z[q] = Pv[q * NC + lane];
#pragma unroll
      for (int l = 0; l < 3; ++l) {
        double s[27];
#pragma unroll
        for (int q = 0; q < NQ; ++q) s[q] = gP[(l * NQ + q) * NC + lane];
        if (l == 0) sf_pass<3, 3, 3, 0, 3>(&p.Dct[0][0], s, zt);
        if (l == 1) sf_pass<3, 3, 3, 1, 3>(&p.Dct[0][0], s, zt);
        if (l == 2) sf_pass<3, 3, 3, 2, 3>(&p.Dct[0][0], s, zt);
#pragma unroll
        for (int q = 0; q < NQ; ++q) z[q] += zt[q];
      }
      double t2[18], t1[12], psi[8];
      sf_pass<3, 3, 3, 2, 2>(&p.Bpt[0][0], z, t2);
      sf_pass<3, 3, 2, 1, 2>(&p.Bpt[0][0], t2, t1);
      sf_pass<3, 2, 2, 0, 2>(&p.Bpt[0][0], t1, psi);
      // mass part: c0 |K| Mp1^3 (sum_a T_ba P_a)
      double mp[8], u1[8], u2[8], mo[8];
#pragma unroll
      for (int j = 0; j < NP; ++j) {
        double s = 0.0;
#pragma unroll
        for (int a = 0; a < K1; ++a) s = fma(p.T[b][a], act ? __ldg(xP + (long long)a * g.block + poff(j)) : 0.0, s);
        mp[j] = s * p.c0_vol;
      }
      sf_pass<2, 2, 2, 0, 2>(&p.Mp1[0][0], mp, u1);
      sf_pass<2, 2, 2, 1, 2>(&p.Mp1[0][0], u1, u2);
      sf_pass<2, 2, 2, 2, 2>(&p.Mp1[0][0], u2, mo);
      if (act) {
        double* yc = Yc + (long long)(b * NE1 + 6 * NQ) * ncell;
#pragma unroll
        for (int j = 0; j < NP; ++j) yc[(long long)j * ncell] = psi[j] + mo[j];
      }
    }
    __syncthreads();   // the shared arrays are refilled for the next Radau node
  }
}

// ------------------------------------------------------------------------------------------- host side -----
static bool inv3(const double A[3][3], double X[3][3]) {
  const double det = A[0][0] * (A[1][1] * A[2][2] - A[1][2] * A[2][1]) - A[0][1] * (A[1][0] * A[2][2] - A[1][2] * A[2][0]) +
                     A[0][2] * (A[1][0] * A[2][1] - A[1][1] * A[2][0]);
  if (det == 0.0) return false;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      const int i1 = (j + 1) % 3, i2 = (j + 2) % 3, j1 = (i + 1) % 3, j2 = (i + 2) % 3;
      X[i][j] = (A[i1][j1] * A[i2][j2] - A[i1][j2] * A[i2][j1]) / det;   // cofactor transpose
    }
  return true;
}

template <int K1>
static bool sf3_consts(const LevelGeom& g, const OpConsts& c, Sf3Consts<K1>& p) {
  double B3[3][3], Bi[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) B3[i][j] = c.B[i][j];
  if (!inv3(B3, Bi)) return false;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      p.B[i][j] = c.B[i][j];
      p.Bt[j][i] = c.B[i][j];
      p.Dm[i][j] = c.Dm[i][j];
      p.Dmt[j][i] = c.Dm[i][j];
      double s = 0.0, m = 0.0;
      for (int k = 0; k < 3; ++k) {
        s += c.Dm[i][k] * Bi[k][j];
        m += c.wg[k] * c.B[k][i] * c.B[k][j];
      }
      p.Dc[i][j] = s;
      p.Dct[j][i] = s;
      p.M1[i][j] = m;
    }
  for (int gq = 0; gq < 3; ++gq)
    for (int j = 0; j < 2; ++j) {
      p.Bp[gq][j] = c.Bp[gq][j];
      p.Bpt[j][gq] = c.Bp[gq][j];
    }
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 2; ++j) {
      double m = 0.0;
      for (int k = 0; k < 3; ++k) m += c.wg[k] * c.Bp[k][i] * c.Bp[k][j];
      p.Mp1[i][j] = m;
    }
  for (int q = 0; q < 27; ++q) p.wq[q] = g.vol * c.wg[q % 3] * c.wg[(q / 3) % 3] * c.wg[q / 9];
  for (int a = 0; a < 3; ++a) p.hinv[a] = 1.0 / g.h[a];
  for (int b = 0; b < K1; ++b) {
    p.th[b] = c.theta[b];
    for (int a = 0; a < K1; ++a) p.T[b][a] = c.T[b][a];
  }
  p.rho = c.rho;
  p.rho_vol = c.rho * g.vol;
  p.c0_vol = c.c0 * g.vol;
  p.alpha = c.alpha;
  p.lam = c.lam;
  p.mu = c.mu;
  for (int i = 0; i < 9; ++i) p.K[i] = c.K[i];
  return true;
}

constexpr size_t kSf3Smem = sizeof(double) * (9 + 3 + 1 + 3) * 27 * 32;

template <int K1>
static cudaError_t launch_sf3(const LevelGeom& g, const int4* tiles, int ntiles, const PatchClass* ecls,
                              const OpConsts& c, const double* x, double* Y, cudaStream_t s) {
  static PerDeviceOnce attr;
  attr.run([] {
    cudaFuncSetAttribute(op_sf3_kernel<K1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSf3Smem);
  });
  Sf3Consts<K1> p;
  if (!sf3_consts<K1>(g, c, p)) return cudaErrorInvalidValue;
  const long long ncell = (long long)g.n[0] * g.n[1] * g.n[2];
  return launch_pdl(op_sf3_kernel<K1>, dim3(ntiles), dim3(96), kSf3Smem, s, g, tiles, ecls, p, x, Y, ncell);
}

bool sf3_supported(int d, int r, int k1) { return d == 3 && r == 2 && (k1 == 2 || k1 == 3); }

cudaError_t launch_op_sf3(const LevelGeom& g, int r, int k1, const int4* tiles, int ntiles, const PatchClass* ecls,
                          const OpConsts& c, const double* x, double* Y, cudaStream_t s) {
  if (ntiles == 0) return cudaSuccess;
  if (g.d == 3 && r == 2 && k1 == 2) return launch_sf3<2>(g, tiles, ntiles, ecls, c, x, Y, s);
  if (g.d == 3 && r == 2 && k1 == 3) return launch_sf3<3>(g, tiles, ntiles, ecls, c, x, Y, s);
  return cudaErrorNotSupported;
}

}  // namespace stgmg
