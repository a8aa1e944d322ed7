// K1 (2D) — matrix-free space-time slab operator, one thread per cell, register sum factorisation (sm_100a, fp64).
//
// Same operator as op_apply.cu (Problem 3.1, Eq:DPQ_A0; forms Def:ACB / Def:ab):
//   (A X)_{phi,b} = sum_a T_ba M_rho U_a - theta_b M_rho V_b
//   (A X)_{chi,b} = sum_a T_ba M_rho V_a + theta_b (A_gamma U_b + C^T P_b)
//   (A X)_{psi,b} = sum_a T_ba M_c  P_a + theta_b (-C V_b + B_gamma P_b)
// Phase 1 (op2d_cell_kernel): one thread per (cell, Radau node b, row block) — row blocks: phi rows, chi rows of
// component 0, chi rows of component 1, psi row — reads its element values through the read-only cache, evaluates
// values / gradients at the (r+1)^2 Gauss points by 1D contractions held in registers (compile-time sizes, fully
// unrolled), forms the pointwise coefficients, integrates back and writes its rows of the element result to a
// cell-major buffer Yc[e][cell] (coalesced; every row written by exactly one thread).
// Phase 2 (op_gather_kernel): one thread per DoF sums the element results of the <= 2^d cells that contain the
// node in a fixed order (deterministic, no atomics) and fuses the residual / RHS combination y = beta*b + alpha*A x.
#include "stgmg_internal.cuh"

namespace stgmg {

template <int R, int K1>
struct T2 {
  static constexpr int NQ1 = R + 1, NP1 = R, NG = R + 1;
  static constexpr int NQ = NQ1 * NQ1, NP = NP1 * NP1, NGP = NG * NG;
  static constexpr int NE1 = 4 * NQ + NP;
  static constexpr int NE = K1 * NE1;
};

constexpr int OP2D_CPB = 32;   // cells per block; block = OP2D_CPB x 4 tasks, grid z = Radau node

// out[x + NX*y] = sum_{i,j} Mx[x][i] My[y][j] in[i + N1*j]     (Mx: NX rows, My: NY rows, row stride kMaxR1)
template <int N1, int NX, int NY>
__device__ __forceinline__ void tp2(const double* in, double* out, const double* Mx, const double* My) {
  double t[NX * N1];
#pragma unroll
  for (int j = 0; j < N1; ++j)
#pragma unroll
    for (int x = 0; x < NX; ++x) {
      double s = 0.0;
#pragma unroll
      for (int i = 0; i < N1; ++i) s = fma(Mx[x * kMaxR1 + i], in[i + N1 * j], s);
      t[x + NX * j] = s;
    }
#pragma unroll
  for (int y = 0; y < NY; ++y)
#pragma unroll
    for (int x = 0; x < NX; ++x) {
      double s = 0.0;
#pragma unroll
      for (int j = 0; j < N1; ++j) s = fma(My[y * kMaxR1 + j], t[x + NX * j], s);
      out[x + NX * y] = s;
    }
}

// out[i + N1*j] += sum_{x,y} Mx[x][i] My[y][j] in[x + NX*y]     (transpose of tp2, accumulating)
template <int N1, int NX, int NY>
__device__ __forceinline__ void tp2T(const double* in, double* out, const double* Mx, const double* My) {
  double t[N1 * NY];
#pragma unroll
  for (int y = 0; y < NY; ++y)
#pragma unroll
    for (int i = 0; i < N1; ++i) {
      double s = 0.0;
#pragma unroll
      for (int x = 0; x < NX; ++x) s = fma(Mx[x * kMaxR1 + i], in[x + NX * y], s);
      t[i + N1 * y] = s;
    }
#pragma unroll
  for (int j = 0; j < N1; ++j)
#pragma unroll
    for (int i = 0; i < N1; ++i) {
      double s = out[i + N1 * j];
#pragma unroll
      for (int y = 0; y < NY; ++y) s = fma(My[y * kMaxR1 + j], t[i + N1 * y], s);
      out[i + N1 * j] = s;
    }
}

template <int R, int K1>
__global__ void __launch_bounds__(OP2D_CPB * 4) op2d_cell_kernel(LevelGeom g, const OpConsts* __restrict__ cdev,
                                                                      const double* __restrict__ x,
                                                                      double* __restrict__ Yc, long long stride,
                                                                      long long ycstride) {
  pdl_trigger();
  using T = T2<R, K1>;
  constexpr int NQ1 = T::NQ1, NP1 = T::NP1, NG = T::NG, NQ = T::NQ, NP = T::NP, NGP = T::NGP, NE1 = T::NE1;
  __shared__ OpConsts c;
  {
    const double* src = reinterpret_cast<const double*>(cdev);
    double* dst = reinterpret_cast<double*>(&c);
    for (int i = threadIdx.x; i < (int)(sizeof(OpConsts) / sizeof(double)); i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  pdl_wait();
  x += blockIdx.y * stride;
  Yc += blockIdx.y * ycstride;
  // thread -> (cell, task), block z -> Radau node b; task 0: phi rows (V slot), 1/2: chi rows component 0/1
  // (U slot), 3: psi row (P slot).  Warp-uniform (b, task); consecutive lanes = consecutive cells.
  const int lc = threadIdx.x % OP2D_CPB;
  const int task = threadIdx.x / OP2D_CPB;
  const int b = blockIdx.z;
  const long long ncell = (long long)g.n[0] * g.n[1];
  const long long cell = (long long)blockIdx.x * OP2D_CPB + lc;
  if (cell >= ncell) return;
  const int cx = (int)(cell % g.n[0]), cy = (int)(cell / g.n[0]);
  const long long qbase = (long long)R * cx * g.qs[0] + (long long)R * cy * g.qs[1];
  const long long pbase = (long long)(R - 1) * cx * g.ps[0] + (long long)(R - 1) * cy * g.ps[1];
  const long long qs1 = g.qs[1], ps1 = g.ps[1];
  // element input (slot, local node j) at Radau node m, read through the read-only cache
  auto XQ = [&](int m, int slot, int j) -> double {
    return __ldg(x + (long long)m * g.block + slot * g.nq + qbase + (j % NQ1) + (j / NQ1) * qs1);
  };
  auto XP = [&](int m, int j) -> double {
    return __ldg(x + (long long)m * g.block + 2 * g.R + pbase + (j % NP1) + (j / NP1) * ps1);
  };
  const double hx = 1.0 / g.h[0], hy = 1.0 / g.h[1];
  const double jac = g.vol;
  const bool bnd = (cx == 0) || (cy == 0) || (cx == g.n[0] - 1) || (cy == g.n[1] - 1);
  const double th = c.theta[b];
  double* yrow = Yc + (long long)b * NE1 * ncell + cell;    // row e of node b at yrow[e * ncell]

  if (task == 0) {
    // ---- phi rows (V slot): M_rho (sum_a T_ba U_a - theta_b V_b)
#pragma unroll 1
    for (int cc = 0; cc < 2; ++cc) {
      double nod[NQ], qv[NGP], out[NQ];
#pragma unroll
      for (int j = 0; j < NQ; ++j) {
        double s = -th * XQ(b, cc, j);
#pragma unroll
        for (int a = 0; a < K1; ++a) s = fma(c.T[b][a], XQ(a, 2 + cc, j), s);
        nod[j] = s;
      }
      tp2<NQ1, NG, NG>(nod, qv, &c.B[0][0], &c.B[0][0]);
#pragma unroll
      for (int q = 0; q < NGP; ++q) qv[q] *= c.rho * jac * c.wg[q % NG] * c.wg[q / NG];
#pragma unroll
      for (int j = 0; j < NQ; ++j) out[j] = 0.0;
      tp2T<NQ1, NG, NG>(qv, out, &c.B[0][0], &c.B[0][0]);
#pragma unroll
      for (int j = 0; j < NQ; ++j) yrow[(long long)(cc * NQ + j) * ncell] = out[j];
    }
    return;
  }
  if (task <= 2) {
    // ---- chi rows (U slot), component cc: M_rho sum_a T_ba V_a + theta_b (sigma(U_b) - alpha P_b I) : grad chi
    const int cc = task - 1;
    double nod[NQ], out[NQ];
    {
      double qv[NGP];
#pragma unroll
      for (int j = 0; j < NQ; ++j) {
        double s = 0.0;
#pragma unroll
        for (int a = 0; a < K1; ++a) s = fma(c.T[b][a], XQ(a, cc, j), s);
        nod[j] = s;
      }
      tp2<NQ1, NG, NG>(nod, qv, &c.B[0][0], &c.B[0][0]);
#pragma unroll
      for (int q = 0; q < NGP; ++q) qv[q] *= c.rho * jac * c.wg[q % NG] * c.wg[q / NG];
#pragma unroll
      for (int j = 0; j < NQ; ++j) out[j] = 0.0;
      tp2T<NQ1, NG, NG>(qv, out, &c.B[0][0], &c.B[0][0]);
    }
    {
      double g00[NGP], g01[NGP], g10[NGP], g11[NGP], pv[NGP], pn[NP];
#pragma unroll
      for (int j = 0; j < NQ; ++j) nod[j] = XQ(b, 2, j);
      tp2<NQ1, NG, NG>(nod, g00, &c.Dm[0][0], &c.B[0][0]);
      tp2<NQ1, NG, NG>(nod, g01, &c.B[0][0], &c.Dm[0][0]);
#pragma unroll
      for (int j = 0; j < NQ; ++j) nod[j] = XQ(b, 3, j);
      tp2<NQ1, NG, NG>(nod, g10, &c.Dm[0][0], &c.B[0][0]);
      tp2<NQ1, NG, NG>(nod, g11, &c.B[0][0], &c.Dm[0][0]);
#pragma unroll
      for (int j = 0; j < NP; ++j) pn[j] = XP(b, j);
      tp2<NP1, NG, NG>(pn, pv, &c.Bp[0][0], &c.Bp[0][0]);
#pragma unroll
      for (int q = 0; q < NGP; ++q) {
        const double w = th * jac * c.wg[q % NG] * c.wg[q / NG];
        const double ux = g00[q] * hx, uy = g01[q] * hy, vx = g10[q] * hx, vy = g11[q] * hy;
        const double tr = ux + vy;
        const double sxy = c.mu * (uy + vx);
        const double d0 = c.lam * tr - c.alpha * pv[q];
        // row cc of (sigma - alpha p I), scaled: gx = sigma_{cc,0} w / h_x, gy = sigma_{cc,1} w / h_y
        if (cc == 0) {
          g00[q] = (2.0 * c.mu * ux + d0) * w * hx;
          g01[q] = sxy * w * hy;
        } else {
          g00[q] = sxy * w * hx;
          g01[q] = (2.0 * c.mu * vy + d0) * w * hy;
        }
      }
      tp2T<NQ1, NG, NG>(g00, out, &c.Dm[0][0], &c.B[0][0]);
      tp2T<NQ1, NG, NG>(g01, out, &c.B[0][0], &c.Dm[0][0]);
    }
    if (bnd) {
      // Nitsche terms of A_gamma (Def:A, Def:agam) and alpha <chi.n, p> of C (Def:C) on Dirichlet u faces
#pragma unroll 1
      for (int f = 0; f < 4; ++f) {
        const int fa = f >> 1, fs = f & 1;
        const int ci = fa == 0 ? cx : cy;
        if (ci != (fs ? g.n[fa] - 1 : 0) || g.bcu[f] != 0) continue;
        const double nrm = fs ? 1.0 : -1.0;
        const double* Vq = fa == 0 ? &c.E[fs][0] : &c.B[0][0];
        const double* Wq = fa == 0 ? &c.B[0][0] : &c.E[fs][0];
        const double* dVq = fa == 0 ? &c.dE[fs][0] : &c.Dm[0][0];
        const double* dWq = fa == 0 ? &c.Dm[0][0] : &c.dE[fs][0];
        const double* Vp = fa == 0 ? &c.Ep[fs][0] : &c.Bp[0][0];
        const double* Wp = fa == 0 ? &c.Bp[0][0] : &c.Ep[fs][0];
        constexpr int NF = NG;
        const double area = jac * (fa == 0 ? hx : hy);
        double fP[NF], pn[NP], U0[NF], U1[NF], a00[NF], a01[NF], a10[NF], a11[NF];
#pragma unroll
        for (int j = 0; j < NP; ++j) pn[j] = XP(b, j);
        if (fa == 0) tp2<NP1, 1, NF>(pn, fP, Vp, Wp); else tp2<NP1, NF, 1>(pn, fP, Vp, Wp);
#pragma unroll
        for (int j = 0; j < NQ; ++j) nod[j] = XQ(b, 2, j);
        if (fa == 0) {
          tp2<NQ1, 1, NF>(nod, U0, Vq, Wq); tp2<NQ1, 1, NF>(nod, a00, dVq, Wq); tp2<NQ1, 1, NF>(nod, a01, Vq, dWq);
        } else {
          tp2<NQ1, NF, 1>(nod, U0, Vq, Wq); tp2<NQ1, NF, 1>(nod, a00, dVq, Wq); tp2<NQ1, NF, 1>(nod, a01, Vq, dWq);
        }
#pragma unroll
        for (int j = 0; j < NQ; ++j) nod[j] = XQ(b, 3, j);
        if (fa == 0) {
          tp2<NQ1, 1, NF>(nod, U1, Vq, Wq); tp2<NQ1, 1, NF>(nod, a10, dVq, Wq); tp2<NQ1, 1, NF>(nod, a11, Vq, dWq);
        } else {
          tp2<NQ1, NF, 1>(nod, U1, Vq, Wq); tp2<NQ1, NF, 1>(nod, a10, dVq, Wq); tp2<NQ1, NF, 1>(nod, a11, Vq, dWq);
        }
        const double pen = c.gamma_a / g.hF[f];
        double cv[NF], cg0[NF], cg1[NF];
#pragma unroll
        for (int q = 0; q < NF; ++q) {
          const double w = th * area * c.wg[q];
          const double G[2][2] = {{a00[q] * hx, a01[q] * hy}, {a10[q] * hx, a11[q] * hy}};
          const double U[2] = {U0[q], U1[q]};
          const double tr = G[0][0] + G[1][1];
          const double un = U[fa] * nrm;
          const double sn = (c.mu * (G[cc][fa] + G[fa][cc]) + (cc == fa ? c.lam * tr : 0.0)) * nrm;
          cv[q] = (-sn + pen * U[cc] + (cc == fa ? c.alpha * fP[q] * nrm : 0.0)) * w;
          const double ni = (cc == fa ? nrm : 0.0);
          cg0[q] = -((cc == 0 ? c.lam * un : 0.0) + c.mu * (U[cc] * (fa == 0 ? nrm : 0.0) + U[0] * ni)) * w * hx;
          cg1[q] = -((cc == 1 ? c.lam * un : 0.0) + c.mu * (U[cc] * (fa == 1 ? nrm : 0.0) + U[1] * ni)) * w * hy;
        }
        if (fa == 0) {
          tp2T<NQ1, 1, NF>(cv, out, Vq, Wq); tp2T<NQ1, 1, NF>(cg0, out, dVq, Wq); tp2T<NQ1, 1, NF>(cg1, out, Vq, dWq);
        } else {
          tp2T<NQ1, NF, 1>(cv, out, Vq, Wq); tp2T<NQ1, NF, 1>(cg0, out, dVq, Wq); tp2T<NQ1, NF, 1>(cg1, out, Vq, dWq);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < NQ; ++j) yrow[(long long)((2 + cc) * NQ + j) * ncell] = out[j];
    return;
  }
  // ---- task 3: psi row (P slot): M_c sum_a T_ba P_a + theta_b (alpha div V_b, K grad P_b) + Nitsche terms
  double po[NP];
  {
    double pn[NP], pval[NGP], px[NGP], py[NGP], dv[NGP], tmp[NGP], nod[NQ];
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      double s = 0.0;
#pragma unroll
      for (int a = 0; a < K1; ++a) s = fma(c.T[b][a], XP(a, j), s);
      pn[j] = s;
    }
    tp2<NP1, NG, NG>(pn, pval, &c.Bp[0][0], &c.Bp[0][0]);
#pragma unroll
    for (int j = 0; j < NP; ++j) pn[j] = XP(b, j);
    tp2<NP1, NG, NG>(pn, px, &c.Dp[0][0], &c.Bp[0][0]);
    tp2<NP1, NG, NG>(pn, py, &c.Bp[0][0], &c.Dp[0][0]);
    // velocity coupled into the p-equation: V_b (DSA, Problem 3.1) or sum_a T_ba U_a (DS, Problem B.1: d_t u)
    const bool ds = c.ds != 0.0;
#pragma unroll
    for (int j = 0; j < NQ; ++j) {
      double s = 0.0;
      if (ds) {
#pragma unroll
        for (int a = 0; a < K1; ++a) s = fma(c.T[b][a], XQ(a, 2, j), s);
      } else {
        s = XQ(b, 0, j);
      }
      nod[j] = s;
    }
    tp2<NQ1, NG, NG>(nod, dv, &c.Dm[0][0], &c.B[0][0]);
#pragma unroll
    for (int j = 0; j < NQ; ++j) {
      double s = 0.0;
      if (ds) {
#pragma unroll
        for (int a = 0; a < K1; ++a) s = fma(c.T[b][a], XQ(a, 3, j), s);
      } else {
        s = XQ(b, 1, j);
      }
      nod[j] = s;
    }
    tp2<NQ1, NG, NG>(nod, tmp, &c.B[0][0], &c.Dm[0][0]);
    const double cth = ds ? 1.0 : th;   // coefficient of the velocity coupling
#pragma unroll
    for (int q = 0; q < NGP; ++q) {
      const double w = jac * c.wg[q % NG] * c.wg[q / NG];
      const double div = dv[q] * hx + tmp[q] * hy;
      pval[q] = (c.c0 * pval[q] + cth * c.alpha * div) * w;
      const double gx = px[q] * hx, gy = py[q] * hy;
      const double kx = c.K[0] * gx + c.K[1] * gy, ky = c.K[3] * gx + c.K[4] * gy;
      px[q] = th * kx * w * hx;
      py[q] = th * ky * w * hy;
    }
#pragma unroll
    for (int j = 0; j < NP; ++j) po[j] = 0.0;
    tp2T<NP1, NG, NG>(pval, po, &c.Bp[0][0], &c.Bp[0][0]);
    tp2T<NP1, NG, NG>(px, po, &c.Dp[0][0], &c.Bp[0][0]);
    tp2T<NP1, NG, NG>(py, po, &c.Bp[0][0], &c.Dp[0][0]);
  }
  if (bnd) {
#pragma unroll 1
    for (int f = 0; f < 4; ++f) {
      const int fa = f >> 1, fs = f & 1;
      const int ci = fa == 0 ? cx : cy;
      if (ci != (fs ? g.n[fa] - 1 : 0)) continue;
      const bool du = g.bcu[f] == 0, dp = g.bcp[f] == 0;
      if (!du && !dp) continue;
      const double nrm = fs ? 1.0 : -1.0;
      const double* Vq = fa == 0 ? &c.E[fs][0] : &c.B[0][0];
      const double* Wq = fa == 0 ? &c.B[0][0] : &c.E[fs][0];
      const double* Vp = fa == 0 ? &c.Ep[fs][0] : &c.Bp[0][0];
      const double* Wp = fa == 0 ? &c.Bp[0][0] : &c.Ep[fs][0];
      const double* dVp = fa == 0 ? &c.dEp[fs][0] : &c.Dp[0][0];
      const double* dWp = fa == 0 ? &c.Dp[0][0] : &c.dEp[fs][0];
      constexpr int NF = NG;
      const double area = jac * (fa == 0 ? hx : hy);
      double fP[NF], pn[NP], psiv[NF], psig0[NF], psig1[NF];
#pragma unroll
      for (int j = 0; j < NP; ++j) pn[j] = XP(b, j);
      if (fa == 0) tp2<NP1, 1, NF>(pn, fP, Vp, Wp); else tp2<NP1, NF, 1>(pn, fP, Vp, Wp);
#pragma unroll
      for (int q = 0; q < NF; ++q) psiv[q] = psig0[q] = psig1[q] = 0.0;
      if (du) {   // -theta alpha <V.n, psi> (Def:C on G_D^u); DS: -alpha <(sum_a T_ba U_a).n, psi>
        const bool ds = c.ds != 0.0;
        double nod[NQ], Vn[NF];
#pragma unroll
        for (int j = 0; j < NQ; ++j) {
          double s = 0.0;
          if (ds) {
#pragma unroll
            for (int a = 0; a < K1; ++a) s = fma(c.T[b][a], XQ(a, 2 + fa, j), s);
          } else {
            s = XQ(b, fa, j);
          }
          nod[j] = s;
        }
        if (fa == 0) tp2<NQ1, 1, NF>(nod, Vn, Vq, Wq); else tp2<NQ1, NF, 1>(nod, Vn, Vq, Wq);
        const double cth = ds ? c.ds_face : th;   // slab RHS (DS): 0, P:L1073 has u_D(t_{n-1}) = 0 there
#pragma unroll
        for (int q = 0; q < NF; ++q) psiv[q] += -c.alpha * Vn[q] * nrm * cth * area * c.wg[q];
      }
      if (dp) {   // B_gamma Nitsche terms (Def:B, Def:bgam)
        double gx[NF], gy[NF];
        if (fa == 0) {
          tp2<NP1, 1, NF>(pn, gx, dVp, Wp); tp2<NP1, 1, NF>(pn, gy, Vp, dWp);
        } else {
          tp2<NP1, NF, 1>(pn, gx, dVp, Wp); tp2<NP1, NF, 1>(pn, gy, Vp, dWp);
        }
        const double pen = c.gamma_b / g.hF[f];
#pragma unroll
        for (int q = 0; q < NF; ++q) {
          const double w = th * area * c.wg[q];
          const double gpn = (c.K[fa * 3 + 0] * gx[q] * hx + c.K[fa * 3 + 1] * gy[q] * hy) * nrm;
          psiv[q] += (-gpn + pen * fP[q]) * w;
          psig0[q] = -fP[q] * c.K[fa * 3 + 0] * nrm * w * hx;
          psig1[q] = -fP[q] * c.K[fa * 3 + 1] * nrm * w * hy;
        }
      }
      if (fa == 0) {
        tp2T<NP1, 1, NF>(psiv, po, Vp, Wp);
        if (dp) { tp2T<NP1, 1, NF>(psig0, po, dVp, Wp); tp2T<NP1, 1, NF>(psig1, po, Vp, dWp); }
      } else {
        tp2T<NP1, NF, 1>(psiv, po, Vp, Wp);
        if (dp) { tp2T<NP1, NF, 1>(psig0, po, dVp, Wp); tp2T<NP1, NF, 1>(psig1, po, Vp, dWp); }
      }
    }
  }
#pragma unroll
  for (int j = 0; j < NP; ++j) yrow[(long long)(4 * NQ + j) * ncell] = po[j];
}

// Phase 2 (node gather) lives in nodal.cu (gather_nodal_kernel).

template <int R, int K1>
static cudaError_t launch2d(const LevelGeom& g, const OpConsts* cdev, const double* x, double* Yc, int batch,
                            long long stride, long long ycstride, cudaStream_t s) {
  const long long ncell = (long long)g.n[0] * g.n[1];
  dim3 grid((unsigned)((ncell + OP2D_CPB - 1) / OP2D_CPB), (unsigned)batch, (unsigned)K1);
  return launch_pdl(op2d_cell_kernel<R, K1>, grid, dim3(OP2D_CPB * 4), 0, s, g, cdev, x, Yc, stride, ycstride);
}

#define OP2D_CASE(R_, K1_) \
  if (r == R_ && k1 == K1_) return launch2d<R_, K1_>(g, cdev, x, Yc, batch, stride, ycstride, s);

cudaError_t launch_op2d_cells(int r, int k1, const LevelGeom& g, const OpConsts* cdev, const double* x, double* Yc,
                              int batch, long long stride, long long ycstride, cudaStream_t s) {
  OP2D_CASE(2, 1)
  OP2D_CASE(2, 2)
  OP2D_CASE(2, 3)
  OP2D_CASE(3, 1)
  OP2D_CASE(3, 2)
  OP2D_CASE(3, 3)
  return cudaErrorNotSupported;
}

}  // namespace stgmg
