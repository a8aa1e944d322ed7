// K1 — matrix-free space-time slab operator  y (+)= sign * A_l x  (sm_100a, fp64).
//
// Definition (Problem 3.1, Eq:DPQ_A0; block form P:L384-431 read per SURVEY reading A5):
//   (A X)_{phi,b} = sum_a T_ba M_rho U_a - theta_b M_rho V_b
//   (A X)_{chi,b} = sum_a T_ba M_rho V_a + theta_b (A_gamma U_b + C^T P_b)
//   (A X)_{psi,b} = sum_a T_ba M_c  P_a + theta_b (-C V_b + B_gamma P_b)
// with the forms of Def:ACB / Def:ab.  Per cell: the temporal mixing is done on the nodal
// values, the spatial forms by sum factorisation on the (r+1)^d Gauss points (values and gradients via 1D
// contractions along each axis), Nitsche face terms on Dirichlet boundary faces at (r+1)^{d-1} points.
//
// Execution: one warp per cell, warp-synchronous shared-memory sum factorisation, cells of one 2^d colour
// per launch so that no two cells of a launch share a node (deterministic, no atomics).  In 3D this kernel
// produces the per-cell-type element matrices at setup (Yc output); the runtime 3D apply multiplies them with
// the gathered cell vectors on the FP64 tensor pipe (grouped K2 GEMM) and sums them with op_gather_kernel.
#include "stgmg_internal.cuh"

namespace stgmg {

__host__ __device__ constexpr int ipow(int b, int e) { return e == 0 ? 1 : b * ipow(b, e - 1); }

template <int D, int R, int K1>
struct Tr {
  static constexpr int NQ1 = R + 1, NP1 = R, NG = R + 1;
  static constexpr int NQ = ipow(NQ1, D), NP = ipow(NP1, D), NGP = ipow(NG, D);
  static constexpr int NE1 = 2 * D * NQ + NP;
  static constexpr int NE = K1 * NE1;
  static constexpr int NQTY = D * D + 3 * D + 3;        // quantities at quadrature points
  static constexpr int NNOD = 4 * D * NQ + 2 * NP;      // mixed nodal arrays
  static constexpr int TMP = NGP > NQ ? NGP : NQ;
  static constexpr int SMEM = NE + NE1 + NNOD + NQTY * NGP + 2 * TMP;   // doubles per warp
};

// Per-axis operator selection for a tensor contraction.
// kind: 0 = values at Gauss points, 1 = derivative at Gauss points, 2 = value at endpoint, 3 = derivative at endpoint
struct AxisOp {
  const double* M;   // row-major, rows = points, cols = nodes, leading dimension kMaxR1
  int npts;
};

// out (+)= contraction of `in` (nodal, dims nn per axis) to points (dims ops[a].npts), or the transpose
// (points -> nodes) when T = true.  Warp-cooperative; ends with __syncwarp().
template <int D, bool TRANSP>
__device__ __forceinline__ void contract(const double* __restrict__ in, double* __restrict__ out, double* t1,
                                         double* t2, const AxisOp* ops, int nn, bool accumulate, double scale,
                                         int lane) {
  int dims[3];
  for (int a = 0; a < D; ++a) dims[a] = TRANSP ? ops[a].npts : nn;
  const double* src = in;
  for (int a = 0; a < D; ++a) {
    const int nin = dims[a];
    const int nout = TRANSP ? nn : ops[a].npts;
    int odims[3] = {dims[0], dims[1], dims[2]};
    odims[a] = nout;
    int total = 1;
    for (int b = 0; b < D; ++b) total *= odims[b];
    const bool last = (a == D - 1);
    double* dst = last ? out : ((a & 1) ? t2 : t1);
    int stride_a = 1;
    for (int b = 0; b < a; ++b) stride_a *= odims[b];   // axes < a already have output dims (== stride in src too)
    for (int idx = lane; idx < total; idx += 32) {
      const int ilow = idx % stride_a;
      const int ia = (idx / stride_a) % nout;
      const int ihigh = idx / (stride_a * nout);
      const int base = ilow + stride_a * nin * ihigh;  // source position with axis-a coordinate 0
      double s = 0.0;
      if (!TRANSP) {
        const double* Mrow = ops[a].M + ia * kMaxR1;
#pragma unroll 4
        for (int j = 0; j < nin; ++j) s = fma(Mrow[j], src[base + j * stride_a], s);
      } else {
#pragma unroll 4
        for (int j = 0; j < nin; ++j) s = fma(ops[a].M[j * kMaxR1 + ia], src[base + j * stride_a], s);
      }
      if (last) {
        s *= scale;
        dst[idx] = accumulate ? dst[idx] + s : s;
      } else {
        dst[idx] = s;
      }
    }
    __syncwarp();
    src = dst;
    for (int b = 0; b < D; ++b) dims[b] = odims[b];
  }
}

template <int D, int R, int K1>
__global__ void __launch_bounds__(128) op_apply_kernel(LevelGeom g, const OpConsts* __restrict__ cdev,
                                                       const double* __restrict__ x, double* __restrict__ y,
                                                       double* __restrict__ Yc, double sign, int color,
                                                       long long stride, long long ycstride) {
  pdl_trigger();
  using T = Tr<D, R, K1>;
  extern __shared__ double smem[];
  __shared__ OpConsts c;
  {
    const double* src = reinterpret_cast<const double*>(cdev);
    double* dst = reinterpret_cast<double*>(&c);
    for (int i = threadIdx.x; i < (int)(sizeof(OpConsts) / sizeof(double)); i += blockDim.x) dst[i] = src[i];
  }
  __syncthreads();
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int wpb = blockDim.x >> 5;
  double* S = smem + (size_t)warp * T::SMEM;
  double* xe = S;                     // [K1][NE1]
  double* ye = xe + T::NE;            // [NE1]
  double* nod = ye + T::NE1;          // mixed nodal arrays
  double* qv = nod + T::NNOD;         // [NQTY][NGP]
  double* t1 = qv + T::NQTY * T::NGP;
  double* t2 = t1 + T::TMP;

  x += blockIdx.y * stride;
  if (y) y += blockIdx.y * stride;
  if (Yc) Yc += blockIdx.y * ycstride;

  // cell of this warp within the colour
  int cnt[3] = {1, 1, 1}, bit[3] = {0, 0, 0};
  long long ncol = 1;
  for (int a = 0; a < D; ++a) {
    bit[a] = (color >> a) & 1;
    cnt[a] = (g.n[a] - bit[a] + 1) / 2;
    ncol *= cnt[a];
  }
  const long long cid = (long long)blockIdx.x * wpb + warp;
  if (cid >= ncol) return;
  int cell[3] = {0, 0, 0};
  {
    long long rem = cid;
    for (int a = 0; a < D; ++a) {
      cell[a] = 2 * (int)(rem % cnt[a]) + bit[a];
      rem /= cnt[a];
    }
  }
  long long qbase = 0, pbase = 0;
  for (int a = 0; a < D; ++a) {
    qbase += (long long)(R * cell[a]) * g.qs[a];
    pbase += (long long)((R - 1) * cell[a]) * g.ps[a];
  }
  // global index of element dof e (0..NE1-1) at time node m
  auto gidx = [&](int m, int e) -> long long {
    long long off = (long long)m * g.block;
    if (e < 2 * D * T::NQ) {
      const int fc = e / T::NQ, j = e % T::NQ;   // fc = f*D + comp  (f: 0 = V, 1 = U)
      long long node = qbase;
      int jj = j;
      for (int a = 0; a < D; ++a) {
        node += (long long)(jj % T::NQ1) * g.qs[a];
        jj /= T::NQ1;
      }
      return off + (long long)fc * g.nq + node;
    } else {
      int jj = e - 2 * D * T::NQ;
      long long node = pbase;
      for (int a = 0; a < D; ++a) {
        node += (long long)(jj % T::NP1) * g.ps[a];
        jj /= T::NP1;
      }
      return off + 2 * g.R + node;
    }
  };
  for (int i = lane; i < T::NE; i += 32) xe[i] = __ldg(x + gidx(i / T::NE1, i % T::NE1));
  __syncwarp();

  const double hinv[3] = {1.0 / g.h[0], D > 1 ? 1.0 / g.h[1] : 0.0, D > 2 ? 1.0 / g.h[2] : 0.0};
  // axis operators
  AxisOp Bq[3], Bp[3];
  for (int a = 0; a < D; ++a) {
    Bq[a] = {&c.B[0][0], T::NG};
    Bp[a] = {&c.Bp[0][0], T::NG};
  }
  // nodal array pointers
  double* Xphi = nod;                 // [D][NQ]
  double* Xchi = Xphi + D * T::NQ;
  double* Ub = Xchi + D * T::NQ;
  double* Vb = Ub + D * T::NQ;
  double* Xpsi = Vb + D * T::NQ;      // [NP]
  double* Pb = Xpsi + T::NP;
  // quantity pointers at quadrature points
  double* q_phi = qv;                       // [D]
  double* q_chi = q_phi + D * T::NGP;       // [D]
  double* gU = q_chi + D * T::NGP;          // [D][D]  gU[c][b] = d_b U_c
  double* divV = gU + D * D * T::NGP;       // [1]
  double* q_psi = divV + T::NGP;            // [1]
  double* Pv = q_psi + T::NGP;              // [1]
  double* gP = Pv + T::NGP;                 // [D]

  int bface[6];
  int nbf = 0;
  for (int a = 0; a < D; ++a) {
    if (cell[a] == 0) bface[nbf++] = 2 * a;
    if (cell[a] == g.n[a] - 1) bface[nbf++] = 2 * a + 1;
  }
  const double jac = g.vol;

  for (int b = 0; b < K1; ++b) {
    const double th = c.theta[b];
    // 1. temporal mixing on nodal values
    for (int i = lane; i < D * T::NQ; i += 32) {
      double sphi = -th * xe[b * T::NE1 + i];                      // -theta_b V_b
      double schi = 0.0;
#pragma unroll
      for (int a = 0; a < K1; ++a) {
        sphi = fma(c.T[b][a], xe[a * T::NE1 + D * T::NQ + i], sphi);  // T_ba U_a
        schi = fma(c.T[b][a], xe[a * T::NE1 + i], schi);              // T_ba V_a
      }
      Xphi[i] = sphi;
      Xchi[i] = schi;
      Ub[i] = xe[b * T::NE1 + D * T::NQ + i];
      if (c.ds != 0.0) {   // DS (Problem B.1): the p-equation couples d_t u = sum_a T_ba U_a instead of V_b
        double s = 0.0;
#pragma unroll
        for (int a = 0; a < K1; ++a) s = fma(c.T[b][a], xe[a * T::NE1 + D * T::NQ + i], s);
        Vb[i] = s;
      } else {
        Vb[i] = xe[b * T::NE1 + i];
      }
    }
    for (int i = lane; i < T::NP; i += 32) {
      double s = 0.0;
#pragma unroll
      for (int a = 0; a < K1; ++a) s = fma(c.T[b][a], xe[a * T::NE1 + 2 * D * T::NQ + i], s);
      Xpsi[i] = s;
      Pb[i] = xe[b * T::NE1 + 2 * D * T::NQ + i];
    }
    __syncwarp();
    // 2. interpolation to the Gauss points
    for (int cc = 0; cc < D; ++cc) {
      contract<D, false>(Xphi + cc * T::NQ, q_phi + cc * T::NGP, t1, t2, Bq, T::NQ1, false, 1.0, lane);
      contract<D, false>(Xchi + cc * T::NQ, q_chi + cc * T::NGP, t1, t2, Bq, T::NQ1, false, 1.0, lane);
      for (int bb = 0; bb < D; ++bb) {
        AxisOp op[3];
        for (int a = 0; a < D; ++a) op[a] = {a == bb ? &c.Dm[0][0] : &c.B[0][0], T::NG};
        contract<D, false>(Ub + cc * T::NQ, gU + (cc * D + bb) * T::NGP, t1, t2, op, T::NQ1, false, hinv[bb], lane);
        if (bb == cc)
          contract<D, false>(Vb + cc * T::NQ, divV, t1, t2, op, T::NQ1, cc > 0, hinv[bb], lane);
      }
    }
    contract<D, false>(Xpsi, q_psi, t1, t2, Bp, T::NP1, false, 1.0, lane);
    contract<D, false>(Pb, Pv, t1, t2, Bp, T::NP1, false, 1.0, lane);
    for (int bb = 0; bb < D; ++bb) {
      AxisOp op[3];
      for (int a = 0; a < D; ++a) op[a] = {a == bb ? &c.Dp[0][0] : &c.Bp[0][0], T::NG};
      contract<D, false>(Pb, gP + bb * T::NGP, t1, t2, op, T::NP1, false, hinv[bb], lane);
    }
    // 3. pointwise: coefficients of the test values / gradients (in place), times JxW
    for (int q = lane; q < T::NGP; q += 32) {
      double w = jac;
      {
        int qq = q;
        for (int a = 0; a < D; ++a) {
          w *= c.wg[qq % T::NG];
          qq /= T::NG;
        }
      }
      double G[3][3], tr = 0.0;
      for (int i = 0; i < D; ++i)
        for (int j = 0; j < D; ++j) G[i][j] = gU[(i * D + j) * T::NGP + q];
      for (int i = 0; i < D; ++i) tr += G[i][i];
      const double p = Pv[q];
      // chi gradient coefficient: theta (sigma(U) - alpha p I) JxW / h_j  (stored in gU)
      for (int i = 0; i < D; ++i)
        for (int j = 0; j < D; ++j) {
          double s = c.mu * (G[i][j] + G[j][i]) + (i == j ? c.lam * tr - c.alpha * p : 0.0);
          gU[(i * D + j) * T::NGP + q] = th * s * w * hinv[j];
        }
      for (int i = 0; i < D; ++i) {
        q_phi[i * T::NGP + q] *= c.rho * w;
        q_chi[i * T::NGP + q] *= c.rho * w;
      }
      // psi value coefficient: (c0 Xpsi + theta alpha div V) JxW ; psi gradient: theta K grad P JxW / h_j
      q_psi[q] = (c.c0 * q_psi[q] + (c.ds != 0.0 ? 1.0 : th) * c.alpha * divV[q]) * w;
      double gp[3];
      for (int j = 0; j < D; ++j) gp[j] = gP[j * T::NGP + q];
      for (int i = 0; i < D; ++i) {
        double s = 0.0;
        for (int j = 0; j < D; ++j) s += c.K[i * 3 + j] * gp[j];
        gP[i * T::NGP + q] = th * s * w * hinv[i];
      }
    }
    __syncwarp();
    // 4. integrate back into ye (element rows at node b: V slot = phi, U slot = chi, P slot = psi)
    for (int cc = 0; cc < D; ++cc) {
      contract<D, true>(q_phi + cc * T::NGP, ye + cc * T::NQ, t1, t2, Bq, T::NQ1, false, 1.0, lane);
      contract<D, true>(q_chi + cc * T::NGP, ye + (D + cc) * T::NQ, t1, t2, Bq, T::NQ1, false, 1.0, lane);
      for (int bb = 0; bb < D; ++bb) {
        AxisOp op[3];
        for (int a = 0; a < D; ++a) op[a] = {a == bb ? &c.Dm[0][0] : &c.B[0][0], T::NG};
        contract<D, true>(gU + (cc * D + bb) * T::NGP, ye + (D + cc) * T::NQ, t1, t2, op, T::NQ1, true, 1.0, lane);
      }
    }
    contract<D, true>(q_psi, ye + 2 * D * T::NQ, t1, t2, Bp, T::NP1, false, 1.0, lane);
    for (int bb = 0; bb < D; ++bb) {
      AxisOp op[3];
      for (int a = 0; a < D; ++a) op[a] = {a == bb ? &c.Dp[0][0] : &c.Bp[0][0], T::NG};
      contract<D, true>(gP + bb * T::NGP, ye + 2 * D * T::NQ, t1, t2, op, T::NP1, true, 1.0, lane);
    }
    // 5. Nitsche face terms on Dirichlet boundary faces (Def:A, Def:C, Def:B, Def:ab)
    for (int fi = 0; fi < nbf; ++fi) {
      const int f = bface[fi], fa = f >> 1, fs = f & 1;
      const bool du = g.bcu[f] == 0, dp = g.bcp[f] == 0;
      if (!du && !dp) continue;
      const double nrm = fs ? 1.0 : -1.0;            // outward normal = nrm * e_fa
      const int NF = ipow(T::NG, D - 1);
      // operators: value / derivative along each axis, endpoint on the face axis
      auto mkop = [&](AxisOp* op, int deriv, bool pres) {
        for (int a = 0; a < D; ++a) {
          if (a == fa)
            op[a] = {pres ? (a == deriv ? &c.dEp[fs][0] : &c.Ep[fs][0]) : (a == deriv ? &c.dE[fs][0] : &c.E[fs][0]), 1};
          else
            op[a] = {pres ? (a == deriv ? &c.Dp[0][0] : &c.Bp[0][0]) : (a == deriv ? &c.Dm[0][0] : &c.B[0][0]), T::NG};
        }
      };
      // face quantities: fU[D], fgU[D][D], fV[D], fP, fgP[D]  (reuse qv storage)
      double* fU = qv;
      double* fgU = fU + D * NF;
      double* fV = fgU + D * D * NF;
      double* fP = fV + D * NF;
      double* fgP = fP + NF;
      AxisOp op[3];
      if (du) {
        for (int cc = 0; cc < D; ++cc) {
          mkop(op, -1, false);
          contract<D, false>(Ub + cc * T::NQ, fU + cc * NF, t1, t2, op, T::NQ1, false, 1.0, lane);
          contract<D, false>(Vb + cc * T::NQ, fV + cc * NF, t1, t2, op, T::NQ1, false, 1.0, lane);
          for (int bb = 0; bb < D; ++bb) {
            mkop(op, bb, false);
            contract<D, false>(Ub + cc * T::NQ, fgU + (cc * D + bb) * NF, t1, t2, op, T::NQ1, false, hinv[bb], lane);
          }
        }
      }
      mkop(op, -1, true);
      contract<D, false>(Pb, fP, t1, t2, op, T::NP1, false, 1.0, lane);
      if (dp) {
        for (int bb = 0; bb < D; ++bb) {
          mkop(op, bb, true);
          contract<D, false>(Pb, fgP + bb * NF, t1, t2, op, T::NP1, false, hinv[bb], lane);
        }
      }
      // pointwise face coefficients (in place):
      //   u-face:  chi val  = theta(-sigma(U) n + gamma_a/hF U + alpha P n) w
      //            chi grad = -theta (lambda (U.n) d_cl + mu (U_c n_l + U_l n_c)) w / h_l
      //            psi val += -theta alpha (V.n) w
      //   p-face:  psi val += theta(-K grad P . n + gamma_b/hF P) w ;  psi grad = -theta P (K n)_l w / h_l
      const double area = g.vol * hinv[fa];
      for (int q = lane; q < NF; q += 32) {
        double w = area;
        {
          int qq = q;
          for (int a = 0; a < D; ++a) {
            if (a == fa) continue;
            w *= c.wg[qq % T::NG];
            qq /= T::NG;
          }
        }
        const double P = fP[q];
        double psi_val = 0.0;
        if (du) {
          double U[3], V[3], G[3][3], tr = 0.0;
          for (int i = 0; i < D; ++i) {
            U[i] = fU[i * NF + q];
            V[i] = fV[i * NF + q];
            for (int j = 0; j < D; ++j) G[i][j] = fgU[(i * D + j) * NF + q];
          }
          for (int i = 0; i < D; ++i) tr += G[i][i];
          const double un = U[fa] * nrm, vn = V[fa] * nrm;
          const double pen = c.gamma_a / g.hF[f];
          for (int i = 0; i < D; ++i) {
            // (sigma(U) n)_i = sigma_{i,fa} nrm
            const double sn = (c.mu * (G[i][fa] + G[fa][i]) + (i == fa ? c.lam * tr : 0.0)) * nrm;
            fU[i * NF + q] = th * (-sn + pen * U[i] + (i == fa ? c.alpha * P * nrm : 0.0)) * w;
            for (int l = 0; l < D; ++l) {
              const double nl = (l == fa ? nrm : 0.0), ni = (i == fa ? nrm : 0.0);
              const double Gc = (i == l ? c.lam * un : 0.0) + c.mu * (U[i] * nl + U[l] * ni);
              fgU[(i * D + l) * NF + q] = -th * Gc * w * hinv[l];
            }
          }
          psi_val += -(c.ds != 0.0 ? c.ds_face : th) * c.alpha * vn * w;
        }
        if (dp) {
          double gpn = 0.0;
          for (int j = 0; j < D; ++j) gpn += c.K[fa * 3 + j] * fgP[j * NF + q];   // (K grad P) . n / nrm
          gpn *= nrm;
          psi_val += th * (-gpn + c.gamma_b / g.hF[f] * P) * w;
          for (int l = 0; l < D; ++l) fgP[l * NF + q] = -th * P * c.K[fa * 3 + l] * nrm * w * hinv[l];
        }
        fP[q] = psi_val;
      }
      __syncwarp();
      if (du) {
        for (int cc = 0; cc < D; ++cc) {
          mkop(op, -1, false);
          contract<D, true>(fU + cc * NF, ye + (D + cc) * T::NQ, t1, t2, op, T::NQ1, true, 1.0, lane);
          for (int bb = 0; bb < D; ++bb) {
            mkop(op, bb, false);
            contract<D, true>(fgU + (cc * D + bb) * NF, ye + (D + cc) * T::NQ, t1, t2, op, T::NQ1, true, 1.0, lane);
          }
        }
      }
      mkop(op, -1, true);
      contract<D, true>(fP, ye + 2 * D * T::NQ, t1, t2, op, T::NP1, true, 1.0, lane);
      if (dp) {
        for (int bb = 0; bb < D; ++bb) {
          mkop(op, bb, true);
          contract<D, true>(fgP + bb * NF, ye + 2 * D * T::NQ, t1, t2, op, T::NP1, true, 1.0, lane);
        }
      }
    }
    // 6. scatter-add the rows of node b (no other cell of this colour touches these nodes), or store the element
    //    result cell-wise: Yc[plin(cell)][b * NE1 + e], plin = lexicographic index of vertex (cell + 1) (setup of
    //    the element matrices, patch-major like the patch results Y)
    if (Yc) {
      long long plin = 0, vs = 1;
      for (int a = 0; a < D; ++a) {
        plin += (long long)(cell[a] + 1) * vs;
        vs *= g.n[a] + 1;
      }
      for (int i = lane; i < T::NE1; i += 32) Yc[plin * T::NE + b * T::NE1 + i] = ye[i];
    } else {
      for (int i = lane; i < T::NE1; i += 32) {
        const long long gi = gidx(b, i);
        y[gi] = fma(sign, ye[i], y[gi]);
      }
    }
    __syncwarp();
  }
}

template <int D, int R, int K1>
static cudaError_t launch_impl(const LevelGeom& g, const OpConsts* cdev, const double* x, double* y, double* Yc,
                               double sign, int batch, long long stride, long long ycstride, cudaStream_t s,
                               int* nlaunch) {
  using T = Tr<D, R, K1>;
  const int wpb = 4;
  const size_t smem = (size_t)wpb * T::SMEM * sizeof(double);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(op_apply_kernel<D, R, K1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr_set = true;
  }
  for (int color = 0; color < (1 << D); ++color) {
    long long ncol = 1;
    for (int a = 0; a < D; ++a) ncol *= (g.n[a] - ((color >> a) & 1) + 1) / 2;
    if (ncol == 0) continue;
    dim3 grid((unsigned)((ncol + wpb - 1) / wpb), (unsigned)batch);
    cudaError_t e = launch_pdl(op_apply_kernel<D, R, K1>, grid, dim3(wpb * 32), smem, s, g, cdev, x, y, Yc, sign, color,
                               stride, ycstride);
    if (nlaunch) ++*nlaunch;
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

#define STGMG_OP_CASE(D_, R_, K1_)                                                                          \
  if (d == D_ && r == R_ && k1 == K1_)                                                                      \
    return launch_impl<D_, R_, K1_>(g, cdev, x, y, Yc, sign, batch, stride, ycstride, s, nlaunch);

cudaError_t launch_op_apply(int d, int r, int k1, const LevelGeom& g, const OpConsts* cdev, const double* x, double* y,
                            double* Yc, double sign, int batch, long long stride, long long ycstride, cudaStream_t s,
                            int* nlaunch) {
  STGMG_OP_CASE(2, 2, 1)
  STGMG_OP_CASE(2, 2, 2)
  STGMG_OP_CASE(2, 2, 3)
  STGMG_OP_CASE(2, 3, 1)
  STGMG_OP_CASE(2, 3, 2)
  STGMG_OP_CASE(2, 3, 3)
  STGMG_OP_CASE(3, 2, 1)
  STGMG_OP_CASE(3, 2, 2)
  return cudaErrorNotSupported;
}

}  // namespace stgmg
