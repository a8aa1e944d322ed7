// Shared pieces of the sum-factorised K1 kernels (op_apply.cu: generic warp-per-cell kernel used at setup and for
// K8; op3d.cu: the runtime 3D Q2 kernel): sizes, the warp-cooperative tensor contraction, and the Nitsche face terms
// of Def:A / Def:C / Def:B / Def:ab on Dirichlet boundary faces.
#pragma once
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

// Nitsche face terms of node b's rows (test slots V: none, U: chi, P: psi) on the Dirichlet faces bface[0..nbf) of
// one cell, accumulated into ye (element order).  Ub, Vb, Pb: the cell's nodal U_b, the velocity coupled into the
// p-equation (V_b, or sum_a T_ba U_a for DS), P_b.  qv: >= (3 D + D^2 + 1) NG^(D-1) doubles of warp scratch; t1, t2:
// contraction scratch.  Warp-cooperative.
template <int D, int R, int K1>
__device__ __forceinline__ void nitsche_faces(const OpConsts& c, const LevelGeom& g, const int* bface, int nbf,
                                              const double* Ub, const double* Vb, const double* Pb, double* ye,
                                              double* qv, double* t1, double* t2, const double* hinv, double th,
                                              int lane) {
  using T = Tr<D, R, K1>;
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
}

}  // namespace stgmg
