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
#include "op_common.cuh"

namespace stgmg {

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
  bool nz = false;
  for (int i = lane; i < T::NE; i += 32) {
    xe[i] = __ldg(x + gidx(i / T::NE1, i % T::NE1));
    nz = nz || xe[i] != 0.0;
  }
  // A cell whose inputs are all zero contributes exactly zero (the operator is linear): skip its work.  At setup the
  // kernel runs on batches of unit vectors (element and mini-level matrices, coarse operator), where all but the <= 2^d
  // cells around the unit vector's node are such cells.
  if (!__any_sync(0xffffffffu, nz)) {
    if (Yc) {
      long long plin = 0, vs = 1;
      for (int a = 0; a < D; ++a) {
        plin += (long long)(cell[a] + 1) * vs;
        vs *= g.n[a] + 1;
      }
      for (int i = lane; i < T::NE; i += 32) Yc[plin * T::NE + i] = 0.0;
    }
    return;
  }
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
    nitsche_faces<D, R, K1>(c, g, bface, nbf, Ub, Vb, Pb, ye, qv, t1, t2, hinv, th, lane);
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
  static PerDeviceOnce attr;
  attr.run([] {
    cudaFuncSetAttribute(op_apply_kernel<D, R, K1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
  });
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
