// on-device load assembly and initial data (sm_100a, fp64).
//   Load functionals (Def:LG) at the Radau nodes t_{n,b} = t_n + tau/2 (t_hat_b + 1) of a slab, scaled by
//   theta_b and placed in the slab layout: U slot (chi rows) theta_b F_gamma(t_{n,b}),
//   P slot (psi rows) theta_b G_gamma(t_{n,b}), V slot 0.  Homogeneous Dirichlet data (readings A26, A31), so only
//     * the body loads of the BASELINE manufactured solution u_i = S sin(2 pi t), p = S cos(2 pi t),
//       S = prod_a sin(pi x_a) (configs 0/1/3): f = rho d_tt u - div sigma(u) + alpha grad p (reading A8),
//       g = c0 d_t p + alpha div d_t u - div(K grad p), in closed form:
//         f_i = sin(2 pi t) [ (mu d pi^2 - 4 pi^2 rho) S - (lambda + mu) sum_j d_i d_j S ] + alpha cos(2 pi t) d_i S
//         g   = -2 pi c0 sin(2 pi t) S + cos(2 pi t) [ 2 pi alpha sum_j d_j S - sum_ij K_ij d_i d_j S ]
//       integrated with the (r+2)^d Gauss rule per cell (reading A10);
//     * the config-4 traction: + sin(pi t / 2) int_{x = hi} chi_{d-1} (reading A23), (r+2)^{d-1} face rule.
//   One thread per (cell, task): tasks 0..d-1 = U-slot component, task d = P slot; element results in the cell-major
//   layout of the 2D operator kernel, summed per node by gather_nodal_kernel (deterministic, no atomics).
// Initial data (reading A20): nodal interpolation of u(t0), v(t0) = d_t u(t0), p(t0) into the LAST Radau block of
// a slab vector (the block stgmg_slab_rhs reads as X_{n-1}); zero elsewhere.
#include "stgmg_internal.cuh"

namespace stgmg {

template <int D>
__device__ __forceinline__ void manufactured_fg(const LoadConsts& c, const double* x, double st, double ct,
                                                double* f, double& g) {
  constexpr double PI = 3.14159265358979323846;
  double sn[3], cs[3];
#pragma unroll
  for (int a = 0; a < D; ++a) sincospi(x[a], &sn[a], &cs[a]);
  double S = 1.0;
#pragma unroll
  for (int a = 0; a < D; ++a) S *= sn[a];
  double dS[3], ddS[3][3];
#pragma unroll
  for (int i = 0; i < D; ++i) {
    double p = PI * cs[i];
#pragma unroll
    for (int k = 0; k < D; ++k)
      if (k != i) p *= sn[k];
    dS[i] = p;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      if (i == j) {
        ddS[i][j] = -PI * PI * S;
      } else {
        double q = PI * PI * cs[i] * cs[j];
#pragma unroll
        for (int k = 0; k < D; ++k)
          if (k != i && k != j) q *= sn[k];
        ddS[i][j] = q;
      }
    }
  }
#pragma unroll
  for (int i = 0; i < D; ++i) {
    double sdd = 0.0;
#pragma unroll
    for (int j = 0; j < D; ++j) sdd += ddS[i][j];
    f[i] = st * ((c.mu * D * PI * PI - 4.0 * PI * PI * c.rho) * S - (c.lam + c.mu) * sdd) + c.alpha * ct * dS[i];
  }
  double sd = 0.0, kdd = 0.0;
#pragma unroll
  for (int i = 0; i < D; ++i) {
    sd += dS[i];
#pragma unroll
    for (int j = 0; j < D; ++j) kdd += c.K[i * 3 + j] * ddS[i][j];
  }
  g = -2.0 * PI * c.c0 * st * S + ct * (2.0 * PI * c.alpha * sd - kdd);
}

template <int D, int R, int K1>
__global__ void __launch_bounds__(128) load_cell_kernel(LevelGeom g, const LoadConsts* __restrict__ lc, int kind,
                                                        double tn, double tau, double* __restrict__ Yc) {
  constexpr int NQ1 = R + 2;                 // load quadrature points per axis (reading A10)
  constexpr int NQE = D == 3 ? (R + 1) * (R + 1) * (R + 1) : (R + 1) * (R + 1);
  constexpr int NPE = D == 3 ? R * R * R : R * R;
  constexpr int NE1 = 2 * D * NQE + NPE;
  constexpr int NPT = D == 3 ? NQ1 * NQ1 * NQ1 : NQ1 * NQ1;
  const LoadConsts c = *lc;
  const long long ncell = (long long)g.n[0] * g.n[1] * (D == 3 ? g.n[2] : 1);
  const long long cell = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const int task = blockIdx.y;               // 0..D-1: U-slot component, D: P slot
  if (cell >= ncell) return;
  int ci[3] = {(int)(cell % g.n[0]), (int)((cell / g.n[0]) % g.n[1]), D == 3 ? (int)(cell / ((long long)g.n[0] * g.n[1])) : 0};
  const bool pres = task == D;
  const int nloc = pres ? NPE : NQE;
  const int n1 = pres ? R : R + 1;
  const double vol = g.vol;
  pdl_wait();
  for (int b = 0; b < K1; ++b) {
    const double t = tn + 0.5 * tau * (c.that[b] + 1.0);
    double acc[NQE];
#pragma unroll
    for (int j = 0; j < NQE; ++j) acc[j] = 0.0;
    if (kind == 0) {   // manufactured body loads
      double st, ct;
      sincospi(2.0 * t, &st, &ct);
      for (int q = 0; q < NPT; ++q) {
        int qa[3] = {q % NQ1, (q / NQ1) % NQ1, D == 3 ? q / (NQ1 * NQ1) : 0};
        double x[3], w = vol;
#pragma unroll
        for (int a = 0; a < D; ++a) {
          x[a] = c.lo[a] + (ci[a] + c.xg[qa[a]]) * g.h[a];
          w *= c.wg[qa[a]];
        }
        double f[3], gg;
        manufactured_fg<D>(c, x, st, ct, f, gg);
        const double val = (pres ? gg : f[task]) * w;
        for (int j = 0; j < nloc; ++j) {
          int rem = j;
          double phi = val;
#pragma unroll
          for (int a = 0; a < D; ++a) {
            const int ja = rem % n1;
            rem /= n1;
            phi *= pres ? c.Bp[qa[a]][ja] : c.Bq[qa[a]][ja];
          }
          acc[j] += phi;
        }
      }
    } else if (kind == 1 && !pres && task == D - 1 && ci[0] == c.xhi_cell) {   // traction on x = hi, comp d-1
      double amp = sinpi(0.5 * t);
      constexpr int NF = D == 3 ? NQ1 * NQ1 : NQ1;
      for (int q = 0; q < NF; ++q) {
        int qa[3] = {0, q % NQ1, D == 3 ? q / NQ1 : 0};
        double w = vol / g.h[0] * amp;
#pragma unroll
        for (int a = 1; a < D; ++a) w *= c.wg[qa[a]];
        for (int j = 0; j < NQE; ++j) {
          int rem = j;
          double phi = w;
#pragma unroll
          for (int a = 0; a < D; ++a) {
            const int ja = rem % (R + 1);
            rem /= (R + 1);
            phi *= a == 0 ? c.Eq[1][ja] : c.Bq[qa[a]][ja];
          }
          acc[j] += phi;
        }
      }
    }
    // element rows of Radau node b: V slots zero, U slot component task / P slot scaled by theta_b
    const double th = c.theta[b];
    if (!pres) {
      for (int j = 0; j < NQE; ++j) {
        Yc[((long long)b * NE1 + task * NQE + j) * ncell + cell] = 0.0;                 // V slot (phi rows)
        Yc[((long long)b * NE1 + (D + task) * NQE + j) * ncell + cell] = th * acc[j];    // U slot (chi rows)
      }
    } else {
      for (int j = 0; j < NPE; ++j) Yc[((long long)b * NE1 + 2 * D * NQE + j) * ncell + cell] = th * acc[j];
    }
  }
}

// initial data into the last Radau block of x (zero elsewhere): V slot v(t0), U slot u(t0), P slot p(t0)
template <int D>
__global__ void initial_state_kernel(LevelGeom g, const LoadConsts* __restrict__ lc, int kind, double t0, int k1,
                                     double* __restrict__ x) {
  constexpr double PI = 3.14159265358979323846;
  const long long mu = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (mu >= g.N) return;
  pdl_wait();
  const int m = (int)(mu / g.block);
  const long long rem = mu - (long long)m * g.block;
  double val = 0.0;
  if (m == k1 - 1 && kind == 0) {
    const LoadConsts& c = *lc;
    const bool pres = rem >= 2 * g.R;
    const long long node = pres ? rem - 2 * g.R : rem % g.nq;
    const int slot = pres ? 2 * D : (int)(rem / g.nq);
    const int deg = pres ? c.r - 1 : c.r;
    long long t = node;
    double S = 1.0;
    for (int a = 0; a < D; ++a) {
      const int na = pres ? g.pn[a] : g.qn[a];
      const int i = (int)(t % na);
      t /= na;
      const int cc = i / deg, l = i - cc * deg;
      const double xa = c.lo[a] + ((double)cc + (pres ? c.gllp[l] : c.gllq[l])) * g.h[a];
      S *= sinpi(xa);
    }
    double st, ct;
    sincospi(2.0 * t0, &st, &ct);
    if (pres) val = S * ct;                       // p(t0)
    else if (slot < D) val = 2.0 * PI * S * ct;   // V slot: v(t0) = d_t u
    else val = S * st;                            // U slot: u(t0)
  }
  x[mu] = val;
}

// Energy helpers: y = 0 except the last Radau block built from x's last block (V, U, P) as
//   mode 0: (0, U, 0)   mode 1: (V, 0, P)   mode 2: (0, V, P)
__global__ void energy_place_kernel(LevelGeom g, int k1, const double* __restrict__ x, double* __restrict__ y, int mode) {
  const long long mu = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (mu >= g.N) return;
  pdl_wait();
  const int m = (int)(mu / g.block);
  const long long rem = mu - (long long)m * g.block;
  double v = 0.0;
  if (m == k1 - 1) {
    const long long o = (long long)m * g.block;
    const int slot = rem < g.R ? 0 : (rem < 2 * g.R ? 1 : 2);   // 0 = V, 1 = U, 2 = P
    if (mode == 0) v = slot == 1 ? x[mu] : 0.0;
    else if (mode == 1) v = slot == 1 ? 0.0 : x[mu];
    else v = slot == 1 ? x[o + (rem - g.R)] : (slot == 2 ? x[mu] : 0.0);
  }
  y[mu] = v;
}

cudaError_t launch_energy_place(const LevelGeom& g, int k1, const double* x, double* y, int mode, cudaStream_t s) {
  return launch_pdl(energy_place_kernel, dim3((unsigned)((g.N + 255) / 256)), dim3(256), 0, s, g, k1, x, y, mode);
}

// Goal quantities (Eq:DefGQ): per face cell, the (r+2)^{d-1}-point face integrals of
// u . n and p of the last Radau block (t_n); partial sums per cell, then one fixed-order reduction (deterministic).
template <int D, int R>
__global__ void face_integrals_kernel(LevelGeom g, const LoadConsts* __restrict__ lc, const double* __restrict__ x,
                                      int k1, int face, int c0, int c1, double* __restrict__ part) {
  constexpr int NQ1 = R + 2, NF = D == 3 ? NQ1 * NQ1 : NQ1;
  const int a = face >> 1, side = face & 1;
  // face cells: the other axes run over all cells (x restricted to the owned range [c0, c1) when a != 0)
  int n1 = 1, n2 = 1, ax1 = 0, ax2 = 0;
  {
    int k = 0;
    for (int b = 0; b < D; ++b)
      if (b != a) {
        if (k == 0) { ax1 = b; n1 = (b == 0 ? c1 - c0 : g.n[b]); } else { ax2 = b; n2 = g.n[b]; }
        ++k;
      }
  }
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n1 * n2) return;
  pdl_wait();
  const LoadConsts& c = *lc;
  int cell[3] = {0, 0, 0};
  cell[a] = side ? g.n[a] - 1 : 0;
  cell[ax1] = t % n1 + (ax1 == 0 ? c0 : 0);
  if (D == 3) cell[ax2] = t / n1;
  const double nrm = side ? 1.0 : -1.0;
  const long long o = (long long)(k1 - 1) * g.block;
  double bu = 0.0, bp = 0.0;
  for (int q = 0; q < NF; ++q) {
    const int qa[3] = {q % NQ1, q / NQ1, 0};
    double w = g.vol / g.h[a];
    int qq = 0;
    int qi[3] = {0, 0, 0};   // quadrature index along each in-face axis
    for (int b = 0; b < D; ++b) {
      if (b == a) continue;
      w *= c.wg[qa[qq]];
      qi[b] = qa[qq++];
    }
    double u = 0.0, p = 0.0;
    // Q_r nodes of the cell
    for (int j = 0; j < (D == 3 ? (R + 1) * (R + 1) * (R + 1) : (R + 1) * (R + 1)); ++j) {
      int rem = j;
      long long node = 0;
      double phi = 1.0;
      for (int b = 0; b < D; ++b) {
        const int jb = rem % (R + 1);
        rem /= (R + 1);
        node += (long long)(R * cell[b] + jb) * g.qs[b];
        phi *= b == a ? c.Eq[side][jb] : c.Bq[qi[b]][jb];
      }
      u += phi * x[o + g.R + (long long)a * g.nq + node];
    }
    for (int j = 0; j < (D == 3 ? R * R * R : R * R); ++j) {
      int rem = j;
      long long node = 0;
      double phi = 1.0;
      for (int b = 0; b < D; ++b) {
        const int jb = rem % R;
        rem /= R;
        node += (long long)((R - 1) * cell[b] + jb) * g.ps[b];
        // Q_{r-1} basis at the face point: endpoint value = Lagrange value at 0 / 1 (GLL nodes include both ends)
        phi *= b == a ? ((side ? (jb == R - 1) : (jb == 0)) ? 1.0 : 0.0) : c.Bp[qi[b]][jb];
      }
      p += phi * x[o + 2 * g.R + node];
    }
    bu += w * nrm * u;
    bp += w * p;
  }
  part[2 * t] = bu;
  part[2 * t + 1] = bp;
}

// out[0..1] = sum over the n partial pairs, fixed order (one block, strided partial sums + fixed tree)
__global__ void sum_pairs_kernel(const double* __restrict__ part, int n, double* __restrict__ out) {
  __shared__ double s0[256], s1[256];
  pdl_wait();
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < n; i += 256) {
    a += part[2 * i];
    b += part[2 * i + 1];
  }
  s0[threadIdx.x] = a;
  s1[threadIdx.x] = b;
  __syncthreads();
  for (int st = 128; st > 0; st >>= 1) {
    if (threadIdx.x < st) {
      s0[threadIdx.x] += s0[threadIdx.x + st];
      s1[threadIdx.x] += s1[threadIdx.x + st];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = s0[0];
    out[1] = s1[0];
  }
}

cudaError_t launch_face_integrals(int d, int r, int k1, const LevelGeom& g, const LoadConsts* lc, const double* x,
                                  int face, int c0, int c1, double* part, int nface_cells, double* out,
                                  cudaStream_t s) {
  const unsigned grid = (unsigned)((nface_cells + 127) / 128);
  cudaError_t e = cudaErrorNotSupported;
  if (d == 2 && r == 2) e = launch_pdl(face_integrals_kernel<2, 2>, dim3(grid), dim3(128), 0, s, g, lc, x, k1, face, c0, c1, part);
  if (d == 2 && r == 3) e = launch_pdl(face_integrals_kernel<2, 3>, dim3(grid), dim3(128), 0, s, g, lc, x, k1, face, c0, c1, part);
  if (d == 3 && r == 2) e = launch_pdl(face_integrals_kernel<3, 2>, dim3(grid), dim3(128), 0, s, g, lc, x, k1, face, c0, c1, part);
  if (d == 3 && r == 3) e = launch_pdl(face_integrals_kernel<3, 3>, dim3(grid), dim3(128), 0, s, g, lc, x, k1, face, c0, c1, part);
  if (e != cudaSuccess) return e;
  return launch_pdl(sum_pairs_kernel, dim3(1), dim3(256), 0, s, (const double*)part, nface_cells, out);
}

cudaError_t launch_load_cells(int d, int r, int k1, const LevelGeom& g, const LoadConsts* lc, int kind, double tn,
                              double tau, double* Yc, cudaStream_t s) {
  const long long ncell = (long long)g.n[0] * g.n[1] * (d == 3 ? g.n[2] : 1);
  const dim3 grid((unsigned)((ncell + 127) / 128), (unsigned)(d + 1));
#define STGMG_LOAD_CASE(D_, R_, K_)                                                                         \
  if (d == D_ && r == R_ && k1 == K_) return launch_pdl(load_cell_kernel<D_, R_, K_>, grid, dim3(128), 0, s, g, lc, \
                                                        kind, tn, tau, Yc);
  STGMG_LOAD_CASE(2, 2, 1) STGMG_LOAD_CASE(2, 2, 2) STGMG_LOAD_CASE(2, 2, 3)
  STGMG_LOAD_CASE(2, 3, 1) STGMG_LOAD_CASE(2, 3, 2) STGMG_LOAD_CASE(2, 3, 3)
  STGMG_LOAD_CASE(3, 2, 1) STGMG_LOAD_CASE(3, 2, 2)
#undef STGMG_LOAD_CASE
  return cudaErrorNotSupported;
}

cudaError_t launch_initial_state(int d, int k1, const LevelGeom& g, const LoadConsts* lc, int kind, double t0, double* x,
                                 cudaStream_t s) {
  const unsigned grid = (unsigned)((g.N + 255) / 256);
  if (d == 3) return launch_pdl(initial_state_kernel<3>, dim3(grid), dim3(256), 0, s, g, lc, kind, t0, k1, x);
  return launch_pdl(initial_state_kernel<2>, dim3(grid), dim3(256), 0, s, g, lc, kind, t0, k1, x);
}

}  // namespace stgmg
