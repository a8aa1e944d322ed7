// the 3D L-shaped benchmark of Sec. 5.2 with the Q_r^d / P_{r-1}^disc pair (sm_100a, fp64).
//
//   Spaces  (Def:VhQh): u, v in continuous Q_r^3, p in the broken space P_{r-1}^disc (per-cell monomials
//           xi^a, |a| <= r-1, xi = 2 x_hat - 1; reading N3-R6).
//   Forms   (Def:ACB / Def:ab): A_gamma with Nitsche terms on Dirichlet faces and the directional form
//           a^d_gamma of Eq:BCd on directional faces; C with alpha <chi.n, q> on both; B_gamma = the
//           symmetric interior penalty option: volume term, -<{K grad q}.n, [psi]> - <[q], {K grad psi}.n> +
//           gamma/h_F <[q], [psi]> on interior faces and on the Dirichlet faces of p (reading N3-R3).
//   Domain  (readings N3-R1/R2): ([0,1] x [0,.5] U [0,.5] x [.5,1]) x [0,.5], 2^ref cells per cube edge;
//           u = 0 on y = 0, directional on x = 0, z = 0, z = .5, traction t_N on y = 1, free elsewhere; p = 0 on
//           y = 1, no flux elsewhere.
//
// This file holds (i) the host-side assembly of the level data at setup — slab operators A_l = T (x) calM +
// diag(theta) (x) calK as CSR (Problem 3.1, reading A5), prolongations (Q_r nodal interpolation and the
// exact restriction of a coarse cell polynomial to its children), vertex patches with their DoF lists
// (Eq:DefPlm, readings A11/A12), the averaging table, the slab-RHS coupling J, the
// traction load and the goal-quantity weights (Eq:DefGQ) — and (ii) the device kernels the hot path
// needs beyond the shared ones (CSR SpMV, averaging table, Gauss–Jordan K4, FGMRES): patch-matrix extraction from
// the CSR operator, the per-patch inverse application (K2u: one explicit inverse per patch, P:L486 — the L-shape
// has no patch classes) and the load / goal-quantity kernels.  Shares no code with the test oracle.
#include <algorithm>
#include <array>
#include <cmath>
#include <cstring>
#include <map>
#include <string>
#include <vector>

#include "../../include/stgmg.h"
#include "stgmg_internal.cuh"

namespace stgmg {

namespace {

constexpr double kTraction = 5.0e9;

struct CooEntry {
  long long r, c;
  double v;
};

// CSR from triplets: rows ascending, columns ascending, duplicates summed in insertion order (stable sort)
static LsHostCsr coo_to_csr(std::vector<CooEntry>& t, long long nrows) {
  std::stable_sort(t.begin(), t.end(), [](const CooEntry& a, const CooEntry& b) {
    return a.r < b.r || (a.r == b.r && a.c < b.c);
  });
  LsHostCsr m;
  m.rp.assign(nrows + 1, 0);
  for (size_t i = 0; i < t.size();) {
    size_t j = i;
    double s = 0.0;
    for (; j < t.size() && t[j].r == t[i].r && t[j].c == t[i].c; ++j) s += t[j].v;
    m.ci.push_back((int)t[i].c);
    m.v.push_back(s);
    m.rp[t[i].r + 1] += 1;
    i = j;
  }
  for (long long r = 0; r < nrows; ++r) m.rp[r + 1] += m.rp[r];
  std::vector<CooEntry>().swap(t);
  return m;
}

// 1D tables on [0,1]
static std::vector<double> gll_nodes(int r) {
  if (r == 2) return {0.0, 0.5, 1.0};
  const double a = 0.5 * (1.0 - 1.0 / std::sqrt(5.0));
  return {0.0, a, 1.0 - a, 1.0};   // r = 3
}

static void gauss01(int n, std::vector<double>& x, std::vector<double>& w) {
  x.assign(n, 0.0);
  w.assign(n, 0.0);
  auto legendre = [n](double z, double* dp) {   // P_n(z) and P_n'(z) by the three-term recurrence
    double p0 = 1.0, p1 = z;
    for (int k = 2; k <= n; ++k) {
      const double p2 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p0) / k;
      p0 = p1;
      p1 = p2;
    }
    *dp = n * (z * p1 - p0) / (z * z - 1.0);
    return p1;
  };
  for (int i = 0; i < n; ++i) {
    double z = std::cos(M_PI * (i + 0.75) / (n + 0.5)), dp = 0.0;   // Newton from the classical initial guess
    for (int it = 0; it < 40; ++it) z -= legendre(z, &dp) / dp;
    legendre(z, &dp);
    x[n - 1 - i] = 0.5 * (z + 1.0);
    w[n - 1 - i] = 1.0 / ((1.0 - z * z) * dp * dp);   // 2 / ((1 - z^2) P_n'^2) on [-1,1], halved for [0,1]
  }
}

static double lag(const std::vector<double>& nd, int j, double x) {
  double v = 1.0;
  for (size_t m = 0; m < nd.size(); ++m)
    if ((int)m != j) v *= (x - nd[m]) / (nd[j] - nd[m]);
  return v;
}

static double dlag(const std::vector<double>& nd, int j, double x) {
  double s = 0.0;
  for (size_t m = 0; m < nd.size(); ++m) {
    if ((int)m == j) continue;
    double t = 1.0 / (nd[j] - nd[m]);
    for (size_t q = 0; q < nd.size(); ++q)
      if ((int)q != j && q != m) t *= (x - nd[q]) / (nd[j] - nd[q]);
    s += t;
  }
  return s;
}

struct Exps {
  std::vector<std::array<int, 3>> e;
};

// P_deg monomial exponents ordered by total degree, then x before y before z (reading N3-R6)
static Exps p_exps(int deg) {
  Exps ex;
  for (int t = 0; t <= deg; ++t) {
    std::vector<std::array<int, 3>> lvl;
    for (int az = 0; az <= t; ++az)
      for (int ay = 0; ay <= t - az; ++ay) {
        const int ax = t - ay - az;
        lvl.push_back({ax, ay, az});
      }
    // order within a degree: (a_z, a_y, a_x) ascending reversed -> x-heavy first
    std::sort(lvl.begin(), lvl.end(), [](const std::array<int, 3>& a, const std::array<int, 3>& b) {
      if (a[2] != b[2]) return a[2] < b[2];
      if (a[1] != b[1]) return a[1] < b[1];
      return a[0] < b[0];
    });
    for (auto& a : lvl) ex.e.push_back(a);
  }
  return ex;
}

static double ipw(double x, int n) {
  double v = 1.0;
  for (int i = 0; i < n; ++i) v *= x;
  return v;
}

// Basis values / gradients at a reference point xh in [0,1]^3 of a cell of side h.
struct BasisAt {
  std::vector<double> q, p;                 // values
  std::vector<std::array<double, 3>> gq, gp;  // physical gradients
};

static BasisAt eval_basis(const std::vector<double>& nd, const Exps& ex, const double xh[3], double h) {
  const int n1 = (int)nd.size(), nb = n1 * n1 * n1;
  BasisAt B;
  B.q.resize(nb);
  B.gq.resize(nb);
  double L[3][4], D[3][4];
  for (int a = 0; a < 3; ++a)
    for (int j = 0; j < n1; ++j) {
      L[a][j] = lag(nd, j, xh[a]);
      D[a][j] = dlag(nd, j, xh[a]) / h;
    }
  for (int k = 0; k < n1; ++k)
    for (int j = 0; j < n1; ++j)
      for (int i = 0; i < n1; ++i) {
        const int J = i + n1 * (j + n1 * k);
        B.q[J] = L[0][i] * L[1][j] * L[2][k];
        B.gq[J] = {D[0][i] * L[1][j] * L[2][k], L[0][i] * D[1][j] * L[2][k], L[0][i] * L[1][j] * D[2][k]};
      }
  const double xi[3] = {2.0 * xh[0] - 1.0, 2.0 * xh[1] - 1.0, 2.0 * xh[2] - 1.0};
  B.p.resize(ex.e.size());
  B.gp.resize(ex.e.size());
  for (size_t s = 0; s < ex.e.size(); ++s) {
    const auto& a = ex.e[s];
    B.p[s] = ipw(xi[0], a[0]) * ipw(xi[1], a[1]) * ipw(xi[2], a[2]);
    for (int b = 0; b < 3; ++b) {
      double g = 0.0;
      if (a[b] > 0) {
        g = a[b] * ipw(xi[b], a[b] - 1) * 2.0 / h;
        for (int c = 0; c < 3; ++c)
          if (c != b) g *= ipw(xi[c], a[c]);
      }
      B.gp[s][b] = g;
    }
  }
  return B;
}

struct Quad {
  std::vector<std::array<double, 3>> x;   // reference points
  std::vector<double> w;                  // weights incl. measure
};

static Quad volume_quad(int n, double h) {
  std::vector<double> x, w;
  gauss01(n, x, w);
  Quad Q;
  for (int k = 0; k < n; ++k)
    for (int j = 0; j < n; ++j)
      for (int i = 0; i < n; ++i) {
        Q.x.push_back({x[i], x[j], x[k]});
        Q.w.push_back(w[i] * w[j] * w[k] * h * h * h);
      }
  return Q;
}

static Quad face_quad(int n, double h, int f) {
  std::vector<double> x, w;
  gauss01(n, x, w);
  const int a = f / 2, s = f % 2;
  Quad Q;
  for (int j = 0; j < n; ++j)
    for (int i = 0; i < n; ++i) {
      std::array<double, 3> p;
      int t = 0;
      const double uv[2] = {x[i], x[j]};
      for (int b = 0; b < 3; ++b) p[b] = (b == a) ? (double)s : uv[t++];
      Q.x.push_back(p);
      Q.w.push_back(w[i] * w[j] * h * h);
    }
  return Q;
}

// Element-local matrices of a cube of side h.  Vector index (c, J) -> c nbq + J; pressure index s.  M[test][trial].
struct ElemMats {
  int nbq = 0, npc = 0;
  std::vector<double> Mq, Mp, A, C, B;   // nbq^2, npc^2, (3nbq)^2, npc x 3nbq, npc^2
};

struct Forms {
  int r = 2;
  double h = 1.0, hF = 1.0, hD = 1.0, hP = 1.0;   // hD: directional faces; hP: SIP (p) faces
  double lam = 1, mu = 1, alpha = 1, rho = 1, c0 = 1, ga = 1, gb = 1, K[3][3] = {{0}};
  std::vector<double> nd;
  Exps ex;
  int nbq = 0, npc = 0;

  ElemMats volume() const {
    ElemMats E;
    E.nbq = nbq;
    E.npc = npc;
    const int nv = 3 * nbq;
    E.Mq.assign(nbq * nbq, 0.0);
    E.Mp.assign(npc * npc, 0.0);
    E.A.assign((size_t)nv * nv, 0.0);
    E.C.assign((size_t)npc * nv, 0.0);
    E.B.assign(npc * npc, 0.0);
    const Quad Q = volume_quad(r + 1, h);
    for (size_t q = 0; q < Q.w.size(); ++q) {
      const double xh[3] = {Q.x[q][0], Q.x[q][1], Q.x[q][2]};
      const BasisAt Bq = eval_basis(nd, ex, xh, h);
      const double w = Q.w[q];
      for (int I = 0; I < nbq; ++I)
        for (int J = 0; J < nbq; ++J) {
          E.Mq[I * nbq + J] += w * Bq.q[I] * Bq.q[J];
          const auto& gI = Bq.gq[I];
          const auto& gJ = Bq.gq[J];
          const double dot = gI[0] * gJ[0] + gI[1] * gJ[1] + gI[2] * gJ[2];
          for (int c = 0; c < 3; ++c)
            for (int d = 0; d < 3; ++d) {
              // sigma(phi_J e_d) : eps(phi_I e_c) = lam d_c I d_d J + mu d_d I d_c J + mu delta_cd grad I . grad J
              double v = lam * gI[c] * gJ[d] + mu * gI[d] * gJ[c];
              if (c == d) v += mu * dot;
              E.A[(size_t)(c * nbq + I) * nv + d * nbq + J] += w * v;
            }
        }
      for (int s = 0; s < npc; ++s) {
        for (int J = 0; J < nbq; ++J)
          for (int d = 0; d < 3; ++d) E.C[(size_t)s * nv + d * nbq + J] += -alpha * w * Bq.gq[J][d] * Bq.p[s];
        for (int t = 0; t < npc; ++t) {
          E.Mp[s * npc + t] += w * Bq.p[s] * Bq.p[t];
          double kg = 0.0;
          for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) kg += Bq.gp[s][a] * K[a][b] * Bq.gp[t][b];
          E.B[s * npc + t] += w * kg;   // symmetric K: <K grad xi_t, grad xi_s>
        }
      }
    }
    return E;
  }

  // Dirichlet (kind 0: Def:A / Def:agam) or directional (kind 1: Eq:BCd, a^d_gamma) face f: A and C parts
  void face_u(int f, int kind, std::vector<double>& A, std::vector<double>& C) const {
    const int nv = 3 * nbq;
    A.assign((size_t)nv * nv, 0.0);
    C.assign((size_t)npc * nv, 0.0);
    const int fa = f / 2;
    const double n[3] = {fa == 0 ? (f % 2 ? 1.0 : -1.0) : 0.0, fa == 1 ? (f % 2 ? 1.0 : -1.0) : 0.0,
                         fa == 2 ? (f % 2 ? 1.0 : -1.0) : 0.0};
    const double pen = ga / (kind == 0 ? hF : hD);
    const Quad Q = face_quad(r + 1, h, f);
    for (size_t q = 0; q < Q.w.size(); ++q) {
      const double xh[3] = {Q.x[q][0], Q.x[q][1], Q.x[q][2]};
      const BasisAt Bq = eval_basis(nd, ex, xh, h);
      const double w = Q.w[q];
      for (int I = 0; I < nbq; ++I) {
        const auto& gI = Bq.gq[I];
        const double dnI = gI[0] * n[0] + gI[1] * n[1] + gI[2] * n[2];
        for (int J = 0; J < nbq; ++J) {
          const auto& gJ = Bq.gq[J];
          const double dnJ = gJ[0] * n[0] + gJ[1] * n[1] + gJ[2] * n[2];
          const double pI = Bq.q[I], pJ = Bq.q[J];
          for (int c = 0; c < 3; ++c)
            for (int d = 0; d < 3; ++d) {
              double v;
              if (kind == 0) {
                // -(sigma(u) n)_c phi_I - phi_J (sigma(v) n)_d + pen delta_cd phi_I phi_J, u = phi_J e_d, v = phi_I e_c
                const double snu = lam * gJ[d] * n[c] + mu * ((c == d ? dnJ : 0.0) + gJ[c] * n[d]);
                const double snv = lam * gI[c] * n[d] + mu * ((c == d ? dnI : 0.0) + gI[d] * n[c]);
                v = -snu * pI - snv * pJ + (c == d ? pen * pI * pJ : 0.0);
              } else {
                // -(sigma(u)n.n)(v.n) - (u.n)(sigma(v)n.n) + pen (u.n)(v.n)
                const double snnu = lam * gJ[d] + 2.0 * mu * n[d] * dnJ;
                const double snnv = lam * gI[c] + 2.0 * mu * n[c] * dnI;
                v = -snnu * pI * n[c] - pJ * n[d] * snnv + pen * pJ * n[d] * pI * n[c];
              }
              A[(size_t)(c * nbq + I) * nv + d * nbq + J] += w * v;
            }
        }
      }
      for (int s = 0; s < npc; ++s)
        for (int J = 0; J < nbq; ++J)
          for (int d = 0; d < 3; ++d) C[(size_t)s * nv + d * nbq + J] += alpha * w * Bq.q[J] * n[d] * Bq.p[s];
    }
  }

  // SIP on a Dirichlet face of p: -<K grad q.n, psi> - <q, K grad psi.n> + gamma/h_F <q, psi>
  std::vector<double> face_p_dir(int f) const {
    std::vector<double> B(npc * npc, 0.0);
    const int fa = f / 2;
    double n[3] = {0, 0, 0};
    n[fa] = f % 2 ? 1.0 : -1.0;
    const double pen = gb / hP;
    const Quad Q = face_quad(r + 1, h, f);
    for (size_t q = 0; q < Q.w.size(); ++q) {
      const double xh[3] = {Q.x[q][0], Q.x[q][1], Q.x[q][2]};
      const BasisAt Bq = eval_basis(nd, ex, xh, h);
      for (int s = 0; s < npc; ++s) {
        double kns = 0.0;
        for (int a = 0; a < 3; ++a)
          for (int b = 0; b < 3; ++b) kns += n[a] * K[a][b] * Bq.gp[s][b];
        for (int t = 0; t < npc; ++t) {
          double knt = 0.0;
          for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) knt += n[a] * K[a][b] * Bq.gp[t][b];
          // test s, trial t
          B[s * npc + t] += Q.w[q] * (-knt * Bq.p[s] - Bq.p[t] * kns + pen * Bq.p[t] * Bq.p[s]);
        }
      }
    }
    return B;
  }

  // SIP on an interior face normal to axis a between K- (lower) and K+ = K- + e_a; n = e_a (outward of K-),
  // [w] = w- - w+.  Blocks Bf[i][j] (test side i, trial side j; 0 = K-, 1 = K+), each npc x npc.
  void face_p_int(int a, std::vector<double> Bf[2][2]) const {
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 2; ++j) Bf[i][j].assign(npc * npc, 0.0);
    double n[3] = {0, 0, 0};
    n[a] = 1.0;
    const double pen = gb / hP, sg[2] = {1.0, -1.0};
    const Quad Qm = face_quad(r + 1, h, 2 * a + 1), Qp = face_quad(r + 1, h, 2 * a);
    for (size_t q = 0; q < Qm.w.size(); ++q) {
      const double xm[3] = {Qm.x[q][0], Qm.x[q][1], Qm.x[q][2]};
      const double xp[3] = {Qp.x[q][0], Qp.x[q][1], Qp.x[q][2]};
      const BasisAt S[2] = {eval_basis(nd, ex, xm, h), eval_basis(nd, ex, xp, h)};
      std::vector<double> kn[2];
      for (int side = 0; side < 2; ++side) {
        kn[side].assign(npc, 0.0);
        for (int s = 0; s < npc; ++s)
          for (int b = 0; b < 3; ++b) kn[side][s] += K[a][b] * S[side].gp[s][b];
      }
      for (int i = 0; i < 2; ++i)
        for (int j = 0; j < 2; ++j)
          for (int s = 0; s < npc; ++s)
            for (int t = 0; t < npc; ++t) {
              // -{K grad q}.n [psi] - [q] {K grad psi}.n + pen [q][psi];  q = trial t on side j, psi = test s on i
              const double v = -0.5 * kn[j][t] * sg[i] * S[i].p[s] - sg[j] * S[j].p[t] * 0.5 * kn[i][s] +
                               pen * sg[i] * sg[j] * S[j].p[t] * S[i].p[s];
              Bf[i][j][s * npc + t] += Qm.w[q] * v;
            }
    }
  }
};

enum { UB_DIRICHLET = 0, UB_DIRECTIONAL = 1, UB_FREE = 2, UB_TRACTION = 3 };

struct LGrid {
  int ref = 0, r = 2, k1 = 2, N = 1;
  int n[3] = {0, 0, 0};
  double h = 1.0;
  std::vector<int> cid;         // structured cell -> active id or -1
  std::vector<std::array<int, 3>> cells;
  std::vector<int> qmap;        // structured Q node -> compact or -1
  int nq = 0, npc = 0, np = 0;
  long long block = 0, ndof = 0;
  int qs[3] = {1, 1, 1};        // structured Q node strides
  std::vector<int> cellq;       // ncell x nbq compact Q nodes

  bool active(int i, int j, int l) const {
    if (i < 0 || j < 0 || l < 0 || i >= n[0] || j >= n[1] || l >= n[2]) return false;
    return !(i >= N && j >= N);
  }
  int cell_id(int i, int j, int l) const { return active(i, j, l) ? cid[i + n[0] * (j + n[1] * l)] : -1; }
  long long off_v(int m, int c) const { return (long long)m * block + (long long)c * nq; }
  long long off_u(int m, int c) const { return (long long)m * block + 3LL * nq + (long long)c * nq; }
  long long off_p(int m) const { return (long long)m * block + 6LL * nq; }

  void build(int ref_, int r_, int k1_, int npc_) {
    ref = ref_;
    r = r_;
    k1 = k1_;
    N = 1 << ref;
    n[0] = 2 * N;
    n[1] = 2 * N;
    n[2] = N;
    h = 0.5 / N;
    cid.assign((size_t)n[0] * n[1] * n[2], -1);
    for (int l = 0; l < n[2]; ++l)
      for (int j = 0; j < n[1]; ++j)
        for (int i = 0; i < n[0]; ++i)
          if (active(i, j, l)) {
            cid[i + n[0] * (j + n[1] * l)] = (int)cells.size();
            cells.push_back({i, j, l});
          }
    const int qn[3] = {r * n[0] + 1, r * n[1] + 1, r * n[2] + 1};
    qs[0] = 1;
    qs[1] = qn[0];
    qs[2] = qn[0] * qn[1];
    std::vector<char> act((size_t)qn[0] * qn[1] * qn[2], 0);
    for (auto& c : cells)
      for (int z = 0; z <= r; ++z)
        for (int y = 0; y <= r; ++y)
          for (int x = 0; x <= r; ++x) act[(r * c[0] + x) + qs[1] * (r * c[1] + y) + qs[2] * (r * c[2] + z)] = 1;
    qmap.assign(act.size(), -1);
    nq = 0;
    for (size_t i = 0; i < act.size(); ++i)
      if (act[i]) qmap[i] = nq++;
    npc = npc_;
    np = npc * (int)cells.size();
    block = 6LL * nq + np;
    ndof = (long long)k1 * block;
    const int nbq = (r + 1) * (r + 1) * (r + 1);
    cellq.resize(cells.size() * nbq);
    for (size_t c = 0; c < cells.size(); ++c)
      for (int z = 0; z <= r; ++z)
        for (int y = 0; y <= r; ++y)
          for (int x = 0; x <= r; ++x)
            cellq[c * nbq + x + (r + 1) * (y + (r + 1) * z)] =
                qmap[(r * cells[c][0] + x) + qs[1] * (r * cells[c][1] + y) + qs[2] * (r * cells[c][2] + z)];
  }

  // boundary part of u on face f of cell c (a boundary face) — reading N3-R2
  int u_bc(const std::array<int, 3>& c, int f) const {
    const int a = f / 2, s = f % 2;
    if (a == 1 && s == 0) return UB_DIRICHLET;
    if (a == 0 && s == 0) return UB_DIRECTIONAL;
    if (a == 2) return UB_DIRECTIONAL;
    if (a == 1 && s == 1 && c[1] == n[1] - 1) return UB_TRACTION;
    return UB_FREE;
  }
  bool p_dir(const std::array<int, 3>& c, int f) const { return f == 3 && c[1] == n[1] - 1; }
  int neighbour(const std::array<int, 3>& c, int f) const {
    int o[3] = {c[0], c[1], c[2]};
    o[f / 2] += (f % 2) ? 1 : -1;
    return cell_id(o[0], o[1], o[2]);
  }
};

}  // namespace

int lshape_build_host(int ref_coarse, int levels, int r, int k, const OpConsts& oc, int hf_mode, LsHost& out,
                      std::string& err) {
  const bool hf_edge = hf_mode == 1;
  if (r != 2 && r != 3) { err = "L-shape: r must be 2 or 3"; return STGMG_ENOTSUP; }
  if (k < 0 || k + 1 > kMaxK1) { err = "L-shape: k out of range"; return STGMG_ENOTSUP; }
  const int k1 = k + 1;
  const Exps ex = p_exps(r - 1);
  const int npc = (int)ex.e.size(), nbq = (r + 1) * (r + 1) * (r + 1), nv = 3 * nbq;
  std::vector<LGrid> G(levels);
  for (int l = 0; l < levels; ++l) G[l].build(ref_coarse + l, r, k1, npc);
  out.lev.assign(levels, LsLevelHost());
  // temporal constants (T[b][a], theta_b, chi_b(-1)) are those of the structured path (make_consts)
  const double* T = &oc.T[0][0];
  auto Tba = [&](int b, int a) { return T[b * kMaxK1 + a]; };
  for (int l = 0; l < levels; ++l) {
    const LGrid& g = G[l];
    LsLevelHost& Lh = out.lev[l];
    Lh.ref = g.ref;
    Lh.N = g.ndof;
    Lh.nq = g.nq;
    Lh.np = g.np;
    Lh.ncell = (int)g.cells.size();
    Forms F;
    F.r = r;
    F.h = g.h;
    // |K|_d (reading A6 / N3-R4; the SIP average on a uniform mesh), or the edge length h (STGMG_HF_EDGE)
    F.hF = hf_edge ? g.h : g.h * g.h * g.h;
    if (hf_mode == 3) {   // mode 3: the FINE level's |K|_d on every level (coarse operators = Galerkin products, pin L5)
      const double hf = G[levels - 1].h;
      F.hF = hf * hf * hf;
    }
    F.hD = (hf_edge || hf_mode == 2) ? g.h : F.hF;   // mode 2: a^d_gamma with the literal h^-1 of P:L778
    F.hP = F.hF;
    // experiments on the grid robustness of Table 4: 4 = h^3 for u, h for the SIP faces of p;
    // 5 = h for u, h^3 for p; 6 = the face measure h^2 for both
    if (hf_mode == 4) { F.hF = F.hD = g.h * g.h * g.h; F.hP = g.h; }
    if (hf_mode == 5) { F.hF = F.hD = g.h; F.hP = g.h * g.h * g.h; }
    if (hf_mode == 6) { F.hF = F.hD = F.hP = g.h * g.h; }
    F.lam = oc.lam;
    F.mu = oc.mu;
    F.alpha = oc.alpha;
    F.rho = oc.rho;
    F.c0 = oc.c0;
    F.ga = oc.gamma_a;
    F.gb = oc.gamma_b;
    for (int a = 0; a < 3; ++a)
      for (int b = 0; b < 3; ++b) F.K[a][b] = oc.K[a * 3 + b];
    F.nd = gll_nodes(r);
    F.ex = ex;
    F.nbq = nbq;
    F.npc = npc;
    const ElemMats E = F.volume();
    std::map<int, std::pair<std::vector<double>, std::vector<double>>> fu;   // (f, kind) -> (A, C)
    std::map<int, std::vector<double>> fpd;
    std::vector<double> fpi[3][2][2];
    for (int a = 0; a < 3; ++a) F.face_p_int(a, fpi[a]);
    // spatial matrices: Mq (nq), A (3nq), C (np x 3nq), B (np), Mp (np) — triplets per cell and face
    std::vector<CooEntry> tM, tA, tC, tB, tP;
    const int nc = (int)g.cells.size();
    std::vector<long long> vd(nv);
    for (int c = 0; c < nc; ++c) {
      const auto& cc = g.cells[c];
      const int* q = &g.cellq[(size_t)c * nbq];
      for (int comp = 0; comp < 3; ++comp)
        for (int J = 0; J < nbq; ++J) vd[comp * nbq + J] = (long long)comp * g.nq + q[J];
      const long long p0 = (long long)c * npc;
      for (int I = 0; I < nbq; ++I)
        for (int J = 0; J < nbq; ++J) tM.push_back({q[I], q[J], E.Mq[I * nbq + J]});
      for (int s = 0; s < npc; ++s)
        for (int t = 0; t < npc; ++t) tP.push_back({p0 + s, p0 + t, E.Mp[s * npc + t]});
      std::vector<double> A = E.A, C = E.C, B = E.B;
      for (int f = 0; f < 6; ++f) {
        const int nb = g.neighbour(cc, f);
        if (nb >= 0) {
          if (f % 2 == 1) {
            const long long pn = (long long)nb * npc, side[2] = {p0, pn};
            for (int i = 0; i < 2; ++i)
              for (int j = 0; j < 2; ++j)
                for (int s = 0; s < npc; ++s)
                  for (int t = 0; t < npc; ++t) tB.push_back({side[i] + s, side[j] + t, fpi[f / 2][i][j][s * npc + t]});
          }
          continue;
        }
        const int ub = g.u_bc(cc, f);
        if (ub == UB_DIRICHLET || ub == UB_DIRECTIONAL) {
          const int key = f * 2 + ub;
          if (!fu.count(key)) F.face_u(f, ub, fu[key].first, fu[key].second);
          const auto& AC = fu[key];
          for (size_t i = 0; i < A.size(); ++i) A[i] += AC.first[i];
          for (size_t i = 0; i < C.size(); ++i) C[i] += AC.second[i];
        }
        if (g.p_dir(cc, f)) {
          if (!fpd.count(f)) fpd[f] = F.face_p_dir(f);
          const auto& Bf = fpd[f];
          for (size_t i = 0; i < B.size(); ++i) B[i] += Bf[i];
        }
      }
      for (int I = 0; I < nv; ++I)
        for (int J = 0; J < nv; ++J) tA.push_back({vd[I], vd[J], A[(size_t)I * nv + J]});
      for (int s = 0; s < npc; ++s) {
        for (int J = 0; J < nv; ++J) tC.push_back({p0 + s, vd[J], C[(size_t)s * nv + J]});
        for (int t = 0; t < npc; ++t) tB.push_back({p0 + s, p0 + t, B[s * npc + t]});
      }
    }
    LsHostCsr Mq = coo_to_csr(tM, g.nq), Mp = coo_to_csr(tP, g.np), SA = coo_to_csr(tA, 3LL * g.nq),
              SC = coo_to_csr(tC, g.np), SB = coo_to_csr(tB, g.np);
    // C^T (3nq x np)
    std::vector<CooEntry> tCT;
    for (int s = 0; s < g.np; ++s)
      for (int e = SC.rp[s]; e < SC.rp[s + 1]; ++e) tCT.push_back({SC.ci[e], s, SC.v[e]});
    LsHostCsr SCT = coo_to_csr(tCT, 3LL * g.nq);
    // slab operator rows (Problem 3.1): row b, test slot; columns a, trial slot
    std::vector<CooEntry> tS;
    for (int b = 0; b < k1; ++b) {
      const double th = oc.theta[b];
      for (int comp = 0; comp < 3; ++comp)
        for (int i = 0; i < g.nq; ++i) {
          const long long rv = g.off_v(b, comp) + i, ru = g.off_u(b, comp) + i;
          for (int e = Mq.rp[i]; e < Mq.rp[i + 1]; ++e) {
            const int j = Mq.ci[e];
            const double m = oc.rho * Mq.v[e];
            tS.push_back({rv, g.off_v(b, comp) + j, -th * m});                      // [phi_b, V_b] = -theta M_rho
            for (int a = 0; a < k1; ++a) {
              tS.push_back({rv, g.off_u(a, comp) + j, Tba(b, a) * m});               // [phi_b, U_a] = T_ba M_rho
              tS.push_back({ru, g.off_v(a, comp) + j, Tba(b, a) * m});               // [chi_b, V_a] = T_ba M_rho
            }
          }
          const long long rowA = (long long)comp * g.nq + i;
          for (int e = SA.rp[rowA]; e < SA.rp[rowA + 1]; ++e)
            tS.push_back({ru, (long long)b * g.block + 3LL * g.nq + SA.ci[e], th * SA.v[e]});   // theta A_gamma
          for (int e = SCT.rp[rowA]; e < SCT.rp[rowA + 1]; ++e)
            tS.push_back({ru, g.off_p(b) + SCT.ci[e], th * SCT.v[e]});                         // theta C^T
        }
      for (int s = 0; s < g.np; ++s) {
        const long long rp_ = g.off_p(b) + s;
        for (int e = SC.rp[s]; e < SC.rp[s + 1]; ++e) tS.push_back({rp_, g.off_v(b, 0) + SC.ci[e], -th * SC.v[e]});
        for (int e = Mp.rp[s]; e < Mp.rp[s + 1]; ++e)
          for (int a = 0; a < k1; ++a) tS.push_back({rp_, g.off_p(a) + Mp.ci[e], Tba(b, a) * oc.c0 * Mp.v[e]});
        for (int e = SB.rp[s]; e < SB.rp[s + 1]; ++e) tS.push_back({rp_, g.off_p(b) + SB.ci[e], th * SB.v[e]});
      }
    }
    if (g.ndof >= (1LL << 31)) { err = "L-shape level too large for 32-bit CSR"; return STGMG_ENOTSUP; }
    Lh.A = coo_to_csr(tS, g.ndof);
    if (l == levels - 1) {   // fine level: slab-RHS coupling, traction load, goal weights
      std::vector<CooEntry> tJ;
      const int kk = k1 - 1;
      for (int b = 0; b < k1; ++b) {
        const double cb = oc.chim1[b];
        for (int comp = 0; comp < 3; ++comp)
          for (int i = 0; i < g.nq; ++i)
            for (int e = Mq.rp[i]; e < Mq.rp[i + 1]; ++e) {
              const double m = cb * oc.rho * Mq.v[e];
              tJ.push_back({g.off_v(b, comp) + i, g.off_u(kk, comp) + Mq.ci[e], m});   // phi_b: M_rho U^{n-1}
              tJ.push_back({g.off_u(b, comp) + i, g.off_v(kk, comp) + Mq.ci[e], m});   // chi_b: M_rho V^{n-1}
            }
        for (int s = 0; s < g.np; ++s)
          for (int e = Mp.rp[s]; e < Mp.rp[s + 1]; ++e)
            tJ.push_back({g.off_p(b) + s, g.off_p(kk) + Mp.ci[e], cb * oc.c0 * Mp.v[e]});   // psi_b: M_c P^{n-1}
      }
      out.J = coo_to_csr(tJ, g.ndof);
      // traction: -<t_N, chi>_{Gamma^N_u}, (r+2)-point Gauss per face axis (reading A10), y component
      out.fN.assign(3 * (size_t)g.nq, 0.0);
      out.wu.assign(g.nq, 0.0);
      out.wp.assign(g.np, 0.0);
      const Quad Qt = face_quad(r + 2, g.h, 3), Qg = face_quad(r + 1, g.h, 1);
      for (int c = 0; c < nc; ++c) {
        const auto& cc = g.cells[c];
        const int* q = &g.cellq[(size_t)c * nbq];
        if (cc[1] == g.n[1] - 1 && g.u_bc(cc, 3) == UB_TRACTION) {
          for (size_t iq = 0; iq < Qt.w.size(); ++iq) {
            const double xh[3] = {Qt.x[iq][0], Qt.x[iq][1], Qt.x[iq][2]};
            const BasisAt Bq = eval_basis(F.nd, ex, xh, g.h);
            const double x = (cc[0] + xh[0]) * g.h, z = (cc[2] + xh[2]) * g.h;
            const double tn = kTraction * (32.0 * x * z - 18.0 * x - 16.0 * z + 10.0);
            for (int J = 0; J < nbq; ++J) out.fN[(size_t)g.nq + q[J]] += -tn * Bq.q[J] * Qt.w[iq];
          }
        }
        if (cc[0] == g.n[0] - 1) {   // Gamma_m = {1} x (0,.5) x (0,.5), n = e_x
          for (size_t iq = 0; iq < Qg.w.size(); ++iq) {
            const double xh[3] = {Qg.x[iq][0], Qg.x[iq][1], Qg.x[iq][2]};
            const BasisAt Bq = eval_basis(F.nd, ex, xh, g.h);
            for (int J = 0; J < nbq; ++J) out.wu[q[J]] += Bq.q[J] * Qg.w[iq];
            for (int s = 0; s < npc; ++s) out.wp[(size_t)c * npc + s] += Bq.p[s] * Qg.w[iq];
          }
        }
      }
    }
    if (l >= 1) {
      // prolongation level l-1 -> l (rows: this level)
      const LGrid& gc = G[l - 1];
      std::vector<CooEntry> tQ;
      const std::vector<double> nd = gll_nodes(r);
      const int qn[3] = {r * g.n[0] + 1, r * g.n[1] + 1, r * g.n[2] + 1};
      for (int z = 0; z < qn[2]; ++z)
        for (int y = 0; y < qn[1]; ++y)
          for (int x = 0; x < qn[0]; ++x) {
            const int fi = g.qmap[x + g.qs[1] * y + g.qs[2] * z];
            if (fi < 0) continue;
            const int idx[3] = {x, y, z};
            int cn[3][4];
            double cw[3][4];
            int cnt[3];
            for (int a = 0; a < 3; ++a) {
              const int cf = std::min(idx[a] / r, g.n[a] - 1), lf = idx[a] - r * cf, ccell = cf / 2;
              const double xh = 0.5 * ((cf % 2) + nd[lf]);
              cnt[a] = 0;
              for (int j = 0; j <= r; ++j) {
                const double w = lag(nd, j, xh);
                if (w == 0.0) continue;
                cn[a][cnt[a]] = r * ccell + j;
                cw[a][cnt[a]] = w;
                ++cnt[a];
              }
            }
            for (int k2 = 0; k2 < cnt[2]; ++k2)
              for (int j2 = 0; j2 < cnt[1]; ++j2)
                for (int i2 = 0; i2 < cnt[0]; ++i2) {
                  const int ci = gc.qmap[cn[0][i2] + gc.qs[1] * cn[1][j2] + gc.qs[2] * cn[2][k2]];
                  if (ci < 0) { err = "L-shape transfer reaches an inactive coarse node"; return STGMG_EINVAL; }
                  tQ.push_back({fi, ci, cw[0][i2] * cw[1][j2] * cw[2][k2]});
                }
          }
      LsHostCsr PQ = coo_to_csr(tQ, g.nq);
      // P_{r-1}^disc: child coefficient of xi_f^beta in the parent monomial xi_c^alpha, xi_c = xi_f / 2 + sg / 2
      auto binom = [](int n_, int k_) {
        double v = 1.0;
        for (int i = 1; i <= k_; ++i) v = v * (n_ - k_ + i) / i;
        return v;
      };
      std::vector<CooEntry> tPP;
      for (int c = 0; c < nc; ++c) {
        const auto& cc = g.cells[c];
        const int pc = gc.cell_id(cc[0] / 2, cc[1] / 2, cc[2] / 2);
        for (int i = 0; i < npc; ++i) {
          const auto& be = ex.e[i];
          for (int j = 0; j < npc; ++j) {
            const auto& al = ex.e[j];
            double v = 1.0;
            for (int a = 0; a < 3 && v != 0.0; ++a) {
              if (be[a] > al[a]) { v = 0.0; break; }
              const double sg = (cc[a] % 2) ? 1.0 : -1.0;
              v *= binom(al[a], be[a]) * ipw(0.5, be[a]) * ipw(0.5 * sg, al[a] - be[a]);
            }
            if (v != 0.0) tPP.push_back({(long long)c * npc + i, (long long)pc * npc + j, v});
          }
        }
      }
      LsHostCsr PP = coo_to_csr(tPP, g.np);
      std::vector<CooEntry> tPr;
      for (int m = 0; m < k1; ++m) {
        for (int f = 0; f < 6; ++f)
          for (int i = 0; i < g.nq; ++i)
            for (int e = PQ.rp[i]; e < PQ.rp[i + 1]; ++e)
              tPr.push_back({(long long)m * g.block + (long long)f * g.nq + i,
                             (long long)m * gc.block + (long long)f * gc.nq + PQ.ci[e], PQ.v[e]});
        for (int i = 0; i < g.np; ++i)
          for (int e = PP.rp[i]; e < PP.rp[i + 1]; ++e)
            tPr.push_back({g.off_p(m) + i, gc.off_p(m) + PP.ci[e], PP.v[e]});
      }
      Lh.P = coo_to_csr(tPr, g.ndof);
      // vertex patches (Eq:DefPlm): active vertices, lexicographic; Z(P) ordered (m, f, c, node) / P ascending
      const int nvx[3] = {g.n[0] + 1, g.n[1] + 1, g.n[2] + 1};
      std::vector<std::vector<int>> lists(g.ndof);
      long long yoff = 0;
      Lh.pzoff.push_back(0);
      for (int vz = 0; vz < nvx[2]; ++vz)
        for (int vy = 0; vy < nvx[1]; ++vy)
          for (int vx = 0; vx < nvx[0]; ++vx) {
            std::vector<int> cl;
            for (int oz = -1; oz <= 0; ++oz)
              for (int oy = -1; oy <= 0; ++oy)
                for (int ox = -1; ox <= 0; ++ox) {
                  const int id = g.cell_id(vx + ox, vy + oy, vz + oz);
                  if (id >= 0) cl.push_back(id);
                }
            if (cl.empty()) continue;
            std::sort(cl.begin(), cl.end());
            std::vector<int> qn_;
            for (int c : cl)
              for (int J = 0; J < nbq; ++J) qn_.push_back(g.cellq[(size_t)c * nbq + J]);
            std::sort(qn_.begin(), qn_.end());
            qn_.erase(std::unique(qn_.begin(), qn_.end()), qn_.end());
            std::vector<long long> z;
            for (int m = 0; m < k1; ++m) {
              for (int comp = 0; comp < 3; ++comp)
                for (int q : qn_) z.push_back(g.off_v(m, comp) + q);
              for (int comp = 0; comp < 3; ++comp)
                for (int q : qn_) z.push_back(g.off_u(m, comp) + q);
              for (int c : cl)
                for (int s = 0; s < npc; ++s) z.push_back(g.off_p(m) + (long long)c * npc + s);
            }
            for (size_t i = 0; i < z.size(); ++i) {
              Lh.pz.push_back((int)z[i]);
              lists[z[i]].push_back((int)(yoff + (long long)i));
            }
            Lh.pcp.push_back((int)z.size());
            Lh.maxcp = std::max(Lh.maxcp, (int)z.size());
            yoff += (long long)z.size();
            Lh.pzoff.push_back((long long)Lh.pz.size());
          }
      Lh.ysize = yoff;
      if (yoff >= (1LL << 31)) { err = "L-shape patch results exceed 32-bit offsets"; return STGMG_ENOTSUP; }
      Lh.k3tab.assign((size_t)27 * g.ndof, -1);
      for (long long mu = 0; mu < g.ndof; ++mu) {
        if (lists[mu].empty()) { err = "L-shape: a DoF lies in no patch"; return STGMG_ECOVER; }
        if (lists[mu].size() > 27) { err = "L-shape: more than 27 patches contain a DoF"; return STGMG_ENOTSUP; }
        for (size_t s = 0; s < lists[mu].size(); ++s) Lh.k3tab[s * g.ndof + mu] = lists[mu][s];
      }
    }
  }
  return 0;
}

// --------------------------------------------------------------------------------------------- kernels -----
// K4 input: A_P[i][j] = A_l[Z_i][Z_j] from the CSR operator (columns ascending: binary search), row-major
// with leading dimension lda, identity padding past C_P.
__global__ void csr_extract_patches_kernel(const int* __restrict__ rp, const int* __restrict__ ci,
                                           const double* __restrict__ v, const int* __restrict__ pz,
                                           const long long* __restrict__ pzoff, const int* __restrict__ pcp,
                                           int p0, double* __restrict__ out, int lda) {
  const int p = blockIdx.y, i = blockIdx.x;
  const int cp = pcp[p0 + p];
  const int* z = pz + pzoff[p0 + p];
  double* o = out + ((long long)p * lda + i) * lda;
  if (i >= cp) {
    for (int j = threadIdx.x; j < lda; j += blockDim.x) o[j] = (i == j) ? 1.0 : 0.0;
    return;
  }
  const int row = z[i], lo = rp[row], hi = rp[row + 1];
  for (int j = threadIdx.x; j < lda; j += blockDim.x) {
    double val = 0.0;
    if (j < cp) {
      const int col = z[j];
      int a = lo, b = hi;
      while (a < b) {
        const int m = (a + b) >> 1;
        if (ci[m] < col) a = m + 1; else b = m;
      }
      if (a < hi && ci[a] == col) val = v[a];
    } else if (j == i) {
      val = 1.0;
    }
    o[j] = val;
  }
}

cudaError_t launch_csr_extract_patches(const int* rp, const int* ci, const double* v, const int* pz,
                                       const long long* pzoff, const int* pcp, int p0, int np, double* out, int lda,
                                       cudaStream_t s) {
  csr_extract_patches_kernel<<<dim3(lda, np), 256, 0, s>>>(rp, ci, v, pz, pzoff, pcp, p0, out, lda);
  return cudaGetLastError();
}

// K2u: y_P = A_P^{-1} r[Z(P)] for every patch (explicit per-patch inverse, row-major lda).  CTA = (row chunk,
// patch); the patch residual is gathered into shared memory once, one warp per row reads the inverse row
// coalesced and reduces with a fixed shuffle tree (deterministic).  HBM-bound on the inverses.
constexpr int K2U_ROWS = 32, K2U_THREADS = 256;

__global__ void __launch_bounds__(K2U_THREADS) patch_gemv_kernel(const int* __restrict__ pz,
                                                                 const long long* __restrict__ pzoff,
                                                                 const int* __restrict__ pcp,
                                                                 const double* __restrict__ inv, int lda,
                                                                 const double* __restrict__ r,
                                                                 double* __restrict__ Y) {
  extern __shared__ double rs[];
  pdl_trigger();
  const int p = blockIdx.y;
  const int cp = __ldg(pcp + p);
  const long long zo = __ldg(pzoff + p);
  const int row0 = blockIdx.x * K2U_ROWS;
  if (row0 >= cp) return;
  pdl_wait();
  for (int j = threadIdx.x; j < cp; j += blockDim.x) rs[j] = __ldg(r + __ldg(pz + zo + j));
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const double* A = inv + (long long)p * lda * lda;
  for (int i = row0 + warp; i < row0 + K2U_ROWS && i < cp; i += K2U_THREADS / 32) {
    const double* a = A + (long long)i * lda;
    double s = 0.0;
    for (int j = lane; j < cp; j += 32) s = fma(__ldg(a + j), rs[j], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) Y[zo + i] = s;
  }
}

cudaError_t launch_patch_gemv(int npatch, int maxcp, const int* pz, const long long* pzoff, const int* pcp,
                              const double* inv, int lda, const double* r, double* Y, cudaStream_t s) {
  const size_t smem = sizeof(double) * (size_t)maxcp;
  static PerDeviceOnce attr;
  attr.run([] {
    cudaFuncSetAttribute(patch_gemv_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  });
  return launch_pdl(patch_gemv_kernel, dim3((maxcp + K2U_ROWS - 1) / K2U_ROWS, npatch), dim3(K2U_THREADS), smem, s,
                    pz, pzoff, pcp, inv, lda, r, Y);
}

// dense row-major copy of a CSR matrix (coarse direct solve setup)
__global__ void csr_to_dense_kernel(int n, const int* __restrict__ rp, const int* __restrict__ ci,
                                    const double* __restrict__ v, double* __restrict__ out) {
  const int i = blockIdx.x;
  for (int j = threadIdx.x; j < n; j += blockDim.x) out[(long long)i * n + j] = 0.0;
  __syncthreads();
  for (int e = rp[i] + threadIdx.x; e < rp[i + 1]; e += blockDim.x) out[(long long)i * n + ci[e]] = v[e];
}

cudaError_t launch_csr_to_dense(int n, const int* rp, const int* ci, const double* v, double* out, cudaStream_t s) {
  csr_to_dense_kernel<<<n, 256, 0, s>>>(n, rp, ci, v, out);
  return cudaGetLastError();
}

// Slab load L_n (Def:L P:L220): chi_b rows (U block of node b) = theta_b sin(8 pi t_{n,b}) F, the rest 0
__global__ void lshape_load_kernel(long long N, long long block, long long R, int k1, const double* __restrict__ fN,
                                   double4 coef, double* __restrict__ L) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const int b = (int)(i / block);
  const long long o = i - (long long)b * block;
  const double cb = b == 0 ? coef.x : (b == 1 ? coef.y : (b == 2 ? coef.z : coef.w));
  L[i] = (o >= R && o < 2 * R) ? cb * fN[o - R] : 0.0;
}

cudaError_t launch_lshape_load(long long N, long long block, long long R, int k1, const double* fN, const double* coef,
                               double* L, cudaStream_t s) {
  const double4 c4 = make_double4(coef[0], k1 > 1 ? coef[1] : 0.0, k1 > 2 ? coef[2] : 0.0, k1 > 3 ? coef[3] : 0.0);
  lshape_load_kernel<<<(unsigned)((N + 255) / 256), 256, 0, s>>>(N, block, R, k1, fN, c4, L);
  return cudaGetLastError();
}

// Goal quantities (Eq:DefGQ): out[0] = wu . U_x, out[1] = wp . P of the last Radau block; one CTA, fixed order.
__global__ void lshape_goal_kernel(const double* __restrict__ x, long long ou, long long op, int nq, int np,
                                   const double* __restrict__ wu, const double* __restrict__ wp,
                                   double* __restrict__ out) {
  __shared__ double su[1024], sp_[1024];
  double a = 0.0, b = 0.0;
  for (int i = threadIdx.x; i < nq; i += blockDim.x) a = fma(wu[i], x[ou + i], a);
  for (int i = threadIdx.x; i < np; i += blockDim.x) b = fma(wp[i], x[op + i], b);
  su[threadIdx.x] = a;
  sp_[threadIdx.x] = b;
  __syncthreads();
  for (int st = blockDim.x / 2; st > 0; st >>= 1) {
    if ((int)threadIdx.x < st) {
      su[threadIdx.x] += su[threadIdx.x + st];
      sp_[threadIdx.x] += sp_[threadIdx.x + st];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[0] = su[0];
    out[1] = sp_[0];
  }
}

cudaError_t launch_lshape_goal(const double* x, long long ou, long long op, int nq, int np, const double* wu,
                               const double* wp, double* out, cudaStream_t s) {
  lshape_goal_kernel<<<1, 1024, 0, s>>>(x, ou, op, nq, np, wu, wp, out);
  return cudaGetLastError();
}

}  // namespace stgmg
