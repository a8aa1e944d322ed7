// Node-mapped, latency-lean versions of the HBM/latency-bound kernels of the V-cycle (sm_100a, fp64):
//   K3  avg_nodal      : Algorithm 1's averaging update (reading A17)  d <- d + omega * sum_P y_P / p
//   K1b gather_nodal   : node sum of element results (the second half of the operator apply / residual, Def:ACB)
//   K5  restrict_nodal : b_c = P^T r_f
//   K5  prolong_nodal  : d_f += P d_c
// One thread per spatial node (Q_r nodes first, then Q_{r-1} pressure nodes) handles every DoF that lives on the
// node — all Radau nodes m and all field components — so the index arithmetic (patch / cell / support lists) is
// done once per node and the k+1 x 2d independent sums give each thread ILP instead of a long serial chain.  All
// index math is 32-bit with compile-time degrees (no 64-bit divisions).  Summation orders are exactly those of the
// DoF-mapped kernels (patches / cells in lexicographic vertex order, supports in the CSR order), so the results are
// bitwise identical to them.
#include "stgmg_internal.cuh"

namespace stgmg {

template <int D>
__device__ __forceinline__ void node_coords(int node, const int* nn, int* idx) {
  idx[0] = node % nn[0];
  const int t = node / nn[0];
  if (D == 3) {
    idx[1] = t % nn[1];
    idx[2] = t / nn[1];
  } else {
    idx[1] = t;
    idx[2] = 0;
  }
}

// ------------------------------------------------------------------------------------------------ K3 --------
template <int D, int R, int K1>
__global__ void __launch_bounds__(128) avg_nodal_kernel(LevelGeom g, const double* __restrict__ Y, int ldy,
                                                        double omega, int zero_init, double* __restrict__ dvec,
                                                        int overwrite) {
  pdl_trigger();
  constexpr int NPMAX = D == 3 ? 27 : 9;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int nq = (int)g.nq, np = (int)g.np;
  if (t >= nq + np) return;
  const bool pres = t >= nq;
  // one (Radau node m, field slot) per grid row: the per-node thread with all 2d K1 slots needed 208 registers
  // (8 warps per SM, ncu: 12 % of the warp slots active)
  const int m = blockIdx.y / (2 * D), sl = blockIdx.y % (2 * D);
  if (pres && sl > 0) return;
  const int node = pres ? t - nq : t;
  int idx[3];
  node_coords<D>(node, pres ? g.pn : g.qn, idx);
  // per-axis candidate patches (vertex w, local index of the node in the patch box, cells of the patch)
  int cnt[3] = {1, 1, 1}, pw[3][3], pl[3][3], pc[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a) { pw[a][0] = 0; pl[a][0] = 0; pc[a][0] = 1; }
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const int i = idx[a], n = g.n[a];
    int c, l;
    if (pres) { c = i / (R - 1); l = i - c * (R - 1); } else { c = i / R; l = i - c * R; }
    const int deg = pres ? R - 1 : R;
    int w0, nw;
    if (l == 0) { w0 = c > 0 ? c - 1 : c; nw = (c > 0 ? 1 : 0) + 1 + (c <= n - 1 ? 1 : 0); }
    else { w0 = c; nw = 2; }
    cnt[a] = nw;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int w = w0 + j;
      const int lo = w > 0 ? w - 1 : 0;
      pw[a][j] = w;
      pl[a][j] = i - deg * lo;
      pc[a][j] = (w > 0 ? 1 : 0) + (w < n ? 1 : 0);
    }
  }
  // per candidate patch: offset of (m = 0, slot 0) of this node in Y, slot stride nQ, Radau stride blk
  int off[NPMAX];
  const int vs1 = g.n[0] + 1, vs2 = (g.n[0] + 1) * (g.n[1] + 1);
#pragma unroll
  for (int i3 = 0; i3 < (D == 3 ? 3 : 1); ++i3)
#pragma unroll
    for (int i2 = 0; i2 < 3; ++i2)
#pragma unroll
      for (int i1 = 0; i1 < 3; ++i1) {
        const int s = (i3 * 3 + i2) * 3 + i1;
        if (s >= NPMAX) continue;
        const bool ok = i1 < cnt[0] && i2 < cnt[1] && (D == 2 || i3 < cnt[2]);
        const int j[3] = {i1, i2, i3};
        int plin = 0, loc = 0, ls = 1, nQ = 1, nP = 1;
#pragma unroll
        for (int a = 0; a < D; ++a) {
          plin += pw[a][j[a]] * (a == 0 ? 1 : (a == 1 ? vs1 : vs2));
          const int qb = R * pc[a][j[a]] + 1, pb = (R - 1) * pc[a][j[a]] + 1;
          loc += pl[a][j[a]] * ls;
          ls *= pres ? pb : qb;
          nQ *= qb;
          nP *= pb;
        }
        // Y offset of (m, slot sl, this node) in patch s (int: npatch * ldy < 2^31 on every level)
        off[s] = ok ? plin * ldy + loc + (pres ? 2 * D * nQ : sl * nQ) + m * (2 * D * nQ + nP) : -1;
      }
  int p = 1;
#pragma unroll
  for (int a = 0; a < D; ++a) p *= cnt[a];
  const long long mu = (long long)m * g.block + (pres ? 2 * g.R + node : (long long)sl * g.nq + node);
  // omega / p_mu (reading A17: d + omega * (sum_P y_P) / p_mu); N2(iii) overwrite: the last patch's y, p = 1
  const double wp = overwrite ? omega : omega / (double)p;
  pdl_wait();
  double v[NPMAX];
#pragma unroll
  for (int s = 0; s < NPMAX; ++s) v[s] = off[s] >= 0 ? __ldg(Y + off[s]) : 0.0;   // absent patch: predicated off
  const double dold = zero_init ? 0.0 : dvec[mu];
  double z = 0.0;
  if (overwrite) {
#pragma unroll
    for (int s = 0; s < NPMAX; ++s) z = off[s] >= 0 ? v[s] : z;   // last patch (lexicographic) wins
  } else {
#pragma unroll
    for (int s = 0; s < NPMAX; ++s) z += off[s] >= 0 ? v[s] : 0.0;
  }
  const double upd = z * wp;
  dvec[mu] = zero_init ? upd : dold + upd;
}

// ------------------------------------------------------------------------------------------------ K1b -------
// y[mu] = beta * base[mu] + alpha * sum_{cells K containing mu} Yc[e(K, mu)], cells in lexicographic order.
// ldpm == 0: Yc[e][cell] (2D cell kernel layout); ldpm > 0: Yc[plin(K)][ldpm] (3D element GEMM, plin = vertex K+1).
template <int D, int R, int K1>
__global__ void __launch_bounds__(128) gather_nodal_kernel(LevelGeom g, const double* __restrict__ Yc,
                                                           const double* base, double* y, double alpha, double beta,
                                                           long long stride, long long ycstride, int ldpm) {
  pdl_trigger();
  constexpr int NQE = D == 3 ? (R + 1) * (R + 1) * (R + 1) : (R + 1) * (R + 1);
  constexpr int NPE = D == 3 ? R * R * R : R * R;
  constexpr int NE1 = 2 * D * NQE + NPE;
  constexpr int NC = 1 << D;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int nq = (int)g.nq, np = (int)g.np;
  if (t >= nq + np) return;
  Yc += blockIdx.y * ycstride;
  y += blockIdx.y * stride;
  if (base) base += blockIdx.y * stride;
  const bool pres = t >= nq;
  const int node = pres ? t - nq : t;
  int idx[3];
  node_coords<D>(node, pres ? g.pn : g.qn, idx);
  int nc[3] = {1, 1, 1}, cc[3][2], li[3][2];
#pragma unroll
  for (int a = 0; a < 3; ++a) { cc[a][0] = cc[a][1] = 0; li[a][0] = li[a][1] = 0; }
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const int i = idx[a];
    int c1, l1;
    if (pres) { c1 = i / (R - 1); l1 = i - c1 * (R - 1); } else { c1 = i / R; l1 = i - c1 * R; }
    const int deg = pres ? R - 1 : R;
    int k = 0;
    if (l1 == 0 && c1 > 0) { cc[a][k] = c1 - 1; li[a][k] = deg; ++k; }
    if (c1 < g.n[a]) { cc[a][k] = c1; li[a][k] = l1; ++k; }
    nc[a] = k;
  }
  int ncell = 1;
#pragma unroll
  for (int a = 0; a < D; ++a) ncell *= g.n[a];
  const int n1 = pres ? R : R + 1;
  const int estride = ldpm ? 1 : ncell;
  int off[NC];
#pragma unroll
  for (int s = 0; s < NC; ++s) {
    const int j[3] = {s & 1, (s >> 1) & 1, (s >> 2) & 1};
    bool ok = true;
    int cell = 0, cs = 1, plin = 0, vs = 1, loc = 0, ls = 1;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      ok = ok && j[a] < nc[a];
      cell += cc[a][j[a]] * cs;
      cs *= g.n[a];
      plin += (cc[a][j[a]] + 1) * vs;
      vs *= g.n[a] + 1;
      loc += li[a][j[a]] * ls;
      ls *= n1;
    }
    const int e0 = loc + (pres ? 2 * D * NQE : 0);
    off[s] = ok ? (ldpm ? plin * ldpm + e0 : e0 * ncell + cell) : -1;
  }
  const long long blockN = g.block;
  const long long node_off = pres ? 2 * g.R + node : (long long)node;
  const double* Yv[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) Yv[c] = Yc + (off[c] >= 0 ? off[c] : 0);
  const int nsl = pres ? 1 : 2 * D;
  pdl_wait();
#pragma unroll
  for (int m = 0; m < K1; ++m) {
    double v[2 * D][NC];
#pragma unroll
    for (int sl = 0; sl < 2 * D; ++sl) {
      const long long eadd = (long long)(m * NE1 + (sl < nsl ? sl : 0) * NQE) * estride;
#pragma unroll
      for (int c = 0; c < NC; ++c) v[sl][c] = __ldg(Yv[c] + eadd);   // absent cell: a valid address (predicating the
                                                                      // loads measured 185 -> 205 us at cfg4 fine)
    }
#pragma unroll
    for (int sl = 0; sl < 2 * D; ++sl) {
      if (sl >= nsl) break;
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < NC; ++c) s += off[c] >= 0 ? v[sl][c] : 0.0;
      const long long mu = m * blockN + node_off + (pres ? 0 : (long long)sl * g.nq);
      y[mu] = (base ? beta * base[mu] : 0.0) + alpha * s;
    }
  }
}

// ------------------------------------------------------------------------------------------------ K3c -------
// Averaging update of the element-wise Vanka smoother: patches are the cells, stored like the 3D
// element results (Y[plin(K + 1)][e(K, mu)]), so d <- d + omega * (sum_{cells K containing mu} y_K) / p_mu with
// p_mu = number of cells containing mu, cells in lexicographic order (reading A17 form).
template <int D, int R, int K1>
__global__ void __launch_bounds__(128) avg_cells_kernel(LevelGeom g, const double* __restrict__ Y, int ldy,
                                                        double omega, int zero_init, double* __restrict__ dvec) {
  constexpr int NQE = D == 3 ? (R + 1) * (R + 1) * (R + 1) : (R + 1) * (R + 1);
  constexpr int NPE = D == 3 ? R * R * R : R * R;
  constexpr int NE1 = 2 * D * NQE + NPE;
  constexpr int NC = 1 << D;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int nq = (int)g.nq, np = (int)g.np;
  if (t >= nq + np) return;
  const bool pres = t >= nq;
  const int node = pres ? t - nq : t;
  int idx[3];
  node_coords<D>(node, pres ? g.pn : g.qn, idx);
  int nc[3] = {1, 1, 1}, cc[3][2], li[3][2];
#pragma unroll
  for (int a = 0; a < 3; ++a) { cc[a][0] = cc[a][1] = 0; li[a][0] = li[a][1] = 0; }
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const int i = idx[a];
    int c1, l1;
    if (pres) { c1 = i / (R - 1); l1 = i - c1 * (R - 1); } else { c1 = i / R; l1 = i - c1 * R; }
    const int deg = pres ? R - 1 : R;
    int k = 0;
    if (l1 == 0 && c1 > 0) { cc[a][k] = c1 - 1; li[a][k] = deg; ++k; }
    if (c1 < g.n[a]) { cc[a][k] = c1; li[a][k] = l1; ++k; }
    nc[a] = k;
  }
  const int n1 = pres ? R : R + 1;
  int off[NC], p = 1;
#pragma unroll
  for (int a = 0; a < D; ++a) p *= nc[a];
#pragma unroll
  for (int s = 0; s < NC; ++s) {
    const int j[3] = {s & 1, (s >> 1) & 1, (s >> 2) & 1};
    bool ok = true;
    int plin = 0, vs = 1, loc = 0, ls = 1;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      ok = ok && j[a] < nc[a];
      plin += (cc[a][j[a]] + 1) * vs;
      vs *= g.n[a] + 1;
      loc += li[a][j[a]] * ls;
      ls *= n1;
    }
    off[s] = ok ? plin * ldy + loc + (pres ? 2 * D * NQE : 0) : -1;
  }
  const double wp = omega / (double)p;
  const long long blockN = g.block;
  const long long node_off = pres ? 2 * g.R + node : (long long)node;
  const int nsl = pres ? 1 : 2 * D;
  pdl_wait();
  for (int m = 0; m < K1; ++m)
    for (int sl = 0; sl < nsl; ++sl) {
      const int eadd = m * NE1 + sl * NQE;
      double z = 0.0;
#pragma unroll
      for (int c = 0; c < NC; ++c)
        if (off[c] >= 0) z += __ldg(Y + off[c] + eadd);
      const long long mu = m * blockN + node_off + (pres ? 0 : (long long)sl * g.nq);
      const double upd = z * wp;
      dvec[mu] = zero_init ? upd : dvec[mu] + upd;
    }
}

// ------------------------------------------------------------------------------------------------ K1e -------
// Residual in "patch-expanded" form for the dense K2 (large levels): r[mu] = beta * base[mu] + alpha * (sum of the
// element results of the cells containing mu, lexicographic) exactly as gather_nodal computes it, then stored at
// every (patch P containing mu, mu_hat) slot of Rexp, the B operand of K2 laid out per class chunk-major and
// bank-swizzled: class block at cls[c].rexp_off, element (column col, mu_hat) at
//   (mu_hat / 16) * ncols * 16 + col * 16 + ((mu_hat % 16) XOR 4 * (col % 4)),
// so every K2 tile reads its B chunk as one contiguous bulk copy (no gather in K2).  Yc == nullptr: r = beta * base.
// Patch classes per axis (App. A.4, as build_patches): n < 4: vertex w is its own class; else {0},{1},{2..n-2},{n-1},{n}.
template <int D, int R, int K1>
__global__ void __launch_bounds__(128) gather_expand_kernel(LevelGeom g, const double* __restrict__ Yc,
                                                            const double* __restrict__ base, double alpha, double beta,
                                                            int ldpm, const PatchClass* __restrict__ cls,
                                                            double* __restrict__ rexp) {
  pdl_trigger();
  constexpr int NQE = D == 3 ? (R + 1) * (R + 1) * (R + 1) : (R + 1) * (R + 1);
  constexpr int NPE = D == 3 ? R * R * R : R * R;
  constexpr int NE1 = 2 * D * NQE + NPE;
  constexpr int NC = 1 << D;
  constexpr int NPMAX = D == 3 ? 27 : 9;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int nq = (int)g.nq, np = (int)g.np;
  if (t >= nq + np) return;
  const bool pres = t >= nq;
  const int node = pres ? t - nq : t;
  const int deg = pres ? R - 1 : R;
  int idx[3];
  node_coords<D>(node, pres ? g.pn : g.qn, idx);
  // ---- cells containing the node (as gather_nodal)
  int nc[3] = {1, 1, 1}, cc[3][2], li[3][2];
#pragma unroll
  for (int a = 0; a < 3; ++a) { cc[a][0] = cc[a][1] = 0; li[a][0] = li[a][1] = 0; }
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const int i = idx[a];
    int c1, l1;
    if (pres) { c1 = i / (R - 1); l1 = i - c1 * (R - 1); } else { c1 = i / R; l1 = i - c1 * R; }
    int k = 0;
    if (l1 == 0 && c1 > 0) { cc[a][k] = c1 - 1; li[a][k] = deg; ++k; }
    if (c1 < g.n[a]) { cc[a][k] = c1; li[a][k] = l1; ++k; }
    nc[a] = k;
  }
  int ncell = 1;
#pragma unroll
  for (int a = 0; a < D; ++a) ncell *= g.n[a];
  const int n1 = pres ? R : R + 1;
  const int estride = ldpm ? 1 : ncell;
  int off[NC];
#pragma unroll
  for (int s = 0; s < NC; ++s) {
    const int j[3] = {s & 1, (s >> 1) & 1, (s >> 2) & 1};
    bool ok = Yc != nullptr;
    int cell = 0, cs = 1, plin = 0, vs = 1, loc = 0, ls = 1;
#pragma unroll
    for (int a = 0; a < D; ++a) {
      ok = ok && j[a] < nc[a];
      cell += cc[a][j[a]] * cs;
      cs *= g.n[a];
      plin += (cc[a][j[a]] + 1) * vs;
      vs *= g.n[a] + 1;
      loc += li[a][j[a]] * ls;
      ls *= n1;
    }
    const int e0 = loc + (pres ? 2 * D * NQE : 0);
    off[s] = ok ? (ldpm ? plin * ldpm + e0 : e0 * ncell + cell) : -1;
  }
  // ---- patches containing the node (as avg_nodal) and their class / column
  int cnt[3] = {1, 1, 1}, pw[3][3], pl[3][3], pc[3][3], pac[3][3], ppos[3][3], pcn[3][3], ncls[3] = {1, 1, 1};
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int j = 0; j < 3; ++j) { pw[a][j] = 0; pl[a][j] = 0; pc[a][j] = 1; pac[a][j] = 0; ppos[a][j] = 0; pcn[a][j] = 1; }
#pragma unroll
  for (int a = 0; a < D; ++a) {
    const int i = idx[a], n = g.n[a];
    ncls[a] = n < 4 ? n + 1 : 5;
    int c, l;
    if (pres) { c = i / (R - 1); l = i - c * (R - 1); } else { c = i / R; l = i - c * R; }
    int w0, nw;
    if (l == 0) { w0 = c > 0 ? c - 1 : c; nw = (c > 0 ? 1 : 0) + 1 + (c <= n - 1 ? 1 : 0); }
    else { w0 = c; nw = 2; }
    cnt[a] = nw;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int w = w0 + j;
      const int lo = w > 0 ? w - 1 : 0;
      pw[a][j] = w;
      pl[a][j] = i - deg * lo;
      pc[a][j] = (w > 0 ? 1 : 0) + (w < n ? 1 : 0);
      if (n < 4) { pac[a][j] = w; ppos[a][j] = 0; pcn[a][j] = 1; }
      else {
        const int ac = w == 0 ? 0 : (w == 1 ? 1 : (w == n ? 4 : (w == n - 1 ? 3 : 2)));
        pac[a][j] = ac;
        ppos[a][j] = ac == 2 ? w - 2 : 0;
        pcn[a][j] = ac == 2 ? n - 3 : 1;
      }
    }
  }
  long long pbase[NPMAX];
  int pcol[NPMAX], pnc[NPMAX], pmh[NPMAX], pnq[NPMAX], pblk[NPMAX];
#pragma unroll
  for (int i3 = 0; i3 < (D == 3 ? 3 : 1); ++i3)
#pragma unroll
    for (int i2 = 0; i2 < 3; ++i2)
#pragma unroll
      for (int i1 = 0; i1 < 3; ++i1) {
        const int s = (i3 * 3 + i2) * 3 + i1;
        if (s >= NPMAX) continue;
        const bool ok = i1 < cnt[0] && i2 < cnt[1] && (D == 2 || i3 < cnt[2]);
        const int j[3] = {i1, i2, i3};
        int loc = 0, ls = 1, nQ = 1, nP = 1, cid = 0, cstr = 1, col = 0, colstr = 1;
#pragma unroll
        for (int a = 0; a < D; ++a) {
          const int qb = R * pc[a][j[a]] + 1, pb = (R - 1) * pc[a][j[a]] + 1;
          loc += pl[a][j[a]] * ls;
          ls *= pres ? pb : qb;
          nQ *= qb;
          nP *= pb;
          cid += pac[a][j[a]] * cstr;
          cstr *= ncls[a];
          col += ppos[a][j[a]] * colstr;
          colstr *= pcn[a][j[a]];
        }
        pbase[s] = ok ? cls[cid].rexp_off : -1;
        pnc[s] = ok ? cls[cid].ncols : 0;
        pcol[s] = col;
        pmh[s] = loc + (pres ? 2 * D * nQ : 0);
        pnq[s] = nQ;
        pblk[s] = 2 * D * nQ + nP;
      }
  const long long blockN = g.block;
  const long long node_off = pres ? 2 * g.R + node : (long long)node;
  const double* Yv[NC];
#pragma unroll
  for (int c = 0; c < NC; ++c) Yv[c] = Yc + (off[c] >= 0 ? off[c] : 0);
  const int nsl = pres ? 1 : 2 * D;
  pdl_wait();
  if constexpr (D == 3) {   // 3D: one (m, slot) at a time (27 patch slots per node: the unrolled form spills)
#pragma unroll 1
    for (int m = 0; m < K1; ++m) {
#pragma unroll 1
      for (int sl = 0; sl < nsl; ++sl) {
        const long long eadd = (long long)(m * NE1 + sl * NQE) * estride;
        double v[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) v[c] = off[c] >= 0 ? __ldg(Yv[c] + eadd) : 0.0;
        double sum = 0.0;
#pragma unroll
        for (int c = 0; c < NC; ++c) sum += off[c] >= 0 ? v[c] : 0.0;
        const long long mu = m * blockN + node_off + (pres ? 0 : (long long)sl * g.nq);
        const double val = beta * base[mu] + alpha * sum;
#pragma unroll
        for (int s = 0; s < NPMAX; ++s) {
          if (pbase[s] < 0) continue;
          const int mh = pmh[s] + m * pblk[s] + (pres ? 0 : sl * pnq[s]);
          rexp[pbase[s] + (long long)(mh >> 4) * pnc[s] * 16 + pcol[s] * 16 + ((mh & 15) ^ ((pcol[s] & 3) << 2))] = val;
        }
      }
    }
  } else {
  // 2D: all loads of the node first (unconditional addresses, so they issue back to back), then sums and stores
  constexpr int NV = K1 * 2 * D;
  double val[NV];
#pragma unroll
  for (int q = 0; q < NV; ++q) {
    const int m = q / (2 * D), sl = q % (2 * D);
    const long long eadd = (long long)(m * NE1 + (sl < nsl ? sl : 0) * NQE) * estride;
    double v[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) v[c] = off[c] >= 0 ? __ldg(Yv[c] + eadd) : 0.0;
    double sum = 0.0;
#pragma unroll
    for (int c = 0; c < NC; ++c) sum += off[c] >= 0 ? v[c] : 0.0;
    const long long mu = m * blockN + node_off + (pres ? 0 : (long long)(sl < nsl ? sl : 0) * g.nq);
    val[q] = beta * __ldg(base + mu) + alpha * sum;
  }
#pragma unroll
  for (int s = 0; s < NPMAX; ++s) {
    if (pbase[s] < 0) continue;
    double* dst = rexp + pbase[s] + pcol[s] * 16;
    const int cst = pnc[s] * 16, swz = (pcol[s] & 3) << 2;
#pragma unroll
    for (int q = 0; q < NV; ++q) {
      const int m = q / (2 * D), sl = q % (2 * D);
      if (sl >= nsl) continue;
      const int mh = pmh[s] + m * pblk[s] + (pres ? 0 : sl * pnq[s]);
      dst[(long long)(mh >> 4) * cst + ((mh & 15) ^ swz)] = val[q];
    }
  }
  }
}

// ------------------------------------------------------------------------------------------------ K5 --------
// b_c = P^T r_f: one thread per coarse node, 1D supports from the coarse-row CSR tables.
template <int D, int K1>
__global__ void __launch_bounds__(128) restrict_nodal_kernel(LevelGeom f, LevelGeom c, TransferTables t,
                                                             const double* __restrict__ rf, double* __restrict__ bc) {
  pdl_trigger();
  constexpr int NS = 2 * D;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int nq = (int)c.nq, np = (int)c.np;
  if (tid >= nq + np) return;
  const bool pres = tid >= nq;
  const int node = pres ? tid - nq : tid;
  int idx[3];
  node_coords<D>(node, pres ? c.pn : c.qn, idx);
  const Interp1D* T = pres ? t.p : t.q;
  int lo[3] = {0, 0, 0}, hi[3] = {1, 1, 1};
#pragma unroll
  for (int a = 0; a < D; ++a) {
    lo[a] = T[a].rp_c[idx[a]];
    hi[a] = T[a].rp_c[idx[a] + 1];
  }
  const int fs1 = pres ? (int)f.ps[1] : (int)f.qs[1];
  const int fs2 = D == 3 ? (pres ? (int)f.ps[2] : (int)f.qs[2]) : 0;
  const long long fbase = pres ? 2 * f.R : 0;
  double acc[K1][NS];
#pragma unroll
  for (int m = 0; m < K1; ++m)
#pragma unroll
    for (int s = 0; s < NS; ++s) acc[m][s] = 0.0;
  pdl_wait();
  for (int e2 = lo[2]; e2 < hi[2]; ++e2) {
    double w2 = 1.0;
    int f2 = 0;
    if (D > 2) { f2 = T[2].ci_c[e2] * fs2; w2 = T[2].v_c[e2]; }
    for (int e1 = lo[1]; e1 < hi[1]; ++e1) {
      const double w1 = w2 * T[1].v_c[e1];
      const int f1 = f2 + T[1].ci_c[e1] * fs1;
      for (int e0 = lo[0]; e0 < hi[0]; ++e0) {
        const double w = w1 * T[0].v_c[e0];
        const long long fn = fbase + f1 + T[0].ci_c[e0];
#pragma unroll
        for (int m = 0; m < K1; ++m)
#pragma unroll
          for (int s = 0; s < NS; ++s) {
            if (pres && s > 0) break;
            acc[m][s] = fma(w, __ldg(rf + m * f.block + fn + (long long)s * f.nq), acc[m][s]);
          }
      }
    }
  }
  const long long node_off = pres ? 2 * c.R + node : (long long)node;
#pragma unroll
  for (int m = 0; m < K1; ++m)
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      if (pres && s > 0) break;
      bc[m * c.block + node_off + (long long)s * c.nq] = acc[m][s];
    }
}

// b_c = P^T r_f axis by axis (P = P_x (x) P_y (x) P_z per Radau node and field): pass a contracts axis a with
// the coarse-row 1D tables; one thread per output element, its <= 2r+1 supports along the axis.  Buffers use the level
// layout with the pass's own node counts (nq, np per (m, slot) block).  Every pass reads and writes coalesced; three
// passes move ~2.5 N_f doubles instead of the per-coarse-node gather of (2r+1)^d supports (latency-bound: ncu 0.05–0.18
// of HBM).  Bitwise 1-vs-n on owned DoFs (each output depends on the window's fine values only).
struct SepDims {
  int q[3], p[3];        // node counts per axis (Q_r, Q_{r-1})
  long long nq, np, blk;
};

template <int D, int K1>
__global__ void __launch_bounds__(256) restrict_pass_kernel(const double* __restrict__ in, SepDims di,
                                                            double* __restrict__ out, SepDims dout, int axis,
                                                            Interp1D tq, Interp1D tp) {
  pdl_trigger();
  // 32-bit index arithmetic (every level vector here has < 2^31 entries; 64-bit divisions dominated the first
  // version of this kernel)
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  const int blk = (int)dout.blk, nq = (int)dout.nq;
  if (idx >= K1 * blk) return;
  const int m = idx / blk;
  const int rem = idx - m * blk;
  const bool pres = rem >= 2 * D * nq;
  const int slot = pres ? 2 * D : rem / nq;
  int node = pres ? rem - 2 * D * nq : rem - slot * nq;
  const int* od = pres ? dout.p : dout.q;
  const int* id = pres ? di.p : di.q;
  int c[3] = {0, 0, 0};
#pragma unroll
  for (int a = 0; a < D - 1; ++a) {
    const int q = node / od[a];
    c[a] = node - q * od[a];
    node = q;
  }
  c[D - 1] = node;
  int base = 0, st = 1, sa = 1;   // input offset without the contracted axis; stride of that axis
#pragma unroll
  for (int a = 0; a < D; ++a) {
    if (a == axis) sa = st;
    else base += c[a] * st;
    st *= id[a];
  }
  const Interp1D& T = pres ? tp : tq;
  const double* src = in + (long long)m * di.blk + (pres ? 2 * D * di.nq : (long long)slot * di.nq) + base;
  const int lo = __ldg(T.rp_c + c[axis]), hi = __ldg(T.rp_c + c[axis] + 1);
  pdl_wait();
  double acc = 0.0;
  for (int e = lo; e < hi; ++e) acc = fma(__ldg(T.v_c + e), __ldg(src + __ldg(T.ci_c + e) * sa), acc);
  out[idx] = acc;
}

// d_f += P d_c: one thread per fine node, 1D supports from the fine-row CSR tables.
template <int D, int K1>
__global__ void __launch_bounds__(128) prolong_nodal_kernel(LevelGeom f, LevelGeom c, TransferTables t,
                                                            const double* __restrict__ dc, double* __restrict__ df) {
  pdl_trigger();
  constexpr int NS = 2 * D;
  const int tid = blockIdx.x * blockDim.x + threadIdx.x;
  const int nq = (int)f.nq, np = (int)f.np;
  if (tid >= nq + np) return;
  const bool pres = tid >= nq;
  const int node = pres ? tid - nq : tid;
  int idx[3];
  node_coords<D>(node, pres ? f.pn : f.qn, idx);
  const Interp1D* T = pres ? t.p : t.q;
  int lo[3] = {0, 0, 0}, hi[3] = {1, 1, 1};
#pragma unroll
  for (int a = 0; a < D; ++a) {
    lo[a] = T[a].rp_f[idx[a]];
    hi[a] = T[a].rp_f[idx[a] + 1];
  }
  const int cs1 = pres ? (int)c.ps[1] : (int)c.qs[1];
  const int cs2 = D == 3 ? (pres ? (int)c.ps[2] : (int)c.qs[2]) : 0;
  const long long cbase = pres ? 2 * c.R : 0;
  double acc[K1][NS];
#pragma unroll
  for (int m = 0; m < K1; ++m)
#pragma unroll
    for (int s = 0; s < NS; ++s) acc[m][s] = 0.0;
  pdl_wait();
  for (int e2 = lo[2]; e2 < hi[2]; ++e2) {
    double w2 = 1.0;
    int c2 = 0;
    if (D > 2) { c2 = T[2].ci_f[e2] * cs2; w2 = T[2].v_f[e2]; }
    for (int e1 = lo[1]; e1 < hi[1]; ++e1) {
      const double w1 = w2 * T[1].v_f[e1];
      const int c1 = c2 + T[1].ci_f[e1] * cs1;
      for (int e0 = lo[0]; e0 < hi[0]; ++e0) {
        const double w = w1 * T[0].v_f[e0];
        const long long cn = cbase + c1 + T[0].ci_f[e0];
#pragma unroll
        for (int m = 0; m < K1; ++m)
#pragma unroll
          for (int s = 0; s < NS; ++s) {
            if (pres && s > 0) break;
            acc[m][s] = fma(w, __ldg(dc + m * c.block + cn + (long long)s * c.nq), acc[m][s]);
          }
      }
    }
  }
  const long long node_off = pres ? 2 * f.R + node : (long long)node;
#pragma unroll
  for (int m = 0; m < K1; ++m)
#pragma unroll
    for (int s = 0; s < NS; ++s) {
      if (pres && s > 0) break;
      const long long mu = m * f.block + node_off + (long long)s * f.nq;
      df[mu] += acc[m][s];
    }
}

// ------------------------------------------------------------------------------------------- launchers ------
static inline unsigned node_blocks(const LevelGeom& g) { return (unsigned)((g.nq + g.np + 127) / 128); }

#define STGMG_DRK(d, r, k1, CALL)                                                            \
  do {                                                                                       \
    if (d == 2 && r == 2 && k1 == 1) { constexpr int D_ = 2, R_ = 2, K_ = 1; CALL; }          \
    if (d == 2 && r == 2 && k1 == 2) { constexpr int D_ = 2, R_ = 2, K_ = 2; CALL; }          \
    if (d == 2 && r == 2 && k1 == 3) { constexpr int D_ = 2, R_ = 2, K_ = 3; CALL; }          \
    if (d == 2 && r == 3 && k1 == 1) { constexpr int D_ = 2, R_ = 3, K_ = 1; CALL; }          \
    if (d == 2 && r == 3 && k1 == 2) { constexpr int D_ = 2, R_ = 3, K_ = 2; CALL; }          \
    if (d == 2 && r == 3 && k1 == 3) { constexpr int D_ = 2, R_ = 3, K_ = 3; CALL; }          \
    if (d == 3 && r == 2 && k1 == 1) { constexpr int D_ = 3, R_ = 2, K_ = 1; CALL; }          \
    if (d == 3 && r == 2 && k1 == 2) { constexpr int D_ = 3, R_ = 2, K_ = 2; CALL; }          \
    if (d == 3 && r == 3 && k1 == 1) { constexpr int D_ = 3, R_ = 3, K_ = 1; CALL; }          \
    if (d == 3 && r == 3 && k1 == 2) { constexpr int D_ = 3, R_ = 3, K_ = 2; CALL; }          \
  } while (0)

cudaError_t launch_vanka_average(const LevelGeom& g, int r, int k1, const double* Y, int ldy, double omega,
                                 int zero_init, double* dvec, cudaStream_t s, int overwrite) {
  STGMG_DRK(g.d, r, k1,
            return launch_pdl(avg_nodal_kernel<D_, R_, K_>, dim3(node_blocks(g), K_ * 2 * D_), dim3(128), 0, s, g, Y,
                              ldy, omega, zero_init, dvec, overwrite));
  return cudaErrorNotSupported;
}

cudaError_t launch_op_gather(const LevelGeom& g, int r, int k1, const double* Yc, const double* base, double* y,
                             double alpha, double beta, int batch, long long stride, long long ycstride,
                             cudaStream_t s, int ldpm) {
  STGMG_DRK(g.d, r, k1,
            return launch_pdl(gather_nodal_kernel<D_, R_, K_>, dim3(node_blocks(g), (unsigned)batch), dim3(128), 0, s,
                              g, Yc, base, y, alpha, beta, stride, ycstride, ldpm));
  return cudaErrorNotSupported;
}

cudaError_t launch_avg_cells(const LevelGeom& g, int r, int k1, const double* Y, int ldy, double omega, int zero_init,
                             double* dvec, cudaStream_t s) {
  STGMG_DRK(g.d, r, k1,
            return launch_pdl(avg_cells_kernel<D_, R_, K_>, dim3(node_blocks(g)), dim3(128), 0, s, g, Y, ldy, omega,
                              zero_init, dvec));
  return cudaErrorNotSupported;
}

cudaError_t launch_gather_expand(const LevelGeom& g, int r, int k1, const double* Yc, const double* base, double alpha,
                                 double beta, int ldpm, const PatchClass* cls, double* rexp, cudaStream_t s) {
  STGMG_DRK(g.d, r, k1,
            return launch_pdl(gather_expand_kernel<D_, R_, K_>, dim3(node_blocks(g)), dim3(128), 0, s, g, Yc, base,
                              alpha, beta, ldpm, cls, rexp));
  return cudaErrorNotSupported;
}

cudaError_t launch_restrict(const LevelGeom& fine, const LevelGeom& coarse, int k1, const TransferTables& t,
                            const double* rf, double* bc, cudaStream_t s) {
  STGMG_DRK(fine.d, 2, k1,
            return launch_pdl(restrict_nodal_kernel<D_, K_>, dim3(node_blocks(coarse)), dim3(128), 0, s, fine, coarse,
                              t, rf, bc));
  return cudaErrorNotSupported;
}

// Separable restriction (above): d passes through tmp (>= the first pass's output, <= N_fine doubles).
cudaError_t launch_restrict_sep(const LevelGeom& fine, const LevelGeom& coarse, int k1, const TransferTables& t,
                                const double* rf, double* bc, double* tmp, cudaStream_t s) {
  const int d = fine.d;
  SepDims dims[4];
  for (int pass = 0; pass <= d; ++pass) {   // dims after `pass` axes were coarsened
    SepDims& q = dims[pass];
    q.nq = 1;
    q.np = 1;
    for (int a = 0; a < 3; ++a) {
      q.q[a] = a < d ? (a < pass ? coarse.qn[a] : fine.qn[a]) : 1;
      q.p[a] = a < d ? (a < pass ? coarse.pn[a] : fine.pn[a]) : 1;
      q.nq *= q.q[a];
      q.np *= q.p[a];
    }
    q.blk = 2 * d * q.nq + q.np;
  }
  const double* in = rf;
  for (int a = 0; a < d; ++a) {
    // pass 1 -> tmp, pass 2 -> tmp + (size of pass 1), ... last pass -> bc
    double* out = a == d - 1 ? bc : (a == 0 ? tmp : tmp + (long long)k1 * dims[1].blk);
    const long long n = (long long)k1 * dims[a + 1].blk;
    const unsigned grid = (unsigned)((n + 255) / 256);
    cudaError_t e = cudaErrorNotSupported;
    if (d == 3 && k1 == 1) e = launch_pdl(restrict_pass_kernel<3, 1>, dim3(grid), dim3(256), 0, s, in, dims[a], out, dims[a + 1], a, t.q[a], t.p[a]);
    if (d == 3 && k1 == 2) e = launch_pdl(restrict_pass_kernel<3, 2>, dim3(grid), dim3(256), 0, s, in, dims[a], out, dims[a + 1], a, t.q[a], t.p[a]);
    if (d == 3 && k1 == 3) e = launch_pdl(restrict_pass_kernel<3, 3>, dim3(grid), dim3(256), 0, s, in, dims[a], out, dims[a + 1], a, t.q[a], t.p[a]);
    if (d == 3 && k1 == 4) e = launch_pdl(restrict_pass_kernel<3, 4>, dim3(grid), dim3(256), 0, s, in, dims[a], out, dims[a + 1], a, t.q[a], t.p[a]);
    if (d == 2 && k1 == 1) e = launch_pdl(restrict_pass_kernel<2, 1>, dim3(grid), dim3(256), 0, s, in, dims[a], out, dims[a + 1], a, t.q[a], t.p[a]);
    if (d == 2 && k1 == 2) e = launch_pdl(restrict_pass_kernel<2, 2>, dim3(grid), dim3(256), 0, s, in, dims[a], out, dims[a + 1], a, t.q[a], t.p[a]);
    if (d == 2 && k1 == 3) e = launch_pdl(restrict_pass_kernel<2, 3>, dim3(grid), dim3(256), 0, s, in, dims[a], out, dims[a + 1], a, t.q[a], t.p[a]);
    if (d == 2 && k1 == 4) e = launch_pdl(restrict_pass_kernel<2, 4>, dim3(grid), dim3(256), 0, s, in, dims[a], out, dims[a + 1], a, t.q[a], t.p[a]);
    if (e != cudaSuccess) return e;
    in = out;
  }
  return cudaSuccess;
}

cudaError_t launch_prolong_add(const LevelGeom& fine, const LevelGeom& coarse, int k1, const TransferTables& t,
                               const double* dc, double* df, cudaStream_t s) {
  STGMG_DRK(fine.d, 2, k1,
            return launch_pdl(prolong_nodal_kernel<D_, K_>, dim3(node_blocks(fine)), dim3(128), 0, s, fine, coarse, t,
                              dc, df));
  return cudaErrorNotSupported;
}

}  // namespace stgmg
