// K1 — the slab operator as FACTORED element GEMMs on the FP64 tensor pipe (sm_100a, mma.sync m8n8k4 -> DMMA).
//
// Operator (Problem 3.1, Eq:DPQ_A0; block form read per SURVEY reading A5 / App. A.1), per cell K of
// type t (interior, or its set of Dirichlet faces) with the element matrices of Def:ACB / Def:ab:
//   (A X)_{phi,b} = sum_a T_ba M_rho U_a - theta_b M_rho V_b
//   (A X)_{chi,b} = sum_a T_ba M_rho V_a + theta_b (A_gamma U_b + C^T P_b)
//   (A X)_{psi,b} = sum_a T_ba M_c  P_a + theta_b (-C V_b + B_gamma P_b)
// Instead of the (k+1)(2d NQ + NP)-square slab element matrix (340^2 in 3D Q2 dG(1)), the temporal structure and the
// component structure are factored out: three small spatial GEMMs per cell and Radau node, the mixing with T and
// theta done in the epilogue:
//   G1 = M_rho/rho-scalar mass (NQ x NQ)            on U_a,c and V_a,c   (all a, c)     -> MU, MV
//   G2 = [A_gamma | C^T]   (d NQ x (d NQ + NP))     on [U_a; P_a]                       -> AU
//   G3 = [-C | B_gamma]    (NP x (d NQ + NP))       on [V_a; P_a],  GP = M_c on P_a      -> BP, MP
// (3D Q2 dG(1): 57k padded flop slots per cell instead of 248k).  G1 and GP are shared by every cell type; G2, G3
// carry the Nitsche face terms of the type.  The element results are written cell-fastest, Y[element DoF][cell]
// (a warp's stores are 64-byte runs), and summed per node by the deterministic gather (gather_nodal_kernel, ldpm 0).
//
// CTA = 32 cells of one type: the cells' element inputs (all k+1 Radau nodes, zero-padded slot blocks) are gathered
// once into shared memory in a B-operand layout (row = element DoF, column = cell, row stride 36 doubles: the m8n8k4
// B fragments of a warp hit 32 distinct bank pairs); warp w < d * NQM/8 owns component c = w / MB and rows
// 8 (w % MB) .. +8 of G1 and G2 for the 32 cells in two passes of 16 (A fragments pre-arranged fragment-major in
// global memory: one coalesced 256-byte load per k-step), and G3 / GP tasks (8 cells, all Radau nodes) follow on the
// first warps.
#include <algorithm>
#include <cstdlib>
#include <functional>

#include "op_common.cuh"

namespace stgmg {

__device__ __forceinline__ void fg_dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

template <int D, int R, int K1, int NCC = 32>
struct FG {
  static constexpr int NQ = ipow(R + 1, D), NP = ipow(R, D);
  static constexpr int NQK = (NQ + 3) / 4 * 4;     // XE rows per Q slot (K padding, zero rows)
  static constexpr int NPK = (NP + 3) / 4 * 4;     // XE rows of the P slot
  static constexpr int NQM = (NQ + 7) / 8 * 8;     // G1 / G2 rows per component (M padding)
  static constexpr int NPM = (NP + 7) / 8 * 8;     // G3 / GP rows
  static constexpr int RA = 2 * D * NQK + NPK;     // XE rows per Radau node: V_0..V_{d-1}, U_0..U_{d-1}, P
  static constexpr int XR = K1 * RA;
  static constexpr int NC = NCC;                   // cells per CTA tile
  static constexpr int XS = NC + 4;                // XE row stride (doubles)
  static constexpr int KS1 = NQK / 4, KS2 = (D * NQK + NPK) / 4, KSP = NPK / 4;
  static constexpr int KSV = D * NQK / 4;          // G3 k-steps over V (then KSP over P)
  static constexpr int MB = NQM / 8, NT = D * MB;  // warps = G1/G2 tasks
  static constexpr int MB3 = NPM / 8, NT3 = (NC / 8) * MB3;
  static constexpr int NE1 = 2 * D * NQ + NP, NE = K1 * NE1;
  static constexpr size_t SMEM = sizeof(double) * (size_t)XR * XS + 3 * sizeof(long long) * NC;
};

// k loop with the A fragments prefetched three k-steps ahead without register moves: rounds of three steps, each
// fragment register is consumed and immediately reloaded with the fragment three steps later (a rotating ring
// f0 = f1 = f2 stalled every move on the outstanding load: ncu long-scoreboard on the moves).
template <int KS, class Body>
__device__ __forceinline__ void fg_kloop(const double* ap, Body body) {
  double fr[3];
#pragma unroll
  for (int j = 0; j < 3; ++j) fr[j] = j < KS ? __ldg(ap + 32 * j) : 0.0;
#pragma unroll 1
  for (int k0 = 0; k0 < KS; k0 += 3) {
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      const int ks = k0 + j;
      if (ks < KS) {
        const double af = fr[j];
        if (ks + 3 < KS) fr[j] = __ldg(ap + 32 * (ks + 3));
        body(ks, af);
      }
    }
  }
}

struct FgMix {   // temporal constants of the epilogue (T[b][a], theta_b)
  double T[kMaxK1][kMaxK1];
  double th[kMaxK1];
};

// Column bases of a tile (threads < NC): lowest Q_r / Q_{r-1} node of each cell and its lexicographic index.
template <int D, int R, int NC = 32>
__device__ __forceinline__ void fg_bases(const LevelGeom& g, const PatchClass& pc, int4 td, long long* qb,
                                         long long* pb, long long* pl) {
  if (threadIdx.x < NC) {   // cell of column j: box of the type (vlo = cell + 1 per axis), x fastest
    const int j = threadIdx.x;
    long long q = 0, p = 0, v = 0, vs = 1;
    if (j < td.z) {
      int rem = td.y + j;
      for (int a = 0; a < D; ++a) {
        const int ca = pc.vlo[a] - 1 + rem % pc.cnt[a];
        rem /= pc.cnt[a];
        q += (long long)(R * ca) * g.qs[a];
        p += (long long)((R - 1) * ca) * g.ps[a];
        v += (long long)ca * vs;
        vs *= g.n[a];
      }
    }
    qb[j] = q;
    pb[j] = p;
    pl[j] = v;
  }
}

// Element DoF e of XE row `row` (-1 for the zero rows that pad each slot block to a multiple of 4).
template <int D, int R, int K1>
__device__ __forceinline__ int fg_row_elem(int row) {
  using F = FG<D, R, K1>;
  const int a = row / F::RA, rr = row % F::RA;
  if (rr < 2 * D * F::NQK) {
    const int slot = rr / F::NQK, j = rr % F::NQK;
    return j < F::NQ ? a * F::NE1 + slot * F::NQ + j : -1;
  }
  const int j = rr - 2 * D * F::NQK;
  return j < F::NP ? a * F::NE1 + 2 * D * F::NQ + j : -1;
}

// The G1 / G2 / G3 GEMMs of one tile from its gathered inputs XE and the epilogue (mixing with T, theta; stores).
template <int D, int R, int K1, int HN, int NC = 32>
__device__ __forceinline__ void fg_compute(const double* XE, const long long* pl, int4 td, const double* __restrict__ A1,
                                           const double* __restrict__ A2, const double* __restrict__ A3,
                                           const double* __restrict__ AP, long long a2stride, long long a3stride,
                                           const FgMix& mix, double* __restrict__ Y, long long ncell) {
  using F = FG<D, R, K1, NC>;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int kl = lane & 3, nl = lane >> 2;
  const double* Bl = XE + kl * F::XS + nl;   // this lane's B element: row k0 + kl, column n0 + nl
  if (warp < F::NT) {
    const int c = warp / F::MB, i = warp % F::MB;
    const double* a2 = A2 + td.x * a2stride + (long long)(c * F::MB + i) * F::KS2 * 32 + lane;
    const double* a1 = A1 + (long long)i * F::KS1 * 32 + lane;
#pragma unroll 1
    for (int h = 0; h < F::NC / 8; h += HN) {
      // G2: AU_a for rows 8i.. of component c, columns (a, cell)
      double acc2[K1][HN][2];
#pragma unroll
      for (int a = 0; a < K1; ++a)
#pragma unroll
        for (int n = 0; n < HN; ++n) acc2[a][n][0] = acc2[a][n][1] = 0.0;
      fg_kloop<F::KS2>(a2, [&](int ks, double af) {
#pragma unroll
        for (int a = 0; a < K1; ++a) {
          const double* bp = Bl + (a * F::RA + D * F::NQK + 4 * ks) * F::XS + 8 * h;
#pragma unroll
          for (int n = 0; n < HN; ++n) fg_dmma(acc2[a][n][0], acc2[a][n][1], af, bp[8 * n]);
        }
      });
      // G1: mass on V_a,c (f = 0) and U_a,c (f = 1) for rows 8i..
      double acc1[2][K1][HN][2];
#pragma unroll
      for (int f = 0; f < 2; ++f)
#pragma unroll
        for (int a = 0; a < K1; ++a)
#pragma unroll
          for (int n = 0; n < HN; ++n) acc1[f][a][n][0] = acc1[f][a][n][1] = 0.0;
      fg_kloop<F::KS1>(a1, [&](int ks, double af) {
#pragma unroll
        for (int f = 0; f < 2; ++f)
#pragma unroll
          for (int a = 0; a < K1; ++a) {
            const double* bp = Bl + (a * F::RA + (f * D + c) * F::NQK + 4 * ks) * F::XS + 8 * h;
#pragma unroll
            for (int n = 0; n < HN; ++n) fg_dmma(acc1[f][a][n][0], acc1[f][a][n][1], af, bp[8 * n]);
          }
      });
      // epilogue: phi_b = sum_a T_ba MU_a - theta_b MV_b, chi_b = sum_a T_ba MV_a + theta_b AU_b
      const int J = 8 * i + nl;
      if (J < F::NQ) {
#pragma unroll
        for (int n = 0; n < HN; ++n)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int col = 8 * (h + n) + 2 * kl + e;
            if (col >= td.z) continue;
            double* y = Y + (long long)(c * F::NQ + J) * ncell + pl[col];
#pragma unroll
            for (int b = 0; b < K1; ++b) {
              double phi = -mix.th[b] * acc1[0][b][n][e], chi = mix.th[b] * acc2[b][n][e];
#pragma unroll
              for (int a = 0; a < K1; ++a) {
                phi = fma(mix.T[b][a], acc1[1][a][n][e], phi);
                chi = fma(mix.T[b][a], acc1[0][a][n][e], chi);
              }
              y[(long long)b * F::NE1 * ncell] = phi;
              y[(long long)(b * F::NE1 + D * F::NQ) * ncell] = chi;
            }
          }
      }
    }
  }
  // G3 / GP: psi_b = sum_a T_ba MP_a + theta_b BP_b for 8 cells and rows 8 m3.. (tasks spread over the warps)
  for (int t3 = warp; t3 < F::NT3; t3 += F::NT) {
    const int cg = t3 % (F::NC / 8), m3 = t3 / (F::NC / 8);
    double acc3[K1][2], accp[K1][2];
#pragma unroll
    for (int a = 0; a < K1; ++a) acc3[a][0] = acc3[a][1] = accp[a][0] = accp[a][1] = 0.0;
    const double* a3 = A3 + td.x * a3stride + (long long)m3 * F::KS2 * 32 + lane;
    fg_kloop<F::KS2>(a3, [&](int ks, double af) {
      const int r0 = ks < F::KSV ? 4 * ks : 2 * D * F::NQK + 4 * (ks - F::KSV);   // V rows, then P rows
#pragma unroll
      for (int a = 0; a < K1; ++a) fg_dmma(acc3[a][0], acc3[a][1], af, Bl[(a * F::RA + r0) * F::XS + 8 * cg]);
    });
    const double* ap = AP + (long long)m3 * F::KSP * 32 + lane;
#pragma unroll
    for (int ks = 0; ks < F::KSP; ++ks) {
      const double af = __ldg(ap + ks * 32);
#pragma unroll
      for (int a = 0; a < K1; ++a)
        fg_dmma(accp[a][0], accp[a][1], af, Bl[(a * F::RA + 2 * D * F::NQK + 4 * ks) * F::XS + 8 * cg]);
    }
    const int s = 8 * m3 + nl;
    if (s < F::NP) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int col = 8 * cg + 2 * kl + e;
        if (col >= td.z) continue;
        double* y = Y + (long long)(2 * D * F::NQ + s) * ncell + pl[col];
#pragma unroll
        for (int b = 0; b < K1; ++b) {
          double psi = mix.th[b] * acc3[b][e];
#pragma unroll
          for (int a = 0; a < K1; ++a) psi = fma(mix.T[b][a], accp[a][e], psi);
          y[(long long)b * F::NE1 * ncell] = psi;
        }
      }
    }
  }
}

template <int D, int R, int K1>
__global__ void __launch_bounds__(FG<D, R, K1>::NT * 32, 2) op_fgemm_kernel(
    LevelGeom g, const int4* __restrict__ tiles, const PatchClass* __restrict__ ecls, const int* __restrict__ relidx,
    const double* __restrict__ A1, const double* __restrict__ A2, const double* __restrict__ A3,
    const double* __restrict__ AP, long long a2stride, long long a3stride, FgMix mix, const double* __restrict__ x,
    double* __restrict__ Y, long long ncell) {
  using F = FG<D, R, K1>;
  pdl_trigger();
  extern __shared__ double smem[];
  double* XE = smem;
  long long* qb = reinterpret_cast<long long*>(XE + (size_t)F::XR * F::XS);
  long long* pb = qb + F::NC;
  long long* pl = pb + F::NC;   // lexicographic cell index (column of Y)
  const int4 td = tiles[blockIdx.x];   // type, first cell of the type's box (lexicographic), cells, -
  const PatchClass& pc = ecls[td.x];
  fg_bases<D, R>(g, pc, td, qb, pb, pl);
  __syncthreads();
  pdl_wait();
  // gather the element inputs: XE[a RA + slot NQK + node][cell]; GU elements per thread and round with all their
  // loads issued before the stores (the loop was bound by one load in flight)
  const int* rel = relidx + pc.rel_off;
  constexpr int GU = 8, TOT = F::XR * F::NC;
  const int nthr = blockDim.x;
  for (int base = threadIdx.x; base < TOT; base += GU * nthr) {
    long long src[GU];
    int dst[GU];
#pragma unroll
    for (int u = 0; u < GU; ++u) {
      const int idx = base + u * nthr;
      src[u] = -1;
      dst[u] = -1;
      if (idx < TOT) {
        const int row = idx / F::NC, col = idx % F::NC;
        const int e = fg_row_elem<D, R, K1>(row);
        dst[u] = row * F::XS + col;
        if (e >= 0 && col < td.z) {
          const int code = __ldg(rel + e);
          src[u] = (code >> 1) + ((code & 1) ? pb[col] : qb[col]);
        }
      }
    }
    double v[GU];
#pragma unroll
    for (int u = 0; u < GU; ++u) v[u] = src[u] >= 0 ? __ldg(x + src[u]) : 0.0;
#pragma unroll
    for (int u = 0; u < GU; ++u)
      if (dst[u] >= 0) XE[dst[u]] = v[u];
  }
  __syncthreads();
  fg_compute<D, R, K1, 2>(XE, pl, td, A1, A2, A3, AP, a2stride, a3stride, mix, Y, ncell);
}

// Persistent form (STGMG_K1_PERSIST=1): one CTA per SM walks the tiles with a double-buffered input stage — the
// next tile's element inputs are gathered by 8-byte cp.async into the other buffer while the current tile's GEMMs
// run, so the gather latency is hidden behind the DMMA work instead of behind a second co-resident CTA.
__device__ __forceinline__ void fg_cp_async8(double* dst, const double* src) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(src) : "memory");
}

template <int D, int R, int K1>
__global__ void __launch_bounds__(FG<D, R, K1, 16>::NT * 32, 2) op_fgemm_persist_kernel(
    LevelGeom g, const int4* __restrict__ tiles, int ntiles, const PatchClass* __restrict__ ecls,
    const int* __restrict__ relidx, const double* __restrict__ A1, const double* __restrict__ A2,
    const double* __restrict__ A3, const double* __restrict__ AP, long long a2stride, long long a3stride, FgMix mix,
    const double* __restrict__ x, double* __restrict__ Y, long long ncell) {
  // half tiles of 16 cells (two per 32-cell tile), two CTAs per SM, each double-buffered
  using F = FG<D, R, K1, 16>;
  extern __shared__ double smem[];
  double* XEb[2] = {smem, smem + (size_t)F::XR * F::XS};
  long long* meta = reinterpret_cast<long long*>(smem + 2 * (size_t)F::XR * F::XS);   // [buf][qb | pb | pl][NC]
  pdl_trigger();
  pdl_wait();
  const int nv = 2 * ntiles;
  auto half = [&](int v) {
    const int4 t = tiles[v >> 1];
    const int h = v & 1;
    return make_int4(t.x, t.y + 16 * h, max(0, min(16, t.z - 16 * h)), 0);
  };
  auto stage = [&](int v, int b) {   // bases, then the asynchronous gather of half tile v into buffer b
    const int4 td = half(v);
    const PatchClass& pc = ecls[td.x];
    long long* qb = meta + (size_t)b * 3 * F::NC;
    fg_bases<D, R, 16>(g, pc, td, qb, qb + F::NC, qb + 2 * F::NC);
    __syncthreads();
    const int* rel = relidx + pc.rel_off;
    double* XE = XEb[b];
    for (int idx = threadIdx.x; idx < F::XR * F::NC; idx += blockDim.x) {
      const int row = idx / F::NC, col = idx % F::NC;
      const int e = fg_row_elem<D, R, K1>(row);
      double* dst = XE + row * F::XS + col;
      if (e >= 0 && col < td.z) {
        const int code = __ldg(rel + e);
        fg_cp_async8(dst, x + (code >> 1) + ((code & 1) ? qb[F::NC + col] : qb[col]));
      } else {
        *dst = 0.0;
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  int v = blockIdx.x, b = 0;
  if (v < nv) stage(v, 0);
  for (; v < nv; v += gridDim.x, b ^= 1) {
    const int vn = v + gridDim.x;
    if (vn < nv) {
      stage(vn, b ^ 1);
      asm volatile("cp.async.wait_group 1;\n" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    }
    __syncthreads();
    const int4 td = half(v);
    if (td.z > 0)
      fg_compute<D, R, K1, 2, 16>(XEb[b], meta + (size_t)b * 3 * F::NC + 2 * F::NC, td, A1, A2, A3, AP, a2stride,
                                  a3stride, mix, Y, ncell);
    __syncthreads();   // buffer b is refilled by the stage of the next iteration
  }
}

// ------------------------------------------------------------------------------------------- host side -----
// Fragment-major copy of a row-major (rows x cols) block M into out[(mb * ksteps + ks) * 32 + lane] = the m8n8k4 A
// fragment element (row 8 mb + lane / 4, k 4 ks + lane % 4) of the padded matrix; the column map kcol (padded k ->
// source column or -1) and row map (padded row -> source row or -1) describe the zero padding.
static void to_fragments(const std::vector<int>& rowmap, const std::vector<int>& kcol,
                         const std::function<double(int, int)>& M, std::vector<double>& out) {
  const int mb = (int)rowmap.size() / 8, ksn = (int)kcol.size() / 4;
  const size_t base = out.size();
  out.resize(base + (size_t)mb * ksn * 32, 0.0);
  for (int m = 0; m < mb; ++m)
    for (int ks = 0; ks < ksn; ++ks)
      for (int l = 0; l < 32; ++l) {
        const int r = rowmap[8 * m + (l >> 2)], k = kcol[4 * ks + (l & 3)];
        out[base + ((size_t)m * ksn + ks) * 32 + l] = (r >= 0 && k >= 0) ? M(r, k) : 0.0;
      }
}

// Builds the factored matrices from the row-major slab element matrices E[t] (lda, element DoF order
// (a, V_c / U_c / P, node)) of every cell type, using (for K1 >= 2) the blocks
//   [phi_0, U_1] = T_01 M_rho,  [chi_0, U_0] = theta_0 A_gamma,  [chi_0, P_0] = theta_0 C^T,
//   [psi_0, V_0] = -theta_0 C,  [psi_0, P_1] = T_01 M_c,  [psi_0, P_0] = T_00 M_c + theta_0 B_gamma.
template <int D, int R, int K1>
static int fgemm_build(const std::vector<double>& E, int ntypes, int lda, const OpConsts& c, FgemmData& out) {
  using F = FG<D, R, K1>;
  static_assert(K1 >= 2, "the factored operator reads M_rho and M_c from the off-diagonal temporal blocks");
  const double T01 = c.T[0][1], T00 = c.T[0][0], th0 = c.theta[0];
  if (T01 == 0.0 || th0 == 0.0) return -1;
  auto el = [&](int t, int row, int col) { return E[((size_t)t * lda + row) * lda + col]; };
  const int oV = 0, oU = D * F::NQ, oP = 2 * D * F::NQ, b1 = F::NE1;   // element offsets; Radau node 1 at NE1
  // G1: scalar mass block of component 0 (rows phi_0 comp 0, cols U_1 comp 0) / T_01
  std::vector<int> rq(F::NQM), kq(F::NQK);
  for (int i = 0; i < F::NQM; ++i) rq[i] = i < F::NQ ? i : -1;
  for (int k = 0; k < F::NQK; ++k) kq[k] = k < F::NQ ? k : -1;
  out.A1.clear();
  to_fragments(rq, kq, [&](int r, int k) { return el(0, oV + r, b1 + oU + k) / T01; }, out.A1);
  // GP: M_c = [psi_0, P_1] / T_01
  std::vector<int> rp(F::NPM), kp(F::NPK);
  for (int i = 0; i < F::NPM; ++i) rp[i] = i < F::NP ? i : -1;
  for (int k = 0; k < F::NPK; ++k) kp[k] = k < F::NP ? k : -1;
  out.AP.clear();
  to_fragments(rp, kp, [&](int r, int k) { return el(0, oP + r, b1 + oP + k) / T01; }, out.AP);
  // G2 per type: rows (component c, node i) padded to NQM per component; k = U_d nodes (NQK each) then P (NPK)
  std::vector<int> r2(D * F::NQM), k2(D * F::NQK + F::NPK);
  for (int cc = 0; cc < D; ++cc)
    for (int i = 0; i < F::NQM; ++i) r2[cc * F::NQM + i] = i < F::NQ ? cc * F::NQ + i : -1;
  for (int d = 0; d < D; ++d)
    for (int j = 0; j < F::NQK; ++j) k2[d * F::NQK + j] = j < F::NQ ? d * F::NQ + j : -1;
  for (int j = 0; j < F::NPK; ++j) k2[D * F::NQK + j] = j < F::NP ? D * F::NQ + j : -1;   // P part
  std::vector<int> r3(F::NPM);
  for (int i = 0; i < F::NPM; ++i) r3[i] = i < F::NP ? i : -1;
  out.A2.clear();
  out.A3.clear();
  for (int t = 0; t < ntypes; ++t) {
    to_fragments(r2, k2, [&](int r, int k) {
      return k < D * F::NQ ? el(t, oU + r, oU + k) / th0 : el(t, oU + r, oP + (k - D * F::NQ)) / th0;
    }, out.A2);
    to_fragments(r3, k2, [&](int r, int k) {
      if (k < D * F::NQ) return el(t, oP + r, oV + k) / th0;                              // -C
      const int s = k - D * F::NQ;
      return (el(t, oP + r, oP + s) - T00 * el(t, oP + r, b1 + oP + s) / T01) / th0;   // B_gamma
    }, out.A3);
  }
  out.a2stride = (long long)D * F::MB * F::KS2 * 32;
  out.a3stride = (long long)F::MB3 * F::KS2 * 32;
  return 0;
}

int fgemm_build_any(int d, int r, int k1, const std::vector<double>& E, int ntypes, int lda, const OpConsts& c,
                    FgemmData& out) {
  if (d == 3 && r == 2 && k1 == 2) return fgemm_build<3, 2, 2>(E, ntypes, lda, c, out);
  if (d == 3 && r == 2 && k1 == 3) return fgemm_build<3, 2, 3>(E, ntypes, lda, c, out);
  if (d == 2 && r == 3 && k1 == 3) return fgemm_build<2, 3, 3>(E, ntypes, lda, c, out);
  return -1;
}

template <int D, int R, int K1>
static cudaError_t launch_fg(const LevelGeom& g, const int4* tiles, int ntiles, const PatchClass* ecls,
                             const int* relidx, const FgemmDev& m, const OpConsts& c, const double* x, double* Y,
                             cudaStream_t s) {
  using F = FG<D, R, K1>;
  static PerDeviceOnce attr;
  attr.run([] {
    cudaFuncSetAttribute(op_fgemm_kernel<D, R, K1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)F::SMEM);
  });
  long long ncell = 1;
  for (int a = 0; a < D; ++a) ncell *= g.n[a];
  FgMix mix;
  for (int b = 0; b < kMaxK1; ++b) {
    mix.th[b] = c.theta[b];
    for (int a = 0; a < kMaxK1; ++a) mix.T[b][a] = c.T[b][a];
  }
  static const bool persist = std::getenv("STGMG_K1_PERSIST") && std::atoi(std::getenv("STGMG_K1_PERSIST")) != 0;
  if (persist) {
    using FH = FG<D, R, K1, 16>;
    const size_t smem = 2 * sizeof(double) * (size_t)FH::XR * FH::XS + 2 * 3 * sizeof(long long) * FH::NC;
    static PerDeviceOnce attrp;
    attrp.run([smem] {
      cudaFuncSetAttribute(op_fgemm_persist_kernel<D, R, K1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    });
    int dev = 0, nsm = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    return launch_pdl(op_fgemm_persist_kernel<D, R, K1>, dim3(std::min(2 * ntiles, 2 * nsm)), dim3(F::NT * 32), smem, s, g,
                      tiles, ntiles, ecls, relidx, m.A1, m.A2, m.A3, m.AP, m.a2stride, m.a3stride, mix, x, Y, ncell);
  }
  return launch_pdl(op_fgemm_kernel<D, R, K1>, dim3(ntiles), dim3(F::NT * 32), F::SMEM, s, g, tiles, ecls, relidx,
                    m.A1, m.A2, m.A3, m.AP, m.a2stride, m.a3stride, mix, x, Y, ncell);
}

cudaError_t launch_op_fgemm(const LevelGeom& g, int r, int k1, const int4* tiles, int ntiles, const PatchClass* ecls,
                            const int* relidx, const FgemmDev& m, const OpConsts& c, const double* x, double* Y,
                            cudaStream_t s) {
  if (g.d == 3 && r == 2 && k1 == 2) return launch_fg<3, 2, 2>(g, tiles, ntiles, ecls, relidx, m, c, x, Y, s);
  if (g.d == 3 && r == 2 && k1 == 3) return launch_fg<3, 2, 3>(g, tiles, ntiles, ecls, relidx, m, c, x, Y, s);
  if (g.d == 2 && r == 3 && k1 == 3) return launch_fg<2, 3, 3>(g, tiles, ntiles, ecls, relidx, m, c, x, Y, s);
  return cudaErrorNotSupported;
}

int fgemm_cells_per_tile() { return 32; }

}  // namespace stgmg
