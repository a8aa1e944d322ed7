// Internal declarations of the B200 space-time GMRES–GMG library (sm_100a, fp64).
// Public ABI: include/stgmg.h.  Paper references: P:Ln = line n of PAPER.md (arXiv:2303.06742).
#pragma once
#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>
#include <mutex>
#include <string>
#include <vector>

namespace stgmg {

// Per-device "done once" flag: function attributes (dynamic shared memory opt-in) belong to each device's context,
// so a second handle on another GPU of the same process must set them again.  Race-free across host threads.
struct PerDeviceOnce {
  std::atomic<unsigned long long> mask{0};
  std::mutex mu;
  // runs f() once per device; concurrent callers wait until it has finished
  template <class F> void run(F f) {
    int d = 0;
    cudaGetDevice(&d);
    const unsigned long long bit = 1ull << (d & 63);
    if (mask.load(std::memory_order_acquire) & bit) return;
    std::lock_guard<std::mutex> g(mu);
    if (mask.load(std::memory_order_relaxed) & bit) return;
    f();
    mask.fetch_or(bit, std::memory_order_release);
  }
};

constexpr int kMaxR1 = 4;   // max nodes per axis of a Q_r cell (r <= 3)
constexpr int kMaxK1 = 4;   // max Radau nodes (k <= 3)

// Reference-element and problem constants passed by value to the operator kernels.
// 1D tables live on the reference interval [0,1]; derivatives are d/dx_hat (scaled by 1/h in the kernels).
struct OpConsts {
  double B[kMaxR1][kMaxR1];    // B[g][j]  = l_j(x_g)   Q_r Lagrange (GLL nodes) at Gauss points
  double Dm[kMaxR1][kMaxR1];   // Dm[g][j] = l_j'(x_g)
  double Bp[kMaxR1][kMaxR1];   // Q_{r-1}
  double Dp[kMaxR1][kMaxR1];
  double E[2][kMaxR1];         // l_j(0), l_j(1)
  double dE[2][kMaxR1];        // l_j'(0), l_j'(1)
  double Ep[2][kMaxR1];
  double dEp[2][kMaxR1];
  double wg[kMaxR1];           // Gauss weights on [0,1]
  double T[kMaxK1][kMaxK1];    // T[b][a] = w_b chi_a'(t_b) + chi_a(-1) chi_b(-1)
  double theta[kMaxK1];        // (tau/2) w_b
  double chim1[kMaxK1];        // chi_b(-1)
  double rho, alpha, c0, lam, mu, gamma_a, gamma_b;
  double K[9];                 // row-major d x d (stride 3)
  double ds;                   // 1: Problem B.1 (DS) — psi rows couple sum_a T_ba U_a instead of theta_b V_b (N4)
  double ds_face;              // DS only: weight of the G_D^u trace term alpha <(sum_a T_ba U_a).n, psi> (1 in the
                               // operator; 0 in the slab-RHS constants: P:L1073 has u_D(t_{n-1}), not u_h^{n-1})
};

// Constants of the on-device load assembly and initial data (csrc/loads.cu).
struct LoadConsts {
  double xg[kMaxR1 + 2], wg[kMaxR1 + 2];     // (r+2)-point Gauss rule on [0,1] (reading A10)
  double Bq[kMaxR1 + 2][kMaxR1];             // Q_r Lagrange basis (GLL nodes) at those points: Bq[q][j]
  double Bp[kMaxR1 + 2][kMaxR1];             // Q_{r-1}
  double Eq[2][kMaxR1];                      // Q_r basis at 0 / 1
  double gllq[kMaxR1], gllp[kMaxR1];         // GLL nodes of Q_r / Q_{r-1} on [0,1] (reading A9)
  double that[kMaxK1], theta[kMaxK1];        // right Radau nodes on [-1,1], theta_b = tau w_b / 2
  double lo[3];                              // physical origin of this rank's (window) fine level
  double rho, alpha, c0, lam, mu, K[9];
  int r, xhi_cell;                           // local index of the cell at x = hi (-1: not on this rank)
};


// Geometry of one structured level (box split into n[a] cells per axis).
struct LevelGeom {
  int d;
  int n[3];
  double h[3];
  double vol;                  // |K|_d
  int qn[3], pn[3];            // Q_r / Q_{r-1} nodes per axis
  long long qs[3], ps[3];      // lexicographic strides
  long long nq, np, R, S, block, N;
  int bcu[6], bcp[6];          // 0 = Dirichlet (Nitsche), 1 = Neumann
  double hF[6];                // penalty length per boundary face on this level
};

// One patch class on a level.  Patches of a class: vertices v with per-axis index in
// [vlo[a], vlo[a] + cnt[a]).  Patch-local layout (m, f, c, node lex in the patch box) (reading A12).
struct PatchClass {
  int cp;                      // C_P
  int ncols;                   // number of patches in the class
  int vlo[3], cnt[3];          // vertices vlo[a] + i * vst, i < cnt[a], per axis
  int vst;                     // vertex stride (1; 4 for the colour sub-classes of the multiplicative smoother)
  int cells[3];                // cells of the patch per axis (1 or 2)
  long long rel_off;           // offset of this class's relidx table (cp entries)
  long long inv_off;           // offset of the class inverse (lda x lda)
  long long rexp_off;          // offset of the class block of the expanded residual (dense K2), -1 if unused
  long long col_off;           // offset of the class's columns in the per-column gather-base table (expand_pull)
};

struct TileDesc {              // one CTA tile of the grouped patch GEMM: rows [m0, m0+BM), columns [n0, n0+nn)
  int cls, m0, n0, nn;
};

#define STGMG_CUDA(call)                                                                   \
  do {                                                                                     \
    cudaError_t _e = (call);                                                               \
    if (_e != cudaSuccess) {                                                               \
      ::stgmg::set_error(std::string(#call) + ": " + cudaGetErrorString(_e));              \
      return -3;                                                                           \
    }                                                                                      \
  } while (0)

void set_error(const std::string& msg);

// Programmatic dependent launch (sm_90+): the next kernel of the stream may begin launching while the previous
// one drains; every hot kernel calls pdl_wait() before it reads what its predecessor wrote.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;\n" ::: "memory"); }
// Let the next kernel of the stream launch now: its CTAs run their prologue (index math, static-table loads) while
// this grid drains and block in pdl_wait() until it has completed.  Safe because no kernel writes global memory
// before its own pdl_wait().
// Measured on B200: early triggers make every kernel a little faster in isolation but the heterogeneous V-cycle chain
// slower (cfg1 V-cycle 1.19 -> 1.46 ms), so they are opt-in (-DSTGMG_PDL_TRIGGER).
#ifndef STGMG_PDL_TRIGGER
__device__ __forceinline__ void pdl_trigger() {}
#else
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;\n" ::: "memory"); }
#endif

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                              Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// ---- kernels launchers (each returns cudaError_t of the launch) ----
// K1 (warp per cell, 2^d colours): y += sign * A_l x, or (Yc != null) element results Yc[plin(cell)][NE].
cudaError_t launch_op_apply(int d, int r, int k1, const LevelGeom& g, const OpConsts* cdev, const double* x, double* y,
                            double* Yc, double sign, int batch, long long stride, long long ycstride, cudaStream_t s,
                            int* nlaunch);
// K2: Y[patch][mu_hat] = Ainv_class * R_P r for all patches (grouped DMMA GEMM); variant = tile shape.
int k2_pick_variant(long long npatch, int maxcp);
void k2_tile_shape(int variant, int* bm, int* bn);
int k2_slots(int variant);   // resident CTA slots on the GPU for a tile variant
// Tiles of a grouped GEMM balanced over the resident CTA slots: cp[c] x ncols[c] per class, BM x (<= BN) tiles;
// consecutive groups of cn tiles share (class, row block) (cn = 1 everywhere since the A multicast was dropped).
std::vector<TileDesc> balanced_tiles(const std::vector<int>& cp, const std::vector<int>& ncols, int bm, int bn,
                                     int slots, int cn);
// A matrices of the grouped GEMM: row-major lda x lda -> chunk-major swizzled (dst needs nmat*lda*lda + slack).
cudaError_t launch_chunk_swizzle(const double* src, double* dst, int nmat, int lda, cudaStream_t s);
constexpr int EXPAND_COLS = 32;      // patch columns per expand_pull block (x 16 slots = 512 elements)
constexpr int kK2Slack = 224 * 16;   // doubles after the last chunk-major matrix (tile rows past lda)
cudaError_t launch_patch_gemm(const LevelGeom& g, int r, int variant, const PatchClass* cls_dev, const TileDesc* tiles,
                              int ntiles, const int* relidx, const double* invc, int lda, const double* rvec,
                              double* Y, int ldy, cudaStream_t s);
// Multiplicative colour-ordered smoother: d[dof(P, mu_hat)] += omega * Y[P][mu_hat] for the patches
// (sub-class, column) of one colour; same-colour patches are DoF-disjoint, so there are no conflicting writes.
cudaError_t launch_colour_update(const LevelGeom& g, int r, const PatchClass* cls, const int2* items, int nitems,
                                 const int* relidx, const double* Y, int ldy, double omega, double* dvec,
                                 cudaStream_t s);
// K2D: dense K2 on the patch-expanded residual (variant 2 = 112 x 32 tiles, 6 = 112 x 64), bulk copies only.
cudaError_t launch_patch_gemm_dense(const LevelGeom& g, int variant, const PatchClass* cls_dev, const TileDesc* tiles,
                                    int ntiles, const double* invc, int lda, const double* rexp, double* Y, int ldy,
                                    cudaStream_t s);
int k2d_slots(int variant);
// K1e: residual written in patch-expanded, class chunk-major swizzled form (B operand of the dense K2).
// Rexp[class block, chunk q, column col, slot] = r[dof(patch col, mu_hat)] for a dense level, one thread per element
// in Rexp order (coalesced stores); blocks = {class, chunk, first column, columns}, colbase[col_off + col] = (bq, bp)
cudaError_t launch_expand_pull(const int4* blocks, int nblocks, const PatchClass* cls, const int* relidx,
                               const int2* colbase, const double* r, double* rexp, cudaStream_t s);
cudaError_t launch_gather_expand(const LevelGeom& g, int r, int k1, const double* Yc, const double* base, double alpha,
                                 double beta, int ldpm, const PatchClass* cls, double* rexp, cudaStream_t s);
cudaError_t launch_load_cells(int d, int r, int k1, const LevelGeom& g, const LoadConsts* lc, int kind, double tn,
                              double tau, double* Yc, cudaStream_t s);
cudaError_t launch_initial_state(int d, int k1, const LevelGeom& g, const LoadConsts* lc, int kind, double t0, double* x,
                                 cudaStream_t s);
// K3 of the element-wise Vanka smoother: cells as patches, Y[plin(K + 1)][element-local index].
cudaError_t launch_avg_cells(const LevelGeom& g, int r, int k1, const double* Y, int ldy, double omega, int zero_init,
                             double* dvec, cudaStream_t s);
// K3: d <- (zero ? 0 : d) + omega * (sum_P Y_P[mu_hat]) / p_mu   (pull form, lexicographic patch order).
cudaError_t launch_vanka_average(const LevelGeom& g, int r, int k1, const double* Y, int ldy, double omega,
                                 int zero_init, double* dvec, cudaStream_t s, int overwrite = 0);
// K4 (setup): gather A_P of each class from the dense mini-level matrix; equilibrated Gauss–Jordan inverse.
cudaError_t launch_extract_patch(const LevelGeom& mini, int r, int k1, const double* Adense, long long ldA,
                                 const int* vrep, int nclass, const int* cps, const long long* rel_offs,
                                 const int* relidx_mini, double* inv, int lda, cudaStream_t s);
struct GjScratch {                     // device scratch of the blocked Gauss–Jordan (ping-pong copy, permutations);
  double* buf = nullptr;               // owned by the caller, grown on demand, reused across calls
  int* pi = nullptr;
  size_t buf_bytes = 0, pi_bytes = 0;
};
int gauss_jordan_inverse(double* mats, int nmat, int n_max, const int* n_each, int lda, int* perm, double* colk,
                         double* scale, int* status, cudaStream_t s, GjScratch* scratch = nullptr);
// K5: restriction / prolongation with per-axis sparse 1D interpolation tables.
struct Interp1D {              // CSR tables of the 1D prolongation for one axis and degree (device)
  const int* rp_f; const int* ci_f; const double* v_f;   // rows = fine nodes
  const int* rp_c; const int* ci_c; const double* v_c;   // rows = coarse nodes (transpose)
  int nz_c;                                               // nonzeros of the coarse-row table
};
struct TransferTables { Interp1D q[3], p[3]; };
cudaError_t launch_restrict(const LevelGeom& fine, const LevelGeom& coarse, int k1, const TransferTables& t,
                            const double* rf, double* bc, cudaStream_t s);
cudaError_t launch_prolong_add(const LevelGeom& fine, const LevelGeom& coarse, int k1, const TransferTables& t,
                               const double* dc, double* df, cudaStream_t s);
cudaError_t launch_restrict_sep(const LevelGeom& fine, const LevelGeom& coarse, int k1, const TransferTables& t,
                                const double* rf, double* bc, double* tmp, cudaStream_t s);
// K6: y = A x dense (coarse solve, row-major lda).
cudaError_t launch_gemv(const double* A, int n, int lda, const double* x, double* y, cudaStream_t s);

// ---- the 3D L-shaped benchmark (csrc/lshape.cu) ----
struct LsHostCsr {
  std::vector<int> rp, ci;
  std::vector<double> v;
};
struct LsLevelHost {                  // one level of the L-shape hierarchy, assembled on the host at setup
  int ref = 0, nq = 0, np = 0, ncell = 0, maxcp = 0;
  long long N = 0, ysize = 0;
  LsHostCsr A;                        // slab operator A_l (N x N)
  LsHostCsr P;                        // prolongation level l-1 -> l (rows: this level); l >= 1
  std::vector<int> pz, pcp;           // vertex patches: concatenated DoF lists Z(P), sizes C_P
  std::vector<long long> pzoff;       // start of Z(P) in pz (= start of y_P in the patch results)
  std::vector<int> k3tab;             // averaging table, 27 x N (Y offsets, lexicographic patches, -1 = none)
};
struct LsHost {
  std::vector<LsLevelHost> lev;
  LsHostCsr J;                        // slab-RHS coupling F = L + J X_{n-1} (fine level)
  std::vector<double> fN;             // -<t_N, chi> per unit sin(8 pi t), U components (3 nq), fine level
  std::vector<double> wu, wp;         // goal weights on Gamma_m: U_x nodes (nq), P DoFs (np)
};
int lshape_build_host(int ref_coarse, int levels, int r, int k, const OpConsts& oc, int hf_mode, LsHost& out,
                      std::string& err);
cudaError_t launch_csr_extract_patches(const int* rp, const int* ci, const double* v, const int* pz,
                                       const long long* pzoff, const int* pcp, int p0, int np, double* out, int lda,
                                       cudaStream_t s);
cudaError_t launch_patch_gemv(int npatch, int maxcp, const int* pz, const long long* pzoff, const int* pcp,
                              const double* inv, int lda, const double* r, double* Y, cudaStream_t s);
cudaError_t launch_csr_to_dense(int n, const int* rp, const int* ci, const double* v, double* out, cudaStream_t s);
cudaError_t launch_lshape_load(long long N, long long block, long long R, int k1, const double* fN, const double* coef,
                               double* L, cudaStream_t s);
cudaError_t launch_lshape_goal(const double* x, long long ou, long long op, int nq, int np, const double* wu,
                               const double* wp, double* out, cudaStream_t s);

// ---- K1 as factored element GEMMs (csrc/op_fgemm.cu) ----
struct FgemmData {                    // fragment-major A operands (host)
  std::vector<double> A1, A2, A3, AP; // mass (shared), [A_gamma | C^T] and [-C | B_gamma] per cell type, M_c (shared)
  long long a2stride = 0, a3stride = 0;
};
struct FgemmDev {
  const double *A1 = nullptr, *A2 = nullptr, *A3 = nullptr, *AP = nullptr;
  long long a2stride = 0, a3stride = 0;
};
int fgemm_build_any(int d, int r, int k1, const std::vector<double>& E, int ntypes, int lda, const OpConsts& c,
                    FgemmData& out);
int fgemm_cells_per_tile();
cudaError_t launch_op_fgemm(const LevelGeom& g, int r, int k1, const int4* tiles, int ntiles, const PatchClass* ecls,
                            const int* relidx, const FgemmDev& m, const OpConsts& c, const double* x, double* Y,
                            cudaStream_t s);   // Y[element DoF][cell] (cell-fastest)
// K1 on the volume-only cell types by sum factorisation (csrc/op_sf3.cu; 3D Q2), same tiles / Y layout as op_fgemm.
bool sf3_supported(int d, int r, int k1);
cudaError_t launch_op_sf3(const LevelGeom& g, int r, int k1, const int4* tiles, int ntiles, const PatchClass* ecls,
                          const OpConsts& c, const double* x, double* Y, cudaStream_t s);

}  // namespace stgmg
