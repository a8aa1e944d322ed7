// C ABI (include/stgmg.h) and host orchestration of the B200 space-time GMRES–GMG slab solver.
//   setup   : level geometry, reference tables (Eq:GF P:L122-128, Def:VhQh P:L148), temporal constants
//             (P:L412-430 read per SURVEY App. A.1), patch classes (Eq:DefPlm, App. A.4), class
//             inverses on the device, coarse inverse, transfer tables, CUDA graph
//             of the V-cycle.
//   vcycle  : P:L435-440 with Algorithm 1 on l = L..1 and the coarse direct solve on T_0.
//   solve   : flexible GMRES(m), right preconditioned (readings A2-A4, A35).
#include <algorithm>
#include <array>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <functional>
#include <memory>

#include <nvtx3/nvToolsExt.h>

#include "../../include/stgmg.h"
#include "dist.cuh"
#include "stgmg_internal.cuh"

namespace stgmg {

// NVTX range for the lifetime of a scope (host-side phases: setup steps, solve, Arnoldi steps, per-level timing
// V-cycle).  Header-only NVTX v3; a no-op unless a profiler is attached.
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }

cudaError_t launch_mgs_dot(double* w, const double* vprev, const double* hprev, const double* vnext, long long n,
                           double* partials, unsigned* counter, double* out, int do_sqrt, const unsigned char* mask,
                           cudaStream_t s);
cudaError_t launch_sqrt(double* v, cudaStream_t s);
cudaError_t launch_scale(double* y, const double* x, const double* sc, int invert, long long n, cudaStream_t s);
cudaError_t launch_givens(double* H, int ldh, double* cs, double* sn, double* gv, int j, double* scal, cudaStream_t s);
cudaError_t launch_givens_cond(double* H, int ldh, double* cs, double* sn, double* gv, int j, double* scal, int* ctl,
                               int has_next, cudaGraphConditionalHandle next, cudaStream_t s);
cudaError_t launch_backsub_ctl(const double* H, int ldh, const double* gv, double* y, const int* ctl, cudaStream_t s);
cudaError_t launch_update_x_ctl(double* x, const double* Z, const double* y, const int* ctl, long long n,
                                cudaStream_t s);
cudaError_t launch_backsub(const double* H, int ldh, const double* gv, double* y, int jn, cudaStream_t s);
cudaError_t launch_update_x(double* x, const double* Z, const double* y, int jn, long long n, cudaStream_t s);
cudaError_t launch_set_scalar(double* dst, const double* src, cudaStream_t s);
cudaError_t launch_identity(double* X, long long n, cudaStream_t s);
cudaError_t launch_noop(int blocks, cudaStream_t s);
cudaError_t launch_csr_spmv(int nrows, int lpr, const int* rp, const int* ci, const double* v, const double* x,
                            const double* base, double* y, double alpha, double beta, cudaStream_t s);
cudaError_t launch_avg_table(int d, int N, const int* tab, const double* Y, double omega, int zero_init, double* dvec,
                             cudaStream_t s, int overwrite = 0);
cudaError_t launch_energy_place(const LevelGeom& g, int k1, const double* x, double* y, int mode, cudaStream_t s);
cudaError_t launch_face_integrals(int d, int r, int k1, const LevelGeom& g, const LoadConsts* lc, const double* x,
                                  int face, int c0, int c1, double* part, int nface_cells, double* out,
                                  cudaStream_t s);
cudaError_t launch_extract_elem(const double* Ycb, long long ycstride, int ne, int ntypes, const long long* rep,
                                const int* mdofs, double* E, int lda, cudaStream_t s);
cudaError_t launch_op2d_cells(int r, int k1, const LevelGeom& g, const OpConsts* cdev, const double* x, double* Yc,
                              int batch, long long stride, long long ycstride, cudaStream_t s);
cudaError_t launch_op_gather(const LevelGeom& g, int r, int k1, const double* Yc, const double* base, double* y,
                             double alpha, double beta, int batch, long long stride, long long ycstride,
                             cudaStream_t s, int ldpm);

// ------------------------------------------------------------------------------ host numerics (1D tables) ----
static void legendre(int n, double x, double& p, double& dp) {
  double p0 = 1.0, p1 = x;
  if (n == 0) { p = 1.0; dp = 0.0; return; }
  for (int k = 2; k <= n; ++k) {
    const double p2 = ((2.0 * k - 1.0) * x * p1 - (k - 1.0) * p0) / k;
    p0 = p1;
    p1 = p2;
  }
  p = p1;
  dp = (std::fabs(x) < 1.0) ? n * (x * p1 - p0) / (x * x - 1.0) : 0.0;
}

// all roots of f in (-1, 1) by sign scan + bisection (n <= 8 roots; robust, to full precision)
static std::vector<double> roots_in(const std::function<double(double)>& f) {
  std::vector<double> out;
  const int M = 20000;
  double xa = -1.0 + 1e-14, fa = f(xa);
  for (int i = 1; i <= M; ++i) {
    const double xb = -1.0 + 2.0 * i / M - (i == M ? 1e-14 : 0.0);
    const double fb = f(xb);
    if (fa == 0.0) out.push_back(xa);
    else if (fa * fb < 0.0) {
      double lo = xa, hi = xb, flo = fa;
      for (int it = 0; it < 200; ++it) {
        const double mid = 0.5 * (lo + hi);
        const double fm = f(mid);
        if (fm == 0.0 || hi - lo < 1e-17) { lo = hi = mid; break; }
        if ((fm < 0) == (flo < 0)) { lo = mid; flo = fm; } else hi = mid;
      }
      out.push_back(0.5 * (lo + hi));
    }
    xa = xb;
    fa = fb;
  }
  return out;
}

static void gauss01(int n, std::vector<double>& x, std::vector<double>& w) {
  auto r = roots_in([n](double t) { double p, dp; legendre(n, t, p, dp); return p; });
  x.clear(); w.clear();
  for (double t : r) {
    // Newton polish
    for (int it = 0; it < 3; ++it) { double p, dp; legendre(n, t, p, dp); t -= p / dp; }
    double p, dp;
    legendre(n, t, p, dp);
    x.push_back(0.5 * (t + 1.0));
    w.push_back(0.5 * 2.0 / ((1.0 - t * t) * dp * dp));
  }
}

static std::vector<double> gll01(int r) {   // Gauss–Lobatto nodes on [0,1] (reading A9)
  std::vector<double> x{0.0};
  if (r >= 2) {
    auto rr = roots_in([r](double t) { double p, dp; legendre(r, t, p, dp); return dp; });
    for (double t : rr) x.push_back(0.5 * (t + 1.0));
  }
  x.push_back(1.0);
  return x;
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
    for (size_t l = 0; l < nd.size(); ++l)
      if ((int)l != j && l != m) t *= (x - nd[l]) / (nd[j] - nd[l]);
    s += t;
  }
  return s;
}

// right Gauss–Radau on [-1,1]: nodes = roots of P_{k+1} - P_k (includes +1); weights (1+t)/((k+1)^2 P_k(t)^2),
// 2/(k+1)^2 at t = 1 (Eq:GF).
static void radau(int k, std::vector<double>& t, std::vector<double>& w) {
  t.clear(); w.clear();
  if (k > 0) {
    auto rr = roots_in([k](double x) { double a, da, b, db; legendre(k + 1, x, a, da); legendre(k, x, b, db); return a - b; });
    for (double x : rr) {
      double pk, dpk;
      legendre(k, x, pk, dpk);
      t.push_back(x);
      w.push_back((1.0 + x) / ((k + 1.0) * (k + 1.0) * pk * pk));
    }
  }
  t.push_back(1.0);
  w.push_back(2.0 / ((k + 1.0) * (k + 1.0)));
}

static OpConsts make_consts(int d, int r, int k, const stgmg_params& p) {
  OpConsts c;
  std::memset(&c, 0, sizeof(c));
  std::vector<double> xg, wg;
  gauss01(r + 1, xg, wg);
  const auto nq = gll01(r), np = gll01(r - 1);
  for (int g = 0; g <= r; ++g) {
    c.wg[g] = wg[g];
    for (int j = 0; j <= r; ++j) {
      c.B[g][j] = lag(nq, j, xg[g]);
      c.Dm[g][j] = dlag(nq, j, xg[g]);
    }
    for (int j = 0; j < r; ++j) {
      c.Bp[g][j] = lag(np, j, xg[g]);
      c.Dp[g][j] = dlag(np, j, xg[g]);
    }
  }
  for (int s = 0; s < 2; ++s) {
    for (int j = 0; j <= r; ++j) {
      c.E[s][j] = lag(nq, j, (double)s);
      c.dE[s][j] = dlag(nq, j, (double)s);
    }
    for (int j = 0; j < r; ++j) {
      c.Ep[s][j] = lag(np, j, (double)s);
      c.dEp[s][j] = dlag(np, j, (double)s);
    }
  }
  std::vector<double> t, w;
  radau(k, t, w);
  for (int b = 0; b <= k; ++b) {
    c.theta[b] = 0.5 * p.tau * w[b];
    c.chim1[b] = lag(t, b, -1.0);
  }
  for (int b = 0; b <= k; ++b)
    for (int a = 0; a <= k; ++a) c.T[b][a] = w[b] * dlag(t, a, t[b]) + c.chim1[a] * c.chim1[b];
  c.rho = p.rho; c.alpha = p.alpha; c.c0 = p.c0; c.lam = p.lambda; c.mu = p.mu;
  c.ds = p.formulation == STGMG_FORM_DS ? 1.0 : 0.0;
  c.ds_face = 1.0;
  c.gamma_a = p.gamma_a < 0 ? 5.0e4 * r * (r + 1) : p.gamma_a;
  c.gamma_b = p.gamma_b < 0 ? 0.5 * r * (r - 1) : p.gamma_b;
  for (int i = 0; i < 9; ++i) c.K[i] = 0.0;
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) c.K[i * 3 + j] = p.K[i * 3 + j];
  return c;
}

static LevelGeom make_geom(int d, const int n[3], const double h[3], int r, int k1, const int bcu[6], const int bcp[6],
                           int hF_mode) {
  LevelGeom g;
  std::memset(&g, 0, sizeof(g));
  g.d = d;
  g.vol = 1.0;
  g.nq = 1; g.np = 1;
  for (int a = 0; a < 3; ++a) {
    g.n[a] = a < d ? n[a] : 1;
    g.h[a] = a < d ? h[a] : 1.0;
    g.qn[a] = a < d ? r * n[a] + 1 : 1;
    g.pn[a] = a < d ? (r - 1) * n[a] + 1 : 1;
  }
  for (int a = 0; a < d; ++a) {
    g.vol *= h[a];
    g.qs[a] = g.nq; g.ps[a] = g.np;
    g.nq *= g.qn[a]; g.np *= g.pn[a];
  }
  g.R = (long long)d * g.nq;
  g.S = g.np;
  g.block = 2 * g.R + g.S;
  g.N = (long long)k1 * g.block;
  for (int f = 0; f < 6; ++f) {
    g.bcu[f] = bcu[f];
    g.bcp[f] = bcp[f];
    g.hF[f] = hF_mode == STGMG_HF_EDGE ? g.h[f / 2] : g.vol;   // h_F = |K|_d on boundary faces
  }
  return g;
}

// 1D prolongation tables for one axis (n_coarse cells, degree deg): CSR by fine rows and by coarse rows.
struct Interp1DHost {
  std::vector<int> rp_f, ci_f, rp_c, ci_c;
  std::vector<double> v_f, v_c;
};

static Interp1DHost make_interp(int nc, int deg) {
  const auto nodes = gll01(deg);
  const int nf_nodes = deg * 2 * nc + 1, nc_nodes = deg * nc + 1;
  std::vector<std::vector<std::pair<int, double>>> rows(nf_nodes);
  for (int f = 0; f < nf_nodes; ++f) {
    const int cf = std::min(f / deg, 2 * nc - 1);   // fine cell holding fine node f
    const int i = f - deg * cf;
    const int cc = cf / 2;
    const double xhat = 0.5 * ((cf % 2) + nodes[i]);
    for (int j = 0; j <= deg; ++j) {
      const double v = lag(nodes, j, xhat);
      if (v != 0.0) rows[f].push_back({deg * cc + j, v});
    }
  }
  Interp1DHost o;
  o.rp_f.push_back(0);
  std::vector<std::vector<std::pair<int, double>>> cols(nc_nodes);
  for (int f = 0; f < nf_nodes; ++f) {
    for (auto& e : rows[f]) {
      o.ci_f.push_back(e.first);
      o.v_f.push_back(e.second);
      cols[e.first].push_back({f, e.second});
    }
    o.rp_f.push_back((int)o.ci_f.size());
  }
  o.rp_c.push_back(0);
  for (int c = 0; c < nc_nodes; ++c) {
    for (auto& e : cols[c]) {
      o.ci_c.push_back(e.first);
      o.v_c.push_back(e.second);
    }
    o.rp_c.push_back((int)o.ci_c.size());
  }
  return o;
}


// The 1D tables of make_interp restricted to x-windows: fine local nodes [0, nf*deg] = global + w0f*deg, coarse
// local nodes [0, nc*deg] = global + w0c*deg (entries outside a window are dropped; they only feed ghost values).
static Interp1DHost make_interp_window(int nc_global, int deg, int w0f, int nf, int w0c, int ncw) {
  const Interp1DHost G = make_interp(nc_global, deg);
  Interp1DHost o;
  o.rp_f.push_back(0);
  for (int f = 0; f <= nf * deg; ++f) {
    const int fg = f + w0f * deg;
    for (int e = G.rp_f[fg]; e < G.rp_f[fg + 1]; ++e) {
      const int J = G.ci_f[e] - w0c * deg;
      if (J >= 0 && J <= ncw * deg) {
        o.ci_f.push_back(J);
        o.v_f.push_back(G.v_f[e]);
      }
    }
    o.rp_f.push_back((int)o.ci_f.size());
  }
  o.rp_c.push_back(0);
  for (int J = 0; J <= ncw * deg; ++J) {
    const int Jg = J + w0c * deg;
    for (int e = G.rp_c[Jg]; e < G.rp_c[Jg + 1]; ++e) {
      const int f = G.ci_c[e] - w0f * deg;
      if (f >= 0 && f <= nf * deg) {
        o.ci_c.push_back(f);
        o.v_c.push_back(G.v_c[e]);
      }
    }
    o.rp_c.push_back((int)o.ci_c.size());
  }
  return o;
}
}  // namespace stgmg

using namespace stgmg;

struct LevelData {
  LevelGeom g;
  double *b = nullptr, *d = nullptr, *r = nullptr, *Y = nullptr;
  int ldy = 0, lda = 0, maxcp = 0, ntiles = 0, k2var = 0;
  long long npatch = 0;
  std::vector<PatchClass> cls;
  PatchClass* cls_dev = nullptr;
  TileDesc* tiles_dev = nullptr;
  int* relidx_dev = nullptr;
  double* inv_dev = nullptr;
  TransferTables tt;
  // 3D operator: per-cell-type element matrices applied as a grouped DMMA GEMM (cells play the role of patches)
  std::vector<PatchClass> ecls;
  PatchClass* ecls_dev = nullptr;
  TileDesc* etiles_dev = nullptr;
  int entiles = 0, elda = 0, ek2var = 0;
  int* erelidx_dev = nullptr;
  double* E_dev = nullptr;
  // K1 as factored element GEMMs (csrc/op_fgemm.cu): tiles {type, first cell, cells} and fragment-major operands
  bool fg = false;
  int4* fg_tiles = nullptr;
  int fg_ntiles = 0;
  int4* sf_tiles = nullptr;        // K1 tiles of the volume-only cell types on the sum-factorised kernel (op_sf3.cu)
  int sf_ntiles = 0;
  FgemmDev fgm;
  // x-slab domain decomposition; a replicated level has part = false, w0 = 0, gnx = n[0]
  bool part = false, has_left = false, has_right = false;
  int gnx = 0, w0 = 0, c0 = 0, c1 = 0;   // global cells along x, window start (global cell), owned cells (local)
  long long npatch_global = 0, ncell_global = 0;
  double *sl = nullptr, *sr = nullptr, *rl = nullptr, *rr = nullptr;   // halo message buffers
  long long nsl = 0, nsr = 0, nrl = 0, nrr = 0;
  double *agsend = nullptr, *agrecv = nullptr;   // transition to an agglomerated (replicated) coarser level
  long long nag = 0;
  // small-level fast path (csrc/small.cu): assembled CSR operator, CSR transfers to/from level l-1, averaging table
  Interp1DHost ih_q[3], ih_p[3];                 // host copies of the 1D transfer tables (CSR assembly)
  int *A_rp = nullptr, *A_ci = nullptr, A_lpr = 32;
  double* A_v = nullptr;
  int *P_rp = nullptr, *P_ci = nullptr, P_lpr = 4;   // prolongation: rows = DoFs of this level
  double* P_v = nullptr;
  int *R_rp = nullptr, *R_ci = nullptr, R_lpr = 8;   // restriction: rows = DoFs of level l-1
  double* R_v = nullptr;
  int* k3tab = nullptr;
  // multiplicative colour-ordered smoother: per vertex colour, the colour's sub-classes, K2 tiles and
  // (sub-class, column) items of the update kernel
  struct Colour {
    PatchClass* cls_dev = nullptr;
    TileDesc* tiles_dev = nullptr;
    int ntiles = 0, k2var = 0;
    int2* items_dev = nullptr;
    int nitems = 0;
  };
  std::vector<Colour> colours;
  // dense K2: the residual expanded per (patch, mu_hat), class chunk-major swizzled (csrc/nodal.cu gather_expand)
  bool dense = false;
  double* Rexp = nullptr;
  long long nrexp = 0;
  int4* exp_blocks = nullptr;   // expand_pull blocks {class, chunk, first column, columns}
  int n_exp_blocks = 0;
  int2* colbase = nullptr;      // per patch column (class-major): gather bases (bq, bp)
  bool exp_fused = false;       // STGMG_EXPAND_FUSED=1: the push-form gather_expand instead
  // unstructured level (SURVEY N3, L-shape): CSR operator / transfers / averaging table above, plus one explicit
  // inverse per vertex patch (K2u, csrc/lshape.cu)
  double* rtmp = nullptr;       // intermediates of the separable restriction (levels with 200k..16M DoFs)
  bool unstr = false;
  int* pz = nullptr;            // concatenated Z(P)
  long long* pzoff = nullptr;   // start of Z(P) and of y_P
  int* pcp = nullptr;           // C_P
  double* pinv = nullptr;       // npatch x plda x plda, row-major
  int plda = 0, pmax = 0;
};

struct stgmg_handle {
  int d = 2, r = 2, k = 1, k1 = 2, L = 1;
  stgmg_params prm;
  OpConsts c;
  std::vector<LevelData> lev;
  double* A0inv = nullptr;
  int n0 = 0;
  // folded coarse sub-cycle: the V-cycle restricted to levels <= fold_lv is a fixed linear map b_f -> d_f; it is
  // assembled at setup (run on every unit vector) and applied as one GEMV (fold_ready once assembled)
  int fold_lv = 0;
  bool fold_ready = false;
  // device-resident Arnoldi loop (single GPU): one graph per restart length m, an IF node per step whose handle the
  // previous step's Givens kernel sets (no host round trip per step)
  cudaGraphExec_t cyc_exec = nullptr;
  int cyc_m = 0;
  // Opt-in (STGMG_SOLVE_GRAPH=1; 2 = V-cycle kernels captured into each step instead of a child graph): measured
  // SLOWER on cfg1 (solve 2.81 -> 3.09 ms): once a graph with conditional nodes is loaded, every launch on the stream,
  // the plain V-cycle graph included, runs about 40 us per V-cycle slower, more than the per-step host round trip
  // (about 36 us) it removes.  Default: the host-checked loop.
  bool cyc_off = true;           // off by default, or the graph could not be built
  bool cyc_inline = false;
  std::vector<int> cyc_step_launches;
  // STGMG_PROFILE_SOLVE=1: device timestamps of the phases of each Arnoldi step, printed after the solve
  bool prof = false;
  cudaEvent_t pev[64] = {};
  int npev = 0;
  int* ctl = nullptr;            // [0] Arnoldi steps of the solve, [1] steps of the current cycle
  double* Vfold = nullptr;
  cudaStream_t s = nullptr;
  bool own_stream = false;
  // Krylov workspace
  int m_alloc = 0;
  double *V = nullptr, *Z = nullptr, *w = nullptr, *rv = nullptr, *H = nullptr, *cs = nullptr, *sn = nullptr,
         *gv = nullptr, *yv = nullptr, *scal = nullptr, *partials = nullptr;
  unsigned* counter = nullptr;
  double* pinned = nullptr;
  double *stage_rhs = nullptr, *stage_x = nullptr, *rhs_int = nullptr;
  cudaGraphExec_t vgraph = nullptr;
  cudaGraph_t vgraph_tmpl = nullptr;
  // V-cycle graphs of the Arnoldi steps with the fine level's b / d bound to v_j / z_j (captured at first use): no
  // copies of v_j in and z_j out around each preconditioner application.  STGMG_STEP_GRAPHS=0: the copying form.
  std::vector<cudaGraphExec_t> vg_step;
  std::vector<int> vg_step_launches;
  int vg_step_m = 0;
  bool step_graphs = true;
  int vgraph_launches = 0;
  long long launches = 0;
  std::vector<void*> allocs;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  OpConsts* c_dev = nullptr;    // operator constants (device copy, read by the 2D cell kernel)
  OpConsts* cj_dev = nullptr;   // slab-RHS variant: T'_ba = chi_b(-1) delta_{a,k}, theta = 0 (K8)
  OpConsts cj;                  // host copy (the sum-factorised K8 takes its constants by value)
  LoadConsts* lc_dev = nullptr; // on-device load assembly / initial data
  OpConsts* ce_dev = nullptr;   // discrete energy (N1, P7): [0] T = 0, theta_k = 1 ; [1] T_kk = 1, theta = 0
  double* Yc = nullptr;         // element results of the 2D cell kernel (largest level)
  double* Ycell = nullptr;      // element results of the 3D element GEMM, patch-major (largest level)
  // multi-GPU
  Transport* tr = nullptr;
  int rank = 0, nranks = 1;
  unsigned char* mask = nullptr;   // owned fine-level DoFs (Krylov inner products)
  bool graphable = true;
  bool op_gemm = false;            // runtime K1 = element GEMM on the tensor pipe + node gather (3D; large 2D elements)
  GjScratch gj;                    // blocked Gauss–Jordan scratch, reused by every setup inverse, freed after setup
  // K4 inverses of stgmg_setup in flight: the coarse inverse and every level's class inverses run on their own
  // non-blocking streams, overlapping each other and the host-side setup of the next levels; finish_inverses joins
  // them (swizzle, singularity check) before the V-cycle graph is captured.  STGMG_SETUP_SERIAL=1: on h->s.
  struct PendingInv {
    int level = 0;                 // 0 = coarse inverse (A0inv), >= 1 = class inverses of that level
    int n = 0, lda = 0;            // matrices, leading dimension
    cudaStream_t st = nullptr;     // owned unless it is h->s
    cudaEvent_t done = nullptr;
    GjScratch scr;
    double* inv_rm = nullptr;      // row-major class inverses (level >= 1), swizzled into Lv.inv_dev at the join
    int* status = nullptr;         // device, n entries (h->allocs)
  };
  std::vector<PendingInv> pend;
  int fg_on = 1;                   // K1 element GEMM in the factored form (STGMG_K1_FGEMM=0: the full element matrix;
                                   // 2: on every element-route level regardless of size, for tests)
  int sf_on = 1;                   // 3D Q2: volume-only cell types by sum factorisation on levels with >= 128k cells
                                   // (STGMG_K1_SF=0: all factored; 2: every factored level, for tests)
  int nsm = 148;                   // SMs of the device (tile balancing)
  // the 3D L-shaped benchmark (stgmg_setup_lshape); levels are unstructured (LevelData::unstr)
  bool lshape = false;
  int ls_nq = 0, ls_np = 0;
  int *J_rp = nullptr, *J_ci = nullptr, J_lpr = 32;   // slab-RHS coupling F = L + J X_{n-1}
  double* J_v = nullptr;
  double *ls_fN = nullptr, *ls_wu = nullptr, *ls_wp = nullptr;
  double ls_that[kMaxK1] = {};     // right Radau nodes on [-1, 1]
  // per-level share of one V-cycle (stgmg_stats.level_seconds): events at entry / before the recursion / after it /
  // exit of every level, recorded by one eager (not graph-launched) V-cycle after the first solve
  bool lvprof = false, lev_ready = false;
  cudaEvent_t lev_ev[16][4] = {};
  double lev_ms[16] = {};

  // Releases everything the handle owns: stgmg_destroy, and every error return of stgmg_setup (whose unique_ptr
  // drops a partly built handle).  The caller's communicator and stream are not owned.
  ~stgmg_handle() {
    if (s) cudaStreamSynchronize(s);
    if (vgraph) cudaGraphExecDestroy(vgraph);
    if (cyc_exec) cudaGraphExecDestroy(cyc_exec);
    if (vgraph_tmpl) cudaGraphDestroy(vgraph_tmpl);
    for (auto g : vg_step)
      if (g) cudaGraphExecDestroy(g);
    for (void* p : allocs) cudaFree(p);
    if (gj.buf) cudaFree(gj.buf);
    if (gj.pi) cudaFree(gj.pi);
    for (auto& p : pend) {
      if (p.st) cudaStreamSynchronize(p.st);
      if (p.st && p.st != s) cudaStreamDestroy(p.st);
      if (p.done) cudaEventDestroy(p.done);
      if (p.scr.buf) cudaFree(p.scr.buf);
      if (p.scr.pi) cudaFree(p.scr.pi);
      if (p.inv_rm) cudaFree(p.inv_rm);
    }
    delete tr;
    if (pinned) cudaFreeHost(pinned);
    if (e0) cudaEventDestroy(e0);
    if (e1) cudaEventDestroy(e1);
    for (auto e : pev)
      if (e) cudaEventDestroy(e);
    for (auto& le : lev_ev)
      for (auto e : le)
        if (e) cudaEventDestroy(e);
    if (own_stream) cudaStreamDestroy(s);
  }
};

static constexpr int kGhost = 3;   // ghost cells per interior side: one halo exchange of d per smoothing sweep


template <typename T>
static int dalloc(stgmg_handle* h, T** p, size_t count) {
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc((void**)p, count * sizeof(T));
  if (e != cudaSuccess) {
    set_error(std::string("cudaMalloc: ") + cudaGetErrorString(e));
    return STGMG_ENOMEM;
  }
  h->allocs.push_back((void*)*p);
  return 0;
}

template <typename T>
static int upload(stgmg_handle* h, T** p, const std::vector<T>& v) {
  int rc = dalloc(h, p, v.size());
  if (rc) return rc;
  if (!v.empty()) STGMG_CUDA(cudaMemcpy(*p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return 0;
}

#define CK(x)                \
  do {                       \
    int _rc = (x);           \
    if (_rc) return _rc;     \
  } while (0)
#define CKE(x)                                                                      \
  do {                                                                              \
    cudaError_t _e = (x);                                                           \
    if (_e != cudaSuccess) {                                                        \
      set_error(std::string(#x) + ": " + cudaGetErrorString(_e));                   \
      return STGMG_ECUDA;                                                           \
    }                                                                               \
  } while (0)

// ------------------------------------------------------------------------------------- operator wrappers ----
static long long cell_count(const LevelGeom& g) {
  long long n = 1;
  for (int a = 0; a < g.d; ++a) n *= g.n[a];
  return n;
}

static long long elem_dofs(const stgmg_handle* h) {
  long long nq = 1, np = 1;
  for (int a = 0; a < h->d; ++a) { nq *= (h->r + 1); np *= h->r; }
  return (long long)h->k1 * (2 * h->d * nq + np);
}

// y = beta * base + alpha * A_g x on an arbitrary geometry (setup: mini levels, batched unit vectors; K8).
// 2D: cell kernel + deterministic node gather; 3D: coloured warp-per-cell kernel.
static int apply_geom(stgmg_handle* h, const LevelGeom& g, const OpConsts* cdev, const double* x, double* y,
                      const double* base, double alpha, double beta, int batch = 1, long long stride = 0,
                      double* Yc = nullptr) {
  if (h->d == 2) {
    double* yc = Yc ? Yc : h->Yc;
    const long long ycs = cell_count(g) * elem_dofs(h);
    cudaError_t e = launch_op2d_cells(h->r, h->k1, g, cdev, x, yc, batch, stride, ycs, h->s);
    if (e == cudaErrorNotSupported) { set_error("(d, r, k) combination not compiled"); return STGMG_ENOTSUP; }
    CKE(e);
    CKE(launch_op_gather(g, h->r, h->k1, yc, base, y, alpha, beta, batch, stride, ycs, h->s, 0));
    h->launches += 2;
    return 0;
  }
  if (base) {
    if (beta != 1.0 || batch != 1) { set_error("3D apply_geom: base needs beta = 1, batch = 1"); return STGMG_EINVAL; }
    CKE(cudaMemcpyAsync(y, base, sizeof(double) * g.N, cudaMemcpyDeviceToDevice, h->s));
  } else {
    CKE(cudaMemsetAsync(y, 0, sizeof(double) * g.N * batch, h->s));
  }
  int nl = 0;
  cudaError_t e = launch_op_apply(h->d, h->r, h->k1, g, cdev, x, y, nullptr, alpha, batch, stride, 0, h->s, &nl);
  h->launches += nl;
  if (e == cudaErrorNotSupported) { set_error("(d, r, k) combination not compiled"); return STGMG_ENOTSUP; }
  CKE(e);
  return 0;
}

// Element results Ycell[vertex(K + 1)][e] of the element-matrix route of K1: the factored element GEMMs (op_fgemm)
// or the full slab element matrix as a grouped GEMM.
// Returns the leading dimension the node gathers take (0: cell-fastest Y[e][cell], ne: Y[vertex(K + 1)][e]).
static int element_results(stgmg_handle* h, LevelData& Lv, const double* x, int* ldpm) {
  const int ne = (int)elem_dofs(h);
  *ldpm = Lv.fg ? 0 : ne;
  if (Lv.fg) {
    if (Lv.sf_ntiles) {
      CKE(launch_op_sf3(Lv.g, h->r, h->k1, Lv.sf_tiles, Lv.sf_ntiles, Lv.ecls_dev, h->c, x, h->Ycell, h->s));
      if (Lv.fg_ntiles) h->launches += 1;
    }
    if (Lv.fg_ntiles)
      CKE(launch_op_fgemm(Lv.g, h->r, h->k1, Lv.fg_tiles, Lv.fg_ntiles, Lv.ecls_dev, Lv.erelidx_dev, Lv.fgm, h->c, x,
                          h->Ycell, h->s));
  } else
    CKE(launch_patch_gemm(Lv.g, h->r, Lv.ek2var, Lv.ecls_dev, Lv.etiles_dev, Lv.entiles, Lv.erelidx_dev, Lv.E_dev,
                          Lv.elda, x, h->Ycell, ne, h->s));
  return 0;
}

// y = beta * base + alpha * A_l x on hierarchy level l (the runtime operator apply, K1).
static int apply_level(stgmg_handle* h, int l, const double* x, double* y, const double* base, double alpha,
                       double beta) {
  if (h->lev[l].A_rp) {   // small level: assembled operator, one SpMV
    const LevelData& Ls = h->lev[l];
    CKE(launch_csr_spmv((int)Ls.g.N, Ls.A_lpr, Ls.A_rp, Ls.A_ci, Ls.A_v, x, base, y, alpha, beta, h->s));
    h->launches += 1;
    return 0;
  }
  if (!h->op_gemm) return apply_geom(h, h->lev[l].g, h->c_dev, x, y, base, alpha, beta);
  LevelData& Lv = h->lev[l];
  int ldpm = 0;
  CK(element_results(h, Lv, x, &ldpm));
  CKE(launch_op_gather(Lv.g, h->r, h->k1, h->Ycell, base, y, alpha, beta, 1, 0, 0, h->s, ldpm));
  h->launches += 2;
  return 0;
}

static int apply_into(stgmg_handle* h, const LevelGeom& g, const double* x, double* y, int batch = 1,
                      long long stride = 0, double* Yc = nullptr) {
  return apply_geom(h, g, h->c_dev, x, y, nullptr, 1.0, 0.0, batch, stride, Yc);
}

static int residual(stgmg_handle* h, int l, const double* b, const double* x, double* r) {
  return apply_level(h, l, x, r, b, -1.0, 1.0);
}

// Ghost refresh of a level vector of the x-slab decomposition (no-op on replicated levels): every rank sends the
// kGhost cells of owned nodes its neighbours hold as ghosts and overwrites its own ghost nodes.
static int exchange(stgmg_handle* h, int l, double* v) {
  LevelData& Lv = h->lev[l];
  if (!Lv.part || h->nranks == 1) return 0;
  const int G = kGhost, dq = h->r, dp = h->r - 1, nloc = Lv.g.n[0];
  if (Lv.has_left) CKE(launch_halo(Lv.g, h->k1, Lv.c0 * dq, G * dq + 1, Lv.c0 * dp, G * dp + 1, v, Lv.sl, 0, h->s));
  if (Lv.has_right)
    CKE(launch_halo(Lv.g, h->k1, (Lv.c1 - G) * dq, G * dq, (Lv.c1 - G) * dp, G * dp, v, Lv.sr, 0, h->s));
  const int rc = h->tr->halo(Lv.sl, Lv.nsl, Lv.sr, Lv.nsr, Lv.rl, Lv.nrl, Lv.rr, Lv.nrr, h->s);
  if (rc) return rc;
  if (Lv.has_left) CKE(launch_halo(Lv.g, h->k1, 0, Lv.c0 * dq, 0, Lv.c0 * dp, v, Lv.rl, 1, h->s));
  if (Lv.has_right)
    CKE(launch_halo(Lv.g, h->k1, Lv.c1 * dq, (nloc - Lv.c1) * dq + 1, Lv.c1 * dp, (nloc - Lv.c1) * dp + 1, v, Lv.rr, 1,
                    h->s));
  h->launches += 2 * ((Lv.has_left ? 1 : 0) + (Lv.has_right ? 1 : 0));
  return 0;
}

// Partitioned fine level lf -> replicated coarse level lf-1: every rank restricted into the global coarse vector
// bc, valid on its owned coarse x-nodes [q oc deg, (q+1) oc deg]; allgather the slabs so that bc is complete.
static int agglomerate(stgmg_handle* h, int lf, double* bc) {
  LevelData& F = h->lev[lf];
  const LevelGeom& gc = h->lev[lf - 1].g;
  const int oc = h->lev[lf - 1].gnx / h->nranks, dq = h->r, dp = h->r - 1;
  CKE(launch_halo(gc, h->k1, h->rank * oc * dq, oc * dq + 1, h->rank * oc * dp, oc * dp + 1, bc, F.agsend, 0, h->s));
  const int rc = h->tr->allgather(F.agsend, F.nag, F.agrecv, h->s);
  if (rc) return rc;
  for (int q = 0; q < h->nranks; ++q)
    CKE(launch_halo(gc, h->k1, q * oc * dq, oc * dq + 1, q * oc * dp, oc * dp + 1, bc, F.agrecv + (long long)q * F.nag, 1,
                    h->s));
  h->launches += 1 + h->nranks;
  return 0;
}

// K5 restriction b_{l-1} = P^T r_l, K5 prolongation d_l += P d_{l-1}, K3 averaging (small levels: table driven)
static int restrict_level(stgmg_handle* h, int l, const double* rf, double* bc) {
  LevelData& Lv = h->lev[l];
  if (Lv.R_rp)
    CKE(launch_csr_spmv((int)h->lev[l - 1].g.N, Lv.R_lpr, Lv.R_rp, Lv.R_ci, Lv.R_v, rf, nullptr, bc, 1.0, 0.0, h->s));
  else if (Lv.rtmp) {   // large levels: axis-by-axis restriction (coalesced passes)
    CKE(launch_restrict_sep(Lv.g, h->lev[l - 1].g, h->k1, Lv.tt, rf, bc, Lv.rtmp, h->s));
    h->launches += h->d - 1;
  } else {
    CKE(launch_restrict(Lv.g, h->lev[l - 1].g, h->k1, Lv.tt, rf, bc, h->s));
  }
  h->launches += 1;
  return 0;
}

static int prolong_level(stgmg_handle* h, int l, const double* dc, double* df) {
  LevelData& Lv = h->lev[l];
  if (Lv.P_rp)
    CKE(launch_csr_spmv((int)Lv.g.N, Lv.P_lpr, Lv.P_rp, Lv.P_ci, Lv.P_v, dc, df, df, 1.0, 1.0, h->s));
  else
    CKE(launch_prolong_add(Lv.g, h->lev[l - 1].g, h->k1, Lv.tt, dc, df, h->s));
  h->launches += 1;
  return 0;
}

static int average_level(stgmg_handle* h, int l, bool zero, double* d) {
  LevelData& L = h->lev[l];
  const int ow = h->prm.smoother == STGMG_SMOOTH_OVERWRITE ? 1 : 0;   // N2(iii): no averaging
  if (h->prm.smoother == STGMG_SMOOTH_ELEMENT)
    CKE(launch_avg_cells(L.g, h->r, h->k1, L.Y, L.ldy, h->prm.omega, zero ? 1 : 0, d, h->s));
  else if (L.k3tab)
    CKE(launch_avg_table(h->d, (int)L.g.N, L.k3tab, L.Y, h->prm.omega, zero ? 1 : 0, d, h->s, ow));
  else
    CKE(launch_vanka_average(L.g, h->r, h->k1, L.Y, L.ldy, h->prm.omega, zero ? 1 : 0, d, h->s, ow));
  h->launches += 1;
  return 0;
}

// Multiplicative colour-ordered sweep: per colour, r = b - A d (r = b for the first colour of a
// sweep from d = 0), the colour's patch solves, d[Z(P)] += omega y_P.
static int sweep_colored(stgmg_handle* h, int l, const double* b, double* d, bool zero_start) {
  LevelData& L = h->lev[l];
  if (zero_start) CKE(cudaMemsetAsync(d, 0, sizeof(double) * L.g.N, h->s));
  bool first = true;
  for (const auto& C : L.colours) {
    if (C.nitems == 0) continue;
    const double* rin = b;
    if (!(zero_start && first)) {
      CK(residual(h, l, b, d, L.r));
      rin = L.r;
    }
    first = false;
    CKE(launch_patch_gemm(L.g, h->r, C.k2var, C.cls_dev, C.tiles_dev, C.ntiles, L.relidx_dev, L.inv_dev, L.lda, rin,
                          L.Y, L.ldy, h->s));
    CKE(launch_colour_update(L.g, h->r, C.cls_dev, C.items_dev, C.nitems, L.relidx_dev, L.Y, L.ldy, h->prm.omega, d,
                             h->s));
    h->launches += 2;
  }
  return 0;
}

// r = b - A_l d written straight into the patch-expanded B operand of the dense K2 (d == nullptr: r = b)
static int residual_expand(stgmg_handle* h, int l, const double* b, const double* d) {
  LevelData& L = h->lev[l];
  if (!L.exp_fused) {   // r = b - A d (node gather), then the pull-form expansion
    const double* src = b;
    if (d) {
      CK(residual(h, l, b, d, L.r));
      src = L.r;
    }
    CKE(launch_expand_pull(L.exp_blocks, L.n_exp_blocks, L.cls_dev, L.relidx_dev, L.colbase, src, L.Rexp, h->s));
    h->launches += 1;
    return 0;
  }
  if (!d) {
    CKE(launch_gather_expand(L.g, h->r, h->k1, nullptr, b, 0.0, 1.0, 0, L.cls_dev, L.Rexp, h->s));
    h->launches += 1;
    return 0;
  }
  if (!h->op_gemm) {
    const long long ycs = cell_count(L.g) * elem_dofs(h);
    CKE(launch_op2d_cells(h->r, h->k1, L.g, h->c_dev, d, h->Yc, 1, 0, ycs, h->s));
    CKE(launch_gather_expand(L.g, h->r, h->k1, h->Yc, b, -1.0, 1.0, 0, L.cls_dev, L.Rexp, h->s));
  } else {
    int ldpm = 0;
    CK(element_results(h, L, d, &ldpm));
    CKE(launch_gather_expand(L.g, h->r, h->k1, h->Ycell, b, -1.0, 1.0, ldpm, L.cls_dev, L.Rexp, h->s));
  }
  h->launches += 2;
  return 0;
}

static int sweep(stgmg_handle* h, int l, const double* b, double* d, bool zero_start) {
  if (h->prm.smoother == STGMG_SMOOTH_COLORED_MULT) return sweep_colored(h, l, b, d, zero_start);
  LevelData& L = h->lev[l];
  if (L.unstr) {   // L-shape level: CSR residual, per-patch inverses (K2u), averaging table
    const double* rin = b;
    if (!zero_start) {
      CK(residual(h, l, b, d, L.r));
      rin = L.r;
    }
    CKE(launch_patch_gemv((int)L.npatch, L.pmax, L.pz, L.pzoff, L.pcp, L.pinv, L.plda, rin, L.Y, h->s));
    h->launches += 1;
    return average_level(h, l, zero_start, d);
  }
  if (L.dense) {
    CK(residual_expand(h, l, b, zero_start ? nullptr : d));
    CKE(launch_patch_gemm_dense(L.g, L.k2var, L.cls_dev, L.tiles_dev, L.ntiles, L.inv_dev, L.lda, L.Rexp, L.Y, L.ldy,
                                h->s));
    h->launches += 1;
    CK(average_level(h, l, zero_start, d));
    return exchange(h, l, d);
  }
  const double* rin = b;
  if (!zero_start) {
    CK(residual(h, l, b, d, L.r));
    rin = L.r;
  }
  CKE(launch_patch_gemm(L.g, h->r, L.k2var, L.cls_dev, L.tiles_dev, L.ntiles, L.relidx_dev, L.inv_dev, L.lda, rin, L.Y,
                        L.ldy, h->s));
  h->launches += 1;
  CK(average_level(h, l, zero_start, d));
  return exchange(h, l, d);
}

// V-cycle on levels top..0: input lev[top].b, output lev[top].d.  Below the fold level the assembled
// sub-cycle matrix replaces the recursion (same linear map, applied as one GEMV).
static int enqueue_levels(stgmg_handle* h, int top) {
  auto mark = [&](int i) -> int {   // per-level timing V-cycle only (never inside a captured graph)
    if (h->lvprof && top < 16) CKE(cudaEventRecord(h->lev_ev[top][i], h->s));
    return 0;
  };
  CK(mark(0));
  if (top == 0) {
    CKE(launch_gemv(h->A0inv, h->n0, h->n0, h->lev[0].b, h->lev[0].d, h->s));
    h->launches += 1;
    return mark(3);
  }
  LevelData& Lv = h->lev[top];
  if (h->fold_ready && top == h->fold_lv) {
    CKE(launch_gemv(h->Vfold, (int)Lv.g.N, (int)Lv.g.N, Lv.b, Lv.d, h->s));
    h->launches += 1;
    return mark(3);
  }
  for (int j = 0; j < h->prm.jmax; ++j) CK(sweep(h, top, Lv.b, Lv.d, j == 0));
  CK(residual(h, top, Lv.b, Lv.d, Lv.r));
  CK(restrict_level(h, top, Lv.r, h->lev[top - 1].b));
  if (Lv.part && h->lev[top - 1].part) CK(exchange(h, top - 1, h->lev[top - 1].b));
  else if (Lv.part) CK(agglomerate(h, top, h->lev[top - 1].b));
  CK(mark(1));
  CK(enqueue_levels(h, top - 1));
  CK(mark(2));
  CK(prolong_level(h, top, h->lev[top - 1].d, Lv.d));
  for (int j = 0; j < h->prm.jmax; ++j) CK(sweep(h, top, Lv.b, Lv.d, false));
  return mark(3);
}

static int enqueue_vcycle(stgmg_handle* h) { return enqueue_levels(h, h->L - 1); }

// Per-level device time of one V-cycle (SPEC SolveStats' per-level smoother timings): level l's own
// work = pre-smoothing, residual, restriction (+ halo / agglomeration) and prolongation + post-smoothing, i.e. the
// time between its entry and exit events minus the coarser levels' recursion; level 0 (or the folded sub-cycle's
// level) is the coarse solve.  Measured once per handle by an eager V-cycle on the levels' own b / d buffers.
static int profile_levels(stgmg_handle* h) {
  NvtxRange nv("stgmg level timing V-cycle");
  if (!h->lev_ev[0][0])
    for (auto& le : h->lev_ev)
      for (auto& e : le) CKE(cudaEventCreate(&e));
  for (int l = 0; l < h->L && l < 16; ++l) h->lev_ms[l] = 0.0;
  h->lvprof = true;
  const long long saved = h->launches;
  const int rc = enqueue_vcycle(h);
  h->lvprof = false;
  h->launches = saved;
  CK(rc);
  CKE(cudaStreamSynchronize(h->s));
  const int lo = h->fold_ready ? h->fold_lv : 0;
  for (int l = lo; l < h->L && l < 16; ++l) {
    float a = 0.f, b = 0.f;
    if (l == lo) {
      CKE(cudaEventElapsedTime(&a, h->lev_ev[l][0], h->lev_ev[l][3]));
    } else {
      CKE(cudaEventElapsedTime(&a, h->lev_ev[l][0], h->lev_ev[l][1]));
      CKE(cudaEventElapsedTime(&b, h->lev_ev[l][2], h->lev_ev[l][3]));
    }
    h->lev_ms[l] = (double)a + (double)b;
  }
  h->lev_ready = true;
  return 0;
}

// Assemble the folded sub-cycle: column i of Vfold (row-major, n x n) = the V-cycle of levels <= fold_lv applied to
// e_i.  Chosen as the finest replicated level l >= 1 with n_l^2 doubles <= STGMG_FOLD_MB (64 MB by default; 0 = off).
static int build_fold(stgmg_handle* h) {
  NvtxRange nv("stgmg setup: fold");
  if (h->lshape) return 0;   // unstructured levels: no fold
  long long budget = 64ll << 20;
  if (const char* ev = std::getenv("STGMG_FOLD_MB")) budget = std::atoll(ev) << 20;
  h->fold_lv = 0;
  for (int l = 1; l < h->L - 1; ++l) {   // never the fine level (the Krylov operator's own smoother)
    const long long n = h->lev[l].g.N;
    if (!h->lev[l].part && n * n * (long long)sizeof(double) <= budget) h->fold_lv = l;
  }
  if (h->fold_lv == 0) return 0;
  LevelData& F = h->lev[h->fold_lv];
  const long long n = F.g.N;
  CK(dalloc(h, &h->Vfold, (size_t)(n * n)));
  double* one = nullptr;
  CK(dalloc(h, &one, 1));
  const double v1 = 1.0;
  CKE(cudaMemcpy(one, &v1, sizeof(double), cudaMemcpyHostToDevice));
  const long long before = h->launches;
  for (long long i = 0; i < n; ++i) {
    CKE(cudaMemsetAsync(F.b, 0, sizeof(double) * n, h->s));
    CKE(cudaMemcpyAsync(F.b + i, one, sizeof(double), cudaMemcpyDeviceToDevice, h->s));
    CK(enqueue_levels(h, h->fold_lv));
    CKE(cudaMemcpy2DAsync(h->Vfold + i, sizeof(double) * n, F.d, sizeof(double), sizeof(double), (size_t)n,
                          cudaMemcpyDeviceToDevice, h->s));
  }
  CKE(cudaStreamSynchronize(h->s));
  h->launches = before;
  h->fold_ready = true;
  return 0;
}

// ------------------------------------------------------------------------------------------ setup pieces ----
// Tiles of the grouped GEMM (K2, and the 3D element GEMM of K1) balanced over the GPU's resident CTA slots.  A
// unit = (class, row block); its columns are cut into tiles of whole 8-column DMMA blocks, the tile count rounded up
// to a multiple of the cluster size cn (the cn CTAs of a cluster share the unit's A rows by multicast).  The minimal
// tiling (BN columns per tile) fixes the number of waves; W, the largest work of any tile, is then the smallest value
// for which the tiles still fit those waves (binary search), so the last wave is as full as the units allow.  The
// split only decides which CTA computes a column, never the arithmetic.
std::vector<TileDesc> stgmg::balanced_tiles(const std::vector<int>& cp, const std::vector<int>& ncols, int bm, int bn,
                                            int slots, int cn) {
  struct Unit { int cls, m0; long long n, ng; double wpc; };
  std::vector<Unit> u;
  double wpcmax = 0.0, wsum = 0.0;
  cn = std::max(cn, 1);
  const long long gpt = std::max(1, bn / 8);   // 8-column groups per full tile
  for (size_t c = 0; c < cp.size(); ++c)
    for (int m0 = 0; m0 < cp[c]; m0 += bm) {
      const double wpc = (double)std::min(bm, cp[c] - m0) * (double)cp[c];
      u.push_back({(int)c, m0, ncols[c], (ncols[c] + 7) / 8, wpc});
      wpcmax = std::max(wpcmax, wpc);
      wsum += wpc * (double)ncols[c];
    }
  auto tiles_of = [&](const Unit& x, double W) {
    const long long gmax = std::max(1LL, std::min(gpt, (long long)std::floor(W / (8.0 * x.wpc))));
    const long long nt = (x.ng + gmax - 1) / gmax;
    return ((nt + cn - 1) / cn) * cn;
  };
  auto count = [&](double W) {
    long long n = 0;
    for (const auto& x : u) n += tiles_of(x, W);
    return n;
  };
  slots = std::max(slots, 1);
  const double whi = 8.0 * (double)gpt * wpcmax * 1.0000001;
  const long long t0 = count(whi);
  long long target = ((t0 + slots - 1) / slots) * (long long)slots;
  if (const char* ev = std::getenv("STGMG_TILE_TARGET")) target = std::max(t0, (long long)std::atoll(ev));
  double lo = 0.0, hi = whi;
  for (int it = 0; it < 60; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (count(mid) <= target) hi = mid; else lo = mid;
  }
  struct Group { double w; std::vector<TileDesc> t; };
  std::vector<Group> groups;
  double wmax_tile = 0.0;
  for (const auto& x : u) {
    const long long nt = tiles_of(x, hi);
    const long long gb = x.ng / nt, gr = x.ng % nt;
    long long n0 = 0;
    Group gcur;
    gcur.w = 0.0;
    for (long long i = 0; i < nt; ++i) {
      const long long nn = std::max(0LL, std::min(8 * (gb + (i < gr ? 1 : 0)), x.n - n0));
      gcur.t.push_back(TileDesc{x.cls, x.m0, (int)std::min(n0, x.n), (int)nn});
      gcur.w = std::max(gcur.w, x.wpc * (double)nn);
      wmax_tile = std::max(wmax_tile, x.wpc * (double)nn);
      n0 += nn;
      if ((long long)gcur.t.size() == cn) {
        groups.push_back(gcur);
        gcur.t.clear();
        gcur.w = 0.0;
      }
    }
  }
  // heaviest first (load balance over the resident slots); among equal weights, column-tile major: the row blocks
  // (m0) of one column tile run back to back, so its B operand (the expanded residual, GBs on the fine 3D levels)
  // comes from DRAM once and from L2 for the other row blocks (ncu, cfg4 fine K2D: 48.2 GB DRAM per launch with
  // m0-major order, 6.3x the algorithmic bytes).  Order only: every tile computes the same sums.
  std::stable_sort(groups.begin(), groups.end(), [](const Group& a, const Group& b) {
    if (a.w != b.w) return a.w > b.w;
    const TileDesc &x = a.t.front(), &y = b.t.front();
    if (x.cls != y.cls) return x.cls < y.cls;
    if (x.n0 != y.n0) return x.n0 < y.n0;
    return x.m0 < y.m0;
  });
  std::vector<TileDesc> out;
  for (const auto& gq : groups)
    for (const auto& t : gq.t) out.push_back(t);
  if (std::getenv("STGMG_TILE_DEBUG"))
    std::fprintf(stderr, "[stgmg] tiles bm=%d bn=%d cn=%d slots=%d minimal=%lld target=%lld tiles=%zu max_work=%.3g "
                         "avg=%.3g\n",
                 bm, bn, cn, slots, t0, target, out.size(), wmax_tile, out.empty() ? 0.0 : wsum / (double)out.size());
  return out;
}

// STGMG_SETUP_TIMES=1: sub-phase marks inside a setup phase (device synchronised), "what: ms since the last mark".
struct SetupMarks {
  bool on = std::getenv("STGMG_SETUP_TIMES") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what, int level) {
    if (!on) return;
    cudaDeviceSynchronize();
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "stgmg setup:   %-28s level %2d  %9.1f ms\n", what, level,
                 std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

// Enqueues the batched Gauss–Jordan inverse (K4) of nmat matrices behind the work already on h->s, on a stream of
// its own (see stgmg_handle::PendingInv); finish_inverses joins it.
static int launch_inverse_async(stgmg_handle* h, int level, double* mats, int nmat, int n_max, const int* n_each,
                                int lda, int* perm, double* colk, double* scale, int* status, double* inv_rm) {
  static const bool serial = std::getenv("STGMG_SETUP_SERIAL") != nullptr;
  h->pend.emplace_back();
  stgmg_handle::PendingInv& p = h->pend.back();
  p.level = level;
  p.n = nmat;
  p.lda = lda;
  p.status = status;
  p.inv_rm = inv_rm;
  CKE(cudaEventCreateWithFlags(&p.done, cudaEventDisableTiming));
  if (serial) {
    p.st = h->s;
  } else {
    CKE(cudaStreamCreateWithFlags(&p.st, cudaStreamNonBlocking));
    CKE(cudaEventRecord(p.done, h->s));   // inputs ready
    CKE(cudaStreamWaitEvent(p.st, p.done, 0));
  }
  if (gauss_jordan_inverse(mats, nmat, n_max, n_each, lda, perm, colk, scale, status, p.st, &p.scr)) {
    set_error(level ? "gauss_jordan_inverse launch failed" : "coarse gauss_jordan_inverse launch failed");
    return STGMG_ECUDA;
  }
  CKE(cudaEventRecord(p.done, p.st));
  return 0;
}

// Joins the inverses launched by launch_inverse_async: class inverses into the chunk-major K2 layout, singular
// matrices reported (level and pivot step), scratch released.
static int finish_inverses(stgmg_handle* h) {
  if (h->pend.empty()) return 0;
  std::vector<std::vector<int>> st(h->pend.size());
  for (size_t i = 0; i < h->pend.size(); ++i) {
    auto& p = h->pend[i];
    CKE(cudaStreamWaitEvent(h->s, p.done, 0));
    if (p.level > 0) CKE(launch_chunk_swizzle(p.inv_rm, h->lev[p.level].inv_dev, p.n, p.lda, h->s));
    st[i].resize(p.n);
    CKE(cudaMemcpyAsync(st[i].data(), p.status, sizeof(int) * p.n, cudaMemcpyDeviceToHost, h->s));
  }
  CKE(cudaStreamSynchronize(h->s));
  std::string err;
  for (size_t i = 0; i < h->pend.size() && err.empty(); ++i) {
    const auto& p = h->pend[i];
    for (int c = 0; c < p.n && err.empty(); ++c)
      if (st[i][c] != 0)
        err = p.level == 0 ? "singular coarse matrix (pivot step " + std::to_string(st[i][c]) + ")"
                           : "singular patch matrix: level " + std::to_string(p.level) + " class " +
                                 std::to_string(c) + " (pivot step " + std::to_string(st[i][c]) + ")";
  }
  for (auto& p : h->pend) {
    if (p.st != h->s) CKE(cudaStreamDestroy(p.st));
    CKE(cudaEventDestroy(p.done));
    if (p.scr.buf) CKE(cudaFree(p.scr.buf));
    if (p.scr.pi) CKE(cudaFree(p.scr.pi));
    if (p.inv_rm) CKE(cudaFree(p.inv_rm));
  }
  h->pend.clear();
  if (!err.empty()) {
    set_error(err);
    return STGMG_ESINGULAR;
  }
  return 0;
}

static int build_patches(stgmg_handle* h, int l) {
  NvtxRange nv("stgmg setup: patch classes + inverses (K4)");
  SetupMarks sm;
  LevelData& Lv = h->lev[l];
  const LevelGeom& g = Lv.g;
  const int d = h->d, r = h->r, k1 = h->k1;
  // per-axis classes: (vlo, cnt, mini vertex, cells)
  struct AxCls { int vlo, cnt, vmini, cells; };
  std::vector<AxCls> ax[3];
  int nmini[3] = {1, 1, 1};
  const bool cellp = h->prm.smoother == STGMG_SMOOTH_ELEMENT;   // element-wise Vanka
  for (int a = 0; a < d; ++a) {
    const int n = g.n[a];
    if (cellp) {   // one patch per cell, "vertex" = cell + 1; per-axis classes {0}, {1..n-2}, {n-1}
      nmini[a] = std::min(n, 3);
      if (n < 3) {
        for (int c = 0; c < n; ++c) ax[a].push_back({c + 1, 1, c + 1, 1});
      } else {
        ax[a].push_back({1, 1, 1, 1});
        ax[a].push_back({2, n - 2, 2, 1});
        ax[a].push_back({n, 1, 3, 1});
      }
      continue;
    }
    nmini[a] = std::min(n, 4);
    if (n < 4) {
      for (int v = 0; v <= n; ++v) ax[a].push_back({v, 1, v, (v > 0 ? 1 : 0) + (v < n ? 1 : 0)});
    } else {
      ax[a].push_back({0, 1, 0, 1});
      ax[a].push_back({1, 1, 1, 2});
      ax[a].push_back({2, n - 3, 2, 2});
      ax[a].push_back({n - 1, 1, 3, 2});
      ax[a].push_back({n, 1, 4, 1});
    }
  }
  if (d < 3) ax[2].push_back({0, 1, 0, 1});
  if (d < 2) ax[1].push_back({0, 1, 0, 1});
  // mini level: same h, same boundary conditions, min(n,4) cells per axis
  LevelGeom mini = make_geom(d, nmini, g.h, r, k1, g.bcu, g.bcp, h->prm.hF_mode);
  std::vector<int> relidx, minidofs, cps;
  std::vector<long long> offs;
  Lv.cls.clear();
  Lv.maxcp = 0;
  Lv.npatch = 1;
  for (int a = 0; a < d; ++a) Lv.npatch *= (g.n[a] + 1);
  for (auto& cz : ax[2])
    for (auto& cy : ax[1])
      for (auto& cx : ax[0]) {
        const AxCls* A3[3] = {&cx, &cy, &cz};
        PatchClass pc;
        std::memset(&pc, 0, sizeof(pc));
        pc.ncols = 1;
        pc.vst = 1;
        long long nQ = 1, nP = 1;
        int qbox[3] = {1, 1, 1}, pbox[3] = {1, 1, 1};
        for (int a = 0; a < 3; ++a) {
          pc.vlo[a] = A3[a]->vlo;
          pc.cnt[a] = A3[a]->cnt;
          pc.cells[a] = A3[a]->cells;
          pc.ncols *= pc.cnt[a];
          if (a < d) {
            qbox[a] = r * pc.cells[a] + 1;
            pbox[a] = (r - 1) * pc.cells[a] + 1;
            nQ *= qbox[a];
            nP *= pbox[a];
          }
        }
        pc.cp = (int)(k1 * (2 * d * nQ + nP));
        pc.rel_off = (long long)relidx.size();
        // mini-level base of the representative patch
        long long mbq = 0, mbp = 0;
        for (int a = 0; a < d; ++a) {
          const int v = A3[a]->vmini;
          const int c0 = v > 0 ? v - 1 : 0;
          mbq += (long long)(r * c0) * mini.qs[a];
          mbp += (long long)((r - 1) * c0) * mini.ps[a];
        }
        offs.push_back((long long)minidofs.size());
        for (int m = 0; m < k1; ++m) {
          for (int slot = 0; slot <= 2 * d; ++slot) {
            const bool pres = slot == 2 * d;
            const int* box = pres ? pbox : qbox;
            const long long tot = pres ? nP : nQ;
            for (long long e = 0; e < tot; ++e) {
              long long rem = e, rel = 0, mrel = 0;
              for (int a = 0; a < d; ++a) {
                const int la = (int)(rem % box[a]);
                rem /= box[a];
                rel += (long long)la * (pres ? g.ps[a] : g.qs[a]);
                mrel += (long long)la * (pres ? mini.ps[a] : mini.qs[a]);
              }
              const long long off = (long long)m * g.block + (pres ? 2 * g.R : (long long)slot * g.nq);
              const long long moff = (long long)m * mini.block + (pres ? 2 * mini.R : (long long)slot * mini.nq);
              relidx.push_back((int)(2 * (off + rel) + (pres ? 1 : 0)));
              minidofs.push_back((int)(moff + mrel + (pres ? mbp : mbq)));
            }
          }
        }
        cps.push_back(pc.cp);
        Lv.maxcp = std::max(Lv.maxcp, pc.cp);
        Lv.cls.push_back(pc);
      }
  const int ncls = (int)Lv.cls.size();
  if (Lv.maxcp > 2048) {
    set_error("patch size C_P > 2048 not supported by the K2 gather table");
    return STGMG_ENOTSUP;
  }
  Lv.lda = (Lv.maxcp + 15) / 16 * 16;
  Lv.ldy = Lv.maxcp;
  for (int c = 0; c < ncls; ++c) Lv.cls[c].inv_off = (long long)c * Lv.lda * Lv.lda;
  // tiles
  std::vector<TileDesc> tiles;
  Lv.k2var = k2_pick_variant(Lv.npatch_global ? Lv.npatch_global : Lv.npatch, Lv.maxcp);
  if (const char* ev = std::getenv("STGMG_K2_VARIANT")) {   // experiments: force a tile variant on the fine level
    if (l == h->L - 1) Lv.k2var = std::atoi(ev);
  }
  {   // experiments: STGMG_K2_VARIANT_L<l>=v forces variant v on level l
    const std::string key = "STGMG_K2_VARIANT_L" + std::to_string(l);
    if (const char* ev = std::getenv(key.c_str())) Lv.k2var = std::atoi(ev);
  }
  int tbm = 0, tbn = 0;
  k2_tile_shape(Lv.k2var, &tbm, &tbn);
  // dense K2 (bulk-copied B from the patch-expanded residual) on the levels of the big / wide tile variants
  // (measured: cfg2 (C_P = 663) / cfg3 (C_P = 1,554) fine K2 34 / 33.5 TF/s, V-cycles 29.4 -> 27 / 63 -> 56 ms;
  // cfg1 (C_P = 218): K2 22.0 -> 17.9 us, the expansion costs about as much, V-cycle 0.809 vs 0.811 ms)
  Lv.dense = (Lv.k2var == 2 || Lv.k2var == 6) &&
             (h->prm.smoother == STGMG_SMOOTH_ADDITIVE || h->prm.smoother == STGMG_SMOOTH_OVERWRITE);
  if (const char* ev = std::getenv("STGMG_K2_DENSE"))   // experiments / tests: 0 = never, 1 = on big / wide levels
    Lv.dense = std::atoi(ev) != 0 && (Lv.k2var == 2 || Lv.k2var == 6) && h->prm.smoother == STGMG_SMOOTH_ADDITIVE;
  {
    long long off = 0, coff = 0;
    for (auto& c : Lv.cls) {
      c.rexp_off = off;
      off += (long long)((c.cp + 15) / 16) * c.ncols * 16;
      c.col_off = coff;
      coff += c.ncols;
    }
    Lv.nrexp = off;
  }
  {
    std::vector<int> cpv, ncv;
    for (const auto& c : Lv.cls) { cpv.push_back(c.cp); ncv.push_back(c.ncols); }
    tiles = balanced_tiles(cpv, ncv, tbm, tbn, Lv.dense ? k2d_slots(Lv.k2var) : k2_slots(Lv.k2var), 1);
  }
  Lv.ntiles = (int)tiles.size();
  if (Lv.dense) {
    CK(dalloc(h, &Lv.Rexp, (size_t)Lv.nrexp));
    CKE(cudaMemsetAsync(Lv.Rexp, 0, sizeof(double) * (size_t)Lv.nrexp, h->s));   // slots past C_P stay zero
    if (const char* ev = std::getenv("STGMG_EXPAND_FUSED")) Lv.exp_fused = std::atoi(ev) != 0;
    std::vector<int4> eb;
    std::vector<int2> cb;
    for (int ci = 0; ci < (int)Lv.cls.size(); ++ci) {
      const PatchClass& c = Lv.cls[ci];
      for (int q = 0; q < (c.cp + 15) / 16; ++q)
        for (int c0 = 0; c0 < c.ncols; c0 += EXPAND_COLS) eb.push_back(make_int4(ci, q, c0, std::min(EXPAND_COLS, c.ncols - c0)));
      for (int col = 0; col < c.ncols; ++col) {   // gather bases of the patch in column col (as the K2 kernels)
        int rem = col, bq = 0, bp = 0;
        for (int a = 0; a < d; ++a) {
          const int v = c.vlo[a] + (rem % c.cnt[a]) * c.vst;
          rem /= c.cnt[a];
          const int c0 = v > 0 ? v - 1 : 0;
          bq += (h->r * c0) * (int)g.qs[a];
          bp += ((h->r - 1) * c0) * (int)g.ps[a];
        }
        cb.push_back(make_int2(bq, bp));
      }
    }
    Lv.n_exp_blocks = (int)eb.size();
    CK(upload(h, &Lv.exp_blocks, eb));
    CK(upload(h, &Lv.colbase, cb));
  }
  CK(upload(h, &Lv.cls_dev, Lv.cls));
  CK(upload(h, &Lv.tiles_dev, tiles));
  CK(upload(h, &Lv.relidx_dev, relidx));
  if (h->prm.smoother == STGMG_SMOOTH_COLORED_MULT) {   // vertex colours v_a mod 4, lexicographic (x fastest)
    constexpr int NCOL = 4;
    int ncol = 1;
    for (int a = 0; a < d; ++a) ncol *= NCOL;
    Lv.colours.assign(ncol, LevelData::Colour());
    for (int c = 0; c < ncol; ++c) {
      int cc[3] = {0, 0, 0};
      for (int a = 0, t = c; a < d; ++a, t /= NCOL) cc[a] = t % NCOL;
      std::vector<PatchClass> sub;
      std::vector<int2> items;
      for (const auto& pc : Lv.cls) {
        PatchClass q = pc;
        q.vst = NCOL;
        q.ncols = 1;
        bool empty = false;
        for (int a = 0; a < 3; ++a) {
          if (a >= d) continue;
          const int v0 = pc.vlo[a] + (((cc[a] - pc.vlo[a]) % NCOL) + NCOL) % NCOL;
          const int last = pc.vlo[a] + pc.cnt[a] - 1;
          q.vlo[a] = v0;
          q.cnt[a] = v0 <= last ? (last - v0) / NCOL + 1 : 0;
          if (q.cnt[a] == 0) empty = true;
          q.ncols *= q.cnt[a];
        }
        if (empty) continue;
        for (int col = 0; col < q.ncols; ++col) items.push_back(make_int2((int)sub.size(), col));
        sub.push_back(q);
      }
      auto& C = Lv.colours[c];
      C.nitems = (int)items.size();
      if (sub.empty()) continue;
      std::vector<int> cpv, ncv;
      for (const auto& q : sub) { cpv.push_back(q.cp); ncv.push_back(q.ncols); }
      C.k2var = k2_pick_variant((long long)items.size(), Lv.maxcp);
      int cbm = 0, cbn = 0;
      k2_tile_shape(C.k2var, &cbm, &cbn);
      std::vector<TileDesc> ct = balanced_tiles(cpv, ncv, cbm, cbn, k2_slots(C.k2var), 1);
      C.ntiles = (int)ct.size();
      CK(upload(h, &C.cls_dev, sub));
      CK(upload(h, &C.tiles_dev, ct));
      CK(upload(h, &C.items_dev, items));
    }
  }
  sm.mark("classes, tiles, tables", l);
  CK(dalloc(h, &Lv.Y, (size_t)Lv.npatch * Lv.ldy));
  double* inv_rm = nullptr;   // row-major inverses (setup scratch); K2 reads the chunk-major copy Lv.inv_dev
  CKE(cudaMalloc(&inv_rm, sizeof(double) * (size_t)ncls * Lv.lda * Lv.lda));
  CK(dalloc(h, &Lv.inv_dev, (size_t)ncls * Lv.lda * Lv.lda + kK2Slack));
  CKE(cudaMemsetAsync(Lv.inv_dev, 0, sizeof(double) * ((size_t)ncls * Lv.lda * Lv.lda + kK2Slack), h->s));
  // dense mini-level operator: column j = A_mini e_j (stream-ordered scratch: a cudaFree would wait for the
  // inverses of the previous levels still running on their own streams)
  const long long Nm = mini.N;
  double *X = nullptr, *Ym = nullptr;
  CKE(cudaMallocAsync(&X, sizeof(double) * Nm * Nm, h->s));
  CKE(cudaMallocAsync(&Ym, sizeof(double) * Nm * Nm, h->s));
  CKE(cudaMemsetAsync(X, 0, sizeof(double) * Nm * Nm, h->s));
  CKE(cudaMemsetAsync(Ym, 0, sizeof(double) * Nm * Nm, h->s));
  CKE(launch_identity(X, Nm, h->s));
  {
    double* Ycb = nullptr;
    if (h->d == 2) CKE(cudaMallocAsync(&Ycb, sizeof(double) * Nm * cell_count(mini) * elem_dofs(h), h->s));
    int rc = apply_into(h, mini, X, Ym, (int)Nm, Nm, Ycb);
    if (Ycb) CKE(cudaFreeAsync(Ycb, h->s));
    if (rc) return rc;
  }
  sm.mark("mini-level dense operator", l);
  int* cps_dev = nullptr;
  long long* offs_dev = nullptr;
  int* mdofs_dev = nullptr;
  CK(upload(h, &cps_dev, cps));
  CK(upload(h, &offs_dev, offs));
  CK(upload(h, &mdofs_dev, minidofs));
  CKE(launch_extract_patch(mini, r, k1, Ym, Nm, nullptr, ncls, cps_dev, offs_dev, mdofs_dev, inv_rm, Lv.lda, h->s));
  int *perm = nullptr, *status = nullptr;
  double *colk = nullptr, *scale = nullptr;
  CK(dalloc(h, &perm, (size_t)ncls * Lv.lda));
  CK(dalloc(h, &status, (size_t)ncls));
  CK(dalloc(h, &colk, (size_t)ncls * Lv.lda));
  CK(dalloc(h, &scale, (size_t)ncls * Lv.lda));
  CKE(cudaMemsetAsync(status, 0, sizeof(int) * ncls, h->s));
  CKE(cudaFreeAsync(X, h->s));
  CKE(cudaFreeAsync(Ym, h->s));
  sm.mark("extraction", l);
  CK(launch_inverse_async(h, l, inv_rm, ncls, Lv.maxcp, cps_dev, Lv.lda, perm, colk, scale, status, inv_rm));
  sm.mark("Gauss-Jordan", l);
  return 0;
}

// 3D operator setup: per-cell-type element matrices (cell types = per-axis {first, interior, last}, every cell its
// own type when n < 3), produced by the warp-per-cell sum-factorisation kernel on a min(n,3)^3-cell mini level with
// the same h and boundary conditions, for every unit vector; applied at run time as a grouped DMMA GEMM.
static int build_cells(stgmg_handle* h, int l, bool gemm, std::vector<double>* Ehost = nullptr) {
  LevelData& Lv = h->lev[l];
  const LevelGeom& g = Lv.g;
  const int d = h->d, r = h->r, k1 = h->k1;
  const int ne = (int)elem_dofs(h);
  struct AxCls { int clo, cnt, rep; };
  std::vector<AxCls> ax[3];
  int nmini[3] = {1, 1, 1};
  for (int a = 0; a < 3; ++a) {
    if (a >= d) { ax[a].push_back({0, 1, 0}); continue; }
    const int n = g.n[a];
    nmini[a] = std::min(n, 3);
    if (n < 3) {
      for (int c = 0; c < n; ++c) ax[a].push_back({c, 1, c});
    } else {
      ax[a].push_back({0, 1, 0});
      ax[a].push_back({1, n - 2, 1});
      ax[a].push_back({n - 1, 1, 2});
    }
  }
  LevelGeom mini = make_geom(d, nmini, g.h, r, k1, g.bcu, g.bcp, h->prm.hF_mode);
  std::vector<int> relidx, mdofs;
  std::vector<long long> reps;
  Lv.ecls.clear();
  for (auto& cz : ax[2])
    for (auto& cy : ax[1])
      for (auto& cx : ax[0]) {
        const AxCls* A3[3] = {&cx, &cy, &cz};
        PatchClass pc;
        std::memset(&pc, 0, sizeof(pc));
        pc.cp = ne;
        pc.ncols = 1;
        pc.vst = 1;
        pc.rel_off = (long long)relidx.size();
        long long mbq = 0, mbp = 0, rp = 0, vs = 1;
        for (int a = 0; a < 3; ++a) {
          pc.vlo[a] = A3[a]->clo + (a < d ? 1 : 0);   // "vertex" = cell + 1, so that the GEMM's lowest cell is the cell
          pc.cnt[a] = A3[a]->cnt;
          pc.cells[a] = 1;
          pc.ncols *= pc.cnt[a];
          if (a < d) {
            mbq += (long long)(r * A3[a]->rep) * mini.qs[a];
            mbp += (long long)((r - 1) * A3[a]->rep) * mini.ps[a];
            rp += (long long)(A3[a]->rep + 1) * vs;
            vs *= nmini[a] + 1;
          }
        }
        reps.push_back(rp);
        for (int m = 0; m < k1; ++m)
          for (int slot = 0; slot <= 2 * d; ++slot) {
            const bool pres = slot == 2 * d;
            const int n1 = pres ? r : r + 1;
            int tot = 1;
            for (int a = 0; a < d; ++a) tot *= n1;
            for (int e = 0; e < tot; ++e) {
              int rem = e;
              long long rel = 0, mrel = 0;
              for (int a = 0; a < d; ++a) {
                const int la = rem % n1;
                rem /= n1;
                rel += (long long)la * (pres ? g.ps[a] : g.qs[a]);
                mrel += (long long)la * (pres ? mini.ps[a] : mini.qs[a]);
              }
              const long long off = (long long)m * g.block + (pres ? 2 * g.R : (long long)slot * g.nq);
              const long long moff = (long long)m * mini.block + (pres ? 2 * mini.R : (long long)slot * mini.nq);
              relidx.push_back((int)(2 * (off + rel) + (pres ? 1 : 0)));
              mdofs.push_back((int)(moff + mrel + (pres ? mbp : mbq)));
            }
          }
        Lv.ecls.push_back(pc);
      }
  const int nt = (int)Lv.ecls.size();
  Lv.elda = (ne + 15) / 16 * 16;
  for (int t = 0; t < nt; ++t) Lv.ecls[t].inv_off = (long long)t * Lv.elda * Lv.elda;
  if (gemm) {   // runtime element GEMM (3D operator): tiles, class records, gather tables, chunk-major matrices
    Lv.ek2var = k2_pick_variant(Lv.ncell_global ? Lv.ncell_global : cell_count(g), ne);
    if (const char* ev = std::getenv("STGMG_EK2_VARIANT")) Lv.ek2var = std::atoi(ev);   // experiments
    int tbm = 0, tbn = 0;
    k2_tile_shape(Lv.ek2var, &tbm, &tbn);
    std::vector<TileDesc> tiles;
    std::vector<int> cpv, ncv;
    for (const auto& c : Lv.ecls) { cpv.push_back(c.cp); ncv.push_back(c.ncols); }
    tiles = balanced_tiles(cpv, ncv, tbm, tbn, k2_slots(Lv.ek2var), 1);
    Lv.entiles = (int)tiles.size();
    CK(upload(h, &Lv.ecls_dev, Lv.ecls));
    CK(upload(h, &Lv.etiles_dev, tiles));
    CK(upload(h, &Lv.erelidx_dev, relidx));
    CK(dalloc(h, &Lv.E_dev, (size_t)nt * Lv.elda * Lv.elda + kK2Slack));
    CKE(cudaMemsetAsync(Lv.E_dev, 0, sizeof(double) * ((size_t)nt * Lv.elda * Lv.elda + kK2Slack), h->s));
  }
  double* E_rm = nullptr;   // row-major element matrices (setup scratch); the GEMM reads the chunk-major Lv.E_dev
  CKE(cudaMallocAsync(&E_rm, sizeof(double) * (size_t)nt * Lv.elda * Lv.elda, h->s));
  // element results of the mini level for every unit vector
  const long long Nm = mini.N;
  long long nvm = 1;
  for (int a = 0; a < d; ++a) nvm *= nmini[a] + 1;
  const long long ycs = nvm * ne;
  double *X = nullptr, *Ycb = nullptr;
  long long* reps_dev = nullptr;
  int* mdofs_dev = nullptr;
  CKE(cudaMallocAsync(&X, sizeof(double) * Nm * Nm, h->s));
  CKE(cudaMallocAsync(&Ycb, sizeof(double) * Nm * ycs, h->s));
  CKE(cudaMemsetAsync(X, 0, sizeof(double) * Nm * Nm, h->s));
  CKE(cudaMemsetAsync(Ycb, 0, sizeof(double) * Nm * ycs, h->s));
  CKE(launch_identity(X, Nm, h->s));
  int nl = 0;
  CKE(launch_op_apply(d, r, k1, mini, h->c_dev, X, nullptr, Ycb, 1.0, (int)Nm, Nm, ycs, h->s, &nl));
  CK(upload(h, &reps_dev, reps));
  CK(upload(h, &mdofs_dev, mdofs));
  CKE(launch_extract_elem(Ycb, ycs, ne, nt, reps_dev, mdofs_dev, E_rm, Lv.elda, h->s));
  if (gemm) CKE(launch_chunk_swizzle(E_rm, Lv.E_dev, nt, Lv.elda, h->s));
  CKE(cudaStreamSynchronize(h->s));
  // factored form (op_fgemm.cu) on the levels where it wins (measured: cfg4/cfg3 3D levels with >= 4096 cells, the
  // 2D Q3 levels with >= 16384 cells; on smaller levels one CTA per 32 cells leaves the GPU idle)
  const long long ncl = Lv.ncell_global ? Lv.ncell_global : cell_count(g);
  if (gemm && h->fg_on && h->c.ds == 0.0 && (h->fg_on == 2 || ncl >= (d == 3 ? 4096 : 16384))) {
    std::vector<double> Eh((size_t)nt * Lv.elda * Lv.elda);
    CKE(cudaMemcpy(Eh.data(), E_rm, sizeof(double) * Eh.size(), cudaMemcpyDeviceToHost));
    FgemmData fd;
    if (fgemm_build_any(d, r, k1, Eh, nt, Lv.elda, h->c, fd) == 0) {
      std::vector<int4> tl, ts;
      const int nc = fgemm_cells_per_tile();
      for (int t = 0; t < nt; ++t) {
        // volume-only type: every domain face its box touches is Neumann for u and p (no Nitsche terms)
        // (measured on B200: faster than the factored GEMMs at cfg4's fine level, 262k cells, slower on 4k-33k cell
        // levels)
        bool vol = sf3_supported(d, r, k1) && (h->sf_on == 2 || (h->sf_on == 1 && ncl >= 131072));
        for (int a = 0; a < d; ++a) {
          const int c0 = Lv.ecls[t].vlo[a] - 1, c1 = c0 + Lv.ecls[t].cnt[a] - 1;
          if (c0 == 0 && (g.bcu[2 * a] == STGMG_BC_DIRICHLET || g.bcp[2 * a] == STGMG_BC_DIRICHLET)) vol = false;
          if (c1 == g.n[a] - 1 && (g.bcu[2 * a + 1] == STGMG_BC_DIRICHLET || g.bcp[2 * a + 1] == STGMG_BC_DIRICHLET))
            vol = false;
        }
        for (int c0 = 0; c0 < Lv.ecls[t].ncols; c0 += nc)
          (vol ? ts : tl).push_back(make_int4(t, c0, std::min(nc, Lv.ecls[t].ncols - c0), 0));
      }
      if (!ts.empty()) CK(upload(h, &Lv.sf_tiles, ts));
      Lv.sf_ntiles = (int)ts.size();
      double *a1 = nullptr, *a2 = nullptr, *a3 = nullptr, *ap = nullptr;
      CK(upload(h, &a1, fd.A1));
      CK(upload(h, &a2, fd.A2));
      CK(upload(h, &a3, fd.A3));
      CK(upload(h, &ap, fd.AP));
      if (!tl.empty()) CK(upload(h, &Lv.fg_tiles, tl));
      Lv.fg_ntiles = (int)tl.size();
      Lv.fgm.A1 = a1;
      Lv.fgm.A2 = a2;
      Lv.fgm.A3 = a3;
      Lv.fgm.AP = ap;
      Lv.fgm.a2stride = fd.a2stride;
      Lv.fgm.a3stride = fd.a3stride;
      Lv.fg = true;
    }
  }
  if (Ehost) {
    Ehost->resize((size_t)nt * Lv.elda * Lv.elda);
    CKE(cudaMemcpy(Ehost->data(), E_rm, sizeof(double) * Ehost->size(), cudaMemcpyDeviceToHost));
  }
  CKE(cudaFreeAsync(E_rm, h->s));   // stream-ordered: no device-wide wait on the inverses in flight
  CKE(cudaFreeAsync(X, h->s));
  CKE(cudaFreeAsync(Ycb, h->s));
  return 0;
}

static int build_coarse(stgmg_handle* h) {
  NvtxRange nv("stgmg setup: coarse inverse");
  const LevelGeom& g = h->lev[0].g;
  const long long N = g.N;
  h->n0 = (int)N;
  double *X = nullptr, *Ym = nullptr;
  CKE(cudaMallocAsync(&X, sizeof(double) * N * N, h->s));
  CKE(cudaMallocAsync(&Ym, sizeof(double) * N * N, h->s));
  CKE(cudaMemsetAsync(X, 0, sizeof(double) * N * N, h->s));
  CKE(cudaMemsetAsync(Ym, 0, sizeof(double) * N * N, h->s));
  CKE(launch_identity(X, N, h->s));
  {
    double* Ycb = nullptr;
    if (h->d == 2) CKE(cudaMallocAsync(&Ycb, sizeof(double) * N * cell_count(g) * elem_dofs(h), h->s));
    int rc = apply_into(h, g, X, Ym, (int)N, N, Ycb);
    if (Ycb) CKE(cudaFreeAsync(Ycb, h->s));
    if (rc) return rc;
  }
  std::vector<int> dofs(N);
  for (long long i = 0; i < N; ++i) dofs[i] = (int)i;
  std::vector<int> cps{(int)N};
  std::vector<long long> offs{0};
  int *cps_dev, *dofs_dev, *perm, *status;
  long long* offs_dev;
  double *colk, *scale;
  CK(upload(h, &cps_dev, cps));
  CK(upload(h, &offs_dev, offs));
  CK(upload(h, &dofs_dev, dofs));
  CK(dalloc(h, &h->A0inv, (size_t)N * N));
  CKE(launch_extract_patch(g, h->r, h->k1, Ym, N, nullptr, 1, cps_dev, offs_dev, dofs_dev, h->A0inv, (int)N, h->s));
  CK(dalloc(h, &perm, (size_t)N));
  CK(dalloc(h, &status, 1));
  CK(dalloc(h, &colk, (size_t)N));
  CK(dalloc(h, &scale, (size_t)N));
  CKE(cudaMemsetAsync(status, 0, sizeof(int), h->s));
  CKE(cudaFreeAsync(X, h->s));
  CKE(cudaFreeAsync(Ym, h->s));
  return launch_inverse_async(h, 0, h->A0inv, 1, (int)N, cps_dev, (int)N, perm, colk, scale, status, nullptr);
}

static int build_transfer(stgmg_handle* h, int l) {
  LevelData& F = h->lev[l];
  const LevelGeom& cg = h->lev[l - 1].g;
  for (int a = 0; a < 3; ++a) {
    for (int pres = 0; pres < 2; ++pres) {
      Interp1D& T = pres ? F.tt.p[a] : F.tt.q[a];
      if (a >= h->d) {
        T = Interp1D{nullptr, nullptr, nullptr, nullptr, nullptr, nullptr, 0};
        continue;
      }
      const int deg = pres ? h->r - 1 : h->r;
      Interp1DHost ih = (a == 0) ? make_interp_window(h->lev[l - 1].gnx, deg, F.w0, F.g.n[0], h->lev[l - 1].w0, cg.n[0])
                                 : make_interp(cg.n[a], deg);
      (pres ? F.ih_p[a] : F.ih_q[a]) = ih;
      int *rpf, *cif, *rpc, *cic;
      double *vf, *vc;
      CK(upload(h, &rpf, ih.rp_f));
      CK(upload(h, &cif, ih.ci_f));
      CK(upload(h, &vf, ih.v_f));
      CK(upload(h, &rpc, ih.rp_c));
      CK(upload(h, &cic, ih.ci_c));
      CK(upload(h, &vc, ih.v_c));
      T = Interp1D{rpf, cif, vf, rpc, cic, vc, (int)ih.ci_c.size()};
    }
  }
  // separable restriction on levels with 200k..16M DoFs (its intermediates hold < N_l doubles);
  // STGMG_RESTRICT_SEP=0: off
  const char* sep_env = std::getenv("STGMG_RESTRICT_SEP");
  const bool sep_off = sep_env && std::atoi(sep_env) == 0;
  // measured (R+P, one B200): cfg2 fine (7.9M) 368 -> 156 us, cfg3 level 3 (441k) 80 -> 31 us, cfg3 fine (3.4M)
  // 97 -> 81 us, but cfg4 fine (26.6M) 489 -> 542 us (its first pass is latency-bound on the table chain): the gather
  // form stays on levels above 16M DoFs
  const bool sep_all = sep_env && std::atoi(sep_env) == 2;   // every level >= 200k DoFs (measurement)
  if (!sep_off && F.g.N >= 200000 && (F.g.N < 16000000 || sep_all)) CK(dalloc(h, &F.rtmp, (size_t)F.g.N));
  return 0;
}

// --------------------------------------------------------------------------- small-level fast path setup ----
// CSR of a sparse matrix from per-row (column, value) lists filled in a fixed order: columns sorted (stable), equal
// columns summed in fill order.
struct HostCsr {
  std::vector<int> rp, ci;
  std::vector<double> v;
};
static HostCsr to_csr(std::vector<std::vector<std::pair<int, double>>>& rows) {
  HostCsr c;
  c.rp.assign(rows.size() + 1, 0);
  for (size_t i = 0; i < rows.size(); ++i) {
    auto& r = rows[i];
    std::stable_sort(r.begin(), r.end(), [](const auto& x, const auto& y) { return x.first < y.first; });
    for (size_t j = 0; j < r.size();) {
      size_t k = j;
      double s = 0.0;
      for (; k < r.size() && r[k].first == r[j].first; ++k) s += r[k].second;
      c.ci.push_back(r[j].first);
      c.v.push_back(s);
      j = k;
    }
    c.rp[i + 1] = (int)c.ci.size();
    std::vector<std::pair<int, double>>().swap(r);
  }
  return c;
}

static int lanes_for(const HostCsr& c) {   // lanes per row of the SpMV: ~ average row length / 4
  const double avg = c.rp.size() > 1 ? (double)c.ci.size() / (double)(c.rp.size() - 1) : 1.0;
  return avg > 64 ? 32 : (avg > 24 ? 16 : (avg > 8 ? 8 : 4));
}

static int upload_csr(stgmg_handle* h, const HostCsr& c, int** rp, int** ci, double** v) {
  CK(upload(h, rp, c.rp));
  CK(upload(h, ci, c.ci));
  CK(upload(h, v, c.v));
  return 0;
}

// DoF index of (Radau node m, field slot, lexicographic node (x, y, z)) on a level
static long long dof_index(const LevelGeom& g, int m, int slot, const int* idx) {
  const bool pres = slot == 2 * g.d;
  long long node = 0;
  for (int a = 0; a < g.d; ++a) node += (long long)idx[a] * (pres ? g.ps[a] : g.qs[a]);
  return (long long)m * g.block + (pres ? 2 * g.R : (long long)slot * g.nq) + node;
}

static long long global_dofs(const stgmg_handle* h, const LevelData& Lv) {
  long long nq = 1, np = 1;
  for (int a = 0; a < h->d; ++a) {
    const int n = (a == 0 && Lv.gnx) ? Lv.gnx : Lv.g.n[a];
    nq *= (long long)h->r * n + 1;
    np *= (long long)(h->r - 1) * n + 1;
  }
  return (long long)h->k1 * (2 * h->d * nq + np);
}

static long long small_threshold() {
  if (const char* ev = std::getenv("STGMG_SMALL_N")) return std::atoll(ev);
  return 40000;
}

// Assembled operator of level l: A[dof(K, e)][dof(K, e')] += E_type(K)[e][e'] over the cells K in lexicographic
// order (the element matrices are those the 3D element GEMM uses, from the sum-factorised kernel on a mini level).
static int build_small_operator(stgmg_handle* h, int l) {
  LevelData& Lv = h->lev[l];
  const LevelGeom& g = Lv.g;
  const int d = h->d, r = h->r, k1 = h->k1;
  const int ne = (int)elem_dofs(h);
  std::vector<double> E;
  CK(build_cells(h, l, false, &E));   // element matrices only (the 3D element GEMM was set up before)
  const int elda = Lv.elda;
  int ntx[3] = {1, 1, 1};
  for (int a = 0; a < d; ++a) ntx[a] = g.n[a] < 3 ? g.n[a] : 3;
  auto axtype = [&](int a, int c) { const int n = g.n[a]; return n < 3 ? c : (c == 0 ? 0 : (c == n - 1 ? 2 : 1)); };
  std::vector<std::vector<std::pair<int, double>>> rows((size_t)g.N);
  std::vector<long long> dofs(ne);
  int c3[3] = {0, 0, 0};
  for (c3[2] = 0; c3[2] < (d > 2 ? g.n[2] : 1); ++c3[2])
    for (c3[1] = 0; c3[1] < g.n[1]; ++c3[1])
      for (c3[0] = 0; c3[0] < g.n[0]; ++c3[0]) {
        const int t = (d > 2 ? axtype(2, c3[2]) * ntx[1] * ntx[0] : 0) + axtype(1, c3[1]) * ntx[0] + axtype(0, c3[0]);
        int e = 0;
        for (int m = 0; m < k1; ++m)
          for (int slot = 0; slot <= 2 * d; ++slot) {
            const int deg = slot == 2 * d ? r - 1 : r;
            const int n1 = deg + 1;
            int tot = 1;
            for (int a = 0; a < d; ++a) tot *= n1;
            for (int j = 0; j < tot; ++j) {
              int rem = j, idx[3] = {0, 0, 0};
              for (int a = 0; a < d; ++a) {
                idx[a] = deg * c3[a] + rem % n1;
                rem /= n1;
              }
              dofs[e++] = dof_index(g, m, slot, idx);
            }
          }
        const double* Et = E.data() + (size_t)t * elda * elda;
        for (int i = 0; i < ne; ++i)
          for (int j = 0; j < ne; ++j) {
            const double v = Et[(size_t)i * elda + j];
            if (v != 0.0) rows[(size_t)dofs[i]].push_back({(int)dofs[j], v});
          }
      }
  const HostCsr c = to_csr(rows);
  Lv.A_lpr = lanes_for(c);
  return upload_csr(h, c, &Lv.A_rp, &Lv.A_ci, &Lv.A_v);
}

// Prolongation level l-1 -> l (rows = fine DoFs) and restriction (rows = coarse DoFs) from the 1D tables, weights
// multiplied in the order of the node-mapped kernels ((w_z * w_y) * w_x), supports in lexicographic order.
static int build_small_transfer(stgmg_handle* h, int l) {
  LevelData& F = h->lev[l];
  const LevelGeom& fg = F.g;
  const LevelGeom& cg = h->lev[l - 1].g;
  const int d = h->d, k1 = h->k1;
  for (int dir = 0; dir < 2; ++dir) {   // 0: P (fine rows), 1: R = P^T (coarse rows)
    const LevelGeom& rg = dir == 0 ? fg : cg;   // row level
    const LevelGeom& cgx = dir == 0 ? cg : fg;  // column level
    std::vector<std::vector<std::pair<int, double>>> rows((size_t)rg.N);
    for (int slot = 0; slot <= 2 * d; ++slot) {
      const bool pres = slot == 2 * d;
      const Interp1DHost* T = pres ? F.ih_p : F.ih_q;
      const int* nn = pres ? rg.pn : rg.qn;
      int idx[3] = {0, 0, 0};
      for (idx[2] = 0; idx[2] < (d > 2 ? nn[2] : 1); ++idx[2])
        for (idx[1] = 0; idx[1] < nn[1]; ++idx[1])
          for (idx[0] = 0; idx[0] < nn[0]; ++idx[0]) {
            int lo[3] = {0, 0, 0}, hi[3] = {1, 1, 1};
            for (int a = 0; a < d; ++a) {
              const auto& rp = dir == 0 ? T[a].rp_f : T[a].rp_c;
              lo[a] = rp[idx[a]];
              hi[a] = rp[idx[a] + 1];
            }
            std::vector<std::pair<int, double>> ent;
            int ci[3] = {0, 0, 0};
            for (int e2 = lo[2]; e2 < hi[2]; ++e2) {
              double w2 = 1.0;
              if (d > 2) {
                ci[2] = dir == 0 ? T[2].ci_f[e2] : T[2].ci_c[e2];
                w2 = dir == 0 ? T[2].v_f[e2] : T[2].v_c[e2];
              }
              for (int e1 = lo[1]; e1 < hi[1]; ++e1) {
                ci[1] = dir == 0 ? T[1].ci_f[e1] : T[1].ci_c[e1];
                const double w1 = w2 * (dir == 0 ? T[1].v_f[e1] : T[1].v_c[e1]);
                for (int e0 = lo[0]; e0 < hi[0]; ++e0) {
                  ci[0] = dir == 0 ? T[0].ci_f[e0] : T[0].ci_c[e0];
                  const double w = w1 * (dir == 0 ? T[0].v_f[e0] : T[0].v_c[e0]);
                  ent.push_back({0, w});
                  long long node = 0;
                  for (int a = 0; a < d; ++a) node += (long long)ci[a] * (pres ? cgx.ps[a] : cgx.qs[a]);
                  ent.back().first = (int)node;
                }
              }
            }
            for (int m = 0; m < k1; ++m) {
              const long long row = dof_index(rg, m, slot, idx);
              const long long cbase = (long long)m * cgx.block + (pres ? 2 * cgx.R : (long long)slot * cgx.nq);
              for (const auto& en : ent) rows[(size_t)row].push_back({(int)(cbase + en.first), en.second});
            }
          }
    }
    const HostCsr c = to_csr(rows);
    if (dir == 0) {
      F.P_lpr = lanes_for(c);
      CK(upload_csr(h, c, &F.P_rp, &F.P_ci, &F.P_v));
    } else {
      F.R_lpr = lanes_for(c);
      CK(upload_csr(h, c, &F.R_rp, &F.R_ci, &F.R_v));
    }
  }
  return 0;
}

// Averaging table of level l: for every DoF the offsets in Y of the patches containing it, lexicographic.
static int build_small_k3(stgmg_handle* h, int l) {
  LevelData& Lv = h->lev[l];
  const LevelGeom& g = Lv.g;
  const int d = h->d, r = h->r, k1 = h->k1;
  const int NS = d == 3 ? 27 : 9;
  std::vector<int> tab((size_t)NS * g.N, -1);
  for (int slot = 0; slot <= 2 * d; ++slot) {
    const bool pres = slot == 2 * d;
    const int deg = pres ? r - 1 : r;
    const int* nn = pres ? g.pn : g.qn;
    int idx[3] = {0, 0, 0};
    for (idx[2] = 0; idx[2] < (d > 2 ? nn[2] : 1); ++idx[2])
      for (idx[1] = 0; idx[1] < nn[1]; ++idx[1])
        for (idx[0] = 0; idx[0] < nn[0]; ++idx[0]) {
          int cnt[3] = {1, 1, 1}, pw[3][3] = {{0}}, pl[3][3] = {{0}}, pc[3][3] = {{1, 1, 1}, {1, 1, 1}, {1, 1, 1}};
          for (int a = 0; a < d; ++a) {
            const int i = idx[a], n = g.n[a], c = i / deg, lrem = i - c * deg;
            int w0, nw;
            if (lrem == 0) { w0 = c > 0 ? c - 1 : c; nw = (c > 0 ? 1 : 0) + 1 + (c <= n - 1 ? 1 : 0); }
            else { w0 = c; nw = 2; }
            cnt[a] = nw;
            for (int j = 0; j < nw; ++j) {
              const int w = w0 + j, lo = w > 0 ? w - 1 : 0;
              pw[a][j] = w;
              pl[a][j] = i - deg * lo;
              pc[a][j] = (w > 0 ? 1 : 0) + (w < n ? 1 : 0);
            }
          }
          int s = 0;
          std::vector<std::array<long long, 3>> pat;   // (Y offset of loc, nQ, blk) per patch, lexicographic
          for (int i3 = 0; i3 < (d > 2 ? cnt[2] : 1); ++i3)
            for (int i2 = 0; i2 < cnt[1]; ++i2)
              for (int i1 = 0; i1 < cnt[0]; ++i1) {
                const int j[3] = {i1, i2, i3};
                long long plin = 0, vs = 1, loc = 0, ls = 1, nQ = 1, nP = 1;
                for (int a = 0; a < d; ++a) {
                  plin += (long long)pw[a][j[a]] * vs;
                  vs *= g.n[a] + 1;
                  const long long qb = (long long)r * pc[a][j[a]] + 1, pb = (long long)(r - 1) * pc[a][j[a]] + 1;
                  loc += (long long)pl[a][j[a]] * ls;
                  ls *= pres ? pb : qb;
                  nQ *= qb;
                  nP *= pb;
                }
                pat.push_back({plin * Lv.ldy + loc + (pres ? 2 * d * nQ : 0), nQ, 2 * d * nQ + nP});
                ++s;
              }
          for (int m = 0; m < k1; ++m) {
            const long long mu = dof_index(g, m, slot, idx);
            for (size_t q = 0; q < pat.size(); ++q)
              tab[(size_t)q * g.N + mu] = (int)(pat[q][0] + m * pat[q][2] + (pres ? 0 : slot * pat[q][1]));
          }
        }
  }
  return upload(h, &Lv.k3tab, tab);
}

// Decisions use global sizes so that every rank of the x-slab decomposition takes the same one (bitwise 1-vs-n).
static int build_small(stgmg_handle* h, int l) {
  LevelData& Lv = h->lev[l];
  if (l < 1) return 0;
  const long long ng = global_dofs(h, Lv);
  const long long thr = small_threshold();
  long long ncell = 1;
  for (int a = 0; a < h->d; ++a) ncell *= (a == 0 && Lv.gnx) ? Lv.gnx : Lv.g.n[a];
  const long long ne = elem_dofs(h);
  // assembled operator: small levels only (its CSR re-reads ~100-600 values per row from L2)
  if (ng <= thr && ncell * ne * ne <= 12000000LL) CK(build_small_operator(h, l));
  // transfer CSR and averaging tables: a few int32 per DoF, cheaper than the node-mapped index math up to ~10 x thr
  if (ng <= 10 * thr) {
    CK(build_small_transfer(h, l));
    if (h->prm.smoother == STGMG_SMOOTH_ADDITIVE || h->prm.smoother == STGMG_SMOOTH_OVERWRITE)
      CK(build_small_k3(h, l));   // vertex-patch averaging table
  }
  return 0;
}

static int capture_vcycle(stgmg_handle* h) {
  NvtxRange nv("stgmg setup: capture V-cycle graph");
  cudaGraph_t graph;
  const long long before = h->launches;
  CKE(cudaStreamBeginCapture(h->s, cudaStreamCaptureModeThreadLocal));
  int rc = enqueue_vcycle(h);
  cudaError_t e = cudaStreamEndCapture(h->s, &graph);
  if (rc) return rc;
  CKE(e);
  CKE(cudaGraphInstantiate(&h->vgraph, graph, 0));
  h->vgraph_tmpl = graph;   // kept: the device-resident FGMRES embeds it as a child graph
  h->vgraph_launches = (int)(h->launches - before);
  h->launches = before;
  return 0;
}

static int ensure_krylov(stgmg_handle* h, int m) {
  if (m <= h->m_alloc) return 0;
  for (auto& g : h->vg_step)   // bound to the old basis
    if (g) {
      cudaGraphExecDestroy(g);
      g = nullptr;
    }
  const long long N = h->lev[h->L - 1].g.N;
  CK(dalloc(h, &h->V, (size_t)(m + 1) * N));
  CK(dalloc(h, &h->Z, (size_t)m * N));
  CK(dalloc(h, &h->H, (size_t)(m + 1) * m));
  CK(dalloc(h, &h->cs, (size_t)m));
  CK(dalloc(h, &h->sn, (size_t)m));
  CK(dalloc(h, &h->gv, (size_t)m + 1));
  CK(dalloc(h, &h->yv, (size_t)m));
  h->m_alloc = m;
  return 0;
}

// ----------------------------------------------------------------------------------------------- C ABI ----
extern "C" {

const char* stgmg_last_error(void) { return g_last_error.c_str(); }

// Setup steps shared by every hierarchy: Krylov / reduction workspace, events, the folded coarse sub-cycle, the
// V-cycle graph.
static int finish_setup(stgmg_handle* h) {
  CK(finish_inverses(h));
  if (h->gj.buf || h->gj.pi) {   // setup scratch of the class inverses
    CKE(cudaStreamSynchronize(h->s));
    if (h->gj.buf) CKE(cudaFree(h->gj.buf));
    if (h->gj.pi) CKE(cudaFree(h->gj.pi));
    h->gj = GjScratch();
  }
  const long long Nf = h->lev[h->L - 1].g.N;
  CK(dalloc(h, &h->w, (size_t)Nf));
  CK(dalloc(h, &h->rv, (size_t)Nf));
  CK(dalloc(h, &h->stage_rhs, (size_t)Nf));
  CK(dalloc(h, &h->stage_x, (size_t)Nf));
  CK(dalloc(h, &h->rhs_int, (size_t)Nf));
  CK(dalloc(h, &h->scal, 16));
  CK(dalloc(h, &h->partials, 2048));
  CK(dalloc(h, &h->counter, 4));
  CKE(cudaMemset(h->counter, 0, 4 * sizeof(unsigned)));
  CKE(cudaMallocHost(&h->pinned, 16 * sizeof(double)));
  CKE(cudaEventCreate(&h->e0));
  CKE(cudaEventCreate(&h->e1));
  CK(build_fold(h));
  if (const char* ev = std::getenv("STGMG_STEP_GRAPHS")) h->step_graphs = std::atoi(ev) != 0;
  if (std::getenv("STGMG_PROFILE_SOLVE")) {
    h->prof = true;
    for (auto& e : h->pev) CKE(cudaEventCreate(&e));
  }
  if (const char* ev = std::getenv("STGMG_SOLVE_GRAPH")) {   // experiment, see cyc_off
    h->cyc_off = std::atoi(ev) == 0;
    h->cyc_inline = std::atoi(ev) == 2;
  }
  CK(dalloc(h, &h->ctl, 2));
  if (h->graphable) CK(capture_vcycle(h));
  CKE(cudaStreamSynchronize(h->s));
  return 0;
}

// STGMG_SETUP_TIMES=1: host wall time of each setup phase (device synchronised) on stderr.
extern "C++" {
template <class F>
static int timed(const char* what, int level, F f) {
  static const bool on = std::getenv("STGMG_SETUP_TIMES") != nullptr;
  if (!on) return f();
  cudaDeviceSynchronize();
  const auto t0 = std::chrono::steady_clock::now();
  const int rc = f();
  cudaDeviceSynchronize();
  const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  std::fprintf(stderr, "stgmg setup: %-15s level %2d  %9.1f ms\n", what, level, ms);
  return rc;
}
}

// Material / discretisation parameters: rho, c0, tau, mu, alpha > 0, lambda >= 0, K symmetric positive
// definite (Eq:PosDefK, Cholesky of the d x d block).
static int check_params(int d, const stgmg_params* params) {
  if (!(params->rho > 0) || !(params->c0 > 0) || !(params->tau > 0) || !(params->mu > 0) || params->lambda < 0 ||
      !(params->alpha > 0)) {
    set_error("rho, c0, tau, mu, alpha must be > 0 and lambda >= 0 (P:L52)");
    return STGMG_EINVAL;
  }
  // K symmetric positive definite (Eq:PosDefK): Cholesky of the d x d block
  {
    double Kd[3][3];
    for (int i = 0; i < d; ++i)
      for (int j = 0; j < d; ++j) Kd[i][j] = params->K[i * 3 + j];
    for (int i = 0; i < d; ++i)
      for (int j = 0; j < d; ++j)
        if (Kd[i][j] != Kd[j][i]) { set_error("K not symmetric"); return STGMG_EINVAL; }
    for (int j = 0; j < d; ++j) {
      double s = Kd[j][j];
      for (int l = 0; l < j; ++l) s -= Kd[j][l] * Kd[j][l];
      if (!(s > 0)) { set_error("K not positive definite (Eq:PosDefK)"); return STGMG_EINVAL; }
      Kd[j][j] = std::sqrt(s);
      for (int i = j + 1; i < d; ++i) {
        double t = Kd[i][j];
        for (int l = 0; l < j; ++l) t -= Kd[i][l] * Kd[j][l];
        Kd[i][j] = t / Kd[j][j];
      }
    }
  }
  return 0;
}

int stgmg_setup(const stgmg_mesh* mesh, int levels, const stgmg_order* order, const stgmg_params* params,
                stgmg_handle** out) {
  NvtxRange nv("stgmg_setup");
  SetupMarks pm;   // STGMG_SETUP_TIMES: the allocation / constant phases before build_cells
  if (!mesh || !order || !params || !out) { set_error("null argument"); return STGMG_EINVAL; }
  const int d = mesh->dim, r = order->r, k = order->k;
  if ((d != 2 && d != 3) || r < 2 || r > 3 || k < 0 || k > 3 || levels < 1 || levels > 16) {
    set_error("invalid dim / order / levels (d in {2,3}, 2 <= r <= 3, 0 <= k <= 3)");
    return STGMG_EINVAL;
  }
  CK(check_params(d, params));
  for (int a = 0; a < d; ++a)
    if (mesh->cells[a] < 1 || mesh->cells[a] % (1 << (levels - 1)) != 0 || !(mesh->hi[a] > mesh->lo[a])) {
      set_error("cells must be divisible by 2^(levels-1) and the box non-degenerate");
      return STGMG_EINVAL;
    }
  const int nranks = params->nranks > 1 ? params->nranks : 1;
  if (params->formulation != STGMG_FORM_DSA && params->formulation != STGMG_FORM_DS) {
    set_error("unknown formulation");
    return STGMG_EINVAL;
  }
  if (params->smoother != STGMG_SMOOTH_ADDITIVE && params->smoother != STGMG_SMOOTH_COLORED_MULT &&
      params->smoother != STGMG_SMOOTH_ELEMENT && params->smoother != STGMG_SMOOTH_OVERWRITE) {
    set_error("unknown smoother");
    return STGMG_EINVAL;
  }
  if (params->smoother != STGMG_SMOOTH_ADDITIVE && nranks > 1) {
    set_error("the smoother variants (colour-ordered multiplicative, element-wise) are single-GPU only");
    return STGMG_ENOTSUP;
  }
  if (nranks > 1 && (params->rank < 0 || params->rank >= nranks || params->nccl_comm == nullptr)) {
    set_error("multi-GPU: need 0 <= rank < nranks and a communicator (nccl_comm) / loopback hub");
    return STGMG_EINVAL;
  }
  auto h = std::make_unique<stgmg_handle>();
  h->nranks = nranks;
  h->rank = nranks > 1 ? params->rank : 0;
  if (nranks > 1) {
    h->tr = params->comm_kind == STGMG_COMM_LOOPBACK ? make_loopback_transport(params->nccl_comm, h->rank)
            : params->comm_kind == STGMG_COMM_SHM    ? make_shm_transport(params->nccl_comm)
                                                     : make_nccl_transport(params->nccl_comm, h->rank, nranks);
    if (!h->tr) return STGMG_ENCCL;
    h->graphable = h->tr->graph_capturable();
  }
  h->d = d; h->r = r; h->k = k; h->k1 = k + 1; h->L = levels;
  h->prm = *params;
  {
    int dev = 0, nsm = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && nsm > 0)
      h->nsm = nsm;
  }
  if (h->prm.omega <= 0) h->prm.omega = 0.7;
  if (h->prm.jmax <= 0) h->prm.jmax = 4;
  if (params->stream) {
    h->s = (cudaStream_t)params->stream;
  } else {
    // a BLOCKING stream: it orders itself after work the caller queued on the legacy default stream (stgmg.h)
    CKE(cudaStreamCreateWithFlags(&h->s, cudaStreamDefault));
    h->own_stream = true;
  }
  h->c = make_consts(d, r, k, h->prm);
  h->lev.resize(levels);
  for (int l = levels - 1; l >= 0; --l) {
    LevelData& Lv = h->lev[l];
    int n[3] = {1, 1, 1};
    double hh[3] = {1, 1, 1};
    for (int a = 0; a < d; ++a) {
      n[a] = mesh->cells[a] >> (levels - 1 - l);
      hh[a] = (mesh->hi[a] - mesh->lo[a]) / n[a];
    }
    Lv.gnx = n[0];
    Lv.npatch_global = 1;
    Lv.ncell_global = 1;
    for (int a = 0; a < d; ++a) {
      Lv.npatch_global *= n[a] + 1;
      Lv.ncell_global *= n[a];
    }
    // x-slab partition: a level is split while every rank owns >= 4 cells along x and all finer
    // levels are split; coarser levels are agglomerated (replicated on every rank).  A split level must own an
    // EVEN number of cells per rank, so that rank q's cells coarsen onto exactly the coarse cells [q oc, (q+1) oc)
    // whether or not the coarser level is split (agglomerate() relies on it).
    const bool finer_part = (l == levels - 1) || h->lev[l + 1].part;
    Lv.part = nranks > 1 && l >= 1 && finer_part && n[0] % (2 * nranks) == 0 && n[0] / nranks >= 4;
    int bcu[6], bcp[6];
    for (int f = 0; f < 6; ++f) { bcu[f] = mesh->bc_u[f]; bcp[f] = mesh->bc_p[f]; }
    if (Lv.part) {
      const int own = n[0] / nranks, c0g = h->rank * own, c1g = c0g + own;
      Lv.has_left = h->rank > 0;
      Lv.has_right = h->rank < nranks - 1;
      Lv.w0 = Lv.has_left ? c0g - kGhost : 0;
      const int w1 = Lv.has_right ? c1g + kGhost : n[0];
      Lv.c0 = c0g - Lv.w0;
      Lv.c1 = c1g - Lv.w0;
      n[0] = w1 - Lv.w0;
      // artificial window faces carry no boundary terms (their ghost values come from the neighbours)
      if (Lv.has_left) { bcu[0] = STGMG_BC_NEUMANN; bcp[0] = STGMG_BC_NEUMANN; }
      if (Lv.has_right) { bcu[1] = STGMG_BC_NEUMANN; bcp[1] = STGMG_BC_NEUMANN; }
    } else {
      Lv.w0 = 0;
      Lv.c0 = 0;
      Lv.c1 = n[0];
    }
    Lv.g = make_geom(d, n, hh, r, h->k1, bcu, bcp, h->prm.hF_mode);
    if (Lv.part) {   // penalty lengths stay those of the physical mesh
      for (int f = 0; f < 6; ++f) Lv.g.hF[f] = make_geom(d, n, hh, r, h->k1, mesh->bc_u, mesh->bc_p, h->prm.hF_mode).hF[f];
    }
    const long long N = Lv.g.N;
    CK(dalloc(h.get(), &Lv.b, (size_t)N));
    CK(dalloc(h.get(), &Lv.d, (size_t)N));
    CK(dalloc(h.get(), &Lv.r, (size_t)N));
    CKE(cudaMemset(Lv.b, 0, sizeof(double) * N));
    CKE(cudaMemset(Lv.d, 0, sizeof(double) * N));
    CKE(cudaMemset(Lv.r, 0, sizeof(double) * N));
  }
  pm.mark("handle, level vectors", -1);
  if (nranks > 1 && !h->lev[levels - 1].part) {
    set_error("multi-GPU: the fine level must split into an even number >= 4 of cells per rank along x "
              "(cells[0] % (2 nranks) == 0)");
    return STGMG_EINVAL;
  }
  if (nranks > 1) {
    const int G = kGhost, dq = r, dp = r - 1;
    for (int l = 0; l < levels; ++l) {
      LevelData& Lv = h->lev[l];
      if (Lv.part) {
        Lv.nsl = Lv.has_left ? halo_count(Lv.g, h->k1, G * dq + 1, G * dp + 1) : 0;
        Lv.nrl = Lv.has_left ? halo_count(Lv.g, h->k1, G * dq, G * dp) : 0;
        Lv.nsr = Lv.has_right ? halo_count(Lv.g, h->k1, G * dq, G * dp) : 0;
        Lv.nrr = Lv.has_right ? halo_count(Lv.g, h->k1, G * dq + 1, G * dp + 1) : 0;
        CK(dalloc(h.get(), &Lv.sl, (size_t)Lv.nsl));
        CK(dalloc(h.get(), &Lv.sr, (size_t)Lv.nsr));
        CK(dalloc(h.get(), &Lv.rl, (size_t)Lv.nrl));
        CK(dalloc(h.get(), &Lv.rr, (size_t)Lv.nrr));
        if (!h->lev[l - 1].part) {   // transition to the agglomerated levels
          const int oc = h->lev[l - 1].gnx / nranks;
          Lv.nag = halo_count(h->lev[l - 1].g, h->k1, oc * dq + 1, oc * dp + 1);
          CK(dalloc(h.get(), &Lv.agsend, (size_t)Lv.nag));
          CK(dalloc(h.get(), &Lv.agrecv, (size_t)Lv.nag * nranks));
        }
      }
    }
    LevelData& F = h->lev[levels - 1];
    CK(dalloc(h.get(), &h->mask, (size_t)F.g.N));
    const bool last = !F.has_right;
    CKE(launch_owned_mask(F.g, F.c0 * dq, F.c1 * dq + (last ? 1 : 0), F.c0 * dp, F.c1 * dp + (last ? 1 : 0), h->mask,
                          h->s));
  }
  {
    OpConsts cj = h->c;
    // DS (Problem B.1, Eq:DPQ_3 P:L1071-1073): the jump data of the p-equation are <c0 p^{n-1} + alpha div u^{n-1},
    // psi^+> - alpha <u_D(t_{n-1}).n, psi^+>_{G_D^u}; u_D = 0 (readings A25/A26), so no trace term of u^{n-1}
    cj.ds_face = 0.0;
    for (int b = 0; b < kMaxK1; ++b) {
      cj.theta[b] = 0.0;
      for (int a = 0; a < kMaxK1; ++a) cj.T[b][a] = (a == h->k1 - 1) ? h->c.chim1[b] : 0.0;
    }
    CK(dalloc(h.get(), &h->c_dev, 1));
    CK(dalloc(h.get(), &h->cj_dev, 1));
    CKE(cudaMemcpy(h->c_dev, &h->c, sizeof(OpConsts), cudaMemcpyHostToDevice));
    CKE(cudaMemcpy(h->cj_dev, &cj, sizeof(OpConsts), cudaMemcpyHostToDevice));
    h->cj = cj;
    {   // energy constants: ce[0] picks theta_k (A_gamma U in the chi rows), ce[1] picks T_kk (mass rows)
      OpConsts ce[2] = {h->c, h->c};
      for (int b = 0; b < kMaxK1; ++b) {
        ce[0].theta[b] = (b == h->k1 - 1) ? 1.0 : 0.0;
        ce[1].theta[b] = 0.0;
        for (int a2 = 0; a2 < kMaxK1; ++a2) {
          ce[0].T[b][a2] = 0.0;
          ce[1].T[b][a2] = (a2 == h->k1 - 1 && b == h->k1 - 1) ? 1.0 : 0.0;
        }
      }
      ce[0].ds = ce[1].ds = 0.0;
      CK(dalloc(h.get(), &h->ce_dev, 2));
      CKE(cudaMemcpy(h->ce_dev, ce, 2 * sizeof(OpConsts), cudaMemcpyHostToDevice));
    }
    {   // load-assembly constants: (r+2)-point Gauss rule, bases, GLL nodes, Radau nodes, data
      LoadConsts lc;
      std::memset(&lc, 0, sizeof(lc));
      std::vector<double> xg, wg;
      gauss01(r + 2, xg, wg);
      const auto nq = gll01(r), npn = gll01(r - 1);
      for (int q = 0; q < r + 2; ++q) {
        lc.xg[q] = xg[q];
        lc.wg[q] = wg[q];
        for (int j = 0; j <= r; ++j) lc.Bq[q][j] = lag(nq, j, xg[q]);
        for (int j = 0; j < r; ++j) lc.Bp[q][j] = lag(npn, j, xg[q]);
      }
      for (int s = 0; s < 2; ++s)
        for (int j = 0; j <= r; ++j) lc.Eq[s][j] = lag(nq, j, (double)s);
      for (int j = 0; j <= r; ++j) lc.gllq[j] = nq[j];
      for (int j = 0; j < r; ++j) lc.gllp[j] = npn[j];
      std::vector<double> tr, wr;
      radau(k, tr, wr);
      for (int b = 0; b <= k; ++b) {
        lc.that[b] = tr[b];
        lc.theta[b] = h->c.theta[b];
      }
      const LevelData& F = h->lev[levels - 1];
      for (int a0 = 0; a0 < 3; ++a0) lc.lo[a0] = mesh->lo[a0] + (a0 == 0 ? F.w0 * F.g.h[0] : 0.0);
      lc.rho = params->rho; lc.alpha = params->alpha; lc.c0 = params->c0; lc.lam = params->lambda; lc.mu = params->mu;
      for (int i = 0; i < 9; ++i) lc.K[i] = params->K[i];
      lc.r = r;
      lc.xhi_cell = (F.w0 + F.g.n[0] == (F.gnx ? F.gnx : F.g.n[0])) ? F.g.n[0] - 1 : -1;
      CK(dalloc(h.get(), &h->lc_dev, 1));
      CKE(cudaMemcpy(h->lc_dev, &lc, sizeof(LoadConsts), cudaMemcpyHostToDevice));
    }
    if (d == 2) CK(dalloc(h.get(), &h->Yc, (size_t)(cell_count(h->lev[levels - 1].g) * elem_dofs(h.get()))));
    // 2D: the register kernel on small elements (cfg1, 80 DoFs: K1 9.5 vs 13.8 us), the element GEMM on large ones
    // (cfg2, r = 3, k = 2, 219 DoFs: fine-level K1 357 -> 303 us, V-cycle 27.0 -> 26.0 ms)
    h->op_gemm = d == 3 || elem_dofs(h.get()) >= 128;
    if (const char* ev = std::getenv("STGMG_K1_FGEMM")) h->fg_on = std::atoi(ev);
    if (const char* ev = std::getenv("STGMG_K1_SF")) h->sf_on = std::atoi(ev);
    if (d == 2)
      if (const char* ev = std::getenv("STGMG_OP2D_GEMM")) h->op_gemm = std::atoi(ev) != 0;
    if (h->op_gemm) {
      long long nv = 1;
      for (int a = 0; a < 3; ++a) nv *= h->lev[levels - 1].g.n[a] + 1;
      CK(dalloc(h.get(), &h->Ycell, (size_t)(nv * elem_dofs(h.get()))));
      pm.mark("constants, element buffer", -1);
      for (int l = 0; l < levels; ++l) CK(timed("build_cells", l, [&] { return build_cells(h.get(), l, true); }));
    }
  }
  CK(timed("build_coarse", 0, [&] { return build_coarse(h.get()); }));
  for (int l = 1; l < levels; ++l) {
    CK(timed("build_patches", l, [&] { return build_patches(h.get(), l); }));
    CK(timed("build_transfer", l, [&] { return build_transfer(h.get(), l); }));
    CK(timed("build_small", l, [&] { return build_small(h.get(), l); }));
  }
  CK(timed("finish_setup", -1, [&] { return finish_setup(h.get()); }));
  *out = h.release();
  return 0;
}

// ------------------------------------------------------------------ the 3D L-shaped benchmark ----
static HostCsr to_host_csr(const LsHostCsr& m) {
  HostCsr c;
  c.rp = m.rp;
  c.ci = m.ci;
  c.v = m.v;
  return c;
}

static HostCsr transpose_csr(const LsHostCsr& m, long long ncols) {
  HostCsr t;
  t.rp.assign(ncols + 1, 0);
  for (int c : m.ci) t.rp[c + 1] += 1;
  for (long long i = 0; i < ncols; ++i) t.rp[i + 1] += t.rp[i];
  t.ci.resize(m.ci.size());
  t.v.resize(m.v.size());
  std::vector<int> pos(t.rp.begin(), t.rp.end() - 1);
  const long long nrows = (long long)m.rp.size() - 1;
  for (long long r = 0; r < nrows; ++r)      // rows ascending: columns of the transpose come out ascending
    for (int e = m.rp[r]; e < m.rp[r + 1]; ++e) {
      const int c = m.ci[e];
      t.ci[pos[c]] = (int)r;
      t.v[pos[c]] = m.v[e];
      ++pos[c];
    }
  return t;
}

// Batched equilibrated explicit inverses (K4) of n matrices already in mats (row-major, lda).
static int invert_batch(stgmg_handle* h, double* mats, int n, int nmax, const int* n_each_dev, int lda,
                        const char* what) {
  int *perm = nullptr, *status = nullptr;
  double *colk = nullptr, *scale = nullptr;
  CKE(cudaMalloc(&perm, sizeof(int) * (size_t)n * lda));
  CKE(cudaMalloc(&status, sizeof(int) * (size_t)n));
  CKE(cudaMalloc(&colk, sizeof(double) * (size_t)n * lda));
  CKE(cudaMalloc(&scale, sizeof(double) * (size_t)n * lda));
  CKE(cudaMemsetAsync(status, 0, sizeof(int) * (size_t)n, h->s));
  if (gauss_jordan_inverse(mats, n, nmax, n_each_dev, lda, perm, colk, scale, status, h->s, &h->gj)) {
    set_error(std::string(what) + ": gauss_jordan_inverse launch failed");
    return STGMG_ECUDA;
  }
  std::vector<int> st(n);
  CKE(cudaMemcpyAsync(st.data(), status, sizeof(int) * (size_t)n, cudaMemcpyDeviceToHost, h->s));
  CKE(cudaStreamSynchronize(h->s));
  cudaFree(perm);
  cudaFree(status);
  cudaFree(colk);
  cudaFree(scale);
  for (int i = 0; i < n; ++i)
    if (st[i] != 0) {
      set_error(std::string(what) + ": singular matrix " + std::to_string(i) + " (pivot " + std::to_string(st[i]) +
                ")");
      return STGMG_ESINGULAR;
    }
  return 0;
}

int stgmg_setup_lshape(int ref_fine, int levels, const stgmg_order* order, const stgmg_params* params,
                       stgmg_handle** out) {
  NvtxRange nv("stgmg_setup_lshape");
  if (!order || !params || !out) { set_error("null argument"); return STGMG_EINVAL; }
  const int r = order->r, k = order->k;
  if (r < 2 || r > 3 || k < 0 || k > 3 || levels < 1 || levels > 8 || ref_fine < levels - 1 || ref_fine > 7) {
    set_error("L-shape: need 2 <= r <= 3, 0 <= k <= 3, 1 <= levels <= ref_fine + 1, ref_fine <= 7");
    return STGMG_EINVAL;
  }
  CK(check_params(3, params));
  if (params->nranks > 1 || params->smoother != STGMG_SMOOTH_ADDITIVE || params->formulation != STGMG_FORM_DSA) {
    set_error("L-shape: single GPU, Algorithm 1 (additive) and Problem 3.1 only");
    return STGMG_ENOTSUP;
  }
  auto h = std::make_unique<stgmg_handle>();
  h->lshape = true;
  h->d = 3; h->r = r; h->k = k; h->k1 = k + 1; h->L = levels;
  h->prm = *params;
  if (h->prm.omega <= 0) h->prm.omega = 0.7;
  if (h->prm.jmax <= 0) h->prm.jmax = 4;
  if (params->stream) {
    h->s = (cudaStream_t)params->stream;
  } else {
    CKE(cudaStreamCreateWithFlags(&h->s, cudaStreamDefault));
    h->own_stream = true;
  }
  h->c = make_consts(3, r, k, h->prm);
  {
    std::vector<double> t, w;
    radau(k, t, w);
    for (int b = 0; b <= k; ++b) h->ls_that[b] = t[b];
  }
  LsHost host;
  {
    NvtxRange nv2("stgmg setup: L-shape host assembly");
    std::string err;
    const int rc = lshape_build_host(ref_fine - levels + 1, levels, r, k, h->c, params->hF_mode, host, err);
    if (rc) { set_error(err); return rc; }
  }
  h->lev.resize(levels);
  for (int l = 0; l < levels; ++l) {
    LevelData& Lv = h->lev[l];
    const LsLevelHost& Hl = host.lev[l];
    std::memset(&Lv.g, 0, sizeof(Lv.g));
    Lv.g.d = 3;
    Lv.g.nq = Hl.nq;
    Lv.g.np = Hl.np;
    Lv.g.R = 3LL * Hl.nq;
    Lv.g.S = Hl.np;
    Lv.g.block = 6LL * Hl.nq + Hl.np;
    Lv.g.N = Hl.N;
    Lv.unstr = l >= 1;
    const long long N = Hl.N;
    CK(dalloc(h.get(), &Lv.b, (size_t)N));
    CK(dalloc(h.get(), &Lv.d, (size_t)N));
    CK(dalloc(h.get(), &Lv.r, (size_t)N));
    CKE(cudaMemset(Lv.b, 0, sizeof(double) * N));
    CKE(cudaMemset(Lv.d, 0, sizeof(double) * N));
    CKE(cudaMemset(Lv.r, 0, sizeof(double) * N));
    const HostCsr A = to_host_csr(Hl.A);
    Lv.A_lpr = lanes_for(A);
    CK(upload_csr(h.get(), A, &Lv.A_rp, &Lv.A_ci, &Lv.A_v));
    if (l == 0) continue;
    const HostCsr P = to_host_csr(Hl.P);
    const HostCsr R = transpose_csr(Hl.P, host.lev[l - 1].N);
    Lv.P_lpr = lanes_for(P);
    Lv.R_lpr = lanes_for(R);
    CK(upload_csr(h.get(), P, &Lv.P_rp, &Lv.P_ci, &Lv.P_v));
    CK(upload_csr(h.get(), R, &Lv.R_rp, &Lv.R_ci, &Lv.R_v));
    Lv.npatch = (long long)Hl.pcp.size();
    Lv.pmax = Hl.maxcp;
    Lv.maxcp = Hl.maxcp;
    Lv.plda = Hl.maxcp;
    CK(upload(h.get(), &Lv.pz, Hl.pz));
    CK(upload(h.get(), &Lv.pzoff, Hl.pzoff));
    CK(upload(h.get(), &Lv.pcp, Hl.pcp));
    CK(upload(h.get(), &Lv.k3tab, Hl.k3tab));
    CK(dalloc(h.get(), &Lv.Y, (size_t)Hl.ysize));
    CKE(cudaMemset(Lv.Y, 0, sizeof(double) * Hl.ysize));
    // per-patch A_P extracted from the CSR operator, equilibrated explicit inverses (K4)
    CK(dalloc(h.get(), &Lv.pinv, (size_t)Lv.npatch * Lv.plda * Lv.plda));
    CKE(launch_csr_extract_patches(Lv.A_rp, Lv.A_ci, Lv.A_v, Lv.pz, Lv.pzoff, Lv.pcp, 0, (int)Lv.npatch, Lv.pinv,
                                   Lv.plda, h->s));
    CK(invert_batch(h.get(), Lv.pinv, (int)Lv.npatch, Lv.pmax, Lv.pcp, Lv.plda, "L-shape patch inverse"));
  }
  {   // coarse direct solve: equilibrated explicit inverse of A_0
    NvtxRange nv3("stgmg setup: coarse inverse");
    LevelData& L0 = h->lev[0];
    h->n0 = (int)L0.g.N;
    CK(dalloc(h.get(), &h->A0inv, (size_t)h->n0 * h->n0));
    CKE(launch_csr_to_dense(h->n0, L0.A_rp, L0.A_ci, L0.A_v, h->A0inv, h->s));
    int* n0dev = nullptr;
    CK(upload(h.get(), &n0dev, std::vector<int>{h->n0}));
    CK(invert_batch(h.get(), h->A0inv, 1, h->n0, n0dev, h->n0, "L-shape coarse inverse"));
  }
  {
    const HostCsr J = to_host_csr(host.J);
    h->J_lpr = lanes_for(J);
    CK(upload_csr(h.get(), J, &h->J_rp, &h->J_ci, &h->J_v));
    CK(upload(h.get(), &h->ls_fN, host.fN));
    CK(upload(h.get(), &h->ls_wu, host.wu));
    CK(upload(h.get(), &h->ls_wp, host.wp));
    h->ls_nq = host.lev[levels - 1].nq;
    h->ls_np = host.lev[levels - 1].np;
  }
  CK(finish_setup(h.get()));
  *out = h.release();
  return 0;
}

int stgmg_destroy(stgmg_handle* h) {
  delete h;   // ~stgmg_handle
  return 0;
}

int stgmg_local_size(const stgmg_handle* h, int level, int64_t* n_owned) {
  if (!h || !n_owned || level < 0 || level >= h->L) { set_error("bad level"); return STGMG_EINVAL; }
  *n_owned = h->lev[level].g.N;
  return 0;
}

int stgmg_info(const stgmg_handle* h, int level, int* n_classes, int* max_patch_dofs, int64_t* n_patches) {
  if (!h || level < 0 || level >= h->L) { set_error("bad level"); return STGMG_EINVAL; }
  if (n_classes) *n_classes = (int)h->lev[level].cls.size();
  if (max_patch_dofs) *max_patch_dofs = h->lev[level].maxcp;
  if (n_patches) *n_patches = h->lev[level].npatch;
  return 0;
}

int64_t stgmg_last_launch_count(const stgmg_handle* h) { return h ? h->launches : 0; }

int stgmg_fold_level(const stgmg_handle* h) { return h && h->fold_ready ? h->fold_lv : 0; }

static int sync_if_own(stgmg_handle* h) {
  if (h->own_stream) CKE(cudaStreamSynchronize(h->s));
  CKE(cudaGetLastError());
  return 0;
}

int stgmg_apply_operator(stgmg_handle* h, int level, const double* x, double* y) {
  if (!h || level < 0 || level >= h->L || !x || !y) { set_error("bad argument"); return STGMG_EINVAL; }
  h->launches = 0;
  CK(apply_level(h, level, x, y, nullptr, 1.0, 0.0));
  return sync_if_own(h);
}

int stgmg_residual(stgmg_handle* h, int level, const double* b, const double* x, double* r) {
  if (!h || level < 0 || level >= h->L || !x || !b || !r) { set_error("bad argument"); return STGMG_EINVAL; }
  h->launches = 0;
  CK(residual(h, level, b, x, r));
  return sync_if_own(h);
}

int stgmg_smooth_sweep(stgmg_handle* h, int level, const double* b, double* d) {
  if (!h || level < 1 || level >= h->L || !b || !d) { set_error("bad argument"); return STGMG_EINVAL; }
  h->launches = 0;
  CK(sweep(h, level, b, d, false));
  return sync_if_own(h);
}

int stgmg_restrict(stgmg_handle* h, int level, const double* rf, double* bc) {
  if (!h || level < 1 || level >= h->L) { set_error("bad level"); return STGMG_EINVAL; }
  CK(restrict_level(h, level, rf, bc));
  return sync_if_own(h);
}

int stgmg_prolong_add(stgmg_handle* h, int level, const double* dc, double* df) {
  if (!h || level < 1 || level >= h->L) { set_error("bad level"); return STGMG_EINVAL; }
  CK(prolong_level(h, level, dc, df));
  return sync_if_own(h);
}

static int vcycle_dev(stgmg_handle* h, const double* b, double* x) {
  LevelData& F = h->lev[h->L - 1];
  const size_t bytes = sizeof(double) * F.g.N;
  CKE(cudaMemcpyAsync(F.b, b, bytes, cudaMemcpyDeviceToDevice, h->s));
  if (h->vgraph) {
    CKE(cudaGraphLaunch(h->vgraph, h->s));
    h->launches += h->vgraph_launches;
  } else {
    CK(enqueue_vcycle(h));
  }
  CKE(cudaMemcpyAsync(x, F.d, bytes, cudaMemcpyDeviceToDevice, h->s));
  return 0;
}

int stgmg_vcycle(stgmg_handle* h, const double* b, double* x) {
  NvtxRange nv("stgmg_vcycle");
  if (!h || !b || !x) { set_error("bad argument"); return STGMG_EINVAL; }
  h->launches = 0;
  CK(vcycle_dev(h, b, x));
  return sync_if_own(h);
}

int stgmg_slab_load(stgmg_handle* h, int kind, double t_n, double* load) {
  if (h && load && h->lshape) {   // Sec. 5.2: chi_b rows = theta_b sin(8 pi t_{n,b}) (-<t_N, chi>)
    if (kind != STGMG_LOAD_LSHAPE_TRACTION) { set_error("L-shape handle: kind must be LSHAPE_TRACTION"); return STGMG_EINVAL; }
    double coef[kMaxK1] = {};
    for (int b = 0; b < h->k1; ++b)
      coef[b] = h->c.theta[b] * std::sin(8.0 * M_PI * (t_n + 0.5 * h->prm.tau * (1.0 + h->ls_that[b])));
    const LevelGeom& g = h->lev[h->L - 1].g;
    CKE(launch_lshape_load(g.N, g.block, g.R, h->k1, h->ls_fN, coef, load, h->s));
    h->launches = 1;
    return sync_if_own(h);
  }
  if (h && h->lshape) { set_error("bad argument"); return STGMG_EINVAL; }
  if (!h || !load || (kind != STGMG_LOAD_MANUFACTURED && kind != STGMG_LOAD_BEAM_TRACTION)) {
    set_error("bad argument");
    return STGMG_EINVAL;
  }
  const LevelGeom& g = h->lev[h->L - 1].g;
  double* yc = h->d == 2 ? h->Yc : h->Ycell;   // element-result scratch (cell-major layout), fine level
  h->launches = 0;
  cudaError_t e = launch_load_cells(h->d, h->r, h->k1, g, h->lc_dev, kind, t_n, h->prm.tau, yc, h->s);
  if (e == cudaErrorNotSupported) { set_error("(d, r, k) combination not compiled"); return STGMG_ENOTSUP; }
  CKE(e);
  CKE(launch_op_gather(g, h->r, h->k1, yc, nullptr, load, 1.0, 0.0, 1, 0, 0, h->s, 0));
  h->launches += 2;
  return sync_if_own(h);
}

int stgmg_initial_state(stgmg_handle* h, int kind, double t0, double* x) {
  if (h && x && h->lshape && kind == STGMG_LOAD_LSHAPE_TRACTION) {   // Sec. 5.2 starts at rest (reading N3-R8)
    CKE(cudaMemsetAsync(x, 0, sizeof(double) * h->lev[h->L - 1].g.N, h->s));
    h->launches = 0;
    return sync_if_own(h);
  }
  if (!h || !x || h->lshape || (kind != STGMG_LOAD_MANUFACTURED && kind != STGMG_LOAD_BEAM_TRACTION)) {
    set_error("bad argument");
    return STGMG_EINVAL;
  }
  const LevelGeom& g = h->lev[h->L - 1].g;
  CKE(launch_initial_state(h->d, h->k1, g, h->lc_dev, kind, t0, x, h->s));
  h->launches = 1;
  return sync_if_own(h);
}

// Goal quantities (Eq:DefGQ): b_u = int_face u . n do, b_p = int_face p do at t_n (last Radau
// block of x) over a whole box face; owned face cells of this rank, summed over the ranks.
int stgmg_goal_quantities(stgmg_handle* h, const double* x, int face, double* bu, double* bp) {
  if (!h || !x || !bu || !bp || face < 0 || face >= 2 * h->d) { set_error("bad argument"); return STGMG_EINVAL; }
  if (h->lshape) {   // Eq:DefGQ on Gamma_m = {1} x (0,.5) x (0,.5) (the x+ face of the L-shape)
    if (face != 1) { set_error("L-shape: the goal face is Gamma_m (face 1, x = 1)"); return STGMG_EINVAL; }
    const LevelGeom& g = h->lev[h->L - 1].g;
    const long long ob = (long long)h->k * g.block;
    CKE(launch_lshape_goal(x, ob + g.R, ob + 2 * g.R, h->ls_nq, h->ls_np, h->ls_wu, h->ls_wp, h->scal + 10, h->s));
    h->launches = 1;
    CKE(cudaMemcpyAsync(h->pinned + 10, h->scal + 10, 2 * sizeof(double), cudaMemcpyDeviceToHost, h->s));
    CKE(cudaStreamSynchronize(h->s));
    *bu = h->pinned[10];
    *bp = h->pinned[11];
    return 0;
  }
  const LevelData& F = h->lev[h->L - 1];
  const LevelGeom& g = F.g;
  const int a = face >> 1, side = face & 1;
  const int gnx = F.gnx ? F.gnx : g.n[0];
  const int c0 = F.part ? F.c0 : 0, c1 = F.part ? F.c1 : g.n[0];
  long long ncells = 1;
  for (int b = 0; b < h->d; ++b)
    if (b != a) ncells *= (b == 0 ? (c1 - c0) : g.n[b]);
  if (a == 0) {   // an x face lives on the rank that owns the first / last global cell column
    const bool here = side ? (F.w0 + c1 == gnx) : (F.w0 + c0 == 0);
    if (!here) ncells = 0;
  }
  h->launches = 0;
  if (ncells > 0) {
    cudaError_t e = launch_face_integrals(h->d, h->r, h->k1, g, h->lc_dev, x, face, c0, c1, h->w, (int)ncells,
                                          h->scal + 10, h->s);
    if (e == cudaErrorNotSupported) { set_error("(d, r) combination not compiled"); return STGMG_ENOTSUP; }
    CKE(e);
    h->launches += 2;
  } else {
    CKE(cudaMemsetAsync(h->scal + 10, 0, 2 * sizeof(double), h->s));
  }
  if (h->nranks > 1) {
    const int rc = h->tr->allreduce_sum(h->scal + 10, 2, h->s);
    if (rc) return rc;
  }
  CKE(cudaMemcpyAsync(h->pinned + 10, h->scal + 10, 2 * sizeof(double), cudaMemcpyDeviceToHost, h->s));
  CKE(cudaStreamSynchronize(h->s));
  *bu = h->pinned[10];
  *bp = h->pinned[11];
  return 0;
}

int stgmg_slab_rhs(stgmg_handle* h, const double* load, const double* x_prev, double* rhs) {
  NvtxRange nv("stgmg_slab_rhs");
  if (!h || !x_prev || !rhs) { set_error("bad argument"); return STGMG_EINVAL; }
  const LevelGeom& g = h->lev[h->L - 1].g;
  h->launches = 0;
  if (h->lshape) {   // F_n = L_n + J X_{n-1} with the assembled coupling (one SpMV)
    CKE(launch_csr_spmv((int)g.N, h->J_lpr, h->J_rp, h->J_ci, h->J_v, x_prev, load, rhs, 1.0, 1.0, h->s));
    h->launches = 1;
    return sync_if_own(h);
  }
  LevelData& F = h->lev[h->L - 1];
  if (F.fg && F.sf_ntiles && h->c.ds == 0.0) {
    // 3D fine level with the sum-factorised K1: J X_{n-1} has theta = 0, so every term of the operator but the mass
    // terms vanishes (the Nitsche face terms carry theta_b too) and the volume-only kernel is exact on EVERY cell
    // type; element results into Ycell, one gather adds the load
    CKE(launch_op_sf3(g, h->r, h->k1, F.sf_tiles, F.sf_ntiles, F.ecls_dev, h->cj, x_prev, h->Ycell, h->s));
    if (F.fg_ntiles) CKE(launch_op_sf3(g, h->r, h->k1, F.fg_tiles, F.fg_ntiles, F.ecls_dev, h->cj, x_prev, h->Ycell, h->s));
    CKE(launch_op_gather(g, h->r, h->k1, h->Ycell, load, rhs, 1.0, 1.0, 1, 0, 0, h->s, 0));
    h->launches = F.fg_ntiles ? 3 : 2;
    return sync_if_own(h);
  }
  CK(apply_geom(h, g, h->cj_dev, x_prev, rhs, load, 1.0, 1.0));
  return sync_if_own(h);
}

// Inner product <w, v> (v == nullptr: ||w||^2, sqrt if norm) over the owned DoFs, summed over the ranks; the MGS
// update w <- w - (*hprev) vprev is fused into the same pass.
static int dot(stgmg_handle* h, double* w, const double* vprev, const double* hprev, const double* vnext, double* out,
               bool norm) {
  const long long N = h->lev[h->L - 1].g.N;
  const bool dist = h->nranks > 1;
  CKE(launch_mgs_dot(w, vprev, hprev, vnext, N, h->partials, h->counter, out, (norm && !dist) ? 1 : 0, h->mask, h->s));
  h->launches += 1;
  if (dist) {
    const int rc = h->tr->allreduce_sum(out, 1, h->s);
    if (rc) return rc;
    if (norm) {
      CKE(launch_sqrt(out, h->s));
      h->launches += 1;
    }
  }
  return 0;
}

// Discrete energy at t_n of a slab solution (P7, Eq:ExUniDS_3 P:L300-306):
//   E = A_gamma(U, U) + <rho V, V> + <c0 P, P>,  (V, U, P) = the last Radau block of x (t_{n,k+1} = t_n).
// Two operator applies with selector constants on placed copies of that block, two owned-DoF inner products.
int stgmg_energy(stgmg_handle* h, const double* x, double* energy) {
  if (!h || !x || !energy) { set_error("bad argument"); return STGMG_EINVAL; }
  if (h->lshape) { set_error("stgmg_energy: not available for the L-shape"); return STGMG_ENOTSUP; }
  const int Lf = h->L - 1;
  const LevelGeom& g = h->lev[Lf].g;
  double *Y = h->w, *O = h->rv, *Zt = h->stage_rhs;
  h->launches = 0;
  // A_gamma(U, U): input (0, U, 0) in the last block, T = 0, theta_k = 1 -> chi rows = A_gamma U
  CKE(launch_energy_place(g, h->k1, x, Y, 0, h->s));
  CK(exchange(h, Lf, Y));
  CK(apply_geom(h, g, h->ce_dev, Y, O, nullptr, 1.0, 0.0));
  CK(dot(h, O, nullptr, nullptr, Y, h->scal + 8, false));
  // <rho V, V> + <c0 P, P>: input (V, 0, P), T_kk = 1, theta = 0 -> chi rows = M_rho V, psi rows = M_c P; test
  // vector (0, V, P) aligns V with the chi rows
  CKE(launch_energy_place(g, h->k1, x, Y, 1, h->s));
  CK(exchange(h, Lf, Y));
  CK(apply_geom(h, g, h->ce_dev + 1, Y, O, nullptr, 1.0, 0.0));
  CKE(launch_energy_place(g, h->k1, x, Zt, 2, h->s));
  CK(dot(h, O, nullptr, nullptr, Zt, h->scal + 9, false));
  h->launches += 3;
  CKE(cudaMemcpyAsync(h->pinned + 8, h->scal + 8, 2 * sizeof(double), cudaMemcpyDeviceToHost, h->s));
  CKE(cudaStreamSynchronize(h->s));
  *energy = h->pinned[8] + h->pinned[9];
  return 0;
}

// The part of Arnoldi step j after the preconditioner: w = A z_j, MGS against v_0..v_j, ||w||, Givens, v_{j+1}.
static int arnoldi_tail(stgmg_handle* h, int j, int m, bool cond, cudaGraphConditionalHandle next) {
  const int Lf = h->L - 1, ldh = m + 1;
  const long long N = h->lev[Lf].g.N;
  double* zj = h->Z + (long long)j * N;
  CK(apply_level(h, Lf, zj, h->w, nullptr, 1.0, 0.0));                 // w = A z_j
  double* hcol = h->H + (long long)j * ldh;
  for (int i = 0; i <= j; ++i)                                         // modified Gram–Schmidt
    CK(dot(h, h->w, i > 0 ? h->V + (long long)(i - 1) * N : nullptr, i > 0 ? hcol + (i - 1) : nullptr,
           h->V + (long long)i * N, hcol + i, false));
  CK(dot(h, h->w, h->V + (long long)j * N, hcol + j, nullptr, hcol + j + 1, true));
  if (cond) CKE(launch_givens_cond(h->H, ldh, h->cs, h->sn, h->gv, j, h->scal, h->ctl, j + 1 < m ? 1 : 0, next, h->s));
  else CKE(launch_givens(h->H, ldh, h->cs, h->sn, h->gv, j, h->scal, h->s));
  CKE(launch_scale(h->V + (long long)(j + 1) * N, h->w, h->scal + 1, 1, N, h->s));   // v_{j+1} = w / h_{j+1,j}
  h->launches += 2;
  return exchange(h, Lf, h->V + (long long)(j + 1) * N);
}

// One Arnoldi step j of FGMRES (O11): z_j = V-cycle(v_j), then arnoldi_tail.  Single GPU: the whole step is one
// CUDA graph captured at first use with the fine level's right-hand side / iterate bound to v_j / z_j (no copies
// around the preconditioner, programmatic dependent launch across the V-cycle / apply / MGS boundary).
// cond: capture mode of the device-resident loop (V-cycle as a child graph, Givens decides step j + 1).
static int enqueue_arnoldi_step(stgmg_handle* h, int j, int m, bool cond, cudaGraphConditionalHandle next) {
  const int Lf = h->L - 1;
  const long long N = h->lev[Lf].g.N;
  double* vj = h->V + (long long)j * N;
  double* zj = h->Z + (long long)j * N;
  LevelData& F = h->lev[Lf];
  if (cond) {
    CKE(cudaMemcpyAsync(F.b, vj, sizeof(double) * N, cudaMemcpyDeviceToDevice, h->s));
    if (h->vgraph_tmpl && !h->cyc_inline) {   // the V-cycle graph as a child node of the capture
      cudaStreamCaptureStatus st;
      cudaGraph_t cg;
      const cudaGraphNode_t* deps = nullptr;
      size_t ndep = 0;
      CKE(cudaStreamGetCaptureInfo(h->s, &st, nullptr, &cg, &deps, &ndep));
      cudaGraphNode_t child;
      CKE(cudaGraphAddChildGraphNode(&child, cg, deps, ndep, h->vgraph_tmpl));
      CKE(cudaStreamUpdateCaptureDependencies(h->s, &child, 1, cudaStreamSetCaptureDependencies));
      h->launches += h->vgraph_launches;
    } else {
      CK(enqueue_vcycle(h));
    }
    CKE(cudaMemcpyAsync(zj, F.d, sizeof(double) * N, cudaMemcpyDeviceToDevice, h->s));
    return arnoldi_tail(h, j, m, true, next);
  }
  // per-step graphs whenever the V-cycle itself is captured: single GPU, or a graph-capturable transport (NCCL: the
  // halo send/recv, the all-reduce of the MGS dots and the all-gather of the agglomeration are captured stream work);
  // the host-synchronising loopback / shared-memory transports never get here (no V-cycle graph)
  if (h->vgraph && h->step_graphs) {
    if (h->vg_step_m != m) {   // H's leading dimension is m + 1: graphs of another restart length are stale
      for (auto& g : h->vg_step)
        if (g) {
          cudaGraphExecDestroy(g);
          g = nullptr;
        }
      h->vg_step_m = m;
    }
    if ((int)h->vg_step.size() <= j) {
      h->vg_step.resize(j + 1, nullptr);
      h->vg_step_launches.resize(j + 1, 0);
    }
    if (!h->vg_step[j]) {
      double* b0 = F.b;
      double* d0 = F.d;
      cudaGraph_t graph;
      const long long before = h->launches;
      CKE(cudaStreamBeginCapture(h->s, cudaStreamCaptureModeThreadLocal));
      F.b = vj;
      F.d = zj;
      int rc = enqueue_vcycle(h);
      F.b = b0;
      F.d = d0;
      if (!rc) rc = arnoldi_tail(h, j, m, false, cudaGraphConditionalHandle());
      cudaError_t e = cudaStreamEndCapture(h->s, &graph);
      h->vg_step_launches[j] = (int)(h->launches - before);
      h->launches = before;
      if (rc) return rc;
      CKE(e);
      e = cudaGraphInstantiate(&h->vg_step[j], graph, 0);
      cudaGraphDestroy(graph);
      CKE(e);
    }
    CKE(cudaGraphLaunch(h->vg_step[j], h->s));
    h->launches += h->vg_step_launches[j];
    return 0;
  }
  CK(vcycle_dev(h, vj, zj));                                          // z_j = M^{-1} v_j
  return arnoldi_tail(h, j, m, false, cudaGraphConditionalHandle());
}

// The device-resident restart cycle: a graph of m IF nodes in a chain, node j's body = Arnoldi step j (captured
// with cudaStreamBeginCaptureToGraph); handle j defaults to (j == 0) at every launch and is set by step j - 1's
// Givens kernel.  Single GPU only (the x-slab decomposition's NCCL exchanges stay on the host loop).
static int build_cycle_graph(stgmg_handle* h, int m) {
  if (h->cyc_exec && h->cyc_m == m) return 0;
  if (h->cyc_exec) {
    cudaGraphExecDestroy(h->cyc_exec);
    h->cyc_exec = nullptr;
  }
  cudaGraph_t G;
  CKE(cudaGraphCreate(&G, 0));
  std::vector<cudaGraphConditionalHandle> hd(m);
  int rc = 0;
  for (int j = 0; j < m && !rc; ++j)
    if (cudaGraphConditionalHandleCreate(&hd[j], G, j == 0 ? 1u : 0u, cudaGraphCondAssignDefault) != cudaSuccess) {
      set_error("cudaGraphConditionalHandleCreate failed");
      rc = STGMG_ECUDA;
    }
  cudaGraphNode_t prev = nullptr;
  const long long before = h->launches;
  h->cyc_step_launches.assign(m, 0);
  for (int j = 0; j < m && !rc; ++j) {
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = hd[j];
    np.conditional.type = cudaGraphCondTypeIf;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    if (cudaGraphAddNode(&node, G, prev ? &prev : nullptr, prev ? 1 : 0, &np) != cudaSuccess) {
      set_error("cudaGraphAddNode (conditional) failed");
      rc = STGMG_ECUDA;
      break;
    }
    cudaGraph_t body = np.conditional.phGraph_out[0];
    if (cudaStreamBeginCaptureToGraph(h->s, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) !=
        cudaSuccess) {
      set_error("cudaStreamBeginCaptureToGraph failed");
      rc = STGMG_ECUDA;
      break;
    }
    const long long l0 = h->launches;
    rc = enqueue_arnoldi_step(h, j, m, true, j + 1 < m ? hd[j + 1] : hd[j]);
    h->cyc_step_launches[j] = (int)(h->launches - l0);
    cudaGraph_t out = nullptr;
    const cudaError_t e = cudaStreamEndCapture(h->s, &out);
    if (!rc && e != cudaSuccess) {
      set_error(std::string("capture of an Arnoldi step: ") + cudaGetErrorString(e));
      rc = STGMG_ECUDA;
    }
    prev = node;
  }
  h->launches = before;
  if (!rc) {
    const cudaError_t e = cudaGraphInstantiate(&h->cyc_exec, G, 0);
    if (e != cudaSuccess) {
      set_error(std::string("cudaGraphInstantiate (Arnoldi cycle): ") + cudaGetErrorString(e));
      h->cyc_exec = nullptr;
      rc = STGMG_ECUDA;
    }
  }
  cudaGraphDestroy(G);
  cudaGetLastError();
  if (!rc) h->cyc_m = m;
  return rc;
}

int stgmg_solve(stgmg_handle* h, const double* rhs, double* x, double tol, int tol_mode, int restart, int maxit,
                stgmg_stats* stats) {
  NvtxRange nv("stgmg_solve");
  if (!h || !rhs || !x || restart < 1 || maxit < 1 || !(tol > 0)) { set_error("bad argument"); return STGMG_EINVAL; }
  CK(ensure_krylov(h, restart));
  const int Lf = h->L - 1;
  const LevelGeom& g = h->lev[Lf].g;
  const long long N = g.N;
  const int m = restart, ldh = m + 1;
  bool graph_ok = h->nranks == 1 && h->graphable && !h->cyc_off;
  if (graph_ok && build_cycle_graph(h, m)) {   // not buildable here: the host-checked loop
    if (std::getenv("STGMG_DEBUG")) std::fprintf(stderr, "stgmg: device-resident FGMRES off: %s\n", g_last_error.c_str());
    h->cyc_off = true;
    graph_ok = false;
    cudaGetLastError();
  }
  h->launches = 0;
  double* scal = h->scal;     // [0] |g_{j+1}|, [1] h_{j+1,j}, [2] beta, [3] ||b||
  double* hp = h->pinned;
  CKE(cudaEventRecord(h->e0, h->s));
  if (h->nranks > 1) {        // ghost values of the right-hand side and of the initial guess
    if (rhs != h->rhs_int) CKE(cudaMemcpyAsync(h->rhs_int, rhs, sizeof(double) * N, cudaMemcpyDeviceToDevice, h->s));
    CK(exchange(h, Lf, h->rhs_int));
    CK(exchange(h, Lf, x));
    rhs = h->rhs_int;
  }
  CK(dot(h, const_cast<double*>(rhs), nullptr, nullptr, nullptr, scal + 3, true));
  CK(residual(h, Lf, rhs, x, h->rv));
  CK(dot(h, h->rv, nullptr, nullptr, nullptr, scal + 2, true));
  CKE(cudaMemcpyAsync(hp, scal, 4 * sizeof(double), cudaMemcpyDeviceToHost, h->s));
  CKE(cudaStreamSynchronize(h->s));
  const double bnorm = hp[3];
  double beta = hp[2];
  const double target = tol_mode == STGMG_TOL_ABS ? tol : tol * bnorm;
  int its = 0, restarts = 0;
  bool converged = beta <= target;
  int* hctl = reinterpret_cast<int*>(hp + 14);
  const bool use_graph = graph_ok && !converged;
  if (use_graph) {   // target, maxit and the step counter of the device loop
    hp[4] = target;
    hp[5] = (double)maxit;
    CKE(cudaMemcpyAsync(scal + 4, hp + 4, 2 * sizeof(double), cudaMemcpyHostToDevice, h->s));
    CKE(cudaMemsetAsync(h->ctl, 0, 2 * sizeof(int), h->s));
  }
  while (!converged && its < maxit) {
    CKE(launch_scale(h->V, h->rv, scal + 2, 1, N, h->s));                 // v_0 = r / beta
    CK(exchange(h, Lf, h->V));
    CKE(cudaMemsetAsync(h->gv, 0, sizeof(double) * (m + 1), h->s));
    CKE(launch_set_scalar(h->gv, scal + 2, h->s));                        // g_0 = beta
    CKE(cudaMemsetAsync(h->H, 0, sizeof(double) * ldh * m, h->s));
    h->launches += 2;
    int jdone = 0;
    if (use_graph) {   // the whole cycle on the device: the Givens kernels chain the steps
      CKE(cudaGraphLaunch(h->cyc_exec, h->s));
      CKE(launch_backsub_ctl(h->H, ldh, h->gv, h->yv, h->ctl, h->s));
      CKE(launch_update_x_ctl(x, h->Z, h->yv, h->ctl, N, h->s));
      h->launches += 2;
      CK(residual(h, Lf, rhs, x, h->rv));
      CK(dot(h, h->rv, nullptr, nullptr, nullptr, scal + 2, true));
      CKE(cudaMemcpyAsync(hp + 2, scal + 2, sizeof(double), cudaMemcpyDeviceToHost, h->s));
      CKE(cudaMemcpyAsync(hctl, h->ctl, 2 * sizeof(int), cudaMemcpyDeviceToHost, h->s));
      CKE(cudaStreamSynchronize(h->s));
      jdone = hctl[1];
      for (int j = 0; j < jdone; ++j) h->launches += h->cyc_step_launches[j];
      its = hctl[0];
      beta = hp[2];
      if (beta <= target) { converged = true; break; }
      if (its >= maxit) break;
      ++restarts;
      continue;
    }
    for (int j = 0; j < m; ++j) {
      if (h->prof) CKE(cudaEventRecord(h->pev[h->npev++ % 64], h->s));
      CK(enqueue_arnoldi_step(h, j, m, false, cudaGraphConditionalHandle()));
      if (h->prof) CKE(cudaEventRecord(h->pev[h->npev++ % 64], h->s));
      CKE(cudaMemcpyAsync(hp, scal, 2 * sizeof(double), cudaMemcpyDeviceToHost, h->s));
      CKE(cudaStreamSynchronize(h->s));
      ++its;
      jdone = j + 1;
      if (hp[0] <= target || hp[1] <= 1e-14 * beta || its >= maxit) break;
    }
    CKE(launch_backsub(h->H, ldh, h->gv, h->yv, jdone, h->s));
    CKE(launch_update_x(x, h->Z, h->yv, jdone, N, h->s));
    h->launches += 2;
    CK(residual(h, Lf, rhs, x, h->rv));
    CK(dot(h, h->rv, nullptr, nullptr, nullptr, scal + 2, true));
    CKE(cudaMemcpyAsync(hp + 2, scal + 2, sizeof(double), cudaMemcpyDeviceToHost, h->s));
    CKE(cudaStreamSynchronize(h->s));
    beta = hp[2];
    if (beta <= target) { converged = true; break; }
    if (its >= maxit) break;
    ++restarts;
  }
  CKE(cudaEventRecord(h->e1, h->s));
  CKE(cudaEventSynchronize(h->e1));
  float ms = 0.f;
  CKE(cudaEventElapsedTime(&ms, h->e0, h->e1));
  if (h->prof && h->npev >= 2 && h->npev <= 64) {   // per Arnoldi step: device time, then the gap to the next step
    float t = 0.f;
    std::fprintf(stderr, "stgmg solve profile (us):");
    cudaEventElapsedTime(&t, h->e0, h->pev[0]);
    std::fprintf(stderr, " start->step0 %.1f;", t * 1e3f);
    for (int i = 0; i + 1 < h->npev; i += 2) {
      float a = 0.f, g = 0.f;
      cudaEventElapsedTime(&a, h->pev[i], h->pev[i + 1]);
      if (i + 2 < h->npev) cudaEventElapsedTime(&g, h->pev[i + 1], h->pev[i + 2]);
      else cudaEventElapsedTime(&g, h->pev[i + 1], h->e1);
      std::fprintf(stderr, " | step %.1f next %.1f", a * 1e3f, g * 1e3f);
    }
    std::fprintf(stderr, "\n");
  }
  h->npev = 0;
  if (stats) {
    if (!h->lev_ready && its > 0) CK(profile_levels(h));   // once per handle, outside the timed solve
    std::memset(stats, 0, sizeof(*stats));
    stats->iterations = its;
    stats->restarts = restarts;
    stats->abs_residual = beta;
    stats->rel_residual = bnorm > 0 ? beta / bnorm : 0.0;
    stats->seconds = ms * 1e-3;
    for (int l = 0; l < h->L && l < 16; ++l) stats->level_seconds[l] = its * h->lev_ms[l] * 1e-3;
  }
  return converged ? STGMG_OK : STGMG_NOT_CONVERGED;
}

int stgmg_solve_host(stgmg_handle* h, const double* rhs_host, double* x_host, double tol, int tol_mode, int restart,
                     int maxit, stgmg_stats* stats) {
  if (!h || !rhs_host || !x_host) { set_error("bad argument"); return STGMG_EINVAL; }
  LevelData& F = h->lev[h->L - 1];
  const size_t bytes = sizeof(double) * F.g.N;
  CK(ensure_krylov(h, restart));
  double* stage_rhs = h->stage_rhs;   // allocated in stgmg_setup
  double* stage_x = h->stage_x;
  CKE(cudaMemcpyAsync(stage_rhs, rhs_host, bytes, cudaMemcpyHostToDevice, h->s));
  CKE(cudaMemcpyAsync(stage_x, x_host, bytes, cudaMemcpyHostToDevice, h->s));
  int rc = stgmg_solve(h, stage_rhs, stage_x, tol, tol_mode, restart, maxit, stats);
  if (rc < 0) return rc;
  CKE(cudaMemcpyAsync(x_host, stage_x, bytes, cudaMemcpyDeviceToHost, h->s));
  CKE(cudaStreamSynchronize(h->s));
  return rc;
}

int stgmg_level_work(const stgmg_handle* h, int level, double* k2_flops, double* k2_bytes, double* k1_bytes) {
  if (h && h->lshape) { set_error("not available for the L-shape"); return STGMG_ENOTSUP; }
  if (!h || level < 0 || level >= h->L) { set_error("bad level"); return STGMG_EINVAL; }
  const LevelData& Lv = h->lev[level];
  double fl = 0.0, sumcp = 0.0, invb = 0.0;
  for (const auto& c : Lv.cls) {
    fl += 2.0 * (double)c.cp * (double)c.cp * (double)c.ncols;
    sumcp += (double)c.cp * (double)c.ncols;
    invb += 8.0 * (double)c.cp * (double)c.cp;
  }
  if (k2_flops) *k2_flops = fl;
  if (k2_bytes) *k2_bytes = 8.0 * 2.0 * sumcp + invb;     // gather R_P r + write Y + read the class inverses
  if (k1_bytes) *k1_bytes = 16.0 * (double)Lv.g.N;         // y = A x: read x, write y
  return 0;
}

int stgmg_kernel_work(const stgmg_handle* h, int kind, int level, double* flops, double* bytes) {
  if (!h || level < 0 || level >= h->L || !flops || !bytes) { set_error("bad argument"); return STGMG_EINVAL; }
  if (h->lshape) {   // K2u: one explicit inverse per patch, streamed once per sweep (HBM-bound GEMV)
    if (kind != 0 || !h->lev[level].unstr) { set_error("L-shape: kind 0 on levels >= 1 only"); return STGMG_ENOTSUP; }
    std::vector<int> cps(h->lev[level].npatch);
    CKE(cudaMemcpy(cps.data(), h->lev[level].pcp, sizeof(int) * cps.size(), cudaMemcpyDeviceToHost));
    double s2 = 0.0, s1 = 0.0;
    for (int c : cps) { s2 += (double)c * c; s1 += c; }
    *flops = 2.0 * s2;
    *bytes = 8.0 * s2 + 16.0 * s1;   // the inverses (C_P^2 each) + gather r, write y
    return 0;
  }
  const LevelData& Lv = h->lev[level];
  const double N = (double)Lv.g.N;
  double sumcp = 0.0, fl2 = 0.0, invb = 0.0;
  for (const auto& c : Lv.cls) {
    fl2 += 2.0 * (double)c.cp * (double)c.cp * (double)c.ncols;
    sumcp += (double)c.cp * (double)c.ncols;
    invb += 8.0 * (double)c.cp * (double)c.cp;
  }
  *flops = 0.0;
  switch (kind) {
    case 0: *flops = fl2; *bytes = 16.0 * sumcp + invb; break;                 // K2
    case 1: {   // K1: read x, write y; flops = SURVEY §8(d)'s sum-factorised count (the algorithmic work, not the
                // padded factored-GEMM flops the kernel issues): (k+1) n_cells [(6d^2+5d) 2 (r+1)^(d+1) + c_pt (r+1)^d]
      *bytes = 16.0 * N;
      const int d = h->d, r1 = h->r + 1;
      double nc = 1.0, rp = 1.0;
      for (int a = 0; a < d; ++a) { nc *= Lv.g.n[a]; rp *= r1; }
      const double cpt = d == 3 ? 100.0 : 60.0;
      *flops = (double)h->k1 * nc * ((6.0 * d * d + 5.0 * d) * 2.0 * rp * r1 + cpt * rp);
      break;
    }
    case 2: *bytes = 16.0 * N + 8.0 * sumcp; break;                            // K3: read Y, read + write d
    case 7: {                                                                  // K5: restrict + prolong-add
      if (level < 1) { set_error("kind 7 needs level >= 1"); return STGMG_EINVAL; }
      const double Nc = (double)h->lev[level - 1].g.N;
      *bytes = 8.0 * N + 8.0 * Nc + 8.0 * Nc + 16.0 * N;
      break;
    }
    case 8: *bytes = 32.0 * N; break;                                          // K7: read w, v_prev, v_next; write w
    default: set_error("no work model for this kind"); return STGMG_EINVAL;
  }
  return 0;
}

int stgmg_time_kernel(stgmg_handle* h, int kind, int level, int reps, double* avg_ms) {
  if (h && h->lshape && kind != 0 && kind != 1 && kind != 2 && kind != 3 && kind != 6) {
    set_error("L-shape: kinds 0 (K2u), 1, 2, 3, 6 only");
    return STGMG_ENOTSUP;
  }
  if (!h || level < 0 || level >= h->L || reps < 1 || !avg_ms) { set_error("bad argument"); return STGMG_EINVAL; }
  if ((kind == 0 || kind == 2 || kind == 6 || kind == 7) && level < 1) {
    set_error("smoother kernels need level >= 1");
    return STGMG_EINVAL;
  }
  if (kind == 8 && (level != h->L - 1 || h->m_alloc < 1)) {
    set_error("kind 8 (MGS pass) needs the fine level and an allocated Krylov basis (run a solve first)");
    return STGMG_EINVAL;
  }
  if (kind == 8) CKE(cudaMemsetAsync(h->scal + 12, 0, sizeof(double), h->s));   // h = 0: w is left unchanged
  LevelData& Lv = h->lev[level];
  auto one = [&]() -> int {
    if (kind == 0) {
      if (Lv.unstr)
        CKE(launch_patch_gemv((int)Lv.npatch, Lv.pmax, Lv.pz, Lv.pzoff, Lv.pcp, Lv.pinv, Lv.plda, Lv.r, Lv.Y, h->s));
      else if (Lv.dense)
        CKE(launch_patch_gemm_dense(Lv.g, Lv.k2var, Lv.cls_dev, Lv.tiles_dev, Lv.ntiles, Lv.inv_dev, Lv.lda, Lv.Rexp,
                                    Lv.Y, Lv.ldy, h->s));
      else
        CKE(launch_patch_gemm(Lv.g, h->r, Lv.k2var, Lv.cls_dev, Lv.tiles_dev, Lv.ntiles, Lv.relidx_dev, Lv.inv_dev,
                              Lv.lda, Lv.r, Lv.Y, Lv.ldy, h->s));
    } else if (kind == 1) {
      CK(apply_level(h, level, Lv.d, Lv.r, nullptr, 1.0, 0.0));
    } else if (kind == 2) {
      CK(average_level(h, level, false, Lv.d));
    } else if (kind == 4) {
      CKE(launch_noop(1, h->s));
    } else if (kind == 5) {
      CKE(launch_noop(148, h->s));
    } else if (kind == 6) {   // one post-smoothing sweep (residual, patch solves, averaging)
      CK(sweep(h, level, Lv.b, Lv.d, false));
    } else if (kind == 7) {   // restriction to and prolongation from level - 1
      CK(restrict_level(h, level, Lv.r, h->lev[level - 1].b));
      CK(prolong_level(h, level, h->lev[level - 1].d, Lv.d));
    } else if (kind == 8) {   // one fused MGS pass of K7 on the fine level: w -= h v_0, <w, v_1>
      CK(dot(h, h->w, h->V, h->scal + 12, h->V + h->lev[h->L - 1].g.N, h->scal + 13, false));
    } else if (h->vgraph) {
      CKE(cudaGraphLaunch(h->vgraph, h->s));
    } else {
      CK(enqueue_vcycle(h));
    }
    return 0;
  };
  CK(one());   // warm-up
  // a graph launch cannot be captured, and a host-synchronising transport (loopback / shared memory) cannot be
  // captured either: time back-to-back launches instead
  if (kind == 3 || !h->graphable) {
    CKE(cudaEventRecord(h->e0, h->s));
    for (int i = 0; i < reps; ++i) CK(one());
    CKE(cudaEventRecord(h->e1, h->s));
    CKE(cudaEventSynchronize(h->e1));
    float ms3 = 0.f;
    CKE(cudaEventElapsedTime(&ms3, h->e0, h->e1));
    *avg_ms = ms3 / reps;
    return 0;
  }
  // capture the reps launches into a CUDA graph so that host launch overhead does not enter the measurement
  cudaGraph_t gr;
  cudaGraphExec_t ge;
  CKE(cudaStreamBeginCapture(h->s, cudaStreamCaptureModeThreadLocal));
  for (int i = 0; i < reps; ++i) {
    int rc = one();
    if (rc) { cudaStreamEndCapture(h->s, &gr); return rc; }
  }
  CKE(cudaStreamEndCapture(h->s, &gr));
  CKE(cudaGraphInstantiate(&ge, gr, 0));
  CKE(cudaGraphLaunch(ge, h->s));
  CKE(cudaEventRecord(h->e0, h->s));
  CKE(cudaGraphLaunch(ge, h->s));
  CKE(cudaEventRecord(h->e1, h->s));
  CKE(cudaEventSynchronize(h->e1));
  float ms = 0.f;
  CKE(cudaEventElapsedTime(&ms, h->e0, h->e1));
  if (h->prof && h->npev >= 4 && h->npev <= 64) {   // per step: [gap] vcycle | apply | MGS + Givens + scale
    float t = 0.f;
    std::fprintf(stderr, "stgmg solve profile (us):");
    cudaEventElapsedTime(&t, h->e0, h->pev[0]);
    std::fprintf(stderr, " start->step0 %.1f;", t * 1e3f);
    for (int i = 0; i + 3 < h->npev; i += 4) {
      float a = 0.f, b = 0.f, c = 0.f, g = 0.f;
      cudaEventElapsedTime(&a, h->pev[i], h->pev[i + 1]);
      cudaEventElapsedTime(&b, h->pev[i + 1], h->pev[i + 2]);
      cudaEventElapsedTime(&c, h->pev[i + 2], h->pev[i + 3]);
      if (i + 4 < h->npev) cudaEventElapsedTime(&g, h->pev[i + 3], h->pev[i + 4]);
      else cudaEventElapsedTime(&g, h->pev[i + 3], h->e1);
      std::fprintf(stderr, " | vc %.1f ap %.1f mgs %.1f next %.1f", a * 1e3f, b * 1e3f, c * 1e3f, g * 1e3f);
    }
    std::fprintf(stderr, "\n");
  }
  h->npev = 0;
  cudaGraphExecDestroy(ge);
  cudaGraphDestroy(gr);
  *avg_ms = ms / reps;
  return 0;
}

int stgmg_partition_plan(const stgmg_mesh* mesh, int levels, int level, int rank, int nranks, int* split, int* gnx,
                         int* w0, int* c0, int* c1, int* nx_window) {
  if (!mesh || levels < 1 || level < 0 || level >= levels || nranks < 1 || rank < 0 || rank >= nranks) {
    set_error("bad argument");
    return STGMG_EINVAL;
  }
  bool finer = true;
  int out[6] = {0, 0, 0, 0, 0, 0};
  for (int l = levels - 1; l >= level; --l) {
    const int n = mesh->cells[0] >> (levels - 1 - l);
    const bool part = nranks > 1 && l >= 1 && finer && n % (2 * nranks) == 0 && n / nranks >= 4;   // as stgmg_setup
    finer = part;
    if (l == level) {
      if (part) {
        const int own = n / nranks, a = rank * own, b = a + own;
        const int ws = rank > 0 ? a - kGhost : 0, we = rank < nranks - 1 ? b + kGhost : n;
        out[0] = 1; out[1] = n; out[2] = ws; out[3] = a - ws; out[4] = b - ws; out[5] = we - ws;
      } else {
        out[0] = 0; out[1] = n; out[2] = 0; out[3] = 0; out[4] = n; out[5] = n;
      }
    }
  }
  if (split) *split = out[0];
  if (gnx) *gnx = out[1];
  if (w0) *w0 = out[2];
  if (c0) *c0 = out[3];
  if (c1) *c1 = out[4];
  if (nx_window) *nx_window = out[5];
  return 0;
}

int stgmg_nccl_unique_id(unsigned char id_out[128]) { return nccl_unique_id(id_out); }
int stgmg_nccl_comm_create(const unsigned char id[128], int nranks, int rank, void** comm_out) {
  return nccl_comm_create(id, nranks, rank, comm_out);
}
int stgmg_nccl_comm_destroy(void* comm) { return nccl_comm_destroy(comm); }
int stgmg_shm_comm_create(const char* name, int nranks, int rank, int64_t cap_doubles, void** comm_out) {
  return shm_comm_create(name, nranks, rank, (long long)cap_doubles, comm_out);
}
int stgmg_shm_comm_destroy(void* comm) { return shm_comm_destroy(comm); }
void* stgmg_loopback_hub_create(int nranks) { return loopback_hub_create(nranks); }
void stgmg_loopback_hub_destroy(void* hub) { loopback_hub_destroy(hub); }

}  // extern "C"
