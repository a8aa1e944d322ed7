/* stgmg.h — C ABI of the B200-native space-time GMRES–GMG slab solver (arXiv:2303.06742 hot path).
 *
 * One call of stgmg_solve solves the algebraic I_n-problem  A_n X_n = F_n  (Problem 4.1, Eq:ALS_In,
 * PAPER.md P:L384-390) of the numerically integrated slab problem (Problem 3.1, Eq:DPQ_A0):
 * flexible GMRES(m) right-preconditioned by one geometric-multigrid V-cycle
 * whose smoother is the additive patch-wise Vanka Algorithm 1 (Def:VankaOP P:L469-485,
 * alg:smoother P:L488-524), with interpolation / transpose grid transfer and a direct coarse solve
 * (P:L438).  Spaces: Taylor–Hood Q_r^d / Q_{r-1} (continuous pressure, P:L148 Def:VhQh) with Nitsche
 * boundary terms (Def:ACB, Def:ab); time: dG(k) with a Lagrange basis at the k+1 right
 * Gauss–Radau nodes (Eq:GF P:L122-128, Eq:TimeExp P:L356-362).  Everything is IEEE binary64.
 *
 * Vector layout (every vector argument; Eq:DefXn): for m = 0..k (Radau node), blocks
 *   V (d components), U (d components), P, each component a lexicographic node array (x fastest);
 *   Q_r nodes per axis r*n_a+1 (n_q in total), Q_{r-1} nodes per axis (r-1)*n_a+1 (n_p in total);
 *   offsets V_c: m*(2R+S) + c*n_q,  U_c: m*(2R+S) + R + c*n_q,  P: m*(2R+S) + 2R,  R = d*n_q, S = n_p,
 *   N_l = (k+1)(2R+S).  Row slots of A_n are aligned with the column slots: the V slot holds the rho-scaled
 *   u-equation (test phi), the U slot the v-equation (test chi), the P slot the p-equation (test psi)
 *   (SURVEY §8(c) reading A5).
 *
 * Return codes: 0 = OK, >0 = soft result, <0 = error (message via stgmg_last_error()).
 * Ownership: every vector pointer is caller-owned DEVICE memory (e.g. torch.Tensor.data_ptr()) of length
 * stgmg_local_size(level), except the *_host entry points, which take caller-owned HOST memory.  The
 * library owns every internal buffer (inverses, Krylov basis, level vectors); all of them are allocated in
 * stgmg_setup and freed in stgmg_destroy; nothing is allocated during a solve.  All device work is
 * enqueued on params.stream (0 = the legacy default stream); stgmg_solve / stgmg_solve_host return after a
 * stream synchronisation with the stats filled.  A handle is not thread-safe: one handle per stream/thread.
 */
#ifndef STGMG_H
#define STGMG_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct stgmg_handle stgmg_handle; /* opaque, owned by the library */

enum {
  STGMG_OK = 0,
  STGMG_NOT_CONVERGED = 1, /* maxit Arnoldi steps reached; stats filled, x = last iterate */
  STGMG_EINVAL = -1,       /* invalid argument: r<2, k<0, cells not divisible by 2^(levels-1), rho/c0/tau<=0, ... */
  STGMG_ENOMEM = -2,       /* device allocation failed */
  STGMG_ECUDA = -3,        /* CUDA runtime error; message carries cudaGetErrorString */
  STGMG_ENCCL = -4,        /* multi-GPU transport error (NCCL call failed / libnccl not loadable); message names it */
  STGMG_ESINGULAR = -5,    /* zero pivot in a patch-class or coarse inverse; message names level and class */
  STGMG_ECOVER = -6,       /* a DoF lies in no patch (p_mu == 0) */
  STGMG_ENOTSUP = -7       /* (d, r, k) combination not compiled into this library */
};
enum { STGMG_BC_DIRICHLET = 0, STGMG_BC_NEUMANN = 1 };
enum { STGMG_HF_MEASURE = 0 /* h_F = |K|_d, P:L205 (default) */, STGMG_HF_EDGE = 1 /* h_F = h normal to F */ };
enum { STGMG_TOL_REL = 0 /* ||r|| <= tol ||b|| (BASELINE) */, STGMG_TOL_ABS = 1 /* ||r|| <= tol */ };
enum { STGMG_SMOOTH_ADDITIVE = 0 /* Alg. 1 with averaging, P:L488-524 (default) */,
       STGMG_SMOOTH_COLORED_MULT = 1 /* Eq:VankaOP0 with successive overwriting, patches
                                        ordered by vertex colour (v mod 4 per axis); single GPU only */,
       STGMG_SMOOTH_ELEMENT = 2 /* Alg. 1 on one patch per CELL (element-wise Vanka, the variant the
                                   Remark after alg:smoother P:L529-531 rejects); single GPU only */,
       STGMG_SMOOTH_OVERWRITE = 3 /* Alg. 1 without averaging, every DoF keeps the update of the last
                                     patch (lexicographic) containing it; single GPU only */ };
enum { STGMG_FORM_DSA = 0 /* Problem 3.1 (Eq:DPQ_A0): p-equation couples v (default) */,
       STGMG_FORM_DS = 1 /* Problem B.1: p-equation couples d_t u through T, slab RHS
                            adds -chi_b(-1) C U^{n-1} (stgmg_slab_rhs) */ };
enum { STGMG_LOAD_MANUFACTURED = 0, STGMG_LOAD_BEAM_TRACTION = 1,   /* stgmg_slab_load */
       STGMG_LOAD_LSHAPE_TRACTION = 2 /* Sec. 5.2 traction on the L-shape (stgmg_setup_lshape handles only) */ };
enum { STGMG_COMM_NCCL = 0 /* nccl_comm is an ncclComm_t */,
       STGMG_COMM_LOOPBACK = 1 /* nccl_comm is an in-process hub (N emulated ranks on one GPU; tests) */,
       STGMG_COMM_SHM = 2 /* nccl_comm is a stgmg_shm_comm_create communicator (one process per rank) */ };

/* Structured box, fine level (nested quad/hex levels, h_l = h_{l-1}/2). */
typedef struct {
  int dim;          /* 2 or 3 */
  int cells[3];     /* fine cells per axis; each divisible by 2^(levels-1); cells[2] ignored for dim 2 */
  double lo[3];     /* box lower corner */
  double hi[3];     /* box upper corner */
  int bc_u[6];      /* per face x-,x+,y-,y+,z-,z+: STGMG_BC_DIRICHLET (Nitsche) or _NEUMANN */
  int bc_p[6];
} stgmg_mesh;

typedef struct {
  int r; /* degree of u, v (Q_r); pressure Q_{r-1}; r >= 2 */
  int k; /* dG(k) in time, k+1 Radau nodes; k >= 0 */
} stgmg_order;

typedef struct {
  double rho, alpha, c0, lambda, mu; /* P:L52; isotropic C from (lambda, mu); all > 0 except lambda >= 0 */
  double K[9];                       /* permeability / conductivity, row-major d x d (upper-left block used) */
  double tau;                        /* slab length tau_n (uniform) */
  double gamma_a, gamma_b;           /* Nitsche penalties; < 0 -> 5e4 r(r+1), r(r-1)/2 */
  int hF_mode;                       /* STGMG_HF_MEASURE (default) | STGMG_HF_EDGE */
  double omega;                      /* Vanka under-relaxation, 0.7; <= 0 -> 0.7 */
  int jmax;                          /* smoothing steps per level, 4; <= 0 -> 4 */
  int smoother;                      /* STGMG_SMOOTH_ADDITIVE (default) | _COLORED_MULT | _ELEMENT | _OVERWRITE */
  void* nccl_comm;                   /* multi-GPU: ncclComm_t (STGMG_COMM_NCCL) or loopback hub; NULL if nranks = 1 */
  int rank, nranks;                  /* x-slab domain decomposition over nranks GPUs */
  void* stream;                      /* cudaStream_t for all work; NULL = a library-owned BLOCKING stream (ordered after
                                        work queued on the legacy default stream; calls sync it before returning) */
  int comm_kind;                     /* STGMG_COMM_NCCL | STGMG_COMM_LOOPBACK */
  int formulation;                   /* STGMG_FORM_DSA (Problem 3.1, default) | STGMG_FORM_DS (Problem B.1) */
} stgmg_params;

typedef struct {
  int iterations;         /* total Arnoldi steps (= V-cycles applied) */
  int restarts;           /* completed restart cycles */
  double rel_residual;    /* true ||b - A x|| / ||b|| at return */
  double abs_residual;    /* true ||b - A x|| at return */
  double seconds;         /* device time of the solve (CUDA events on params.stream) */
  double level_seconds[16];/* [l] = iterations x device time of level l's share of one V-cycle (its sweeps, residual,
                              transfers; level 0 / the folded level: the coarse solve), measured once per handle by an
                              event-bracketed eager V-cycle after the first solve (outside `seconds`); 0 above L-1 and
                              below the folded level (SPEC SolveStats) */
} stgmg_stats;

/* Build the level hierarchy, the matrix-free operators, the patch-class inverses (equilibrated LU /
 * Gauss–Jordan on the device) and the coarse inverse; capture the V-cycle as a CUDA graph.
 * levels counts the coarse level (levels = 1: direct solve only).  *out receives the handle.
 * Errors: EINVAL (parameters), ENOMEM, ECUDA, ESINGULAR, ECOVER, ENOTSUP. */
int stgmg_setup(const stgmg_mesh* mesh, int levels, const stgmg_order* order, const stgmg_params* params,
                stgmg_handle** out);

/* the 3D L-shaped benchmark of Sec. 5.2 with the Q_r^d / P_{r-1}^disc pair
 * (Def:VhQh P:L130-148; B_gamma = the symmetric interior penalty option of Def:B; directional conditions
 * Eq:BCd P:L757-781).  Domain ([0,1] x [0,.5] U [0,.5] x [.5,1]) x [0,.5] with 2^ref_fine cells per cube edge on the
 * fine level; levels = ref_fine - ref_coarse + 1 (Table 4: coarse level ref_1).  Boundary parts as DESIGN.md
 * readings N3-R1/R2: u = 0 on y = 0; directional on x = 0 and z = 0, .5; traction t_N on y = 1 (x < .5); free on
 * x = 1 and the re-entrant faces; p = 0 on y = 1 (x < .5), no flux elsewhere.  params: rho, alpha, c0, lambda, mu, K,
 * tau, gamma_a, gamma_b (gamma = gamma_b of the SIP term), hF_mode (penalty length of the Nitsche, directional and
 * SIP terms: cell measure h^3 by default, reading A6; STGMG_HF_EDGE: h; 2: h^3 but h for the directional faces;
 * 3: the fine level's h^3 on every level — coarse operators = Galerkin products; experiments on the grid robustness of
 * Table 4: 4: h^3 for u, h for the SIP faces of p; 5: h for u, h^3 for p; 6: the face measure h^2 for
 * both), omega, jmax, stream (mesh, bc, smoother,
 * formulation and nranks are not used: single GPU, Alg. 1, Problem 3.1).  Level operators are assembled (CSR) on the
 * host at setup from element integrals; every patch has its own explicit inverse (K4 on the device).  Vector layout per
 * Radau node: V_0..V_2, U_0..U_2 on the active Q_r nodes (lexicographic over the (2 r 2^ref + 1)^2 (r 2^ref + 1) node
 * grid, x fastest), then P (dim P_{r-1} monomials per active cell, cells lexicographic).  All other entry points
 * accept the handle except stgmg_energy / stgmg_level_work (ENOTSUP); stgmg_time_kernel takes kinds 0 (K2u, the
 * per-patch inverse GEMV), 1, 2, 3, 6 and stgmg_kernel_work kind 0 (8 sum C_P^2 + 16 sum C_P bytes, 2 sum C_P^2 flops);
 * stgmg_slab_load takes STGMG_LOAD_LSHAPE_TRACTION, stgmg_goal_quantities face 1 (Gamma_m, Eq:DefGQ).
 * Errors: EINVAL, ENOTSUP (r, k, nranks > 1, smoother / formulation variants), ENOMEM, ECUDA, ESINGULAR, ECOVER. */
int stgmg_setup_lshape(int ref_fine, int levels, const stgmg_order* order, const stgmg_params* params,
                       stgmg_handle** out);

/* Number of slab DoFs N_l of a level (0 = coarse .. levels-1 = fine).  Multi-GPU: the DoFs of the rank's x-window
 * (owned cells plus 3 ghost cells per interior side); vectors passed to the library use this local numbering. */
int stgmg_local_size(const stgmg_handle* h, int level, int64_t* n_owned);

/* Multi-GPU partition of level l (host-only, no GPU needed): global cells along x, window start (global cell),
 * owned cells [c0, c1) in window-local cell indices, window cells along x, and whether the level is split
 * (1) or agglomerated / replicated (0).  A level is split while every rank owns an even number >= 4 of cells along x
 * and all finer levels are split. */
int stgmg_partition_plan(const stgmg_mesh* mesh, int levels, int level, int rank, int nranks, int* split,
                         int* gnx, int* w0, int* c0, int* c1, int* nx_window);

/* y = A_l x on level l (matrix-free, Problem 3.1 rediscretised on T_l; reading A14).  x, y: device. */
int stgmg_apply_operator(stgmg_handle* h, int level, const double* x, double* y);

/* r = b - A_l x on level l.  b, x, r: device, r may not alias x. */
int stgmg_residual(stgmg_handle* h, int level, const double* b, const double* x, double* r);

/* One smoothing sweep of Algorithm 1 on level l >= 1: d <- d + omega (sum_P E_P A_P^-1 R_P
 * (b - A_l d)) / p.  d is updated in place.  Exposed for kernel-level parity tests. */
int stgmg_smooth_sweep(stgmg_handle* h, int level, const double* b, double* d);

/* x = V-cycle(b) on the fine level: the preconditioner application M^{-1} b. */
int stgmg_vcycle(stgmg_handle* h, const double* b, double* x);

/* Restriction b_c = P_l^T r_f (level l -> l-1) and prolongation-add d_f += P_l d_c. */
int stgmg_restrict(stgmg_handle* h, int level, const double* r_fine, double* b_coarse);
int stgmg_prolong_add(stgmg_handle* h, int level, const double* d_coarse, double* d_fine);

/* FGMRES(restart) with x as initial guess (x = 0 for the paper's setting).  tol_mode: STGMG_TOL_*.
 * maxit counts Arnoldi steps (reading A35).  Returns OK, NOT_CONVERGED or an error; stats may be NULL. */
int stgmg_solve(stgmg_handle* h, const double* rhs, double* x, double tol, int tol_mode, int restart, int maxit,
                stgmg_stats* stats);

/* Same as stgmg_solve with HOST buffers: copies rhs host->device and x both ways inside the call. */
int stgmg_solve_host(stgmg_handle* h, const double* rhs_host, double* x_host, double tol, int tol_mode,
                     int restart, int maxit, stgmg_stats* stats);

/* SURVEY §8(f) N1, on-device load assembly: load = L_n of the slab (t_n, t_n + tau] in the slab layout — at Radau
 * node b, U slot (chi rows) theta_b F_gamma(t_{n,b}), P slot (psi rows) theta_b G_gamma(t_{n,b}), V slot 0, with
 * t_{n,b} = t_n + tau/2 (t_hat_b + 1) (Def:LG P:L215-228).  kind STGMG_LOAD_MANUFACTURED: the body loads
 * of the BASELINE manufactured solution u_i = S sin(2 pi t), p = S cos(2 pi t), S = prod sin(pi x_a) (configs 0/1/3;
 * reading A8), (r+2)^d Gauss points per cell (reading A10); STGMG_LOAD_BEAM_TRACTION: + sin(pi t/2) int_{x=hi}
 * chi_{d-1} (config 4, reading A23).  Homogeneous Dirichlet data only (readings A26, A31).  load: caller-owned device
 * vector of stgmg_local_size(fine); F_n = stgmg_slab_rhs(load, X_{n-1}). */
int stgmg_slab_load(stgmg_handle* h, int kind, double t_n, double* load);

/* x = 0 except its LAST Radau block = nodal interpolation of (v(t0), u(t0), p(t0)) of the manufactured
 * solution (reading A20; zero for STGMG_LOAD_BEAM_TRACTION), i.e. the X_0 that stgmg_slab_rhs reads for slab 1. */
int stgmg_initial_state(stgmg_handle* h, int kind, double t0, double* x);

/* SURVEY N1 / P7 (Eq:ExUniDS_3): discrete energy at t_n of the slab solution x (its last Radau block
 * (V, U, P)): *energy = A_gamma(U, U) + <rho V, V> + <c0 P, P> (host scalar; owned DoFs summed over the ranks).
 * With zero loads it is non-increasing from slab to slab. */
int stgmg_energy(stgmg_handle* h, const double* x, double* energy);

/* SURVEY N1, goal quantities of Eq:DefGQ on a whole box face (0..2d-1 = x-, x+, y-, y+, z-, z+) at t_n:
 * *b_u = int_face u . n do and *b_p = int_face p do of the last Radau block of x ((r+2)^{d-1} Gauss points per face
 * cell; host scalars; owned face cells summed over the ranks).  EINVAL for a face index outside 0..2d-1. */
int stgmg_goal_quantities(stgmg_handle* h, const double* x, int face, double* b_u, double* b_p);

/* Slab RHS: rhs = load + J X_prev, where X_prev is the previous slab's full vector (its last
 * Radau block is the state at t_{n-1}) and J puts chi_b(-1) M_rho U, chi_b(-1) M_rho V,
 * chi_b(-1) M_c P into the V, U, P slots of node b.  load: the theta_b-scaled load part (may be NULL). */
int stgmg_slab_rhs(stgmg_handle* h, const double* load, const double* x_prev, double* rhs);

int stgmg_destroy(stgmg_handle* h);

/* Thread-local message of the last error. */
const char* stgmg_last_error(void);

/* NCCL bootstrap (libnccl.so.2 is loaded on first use): rank 0 creates the 128-byte id, the caller broadcasts it
 * (e.g. torch.distributed), every rank creates its communicator; the caller owns and destroys it. */
int stgmg_nccl_unique_id(unsigned char id_out[128]);
int stgmg_nccl_comm_create(const unsigned char id[128], int nranks, int rank, void** comm_out);
int stgmg_nccl_comm_destroy(void* comm);

/* In-process loopback hub for N emulated ranks on one GPU (tests of the decomposition; one host thread per rank,
 * each with its own handle and stream; the host synchronises at every exchange). */
void* stgmg_loopback_hub_create(int nranks);
void stgmg_loopback_hub_destroy(void* hub);

/* Process-separated shared-memory communicator (comm_kind STGMG_COMM_SHM): one PROCESS per rank (as under torchrun),
 * on one GPU or several, without NCCL.  Messages are staged through a POSIX shared-memory segment /<name> (rank 0
 * creates and finally unlinks it; the others attach, waiting up to ~20 s) with a mailbox of cap_doubles doubles per
 * message slot; a sense-reversing barrier on process-shared atomics orders the exchanges (host-synchronised, not
 * graph-capturable).  Every rank passes the same name, nranks and cap; comm_out is owned by the caller, who destroys it
 * (collectively) after the handle.  Errors: -1 bad argument, -4 (ENCCL) segment not created / attached. */
int stgmg_shm_comm_create(const char* name, int nranks, int rank, int64_t cap_doubles, void** comm_out);
int stgmg_shm_comm_destroy(void* comm);

/* Diagnostics: number of patch classes on level l, their sizes C_P and the number of kernels launched by
 * the last stgmg_solve (for the bench's gpu_launches field). */
int stgmg_info(const stgmg_handle* h, int level, int* n_classes, int* max_patch_dofs, int64_t* n_patches);
int64_t stgmg_last_launch_count(const stgmg_handle* h);
/* The folded coarse sub-cycle (csrc/api.cu build_fold): the finest level f whose V-cycle (levels f..0: Alg. 1
 * sweeps, transfers, coarse solve) is applied as its assembled n_f x n_f matrix, 0 if none (exact up to
 * rounding; environment STGMG_FOLD_MB=0 at setup disables it). */
int stgmg_fold_level(const stgmg_handle* h);

/* Algorithmic work of one launch on level l (measurement): K2 flops = 2 sum_P C_P^2,
 * K2 bytes = 8 (2 sum_P C_P) + 8 sum_classes C_P^2 (gather, Y write, class inverses), K1 bytes = 16 N_l. */
int stgmg_level_work(const stgmg_handle* h, int level, double* k2_flops, double* k2_bytes, double* k1_bytes);

/* Times reps back-to-back launches of one hot-path kernel on level l with CUDA events on params.stream:
 * kind 0 = K2 patch GEMM, 1 = K1 operator apply (all colours), 2 = K3 averaging, 3 = whole V-cycle graph,
 * 4 / 5 = empty kernel on 1 / 148 CTAs, 6 = one smoothing sweep (level >= 1), 7 = restriction + prolongation,
 * 8 = one fused MGS pass of K7 (fine level only, after a solve has allocated the Krylov basis).
 * Operates on the level's internal work buffers (their contents are overwritten). */
int stgmg_time_kernel(stgmg_handle* h, int kind, int level, int reps, double* avg_ms);

/* Algorithmic work of one launch of stgmg_time_kernel's kind on level l (SURVEY §8(d) "Binding roofline"):
 * kind 0 (K2): flops 2 sum_P C_P^2, bytes 16 sum_P C_P + 8 sum_classes C_P^2; kind 1 (K1, y = A x): 16 N_l bytes
 * and the sum-factorised flop count (k+1) n_cells [(6d^2+5d) 2 (r+1)^(d+1) + c_pt (r+1)^d], c_pt = 60 (2D) / 100 (3D);
 * kind 2 (K3): 16 N_l + 8 sum_P C_P bytes (read Y, read and write d; 1/p is structural); kind 7 (K5 restrict +
 * prolong-add): 24 N_l + 16 N_{l-1} bytes; kind 8 (K7 fused MGS pass): 32 N bytes.  flops = 0 for kinds 2, 7, 8.
 * EINVAL for other kinds. */
int stgmg_kernel_work(const stgmg_handle* h, int kind, int level, double* flops, double* bytes);

#ifdef __cplusplus
}
#endif
#endif /* STGMG_H */
