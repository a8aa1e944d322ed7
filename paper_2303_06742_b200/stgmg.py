"""Thin ctypes binding of the C ABI in include/stgmg.h (argument marshalling only).

Every step of the hot path runs in the CUDA kernels of libstgmg.so; this module only converts Python /
torch arguments to the plain pointers and structs of the ABI.  It never falls back to a CPU path: if the
library or a CUDA device is missing, it raises.
"""
import ctypes
import os

from .build import LIB, build, needs_build

STGMG_OK, STGMG_NOT_CONVERGED = 0, 1
TOL_REL, TOL_ABS = 0, 1
BC_DIRICHLET, BC_NEUMANN = 0, 1
HF_MEASURE, HF_EDGE = 0, 1
SMOOTH_ADDITIVE, SMOOTH_COLORED_MULT, SMOOTH_ELEMENT, SMOOTH_OVERWRITE = 0, 1, 2, 3
LOAD_MANUFACTURED, LOAD_BEAM_TRACTION, LOAD_LSHAPE_TRACTION = 0, 1, 2
FORM_DSA, FORM_DS = 0, 1


class Mesh(ctypes.Structure):
    _fields_ = [("dim", ctypes.c_int), ("cells", ctypes.c_int * 3), ("lo", ctypes.c_double * 3),
                ("hi", ctypes.c_double * 3), ("bc_u", ctypes.c_int * 6), ("bc_p", ctypes.c_int * 6)]


class Order(ctypes.Structure):
    _fields_ = [("r", ctypes.c_int), ("k", ctypes.c_int)]


class Params(ctypes.Structure):
    _fields_ = [("rho", ctypes.c_double), ("alpha", ctypes.c_double), ("c0", ctypes.c_double),
                ("lambda_", ctypes.c_double), ("mu", ctypes.c_double), ("K", ctypes.c_double * 9),
                ("tau", ctypes.c_double), ("gamma_a", ctypes.c_double), ("gamma_b", ctypes.c_double),
                ("hF_mode", ctypes.c_int), ("omega", ctypes.c_double), ("jmax", ctypes.c_int),
                ("smoother", ctypes.c_int), ("nccl_comm", ctypes.c_void_p), ("rank", ctypes.c_int),
                ("nranks", ctypes.c_int), ("stream", ctypes.c_void_p), ("comm_kind", ctypes.c_int),
                ("formulation", ctypes.c_int)]


class Stats(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int), ("restarts", ctypes.c_int), ("rel_residual", ctypes.c_double),
                ("abs_residual", ctypes.c_double), ("seconds", ctypes.c_double),
                ("level_seconds", ctypes.c_double * 16)]

    def as_dict(self):
        return dict(iterations=self.iterations, restarts=self.restarts, rel_residual=self.rel_residual,
                    abs_residual=self.abs_residual, seconds=self.seconds, level_seconds=list(self.level_seconds))


# name -> (restype, argtypes) — every symbol declared in include/stgmg.h
_P = ctypes.c_void_p
SIGNATURES = {
    "stgmg_setup": (ctypes.c_int, [ctypes.POINTER(Mesh), ctypes.c_int, ctypes.POINTER(Order), ctypes.POINTER(Params),
                                   ctypes.POINTER(_P)]),
    "stgmg_setup_lshape": (ctypes.c_int, [ctypes.c_int, ctypes.c_int, ctypes.POINTER(Order), ctypes.POINTER(Params),
                                          ctypes.POINTER(_P)]),
    "stgmg_local_size": (ctypes.c_int, [_P, ctypes.c_int, ctypes.POINTER(ctypes.c_int64)]),
    "stgmg_apply_operator": (ctypes.c_int, [_P, ctypes.c_int, _P, _P]),
    "stgmg_residual": (ctypes.c_int, [_P, ctypes.c_int, _P, _P, _P]),
    "stgmg_smooth_sweep": (ctypes.c_int, [_P, ctypes.c_int, _P, _P]),
    "stgmg_vcycle": (ctypes.c_int, [_P, _P, _P]),
    "stgmg_restrict": (ctypes.c_int, [_P, ctypes.c_int, _P, _P]),
    "stgmg_prolong_add": (ctypes.c_int, [_P, ctypes.c_int, _P, _P]),
    "stgmg_solve": (ctypes.c_int, [_P, _P, _P, ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                   ctypes.POINTER(Stats)]),
    "stgmg_solve_host": (ctypes.c_int, [_P, _P, _P, ctypes.c_double, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                        ctypes.POINTER(Stats)]),
    "stgmg_slab_rhs": (ctypes.c_int, [_P, _P, _P, _P]),
    "stgmg_slab_load": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_double, _P]),
    "stgmg_initial_state": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_double, _P]),
    "stgmg_energy": (ctypes.c_int, [_P, _P, ctypes.POINTER(ctypes.c_double)]),
    "stgmg_goal_quantities": (ctypes.c_int, [_P, _P, ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                             ctypes.POINTER(ctypes.c_double)]),
    "stgmg_destroy": (ctypes.c_int, [_P]),
    "stgmg_last_error": (ctypes.c_char_p, []),
    "stgmg_info": (ctypes.c_int, [_P, ctypes.c_int, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                  ctypes.POINTER(ctypes.c_int64)]),
    "stgmg_last_launch_count": (ctypes.c_int64, [_P]),
    "stgmg_fold_level": (ctypes.c_int, [_P]),
    "stgmg_level_work": (ctypes.c_int, [_P, ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                        ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]),
    "stgmg_time_kernel": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                         ctypes.POINTER(ctypes.c_double)]),
    "stgmg_kernel_work": (ctypes.c_int, [_P, ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                         ctypes.POINTER(ctypes.c_double)]),
    "stgmg_partition_plan": (ctypes.c_int, [ctypes.POINTER(Mesh), ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                            ctypes.c_int] + [ctypes.POINTER(ctypes.c_int)] * 6),
    "stgmg_nccl_unique_id": (ctypes.c_int, [ctypes.c_char_p]),
    "stgmg_nccl_comm_create": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.POINTER(_P)]),
    "stgmg_nccl_comm_destroy": (ctypes.c_int, [_P]),
    "stgmg_loopback_hub_create": (_P, [ctypes.c_int]),
    "stgmg_shm_comm_create": (ctypes.c_int, [ctypes.c_char_p, ctypes.c_int, ctypes.c_int, ctypes.c_int64,
                                             ctypes.POINTER(_P)]),
    "stgmg_shm_comm_destroy": (ctypes.c_int, [_P]),
    "stgmg_loopback_hub_destroy": (None, [_P]),
}

_lib = None


def load_library(path=None, rebuild=False):
    """Load libstgmg.so (building it in-tree first if it is missing or stale)."""
    global _lib
    if _lib is not None and not rebuild:
        return _lib
    path = path or os.environ.get("STGMG_LIB") or LIB   # STGMG_LIB: experiment builds (A/B timing)
    if rebuild or needs_build():
        build()
    if not os.path.exists(path):
        raise RuntimeError("libstgmg.so not found at %s (build with paper_2303_06742_b200.build)" % path)
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class StgmgError(RuntimeError):
    pass


def _check(rc, what):
    if rc < 0:
        raise StgmgError("%s failed (%d): %s" % (what, rc, _lib.stgmg_last_error().decode()))
    return rc


def _ptr(t, n=None, device=None):
    """Device pointer of a contiguous CUDA float64 torch tensor, checked against the ABI's expectations: exactly n
    elements (the level's stgmg_local_size) on the solver's device.  Wrong arguments raise instead of letting the
    library read or write out of bounds."""
    import torch
    if not isinstance(t, torch.Tensor):
        raise TypeError("expected a torch.Tensor")
    if not t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous():
        raise TypeError("expected a contiguous CUDA float64 tensor")
    if n is not None and t.numel() != n:
        raise ValueError("tensor has %d elements, the level vector has %d" % (t.numel(), n))
    if device is not None and t.device != device:
        raise ValueError("tensor on %s, solver on %s" % (t.device, device))
    return ctypes.c_void_p(t.data_ptr())


def _host_ptr(a, n):
    """Host pointer of a C-contiguous float64 CPU array (numpy or torch) of exactly n elements."""
    import numpy as np
    try:
        import torch
        if isinstance(a, torch.Tensor):
            if a.is_cuda or a.dtype != torch.float64 or not a.is_contiguous():
                raise TypeError("expected a contiguous CPU float64 tensor")
            if a.numel() != n:
                raise ValueError("host tensor has %d elements, expected %d" % (a.numel(), n))
            return ctypes.c_void_p(a.data_ptr())
    except ImportError:
        pass
    if not isinstance(a, np.ndarray) or a.dtype != np.float64 or not a.flags["C_CONTIGUOUS"]:
        raise TypeError("expected a C-contiguous float64 numpy array or CPU tensor")
    if a.size != n:
        raise ValueError("host array has %d elements, expected %d" % (a.size, n))
    if not a.flags["WRITEABLE"]:
        raise ValueError("host array must be writeable")
    return a.ctypes.data_as(ctypes.c_void_p)


COMM_NCCL, COMM_LOOPBACK, COMM_SHM = 0, 1, 2


def make_mesh(cfg):
    d = cfg["dim"]
    m = Mesh()
    m.dim = d
    for a in range(3):
        m.cells[a] = int(cfg["cells"][a]) if a < d else 1
        m.lo[a] = float(cfg["lo"][a])
        m.hi[a] = float(cfg["hi"][a])
    for f in range(6):
        m.bc_u[f] = int(cfg["bc_u"][f])
        m.bc_p[f] = int(cfg["bc_p"][f])
    return m


def setup_args(cfg, tau=None, omega=0.7, jmax=4, hF_mode=HF_MEASURE, rank=0, nranks=1, comm=None,
               comm_kind=COMM_NCCL, smoother=0, formulation=0):
    """(stgmg_mesh, stgmg_order, stgmg_params) of a configuration dict (stream left NULL)."""
    m = make_mesh(cfg)
    o = Order(int(cfg["r"]), int(cfg["k"]))
    p = Params()
    pr = cfg["params"]
    p.rho, p.alpha, p.c0, p.lambda_, p.mu = pr["rho"], pr["alpha"], pr["c0"], pr["lam"], pr["mu"]
    K = list(pr["K"])
    if len(K) == 4:
        K = [K[0], K[1], 0, K[2], K[3], 0, 0, 0, 0]
    for i in range(9):
        p.K[i] = float(K[i])
    p.tau = float(tau if tau is not None else cfg["tau"])
    p.gamma_a = float(pr.get("gamma_a", -1.0) or -1.0)
    p.gamma_b = float(pr.get("gamma_b", -1.0) or -1.0)
    p.hF_mode = hF_mode
    p.omega = omega
    p.jmax = jmax
    p.smoother = int(smoother)         # SMOOTH_ADDITIVE (Alg. 1) | _COLORED_MULT | _ELEMENT | _OVERWRITE (N2)
    p.formulation = int(formulation)   # FORM_DSA (Problem 3.1) | FORM_DS (Problem B.1)
    p.nccl_comm = comm
    p.rank, p.nranks = int(rank), int(nranks)
    p.comm_kind = int(comm_kind)
    return m, o, p


def partition_plan(cfg, level, rank, nranks):
    """Host-only partition of a level (no GPU): dict(split, gnx, w0, c0, c1, nx_window)."""
    lib = load_library()
    outs = [ctypes.c_int() for _ in range(6)]
    _check(lib.stgmg_partition_plan(ctypes.byref(make_mesh(cfg)), int(cfg["levels"]), level, rank, nranks,
                                    *[ctypes.byref(o) for o in outs]), "stgmg_partition_plan")
    return dict(zip(["split", "gnx", "w0", "c0", "c1", "nx_window"], [o.value for o in outs]))


def nccl_unique_id():
    lib = load_library()
    buf = ctypes.create_string_buffer(128)
    _check(lib.stgmg_nccl_unique_id(buf), "stgmg_nccl_unique_id")
    return bytes(buf.raw)


def nccl_comm_create(uid, nranks, rank):
    lib = load_library()
    comm = ctypes.c_void_p()
    _check(lib.stgmg_nccl_comm_create(ctypes.c_char_p(bytes(uid)), nranks, rank, ctypes.byref(comm)),
           "stgmg_nccl_comm_create")
    return comm


def nccl_comm_destroy(comm):
    load_library().stgmg_nccl_comm_destroy(comm)


def shm_comm_create(name, nranks, rank, cap_doubles=1 << 22):
    """Process-separated shared-memory communicator (one process per rank; stgmg_shm_comm_create)."""
    lib = load_library()
    comm = ctypes.c_void_p()
    _check(lib.stgmg_shm_comm_create(name.encode(), int(nranks), int(rank), int(cap_doubles), ctypes.byref(comm)),
           "stgmg_shm_comm_create")
    return comm


def shm_comm_destroy(comm):
    load_library().stgmg_shm_comm_destroy(comm)


def loopback_hub(nranks):
    return ctypes.c_void_p(load_library().stgmg_loopback_hub_create(nranks))


def loopback_hub_destroy(hub):
    load_library().stgmg_loopback_hub_destroy(hub)


class Solver:
    """One slab system A_n X_n = F_n of a structured configuration (see stgmg_inputs.CONFIGS).

    Multi-GPU (x-slab decomposition): pass rank, nranks and comm (an NCCL communicator from nccl_comm_create, or a
    loopback hub with comm_kind=COMM_LOOPBACK); vectors are then the rank's window vectors (stgmg_local_size)."""

    def __init__(self, cfg, stream=None, tau=None, omega=0.7, jmax=4, hF_mode=HF_MEASURE, levels=None,
                 rank=0, nranks=1, comm=None, comm_kind=COMM_NCCL, smoother=0, formulation=0):
        import torch
        if not torch.cuda.is_available():
            raise StgmgError("no CUDA device: the stgmg product path has no CPU fallback")
        self.lib = load_library()
        self.cfg = cfg
        m, o, p = setup_args(cfg, tau, omega, jmax, hF_mode, rank, nranks, comm, comm_kind, smoother, formulation)
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        p.stream = ctypes.c_void_p(self.stream.cuda_stream)
        self.levels = int(levels or cfg["levels"])
        h = ctypes.c_void_p()
        _check(self.lib.stgmg_setup(ctypes.byref(m), self.levels, ctypes.byref(o), ctypes.byref(p), ctypes.byref(h)),
               "stgmg_setup")
        self.h = h
        self.device = self.stream.device
        self._n = []
        for lev in range(self.levels):
            n = ctypes.c_int64()
            _check(self.lib.stgmg_local_size(self.h, lev, ctypes.byref(n)), "stgmg_local_size")
            self._n.append(n.value)

    def _lev(self, level):
        lev = self.levels - 1 if level is None else int(level)
        if not 0 <= lev < self.levels:
            raise ValueError("level %d outside 0..%d" % (lev, self.levels - 1))
        return lev

    def _p(self, t, level=None):
        return _ptr(t, self._n[self._lev(level)], self.device)

    def close(self):
        if getattr(self, "h", None):
            self.lib.stgmg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def size(self, level=None):
        n = ctypes.c_int64()
        lev = self.levels - 1 if level is None else level
        _check(self.lib.stgmg_local_size(self.h, lev, ctypes.byref(n)), "stgmg_local_size")
        return n.value

    def info(self, level):
        nc, mx, npat = ctypes.c_int(), ctypes.c_int(), ctypes.c_int64()
        _check(self.lib.stgmg_info(self.h, level, ctypes.byref(nc), ctypes.byref(mx), ctypes.byref(npat)), "stgmg_info")
        return dict(n_classes=nc.value, max_patch_dofs=mx.value, n_patches=npat.value)

    def apply(self, x, y, level=None):
        lev = self._lev(level)
        _check(self.lib.stgmg_apply_operator(self.h, lev, self._p(x, lev), self._p(y, lev)), "stgmg_apply_operator")

    def residual(self, b, x, r, level=None):
        lev = self._lev(level)
        _check(self.lib.stgmg_residual(self.h, lev, self._p(b, lev), self._p(x, lev), self._p(r, lev)),
               "stgmg_residual")

    def smooth_sweep(self, b, d, level=None):
        lev = self._lev(level)
        _check(self.lib.stgmg_smooth_sweep(self.h, lev, self._p(b, lev), self._p(d, lev)), "stgmg_smooth_sweep")

    def restrict(self, level, rf, bc):
        lev = self._lev(level)
        if lev < 1:
            raise ValueError("restriction needs level >= 1")
        _check(self.lib.stgmg_restrict(self.h, lev, self._p(rf, lev), self._p(bc, lev - 1)), "stgmg_restrict")

    def prolong_add(self, level, dc, df):
        lev = self._lev(level)
        if lev < 1:
            raise ValueError("prolongation needs level >= 1")
        _check(self.lib.stgmg_prolong_add(self.h, lev, self._p(dc, lev - 1), self._p(df, lev)), "stgmg_prolong_add")

    def vcycle(self, b, x):
        _check(self.lib.stgmg_vcycle(self.h, self._p(b), self._p(x)), "stgmg_vcycle")

    def solve(self, rhs, x, tol=None, tol_mode=TOL_REL, restart=None, maxit=1000):
        st = Stats()
        rc = _check(self.lib.stgmg_solve(self.h, self._p(rhs), self._p(x), float(tol if tol else self.cfg["rtol"]),
                                         tol_mode, int(restart or self.cfg["restart"]), int(maxit), ctypes.byref(st)),
                    "stgmg_solve")
        out = st.as_dict()
        out["converged"] = rc == STGMG_OK
        return out

    def solve_host(self, rhs_host, x_host, tol=None, tol_mode=TOL_REL, restart=None, maxit=1000):
        """rhs_host, x_host: contiguous float64 CPU tensors (pinned for speed) or numpy arrays."""
        st = Stats()
        n = self._n[-1]
        rc = _check(self.lib.stgmg_solve_host(self.h, _host_ptr(rhs_host, n), _host_ptr(x_host, n),
                                              float(tol if tol else self.cfg["rtol"]),
                                              tol_mode, int(restart or self.cfg["restart"]), int(maxit),
                                              ctypes.byref(st)), "stgmg_solve_host")
        out = st.as_dict()
        out["converged"] = rc == STGMG_OK
        return out

    def slab_rhs(self, load, x_prev, rhs):
        lp = self._p(load) if load is not None else None
        _check(self.lib.stgmg_slab_rhs(self.h, lp, self._p(x_prev), self._p(rhs)), "stgmg_slab_rhs")

    def slab_load(self, kind, t_n, load):
        """L_n of the slab (t_n, t_n + tau] assembled on the device (LOAD_MANUFACTURED / LOAD_BEAM_TRACTION)."""
        _check(self.lib.stgmg_slab_load(self.h, int(kind), float(t_n), self._p(load)), "stgmg_slab_load")

    def initial_state(self, kind, t0, x):
        """x = 0 except the last Radau block = interpolated initial data (reading A20)."""
        _check(self.lib.stgmg_initial_state(self.h, int(kind), float(t0), self._p(x)), "stgmg_initial_state")

    def energy(self, x):
        """A_gamma(U,U) + <rho V,V> + <c0 P,P> of the last Radau block of x (host float)."""
        e = ctypes.c_double()
        _check(self.lib.stgmg_energy(self.h, self._p(x), ctypes.byref(e)), "stgmg_energy")
        return e.value

    def goal_quantities(self, x, face):
        """SURVEY N1 / Eq:DefGQ: (b_u, b_p) = (int_face u.n, int_face p) of the last Radau block of x."""
        bu, bp = ctypes.c_double(), ctypes.c_double()
        _check(self.lib.stgmg_goal_quantities(self.h, self._p(x), int(face), ctypes.byref(bu), ctypes.byref(bp)),
               "stgmg_goal_quantities")
        return bu.value, bp.value

    def level_work(self, level=None):
        lev = self.levels - 1 if level is None else level
        f, bb, b1 = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        _check(self.lib.stgmg_level_work(self.h, lev, ctypes.byref(f), ctypes.byref(bb), ctypes.byref(b1)),
               "stgmg_level_work")
        return dict(k2_flops=f.value, k2_bytes=bb.value, k1_bytes=b1.value)

    def time_kernel(self, kind, level=None, reps=20):
        """Average ms of one launch (kind 0 = K2 patch GEMM, 1 = K1 apply, 2 = K3 average, 3 = V-cycle,
        4 / 5 = empty kernel, 6 = one smoothing sweep, 7 = restriction + prolongation, 8 = one MGS pass)."""
        lev = self.levels - 1 if level is None else level
        ms = ctypes.c_double()
        _check(self.lib.stgmg_time_kernel(self.h, kind, lev, reps, ctypes.byref(ms)), "stgmg_time_kernel")
        return ms.value

    def kernel_work(self, kind, level=None):
        """Algorithmic (flops, bytes) of one launch of time_kernel's kind (stgmg_kernel_work)."""
        lev = self.levels - 1 if level is None else level
        f, b = ctypes.c_double(), ctypes.c_double()
        _check(self.lib.stgmg_kernel_work(self.h, int(kind), lev, ctypes.byref(f), ctypes.byref(b)),
               "stgmg_kernel_work")
        return f.value, b.value

    def launch_count(self):
        return int(self.lib.stgmg_last_launch_count(self.h))

    def fold_level(self):
        return int(self.lib.stgmg_fold_level(self.h))


class LShapeSolver(Solver):
    """The 3D L-shaped benchmark of Sec. 5.2 (stgmg_setup_lshape): Q_r^3 / P_{r-1}^disc on the 3-cube
    L-shape with 2^ref_fine cells per cube edge, levels ref_fine - levels + 1 .. ref_fine.  params: dict with rho,
    alpha, c0, lam, mu, K (9 entries), gamma_a, gamma_b (< 0: defaults of P:L209-211)."""

    def __init__(self, ref_fine, levels, r, k, tau, params, stream=None, omega=0.7, jmax=4, hF_mode=HF_MEASURE):
        import torch
        if not torch.cuda.is_available():
            raise StgmgError("no CUDA device: the stgmg product path has no CPU fallback")
        self.lib = load_library()
        self.cfg = dict(rtol=1e-8, restart=30, levels=levels, lshape=True)
        o = Order(int(r), int(k))
        p = Params()
        p.rho, p.alpha, p.c0, p.lambda_, p.mu = params["rho"], params["alpha"], params["c0"], params["lam"], params["mu"]
        for i in range(9):
            p.K[i] = float(params["K"][i])
        p.tau = float(tau)
        p.gamma_a = float(params.get("gamma_a", -1.0))
        p.gamma_b = float(params.get("gamma_b", -1.0))
        p.omega, p.jmax = omega, jmax
        p.hF_mode = int(hF_mode)
        p.nranks, p.rank = 1, 0
        self.stream = stream if stream is not None else torch.cuda.current_stream()
        p.stream = ctypes.c_void_p(self.stream.cuda_stream)
        self.levels = int(levels)
        h = ctypes.c_void_p()
        _check(self.lib.stgmg_setup_lshape(int(ref_fine), self.levels, ctypes.byref(o), ctypes.byref(p),
                                           ctypes.byref(h)), "stgmg_setup_lshape")
        self.h = h
        self.device = self.stream.device
        self._n = []
        for lev in range(self.levels):
            n = ctypes.c_int64()
            _check(self.lib.stgmg_local_size(self.h, lev, ctypes.byref(n)), "stgmg_local_size")
            self._n.append(n.value)
