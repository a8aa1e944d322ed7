"""CPU-side checks of the boundary: libstgmg.so loads without a GPU and exports every symbol that
include/stgmg.h declares; the binding's signature table covers the header (no compute calls here)."""
import ctypes
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "stgmg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(stgmg_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_boundary_calls():
    names = header_functions()
    for required in ("stgmg_setup", "stgmg_apply_operator", "stgmg_vcycle", "stgmg_solve", "stgmg_destroy"):
        assert required in names


def test_library_exports_every_declared_symbol():
    from paper_2303_06742_b200.build import build, LIB
    build()
    lib = ctypes.CDLL(LIB)
    for name in header_functions():
        assert hasattr(lib, name), name


def test_binding_covers_header():
    from paper_2303_06742_b200.stgmg import SIGNATURES
    assert sorted(SIGNATURES) == header_functions()


def test_product_package_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2303_06742_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle", txt, flags=re.M), f
                assert "oracle/" not in txt, f


def test_solver_requires_gpu_no_fallback():
    import torch
    if torch.cuda.is_available():
        return
    from paper_2303_06742_b200 import Solver, StgmgError
    from stgmg_inputs import config
    try:
        Solver(config(0))
    except StgmgError:
        return
    raise AssertionError("Solver constructed without a GPU")


def _setup_rc(mutate, levels=None):
    """stgmg_setup on a mutated config-0 argument set: (return code, last error).  Argument validation happens
    before any CUDA call, so invalid input is rejected on a machine without a GPU (include/stgmg.h: EINVAL)."""
    from paper_2303_06742_b200.stgmg import load_library, setup_args
    from stgmg_inputs import config
    lib = load_library()
    cfg = config(0)
    m, o, p = setup_args(cfg)
    lv = cfg["levels"] if levels is None else levels
    mutate(m, o, p)
    h = ctypes.c_void_p()
    rc = lib.stgmg_setup(ctypes.byref(m), lv, ctypes.byref(o), ctypes.byref(p), ctypes.byref(h))
    return rc, lib.stgmg_last_error().decode()


def _set(obj, **kw):
    for k, v in kw.items():
        setattr(obj, k, v)


import pytest  # noqa: E402

INVALID = {
    "r<2 (P:L148 Taylor-Hood needs r>=2)": lambda m, o, p: _set(o, r=1),
    "k<0": lambda m, o, p: _set(o, k=-1),
    "cells not divisible by 2^(levels-1)": lambda m, o, p: m.cells.__setitem__(0, 5),
    "rho<=0 (P:L52)": lambda m, o, p: _set(p, rho=0.0),
    "c0<=0 (P:L52)": lambda m, o, p: _set(p, c0=-1.0),
    "tau<=0": lambda m, o, p: _set(p, tau=0.0),
    "K not symmetric (Eq:PosDefK)": lambda m, o, p: p.K.__setitem__(1, 0.5),
    "K not positive definite (Eq:PosDefK)": lambda m, o, p: p.K.__setitem__(4, -1.0),
    "dim 4": lambda m, o, p: _set(m, dim=4),
    "unknown smoother": lambda m, o, p: _set(p, smoother=9),
    "unknown formulation": lambda m, o, p: _set(p, formulation=7),
    "multi-rank without communicator": lambda m, o, p: _set(p, nranks=2, rank=0, nccl_comm=None),
}


@pytest.mark.parametrize("case", sorted(INVALID))
def test_setup_rejects_invalid_arguments(case):
    rc, msg = _setup_rc(INVALID[case])
    assert rc == -1, (case, rc, msg)      # STGMG_EINVAL
    assert msg


def test_setup_rejects_bad_level_count():
    assert _setup_rc(lambda m, o, p: None, levels=0)[0] == -1
    assert _setup_rc(lambda m, o, p: None, levels=17)[0] == -1


def test_partition_plan_even_split_feeds_agglomeration():
    """stgmg_partition_plan (host-only): a split level owns an even number >= 4 of cells per rank, so rank q's fine
    cells coarsen onto exactly the coarse cells [q oc, (q+1) oc) (agglomerate(); 40 cells, 4 levels,
    2 ranks used to split the 10-cell level into 5 + 5 with oc = 2).  Windows tile the global level."""
    from paper_2303_06742_b200.stgmg import partition_plan
    from stgmg_inputs import config
    cfg = config(4)
    cases = [(40, 4, 2), (256, 6, 8), (256, 6, 2), (48, 4, 3), (24, 3, 2), (96, 5, 4)]
    for nx, levels, P in cases:
        cfg = dict(cfg, cells=(nx, 4, 4), levels=levels)
        splits = []
        for lev in range(levels):
            plans = [partition_plan(cfg, lev, q, P) for q in range(P)]
            split = plans[0]["split"]
            assert all(p["split"] == split for p in plans)
            n = nx >> (levels - 1 - lev)
            if split:
                own = [p["c1"] - p["c0"] for p in plans]
                assert own == [n // P] * P and (n // P) % 2 == 0 and n // P >= 4, (nx, levels, P, lev, own)
                assert [p["w0"] + p["c0"] for p in plans] == [q * (n // P) for q in range(P)]
            splits.append(split)
        # split levels form a suffix (fine end) of the hierarchy, never level 0
        assert splits[0] == 0 and splits == sorted(splits)
    cfg = dict(cfg, cells=(40, 4, 4), levels=4)
    assert [partition_plan(cfg, l, 0, 2)["split"] for l in range(4)] == [0, 0, 1, 1]
