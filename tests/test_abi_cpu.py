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
