"""The folded coarse sub-cycle (csrc/api.cu build_fold): below the fold level the V-cycle of Alg. 1 sweeps,
transfers and the coarse solve is a fixed linear map b_f -> d_f, assembled at setup by running it on every unit
vector and applied as one GEMV.  Checks (-m gpu): the folded and the unfolded (STGMG_FOLD_MB=0) V-cycles agree to
rounding (1e-12) on the bench configuration and two shrunken ones, and so do the FGMRES solves (same iteration
count, 1e-10).  The oracle parity of the folded V-cycle itself is in test_gpu_parity.py / test_gpu_bench_config.py."""
import os

import numpy as np
import pytest

from stgmg_inputs import config, uniform_load, random_vector
from tests.gpu_common import small_config

pytestmark = pytest.mark.gpu


def make(cfg, fold_mb=None):
    from paper_2303_06742_b200 import Solver
    saved = os.environ.get("STGMG_FOLD_MB")
    if fold_mb is not None:
        os.environ["STGMG_FOLD_MB"] = str(fold_mb)
    try:
        return Solver(cfg)
    finally:
        if saved is None:
            os.environ.pop("STGMG_FOLD_MB", None)
        else:
            os.environ["STGMG_FOLD_MB"] = saved


@pytest.mark.parametrize("which", ["cfg1", "cfg1s", "cfg2s"])
def test_folded_vcycle_equals_unfolded(which):
    import torch
    cfg = config(1) if which == "cfg1" else small_config(int(which[3]))
    a, b = make(cfg), make(cfg, 0)
    N = a.size()
    for seed in (1, 2):
        rhs = torch.as_tensor(uniform_load(N, seed) if seed == 1 else random_vector(N, 77), device="cuda")
        xa, xb = torch.zeros_like(rhs), torch.zeros_like(rhs)
        a.vcycle(rhs, xa)
        b.vcycle(rhs, xb)
        torch.cuda.synchronize()
        d = (xa - xb).norm().item() / xb.norm().item()
        assert d < 1e-12, d
    sa = a.solve(rhs, xa.zero_(), tol=cfg["rtol"], restart=cfg["restart"])
    sb = b.solve(rhs, xb.zero_(), tol=cfg["rtol"], restart=cfg["restart"])
    assert sa["iterations"] == sb["iterations"]
    assert (xa - xb).norm().item() <= 1e-10 * xb.norm().item()
    a.close()
    b.close()
