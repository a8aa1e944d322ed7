"""The axis-by-axis restriction (nodal.cu restrict_pass_kernel, levels with >= 200k DoFs) against the per-coarse-node
gather form (STGMG_RESTRICT_SEP=0) on the full cfg3 and cfg2 fine levels (-m gpu): b_c = P^T r_f in both;
only the summation order differs (1e-14 relative).  The V-cycle parity at full size (test_gpu_fullsize*.py) covers it
against the oracle."""
import os

import numpy as np
import pytest

from stgmg_inputs import config, random_vector
from tests.gpu_common import to_gpu, to_np

pytestmark = pytest.mark.gpu


def _solver(cfg, sep):
    from paper_2303_06742_b200 import Solver
    old = os.environ.get("STGMG_RESTRICT_SEP")
    os.environ["STGMG_RESTRICT_SEP"] = "1" if sep else "0"
    try:
        return Solver(cfg)
    finally:
        if old is None:
            del os.environ["STGMG_RESTRICT_SEP"]
        else:
            os.environ["STGMG_RESTRICT_SEP"] = old


@pytest.mark.parametrize("ci", [3, 2])
def test_separable_restriction_equals_gather_form(ci):
    import torch
    cfg = config(ci)
    a, b = _solver(cfg, True), _solver(cfg, False)
    L = cfg["levels"] - 1
    rf = to_gpu(random_vector(a.size(L), 77))
    ya = torch.zeros(a.size(L - 1), dtype=torch.float64, device="cuda")
    yb = torch.zeros_like(ya)
    a.restrict(L, rf, ya)
    b.restrict(L, rf, yb)
    torch.cuda.synchronize()
    u, v = to_np(ya), to_np(yb)
    assert np.linalg.norm(u - v) <= 1e-14 * np.linalg.norm(v)
    a.close()
    b.close()
