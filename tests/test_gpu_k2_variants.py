"""GPU parity of every K2 tile variant forced onto every smoothed level (STGMG_K2_VARIANT_L<l>, read at setup):
K2S shared-B (9), K2L latency 32x8 / 32x16 / 32x32 (4 / 7 / 8), pipelined small / medium / big / wide (0 / 1 / 2 / 6),
against the oracle's Alg. 1 sweep and V-cycle (-m gpu).  The variants differ only in tiling and summation grouping,
so the north-star tolerances of test_gpu_parity.py apply.  3D (cfg3s) runs the variants whose tiles fit its C_P."""
import os

import numpy as np
import pytest

from stgmg_inputs import uniform_load, random_vector
from tests.gpu_common import small_config, oracle_hierarchy, cfg_key, to_gpu, to_np

pytestmark = pytest.mark.gpu

CASES = [(c, v) for c in (1,) for v in (9, 4, 7, 8, 0, 1, 2, 6)] + [(3, v) for v in (4, 0, 2)]


@pytest.fixture(scope="module", params=CASES, ids=["cfg%ds_v%d" % c for c in CASES])
def pair(request):
    import torch
    from paper_2303_06742_b200 import Solver
    ci, var = request.param
    cfg = small_config(ci)
    keys = ["STGMG_K2_VARIANT_L%d" % l for l in range(1, cfg["levels"])] + ["STGMG_K2_DENSE"]
    saved = {k: os.environ.get(k) for k in keys}
    for k in keys[:-1]:
        os.environ[k] = str(var)
    os.environ["STGMG_K2_DENSE"] = "0"
    try:
        s = Solver(cfg)
    finally:
        for k, v in saved.items():
            if v is None:
                del os.environ[k]
            else:
                os.environ[k] = v
    H = oracle_hierarchy(cfg_key(cfg))
    yield cfg, s, H
    s.close()
    torch.cuda.synchronize()


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def test_sweep_every_level(pair):
    import torch
    cfg, s, H = pair
    for l in range(1, len(H.levels)):
        N = H.levels[l].N
        b, d0 = random_vector(N, 610 + l), random_vector(N, 620 + l, 1e-3)
        d = to_gpu(d0)
        s.smooth_sweep(to_gpu(b), d, level=l)
        torch.cuda.synchronize()
        assert rel(to_np(d), H.smoothers[l].sweep(b, d0)) < 1e-9, l


def test_vcycle(pair):
    import torch
    cfg, s, H = pair
    b = uniform_load(H.fine.N, 5)
    x = torch.zeros(H.fine.N, dtype=torch.float64, device="cuda")
    s.vcycle(to_gpu(b), x)
    torch.cuda.synchronize()
    assert rel(to_np(x), H.vcycle(b)) < 1e-8
