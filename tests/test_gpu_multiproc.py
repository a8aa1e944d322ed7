"""Multi-PROCESS parity of the x-slab decomposition on one GPU (-m gpu): every rank is its own
process with its own CUDA context, handle and stream — the bootstrap and per-rank state of a torchrun launch — and the
ranks exchange halos, reductions and the coarse agglomeration through the library's process-separated shared-memory
transport (stgmg_shm_comm_create; host-staged, no kernel waits on another rank).  The solution and the V-cycle must
match the 1-GPU solve (1e-10 / 1e-12) with the same iteration count (+-1)."""
import os
import subprocess
import sys
import uuid

import numpy as np
import pytest

from stgmg_inputs import uniform_load, dof_count
from tests.gpu_common import small_config, to_gpu, to_np

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("ci,P", [(3, 2), (4, 2), (4, 4)])
def test_multiprocess_solve_matches_single_gpu(tmp_path, ci, P):
    import torch
    from paper_2303_06742_b200 import Solver
    name = "stgmg_test_" + uuid.uuid4().hex[:12]
    outs = [str(tmp_path / ("r%d.npz" % q)) for q in range(P)]
    procs = [subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "mp_worker.py"), "--rank", str(q),
                               "--nranks", str(P), "--name", name, "--cfg", str(ci), "--out", outs[q]],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT) for q in range(P)]
    logs = [p.communicate(timeout=600)[0].decode() for p in procs]
    for p, log in zip(procs, logs):
        assert p.returncode == 0, log[-3000:]
    cfg = small_config(ci)
    if ci == 4:
        cfg = dict(cfg, cells=(32, 4, 4), hi=(4.0, 1.0, 1.0))
    N = dof_count(cfg)
    s = Solver(cfg)
    b = uniform_load(N, 304)
    xref = torch.zeros(N, dtype=torch.float64, device="cuda")
    st = s.solve(to_gpu(b), xref, tol=cfg["rtol"], restart=cfg["restart"])
    vref = torch.zeros_like(xref)
    s.vcycle(to_gpu(b), vref)
    torch.cuda.synchronize()
    x, v = np.zeros(N), np.zeros(N)
    covered = np.zeros(N, dtype=bool)
    its = set()
    for o in outs:
        z = np.load(o)
        x[z["idx"]] = z["x"]
        v[z["idx"]] = z["v"]
        covered[z["idx"]] = True
        its.add(int(z["its"]))
        assert bool(z["conv"])
    assert covered.all()
    assert len(its) == 1 and abs(its.pop() - st["iterations"]) <= 1
    xr, vr = to_np(xref), to_np(vref)
    assert np.linalg.norm(x - xr) <= 1e-10 * np.linalg.norm(xr)
    assert np.abs(v - vr).max() <= 1e-12 * np.abs(vr).max()
    s.close()
