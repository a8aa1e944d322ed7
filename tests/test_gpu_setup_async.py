"""K4 setup: the class inverses of every level and the coarse inverse run on streams of their own (overlapping each
other and the host-side setup of the next levels, api.cu launch_inverse_async / finish_inverses).  The result must
not depend on that overlap: solves after an asynchronous setup are bitwise identical to solves after the serial
setup (STGMG_SETUP_SERIAL=1, every inverse on the handle's stream); every parity suite runs on the
asynchronous default."""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r"""
import sys, numpy as np, torch
sys.path.insert(0, %(root)r)
sys.path.insert(0, %(root)r + "/tests")
from paper_2303_06742_b200 import Solver
from stgmg_inputs import uniform_load
from gpu_common import small_config
out = []
for i in (3, 4):
    cfg = small_config(i)
    s = Solver(cfg)
    b = torch.as_tensor(uniform_load(s.size(), 7), device="cuda:0")
    x = torch.zeros_like(b)
    st = s.solve(b, x, tol=cfg["rtol"], restart=cfg["restart"])
    assert st["converged"], st
    out.append(x.cpu().numpy())
    s.close()
np.savez(sys.argv[1], *out)
"""


def _run(tmp_path, serial):
    env = dict(os.environ)
    env.pop("STGMG_SETUP_SERIAL", None)
    if serial:
        env["STGMG_SETUP_SERIAL"] = "1"
    f = str(tmp_path / ("serial.npz" if serial else "async.npz"))
    subprocess.run([sys.executable, "-c", WORKER % {"root": ROOT}, f], env=env, check=True, timeout=600)
    z = np.load(f)
    return [z[k] for k in sorted(z.files)]


@pytest.mark.gpu
def test_async_setup_equals_serial_setup(tmp_path):
    a = _run(tmp_path, False)
    s = _run(tmp_path, True)
    assert len(a) == len(s) == 2
    for xa, xs in zip(a, s):
        assert np.array_equal(xa, xs)
