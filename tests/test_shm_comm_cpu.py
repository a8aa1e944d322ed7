"""Host-side bootstrap of the process-separated shared-memory communicator (stgmg_shm_comm_create, CPU only): N
processes attach to one named segment (rank 0 creates it, the others wait for it), pass the attach barrier, and
tear it down collectively; mismatched rank counts are rejected; the segment name is unlinked afterwards."""
import os
import subprocess
import sys
import uuid

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r"""
import sys
sys.path.insert(0, %r)
from paper_2303_06742_b200.stgmg import shm_comm_create, shm_comm_destroy, StgmgError
name, P, q = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
c = shm_comm_create(name, P, q, cap_doubles=1024)
shm_comm_destroy(c)
print("ok", q)
"""


def _run(name, P):
    code = WORKER % ROOT
    ps = [subprocess.Popen([sys.executable, "-c", code, name, str(P), str(q)], stdout=subprocess.PIPE,
                           stderr=subprocess.STDOUT) for q in range(P)]
    return [(p.wait(timeout=120), p.stdout.read().decode()) for p in ps]


def test_shm_comm_bootstrap_and_teardown():
    from paper_2303_06742_b200.build import build
    build()
    for P in (2, 3):
        name = "stgmg_cpu_" + uuid.uuid4().hex[:10]
        res = _run(name, P)
        assert all(rc == 0 for rc, _ in res), res
        assert not os.path.exists("/dev/shm/" + name)


def test_shm_comm_rejects_bad_arguments():
    import pytest
    from paper_2303_06742_b200.stgmg import shm_comm_create, StgmgError
    with pytest.raises(StgmgError):
        shm_comm_create("x", 2, 5)
    with pytest.raises(StgmgError):
        shm_comm_create("x", 0, 0)
