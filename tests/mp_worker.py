"""Worker of tests/test_gpu_multiproc.py: ONE rank of the x-slab decomposition in its own process (as under torchrun),
talking to the other ranks through the library's shared-memory transport (stgmg_shm_comm_create).  Writes the rank's
owned solution entries, its iteration count and its V-cycle to an .npz file.  Not a test module (no test_ prefix)."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--rank", type=int)
    ap.add_argument("--nranks", type=int)
    ap.add_argument("--name")
    ap.add_argument("--cfg", type=int)
    ap.add_argument("--out")
    a = ap.parse_args()
    import numpy as np
    import torch
    from stgmg_inputs import uniform_load
    from tests.gpu_common import small_config
    from paper_2303_06742_b200.stgmg import (Solver, partition_plan, shm_comm_create, shm_comm_destroy, COMM_SHM,
                                             load_library)
    from paper_2303_06742_b200.partition import window_index
    load_library()
    cfg = small_config(a.cfg)
    if a.cfg == 4:
        cfg = dict(cfg, cells=(32, 4, 4), hi=(4.0, 1.0, 1.0))
    fine = cfg["levels"] - 1
    idx, own = window_index(cfg, fine, partition_plan(cfg, fine, a.rank, a.nranks))
    comm = shm_comm_create(a.name, a.nranks, a.rank)
    s = Solver(cfg, rank=a.rank, nranks=a.nranks, comm=comm, comm_kind=COMM_SHM)
    Ng = int(idx.max()) + 1
    # the global vector length: every rank reads the same global draw
    from stgmg_inputs import dof_count
    b = uniform_load(dof_count(cfg), 304)
    x = torch.zeros(len(idx), dtype=torch.float64, device="cuda")
    st = s.solve(torch.as_tensor(b[idx], device="cuda"), x, tol=cfg["rtol"], restart=cfg["restart"])
    v = torch.zeros_like(x)
    s.vcycle(torch.as_tensor(b[idx], device="cuda"), v)
    torch.cuda.synchronize()
    np.savez(a.out, idx=idx[own], x=x.cpu().numpy()[own], v=v.cpu().numpy()[own], its=st["iterations"],
             conv=st["converged"], n=Ng)
    s.close()
    shm_comm_destroy(comm)


if __name__ == "__main__":
    main()
