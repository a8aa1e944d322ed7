"""Host side of the N > 1 path (bench.py under torchrun) on CPU with the gloo backend, world size 2:
the x-slab partition plan and window maps of every rank cover each global DoF exactly once (owned) and every ghost
DoF is owned by a neighbour; the 128-byte NCCL id bootstrap broadcast and the max-over-ranks timing reduction that
bench.py performs.  No GPU: the partition plan is a host function of libstgmg.so."""
import os
import socket

import numpy as np
import pytest

from stgmg_inputs import config, dof_count

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, port, cfg_ids, out_dir):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=WORLD)
    from paper_2303_06742_b200.stgmg import partition_plan
    from paper_2303_06742_b200.partition import window_index
    res = {}
    for ci in cfg_ids:
        cfg = config(ci)
        for level in range(cfg["levels"]):
            plan = partition_plan(cfg, level, rank, WORLD)
            idx, own = window_index(cfg, level, plan)
            res[(ci, level)] = (plan, idx, own)
    # NCCL-id bootstrap exactly as bench.py does it (here over gloo, CPU tensor)
    uid = torch.tensor(list(range(128)) if rank == 0 else [0] * 128, dtype=torch.uint8)
    dist.broadcast(uid, 0)
    # max-over-ranks timing
    t = torch.tensor([1.0 + rank], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    np.save(os.path.join(out_dir, "r%d.npy" % rank),
            np.array([res, bytes(uid.tolist()), float(t.item())], dtype=object), allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()


@pytest.fixture(scope="module")
def gloo_results(tmp_path_factory):
    import torch.multiprocessing as mp
    out = tmp_path_factory.mktemp("gloo")
    port = _free_port()
    mp.start_processes(_worker, args=(port, (1, 2, 4), str(out)), nprocs=WORLD, join=True, start_method="spawn")
    return [np.load(os.path.join(out, "r%d.npy" % q), allow_pickle=True) for q in range(WORLD)]


@pytest.mark.parametrize("ci", [1, 2, 4])
def test_owned_dofs_partition_global_vector(gloo_results, ci):
    cfg = config(ci)
    for level in range(cfg["levels"]):
        N = dof_count(cfg, cfg["levels"] - 1 - level)
        plans = [gloo_results[q][0][(ci, level)][0] for q in range(WORLD)]
        if not plans[0]["split"]:
            # replicated (agglomerated) level: every rank holds the whole vector
            for q in range(WORLD):
                idx, own = gloo_results[q][0][(ci, level)][1:]
                assert len(idx) == N and own.all()
            continue
        count = np.zeros(N, dtype=int)
        for q in range(WORLD):
            idx, own = gloo_results[q][0][(ci, level)][1:]
            assert len(np.unique(idx)) == len(idx)
            count[idx[own]] += 1
        assert (count == 1).all(), (ci, level)
        # every ghost DoF of a rank is owned by another rank
        owned = [set(gloo_results[q][0][(ci, level)][1][gloo_results[q][0][(ci, level)][2]].tolist())
                 for q in range(WORLD)]
        for q in range(WORLD):
            idx, own = gloo_results[q][0][(ci, level)][1:]
            ghosts = set(idx[~own].tolist())
            assert ghosts <= set().union(*[owned[p] for p in range(WORLD) if p != q])


def test_bootstrap_broadcast_and_max_timing(gloo_results):
    for q in range(WORLD):
        assert gloo_results[q][1] == bytes(range(128))
        assert gloo_results[q][2] == float(WORLD)
