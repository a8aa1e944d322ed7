"""Shared helpers of the GPU parity tests: build the CUDA path and the oracle for the same configuration."""
import functools

import numpy as np

from stgmg_inputs import config


def small_config(i):
    """Shrunken versions of the BASELINE configs (same spaces, parameters, BCs; fewer cells / levels) for
    element-by-element parity against the oracle in seconds; several tiles, ragged tails, every patch class."""
    c = config(i)
    if i == 2:
        c.update(cells=(16, 16, 1), levels=3)
    elif i == 3:
        c.update(cells=(8, 8, 8), levels=3)
    elif i == 4:
        c.update(cells=(16, 4, 4), hi=(2.0, 1.0, 1.0), levels=3)
    elif i == 1:
        c.update(cells=(16, 16, 1), levels=4)
    return c


def oracle_params(cfg):
    p = dict(cfg["params"])
    d = cfg["dim"]
    K = np.array(p["K"], dtype=float).reshape(3, 3)[:d, :d]
    p["K"] = K.ravel().tolist()
    return p


@functools.lru_cache(maxsize=8)
def oracle_hierarchy(key):
    from oracle.mg import Hierarchy
    cfg = _cfg_from_key(key)
    d = cfg["dim"]
    return Hierarchy(d, cfg["cells"][:d], cfg["lo"][:d], cfg["hi"][:d], cfg["r"], cfg["k"], cfg["levels"],
                     oracle_params(cfg), cfg["tau"], bc_u=list(cfg["bc_u"][:2 * d]), bc_p=list(cfg["bc_p"][:2 * d]))


_CFGS = {}


def cfg_key(cfg):
    key = repr(sorted((k, repr(v)) for k, v in cfg.items()))
    _CFGS[key] = cfg
    return key


def _cfg_from_key(key):
    return _CFGS[key]


def to_gpu(x):
    import torch
    return torch.as_tensor(np.ascontiguousarray(x), dtype=torch.float64, device="cuda")


def to_np(t):
    return t.detach().cpu().numpy()
