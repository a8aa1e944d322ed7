"""Host-side index bookkeeping of the x-slab domain decomposition: map a global level vector to a
rank's window vector (owned cells + ghost cells, stgmg_partition_plan) and back.  Used by bench.py (N > 1) to hand
every rank its slice of the global load and by the multi-rank tests; no arithmetic of the method."""
import numpy as np


def level_shape(cfg, level):
    d = cfg["dim"]
    return [cfg["cells"][a] >> (cfg["levels"] - 1 - level) for a in range(d)]


def window_index(cfg, level, plan):
    """(local -> global index array, owned mask over local DoFs) for one rank's window of a level."""
    d, r, k = cfg["dim"], cfg["r"], cfg["k"]
    n = level_shape(cfg, level)
    w0, nxw, c0, c1 = plan["w0"], plan["nx_window"], plan["c0"], plan["c1"]
    last = plan["w0"] + plan["nx_window"] == plan["gnx"]
    nl = [nxw] + n[1:]

    def nodes(deg, cells):
        return [deg * c + 1 for c in cells]

    gq, gp = nodes(r, n), nodes(r - 1, n)
    lq, lp = nodes(r, nl), nodes(r - 1, nl)
    nq_g, np_g, nq_l, np_l = int(np.prod(gq)), int(np.prod(gp)), int(np.prod(lq)), int(np.prod(lp))
    Rg, Rl = d * nq_g, d * nq_l
    bg, bl = 2 * Rg + np_g, 2 * Rl + np_l

    def field(deg, gshape, lshape):
        # global node index of every local node (lexicographic, x fastest)
        axes = [np.arange(lshape[0]) + w0 * deg] + [np.arange(s) for s in lshape[1:]]
        grids = np.meshgrid(*axes, indexing="ij")
        strides = np.cumprod([1] + list(gshape[:-1]))
        gidx = sum(g * s for g, s in zip(grids, strides)).ravel(order="F")
        xl = np.meshgrid(*[np.arange(s) for s in lshape], indexing="ij")[0].ravel(order="F")
        own = (xl >= c0 * deg) & ((xl < c1 * deg) | (last & (xl == c1 * deg)))
        return gidx, own

    gq_idx, q_own = field(r, gq, lq)
    gp_idx, p_own = field(r - 1, gp, lp)
    idx, own = [], []
    for m in range(k + 1):
        for slot in range(2 * d):
            idx.append(m * bg + slot * nq_g + gq_idx)
            own.append(q_own)
        idx.append(m * bg + 2 * Rg + gp_idx)
        own.append(p_own)
    idx, own = np.concatenate(idx), np.concatenate(own)
    assert len(idx) == (k + 1) * bl
    return idx, own


def scatter_owned(global_vec, local_vec, idx, own):
    global_vec[idx[own]] = local_vec[own]


def gather_owned(local_vecs, maps, n_global):
    """Assemble a global vector from every rank's window vector (owned DoFs only)."""
    out = np.zeros(n_global)
    for v, (idx, own) in zip(local_vecs, maps):
        scatter_owned(out, v, idx, own)
    return out
