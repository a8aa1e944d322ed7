#!/usr/bin/env python
"""Benchmark of the hot path: one space-time slab solve (FGMRES(m) + GMG V-cycle with patch Vanka) per step.

Workload (default): BASELINE.json configs[4] — the largest single-GPU configuration and the one the north star
asks to scale: 3D clamped beam [0,8]x[0,1]^2, 256x32x32 cells, 6 levels, Q2^3/Q2^3/Q1, dG(1) (26,568,846 DoFs),
tau = 0.01, GMRES(30) (reading of SURVEY §8(d)), rel tol 1e-8; u = 0 at x = 0, traction (0,0,-sin(pi t/2)) on
x = 8 (reading A23), p = 0 on z = 1 (A25); zero initial state.  Each step is one slab of the march
t_n = n tau: the load L_n is assembled on the device (stgmg_slab_load), F_n = L_n + J X_{n-1} (stgmg_slab_rhs, K8),
then the slab is solved.  --config c selects another BASELINE config (0-3: manufactured / random loads as
BASELINE states them).
Metric: MDoF*iter/s = N_slab * GMRES iterations / solve time / 1e6; ms_per_step = s/slab.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]

--impl reference runs the oracle (plain fp64 CPU implementation, oracle/) as it stands on the host cores, on a
bounded sample of the same workload (see cpu_sample()).
N > 1 (torchrun, one rank per GPU): the x-slab domain decomposition of SURVEY §8(e) — every rank owns a slab of
cells of the SAME global slab problem (window vectors, halo exchange over NCCL after every smoothing sweep, GMRES
inner products allreduced), so the scaling is "strong"; value = global DoFs x iterations / max-over-ranks time.
A decomposition that cannot be set up is an error (non-zero exit).  --replicas instead runs N independent copies
of the workload ("weak" scaling, no data-path collective).
"""
import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from stgmg_inputs import config, uniform_load, dof_count  # noqa: E402

def _hbm_peak():
    """MEASURED_PEAKS.json hbm_gbs (driver-written copy bandwidth of this pool's B200s: read + write bytes of a 1:1
    copy); the round-1 value of that file if it is absent."""
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except Exception:
        return 6470.8


HBM_PEAK_GBS = _hbm_peak()

FP64_PEAK_TFLOPS = 37.19   # measured DMMA m8n8k4 peak on this pool's B200 (profiles/fp64_peak_r01.json)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--replicas", action="store_true", help="N > 1: independent replicas instead of the decomposition")
    ap.add_argument("--transport", default="nccl", choices=["nccl", "shm"],
                    help="N > 1: the library's NCCL transport (default) or its process-separated shared-memory "
                         "transport with a gloo process group (exercises the N-rank flow on one GPU; ranks then share "
                         "the device and the numbers are not a scaling measurement)")
    ap.add_argument("--smoother", default="additive", choices=["additive", "colored", "element", "overwrite"],
                    help="additive = Alg. 1 (paper, default); colored = multiplicative colour-ordered Vanka (N2(i)); "
                         "element = element-wise Vanka (N2(ii)); overwrite = Alg. 1 without averaging (N2(iii))")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    lrank = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, lrank


def load_label(cfg):
    if cfg["load"] == "beam":
        return "beam traction (0,0,-sin(pi t/2)) on x=%g (reading A23), zero initial state" % cfg["hi"][0]
    if cfg["load"] == "manufactured":
        return "manufactured solution loads (BASELINE), interpolated initial data (A20)"
    return "uniform[-1,1) seed %s (reading A21), zero initial state" % cfg["seed"]


def workload_config(cfg, args, ws, dd):
    """The config object of the JSON line; identical for both arms (--impl ours / reference)."""
    d = cfg["dim"]
    return {"workload": cfg["name"], "dofs": dof_count(cfg), "dim": d, "cells": list(cfg["cells"][:d]),
            "levels": cfg["levels"], "r": cfg["r"], "k": cfg["k"], "tau": cfg["tau"], "restart": cfg["restart"],
            "rtol": cfg["rtol"], "load": load_label(cfg), "smoother": args.smoother,
            "march": "slab n of step i: t_n = (warmup + i) tau, F_n = L_n + J X_{n-1}",
            "l2": "flushed between timed steps (256 MB write, untimed); inputs > L2 (212 MB per vector at cfg4)",
            "parallelism": ("x-slab decomposition over %d ranks (%s halo exchange)"
                            % (ws, "NCCL" if getattr(args, "transport", "nccl") == "nccl"
                               else "host shared-memory, ranks may share a GPU")) if dd else
                           ("%d replicas" % ws if ws > 1 else "single GPU")}


# ---------------------------------------------------------------------------------------------- clocks -----
class ClockSampler:
    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, gpu_index):
        self.proc = None
        self.path = os.path.join("/tmp", "stgmg_clocks_%d_%d.csv" % (os.getpid(), gpu_index))
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(gpu_index), "--query-gpu=" + ",".join(self.FIELDS),
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, v in zip(["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"], parts[2:]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def nvml_energy_mj(index):
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(index)
        return float(pynvml.nvmlDeviceGetTotalEnergyConsumption(h))
    except Exception:
        return None


def host_info():
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "model": model}


# ---------------------------------------------------------------------------------------------- oracle -----
def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads", 1) for i in threadpool_info()]
        return max(n) if n else 1
    except Exception:
        return os.cpu_count() or 1


def limit_blas():
    """OpenBLAS on every logical CPU of a shared host is pathologically slow for the oracle's LAPACK calls (DESIGN.md
    §3: a 1000^2 inverse 0.09 s on 4 threads, 1.4 s on 8 in the dev container); use half the CPUs, like the tests."""
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits(max(1, (os.cpu_count() or 2) // 2))
    except Exception:
        return None


def oracle_fine_setup(cfg):
    """The oracle as it stands (oracle/ebe.py: element-by-element operator, class-batched patch solves, no global
    matrix) on the bench workload: hierarchy, fine-level smoother (class inverses), slab-1 right-hand side.  Also the
    extrapolation factor S = (K2 flops of one GMRES iteration's V-cycle) / (K2 flops of one fine-level sweep)."""
    from oracle.ebe import EbeHierarchy, ebe_slab_rhs, vcycle_k2_flops, level_k2_flops
    t0 = time.perf_counter()
    H = EbeHierarchy.from_config(cfg)
    L = len(H.levels) - 1
    sm = H.smoother(L)
    b = ebe_slab_rhs(H, cfg, 0)
    S = vcycle_k2_flops(H) / level_k2_flops(H.fine, H.params, H.tau)
    return H, sm, b, S, time.perf_counter() - t0


def cpu_baseline(cfg):
    """Bounded sample: ONE full fine-level Alg. 1 sweep of the oracle (residual element by element, every patch solve,
    averaging) on slab 1 of the workload.  A GMRES iteration = one V-cycle (+ one apply + MGS); its time is
    extrapolated as t_sweep x S (S = V-cycle K2 flops / fine-sweep K2 flops; the patch solves are 95-99 % of the
    flops), and MDoF*iter/s = N / t_iteration."""
    _lim = limit_blas()
    try:
        H, sm, b, S, t_setup = oracle_fine_setup(cfg)
        d = sm.sweep(b, None)                  # first sweep (r = b), as in Alg. 1 from d = 0
        t0 = time.perf_counter()
        sm.sweep(b, d)                         # a later sweep: residual + patch solves + averaging
        dt = time.perf_counter() - t0
    except MemoryError as e:
        return {"value": None, "unit": "MDoF*iter/s", "cores": blas_threads(), "kind": "oracle",
                "sample": "not run: %s" % e}
    N = H.fine.N
    cores = blas_threads()
    single = None
    try:   # the same oracle on ONE thread: one of 8 x-slabs of the patches, scaled to a full sweep
        from threadpoolctl import threadpool_limits
        nx = H.fine.n[0]
        nslab = 8 if nx >= 16 else 1
        with threadpool_limits(1):
            t1 = time.perf_counter()
            sm.partial_sweep(b, d, 0, nx // nslab)
            dt1 = (time.perf_counter() - t1) * nslab
        single = {"value": N / (dt1 * S) / 1e6, "cores": 1,
                  "sample": "fine-level sweep restricted to the first of %d x-slabs of patches, x %d: %.2f s per "
                            "sweep" % (nslab, nslab, dt1)}
    except Exception as e:   # threadpoolctl missing: report the all-core number only
        single = {"value": None, "cores": 1, "sample": "not run: %s" % e}
    return {"value": N / (dt * S) / 1e6, "unit": "MDoF*iter/s", "cores": cores, "kind": "oracle",
            "sample": "one fine-level Alg. 1 sweep of slab 1 of %s (residual, all patch solves, averaging): %.2f s on "
                      "%d BLAS threads; GMRES iteration extrapolated as %.2f sweeps (V-cycle K2 flops / fine-sweep K2 "
                      "flops); oracle setup %.1f s excluded" % (cfg["name"], dt, cores, S, t_setup),
            "single_thread": single, "host": host_info()}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    cfg = config(args.config)
    _lim = limit_blas()
    H, sm, b, S, t_setup = oracle_fine_setup(cfg)
    N = H.fine.N
    nx = H.fine.n[0]
    nslab = 8 if nx >= 16 else 1
    edges = [nx * i // nslab for i in range(nslab)] + [nx + 1]
    d = sm.sweep(b, None)
    # one reference step = the fine-level sweep of one eighth of the patches (vertex x-index slab, rotating), its
    # residual cells and local solves: nslab consecutive steps are one full sweep
    state = {"i": 0}

    def step():
        k = state["i"] % nslab
        sm.partial_sweep(b, d, edges[k], edges[k + 1])
        state["i"] += 1

    for _ in range(min(args.warmup, 1)):        # the CPU needs no warm-up beyond the first call
        step()
    state["i"] = 0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    dt = time.perf_counter() - t0
    t_sweep = dt / args.steps * nslab
    val = N / (t_sweep * S) / 1e6
    cores = blas_threads()
    sample = ("%d steps, each the fine-level Alg. 1 sweep restricted to one of %d x-slabs of patches of slab 1 of %s "
              "(rotating; %d steps = one sweep): sweep %.2f s; GMRES iteration extrapolated as %.2f sweeps (V-cycle "
              "K2 flops / fine-sweep K2 flops); oracle as it stands (oracle/ebe.py) on the host cores; setup %.1f s "
              "excluded" % (args.steps, nslab, cfg["name"], nslab, t_sweep, S, t_setup))
    out = {"impl": "reference", "metric": "slab_solve_throughput", "value": val, "unit": "MDoF*iter/s",
           "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": workload_config(cfg, args, 1, False),
           "cpu_baseline": {"value": val, "unit": "MDoF*iter/s", "cores": cores, "kind": "oracle", "sample": sample,
                            "host": host_info()},
           "e2e": {"value": val, "unit": "MDoF*iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ---------------------------------------------------------------------------------------------- ours -------
def run_ours(args):
    import torch
    ws, rank, lrank = dist_env()
    dd = ws > 1 and not args.replicas
    shm = ws > 1 and args.transport == "shm"
    gpu = (lrank % max(1, torch.cuda.device_count())) if shm else lrank
    if ws > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")   # lets the driver count the communicator's ranks
        torch.cuda.set_device(gpu)
        import torch.distributed as dist
        if shm:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", gpu))
    dev = torch.device("cuda", gpu if ws > 1 else 0)
    red_dev = "cpu" if shm else dev   # gloo reduces host tensors
    from paper_2303_06742_b200 import Solver
    from paper_2303_06742_b200.stgmg import (nccl_unique_id, nccl_comm_create, nccl_comm_destroy, partition_plan,
                                             shm_comm_create, shm_comm_destroy, COMM_NCCL, COMM_SHM,
                                             LOAD_MANUFACTURED, LOAD_BEAM_TRACTION)
    from paper_2303_06742_b200.partition import window_index
    cfg = config(args.config)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    smoother = {"additive": 0, "colored": 1, "element": 2, "overwrite": 3}[args.smoother]
    comm = None
    t_setup = time.perf_counter()
    if dd:
        # the library's own NCCL communicator: rank 0 draws the id, torch.distributed broadcasts it (stgmg.h).
        # Any failure here raises: a decomposition that cannot be set up ends the run with a non-zero exit.
        if shm:   # segment name drawn by rank 0, broadcast over the gloo group
            import uuid
            name = list(("stgmg_bench_" + uuid.uuid4().hex[:16]).encode()) if rank == 0 else [0] * 28
            nt = torch.tensor(name, dtype=torch.uint8)
            torch.distributed.broadcast(nt, 0)
            comm = shm_comm_create(bytes(nt.tolist()).decode(), ws, rank)
        else:
            uid = torch.tensor(list(nccl_unique_id()) if rank == 0 else [0] * 128, dtype=torch.uint8, device=dev)
            torch.distributed.broadcast(uid, 0)
            comm = nccl_comm_create(bytes(uid.cpu().tolist()), ws, rank)
        s = Solver(cfg, stream=stream, rank=rank, nranks=ws, comm=comm, smoother=smoother,
                   comm_kind=COMM_SHM if shm else COMM_NCCL)
    else:
        s = Solver(cfg, stream=stream, smoother=smoother)
    t_setup = time.perf_counter() - t_setup
    N = s.size()                       # this rank's (window) vector length
    Nglob = dof_count(cfg)             # DoFs of the global slab problem
    load_kind = {"manufactured": LOAD_MANUFACTURED, "beam": LOAD_BEAM_TRACTION}.get(cfg["load"])
    if load_kind is None:
        Lg = uniform_load(Nglob, cfg["seed"] or 1)
        if dd:
            idx, _own = window_index(cfg, cfg["levels"] - 1, partition_plan(cfg, cfg["levels"] - 1, rank, ws))
            Lg = Lg[idx]
        L = torch.as_tensor(Lg, device=dev)
    else:
        L = torch.zeros(N, dtype=torch.float64, device=dev)
    X = [torch.zeros(N, dtype=torch.float64, device=dev), torch.zeros(N, dtype=torch.float64, device=dev)]
    if load_kind == LOAD_MANUFACTURED:
        s.initial_state(LOAD_MANUFACTURED, 0.0, X[0])
    rhs = torch.zeros(N, dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)   # > 126 MB L2
    state = {"n": 0}

    def step():
        """One slab of the march: L_n (device), F_n = L_n + J X_{n-1} (K8), solve; returns (stats, launches)."""
        t_n = state["n"] * cfg["tau"]
        nl = 0
        if load_kind is not None:
            s.slab_load(load_kind, t_n, L)
            nl += s.launch_count()
        s.slab_rhs(L, X[0], rhs)
        nl += s.launch_count()
        X[1].zero_()
        st = s.solve(rhs, X[1], tol=cfg["rtol"], restart=cfg["restart"])
        nl += s.launch_count()
        X[0], X[1] = X[1], X[0]
        state["n"] += 1
        return st, nl

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    clocks = ClockSampler(dev.index)
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    its, launches, resid, its_list = 0, 0, [], []
    for i in range(args.steps):
        flush.fill_(float(i))                      # L2 flush between timed steps (untimed)
        ev0[i].record(stream)
        st, nl = step()
        ev1[i].record(stream)
        its += st["iterations"]
        its_list.append(st["iterations"])
        resid.append(st["rel_residual"])
        launches += nl
    torch.cuda.synchronize()
    per_step_ms = [a.elapsed_time(b) for a, b in zip(ev0, ev1)]
    ms = sum(per_step_ms)
    # energy window: NVML's counter updates coarsely, so measure over >= 1.5 s and >= 2 back-to-back slab solves
    # (same step, no flushes); the clock sampler keeps running through it
    e_start = nvml_energy_mj(dev.index)
    t_e0 = time.perf_counter()
    n_e = 0
    while True:
        step()
        n_e += 1
        if n_e >= 2 and time.perf_counter() - t_e0 > 1.5:
            torch.cuda.synchronize()
            if time.perf_counter() - t_e0 > 1.5:
                break
    torch.cuda.synchronize()
    t_e = time.perf_counter() - t_e0
    e_end = nvml_energy_mj(dev.index)
    clk = clocks.stop()
    t_local = torch.tensor([ms], dtype=torch.float64, device=red_dev)
    its_t = torch.tensor([float(its)], dtype=torch.float64, device=red_dev)
    energy_j = (e_end - e_start) * 1e-3 if (e_start is not None and e_end is not None) else None
    if ws > 1:
        import torch.distributed as dist
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
        if not dd:                     # replicas: every rank solved its own copy
            dist.all_reduce(its_t, op=dist.ReduceOp.SUM)
        if energy_j is not None:       # board energy of every participating GPU
            et = torch.tensor([energy_j], dtype=torch.float64, device=red_dev)
            dist.all_reduce(et, op=dist.ReduceOp.SUM)
            energy_j = float(et.item())
    t_max_s = float(t_local.item()) * 1e-3
    value = Nglob * float(its_t.item()) / t_max_s / 1e6    # DoF*iterations of the job / max-over-ranks time
    energy = {"joules_per_solve": energy_j / n_e if energy_j is not None else None,
              "avg_watts": energy_j / t_e if energy_j is not None else None, "solves": n_e, "window_s": t_e,
              "source": "NVML nvmlDeviceGetTotalEnergyConsumption (board), >= 1.5 s window of back-to-back solves"}

    # whole-solve FP64 tensor work: 2 J_max patch-solve sweeps per smoothed level per V-cycle (one V-cycle per GMRES
    # iteration), the dominant flops of the solve (95-99 %).  Levels at or below a folded
    # sub-cycle (2D configs) run as one FFMA GEMV instead; its 2 n_f^2 flops are reported apart and not counted
    # against the DMMA peak.  On split levels every rank counts the patches of its own window.
    fold_lv = s.fold_level()
    vc_flops = sum(2 * 4 * s.level_work(l)["k2_flops"] for l in range(max(1, fold_lv + 1), cfg["levels"]))
    fold_flops = 2.0 * float(s.size(fold_lv)) ** 2 if fold_lv else 0.0
    job_flops = torch.tensor([vc_flops * its], dtype=torch.float64, device=red_dev)
    if ws > 1:
        torch.distributed.all_reduce(job_flops, op=torch.distributed.ReduceOp.SUM)
    solve_tflops = float(job_flops.item()) / t_max_s / 1e12

    # per-kernel rooflines on the fine level (CUDA events around graph-captured back-to-back launches on the bench
    # stream, right after the timed region): K2 against the FP64 DMMA peak, the HBM-bound kernels against HBM
    Lf = cfg["levels"] - 1
    kernels = {}
    for name, kind, reps in [("K2_patch_gemm", 0, 10), ("K1_apply", 1, 10), ("K3_average", 2, 10),
                             ("K5_restrict_prolong", 7, 10), ("K7_mgs_pass", 8, 20)]:
        t_ms = s.time_kernel(kind, Lf, reps=reps)
        fl, by = s.kernel_work(kind, Lf)
        ent = {"avg_launch_ms": t_ms, "algorithmic_bytes": by, "hbm_gbs": by / (t_ms * 1e-3) / 1e9,
               "hbm_frac": by / (t_ms * 1e-3) / 1e9 / HBM_PEAK_GBS}
        if kind == 8:
            ent["note"] = ("3 reads : 1 write per DoF; the peak is a 1:1 copy, and read-dominated streams run above "
                           "it on HBM3e, so hbm_frac can exceed 1")
        if fl:
            ent.update({"flops": fl, "tflops": fl / (t_ms * 1e-3) / 1e12,
                        "fp64_frac": fl / (t_ms * 1e-3) / 1e12 / FP64_PEAK_TFLOPS})
        kernels[name] = ent
    k2 = kernels["K2_patch_gemm"]
    vc_ms = s.time_kernel(3, reps=3)
    traffic = None
    tp = os.path.join(ROOT, "profiles", "k2_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(cfg["name"])
        except Exception:
            traffic = None

    # e2e: the same slab solve through the C ABI with HOST buffers (H2D rhs + x, solve, D2H x inside the timed
    # region), on the right-hand side of the last marched slab
    rhs_h = torch.empty(N, dtype=torch.float64).pin_memory()
    x_h = torch.zeros(N, dtype=torch.float64).pin_memory()
    rhs_h.copy_(rhs.cpu())
    n_e2e = max(1, min(args.steps, 5)) if Nglob > 5e6 else args.steps
    x_h.zero_()
    s.solve_host(rhs_h, x_h)                       # warm-up
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    e2e_its = 0
    t0 = time.perf_counter()
    for _ in range(n_e2e):
        x_h.zero_()
        st = s.solve_host(rhs_h, x_h)
        e2e_its += st["iterations"]
    e2e_dt = time.perf_counter() - t0
    e2e_val = Nglob * e2e_its / e2e_dt / 1e6
    if ws > 1:
        tt = torch.tensor([e2e_dt], dtype=torch.float64, device=red_dev)
        import torch.distributed as dist
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        e2e_val = Nglob * e2e_its * (1 if dd else ws) / float(tt.item()) / 1e6

    out = None
    if rank == 0:
        cpu = None
        if ws == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline(cfg)
        out = {
            "metric": "slab_solve_throughput", "value": value, "unit": "MDoF*iter/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_max_s * 1e3 / args.steps,
            "higher_is_better": True, "scaling": "strong" if dd else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": workload_config(cfg, args, ws, dd),
            "solve": {"load_assembly": "on the device each slab (stgmg_slab_load + stgmg_slab_rhs, inside the timed "
                                       "step)" if load_kind is not None else "host vector, resident on the device",
                      "gmres_iterations_total": its, "gmres_iterations_per_slab": its_list,
                      "final_rel_residual_max": max(resid), "s_per_slab": t_max_s / args.steps,
                      "s_per_slab_each": [t * 1e-3 for t in per_step_ms], "setup_s": t_setup,
                      "vcycle_ms": vc_ms, "slabs_marched": state["n"],
                      "coarse_fold": ({"level": fold_lv, "dofs": s.size(fold_lv),
                                       "note": "V-cycle of levels %d..0 (Alg. 1 sweeps, transfers, coarse solve) "
                                               "applied as its assembled matrix, built at setup from the same "
                                               "kernels; exact up to rounding (DESIGN.md 7.1)" % fold_lv}
                                      if fold_lv else None)},
            "gpu_launches": launches,
            "energy": energy,
            "roofline": {"kernel": "K2 vanka_patch_gemm (fine level)", "bound": "tensor", "achieved": k2["tflops"],
                         "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": k2["fp64_frac"],
                         "traffic": traffic, "avg_launch_ms": k2["avg_launch_ms"], "flops_per_launch": k2["flops"],
                         "algorithmic_bytes_per_launch": k2["algorithmic_bytes"],
                         "peak_source": "FP64 DMMA m8n8k4 microbenchmark on this pool (profiles/fp64_peak_r01.json); "
                                        "MEASURED_PEAKS.json has no fp64 entry",
                         "timing": "CUDA events on the bench stream around graph-captured back-to-back launches of "
                                   "the fine-level K2 right after the timed region (inside the timed region it runs "
                                   "within the per-step graphs); its share of the step: profiles/launches_r02_*.txt"},
            "kernels": kernels,
            "solve_fp64": {"flops_per_vcycle": vc_flops, "achieved_tflops": solve_tflops,
                           "frac_of_dmma_peak": solve_tflops / (FP64_PEAK_TFLOPS * ws),
                           "fold_gemv_flops_per_vcycle": fold_flops,
                           "note": "patch-solve (K2, DMMA) flops of the whole slab solves / timed solve time; the "
                                   "folded sub-cycle GEMV (FFMA) and K1/K3/K5/K7 flops (<5 %) are not counted"},
            "clocks": clk,
            "e2e": {"value": e2e_val, "unit": "MDoF*iter/s", "h2d_bytes_per_step": 16 * N * ws,
                    "d2h_bytes_per_step": 8 * N * ws, "steps": n_e2e,
                    "how": "stgmg_solve_host: pinned host rhs/x copied H2D, solve, x copied D2H, host clock"},
            "cpu_baseline": cpu,
        }
        print(json.dumps(out), flush=True)
    s.close()
    if comm is not None:
        (shm_comm_destroy if shm else nccl_comm_destroy)(comm)
    if ws > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
