#!/usr/bin/env python
"""Benchmark of the hot path: one space-time slab solve (FGMRES(m) + GMG V-cycle with patch Vanka) per step.

Workload (default): BASELINE.json configs[1] — 2D unit square, 64x64 cells, 6 levels, Q2^2/Q2^2/Q1, dG(1)
(141,578 DoFs), tau = 0.01, GMRES(30), rel tol 1e-8, load = i.i.d. U[-1,1) seed 1 (reading A21), zero initial
state; each step forms the slab RHS F_n = L + J X_{n-1} on the device (K8) and solves (slab marching).
Metric: MDoF*iter/s = N_slab * GMRES iterations / solve time / 1e6; ms_per_step = s/slab.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 1] [--impl ours|reference]

--impl reference runs the oracle (plain fp64 CPU implementation, oracle/) as it stands on the host cores.
N > 1 (torchrun, one rank per GPU): the x-slab domain decomposition of SURVEY §8(e) — every rank owns a slab of
cells of the SAME global slab problem (window vectors, halo exchange over NCCL after every smoothing sweep, GMRES
inner products allreduced), so the scaling is "strong"; value = global DoFs x iterations / max-over-ranks time.
--replicas instead runs N independent copies of the workload ("weak" scaling, no data-path collective).
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

FP64_PEAK_TFLOPS = 37.19   # measured DMMA m8n8k4 peak on this pool's B200 (profiles/fp64_peak_r01.json)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--replicas", action="store_true", help="N > 1: independent replicas instead of the decomposition")
    ap.add_argument("--smoother", default="additive", choices=["additive", "colored", "element", "overwrite"],
                    help="additive = Alg. 1 (paper, default); colored = multiplicative colour-ordered Vanka (N2(i)); "
                         "element = element-wise Vanka (N2(ii)); overwrite = Alg. 1 without averaging (N2(iii))")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    lrank = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, lrank


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


# ---------------------------------------------------------------------------------------------- oracle -----
def oracle_slab_solver(cfg):
    """The oracle as it stands (CPU), for the cpu_baseline / --impl reference legs."""
    from oracle.mg import Hierarchy
    from oracle.gmres import fgmres
    from oracle.loads import slab_rhs, end_state
    d = cfg["dim"]
    p = dict(cfg["params"])
    p["K"] = np.array(p["K"], dtype=float).reshape(3, 3)[:d, :d].ravel().tolist()
    H = Hierarchy(d, cfg["cells"][:d], cfg["lo"][:d], cfg["hi"][:d], cfg["r"], cfg["k"], cfg["levels"], p, cfg["tau"],
                  bc_u=list(cfg["bc_u"][:2 * d]), bc_p=list(cfg["bc_p"][:2 * d]))
    S = H.ops[-1].assemble_spatial()
    lev, op, A = H.fine, H.ops[-1], H.A[-1]
    L = uniform_load(lev.N, cfg["seed"] or 1)
    state = {"X": np.zeros(lev.N)}

    def step():
        U, V, P = end_state(lev, state["X"])
        b = slab_rhs(lev, S, op.chi_m1, op.th, U, V, P, None, None) + L
        x, info = fgmres(lambda v: A @ v, b, H.vcycle, tol=cfg["rtol"], restart=cfg["restart"])
        state["X"] = x
        return info["iterations"]

    return lev.N, step


def blas_threads():
    try:
        from threadpoolctl import threadpool_info
        n = [i.get("num_threads", 1) for i in threadpool_info()]
        return max(n) if n else 1
    except Exception:
        return os.cpu_count() or 1


def cpu_baseline(cfg, budget_s=25.0):
    N, step = oracle_slab_solver(cfg)
    t0 = time.perf_counter()
    its, n = 0, 0
    while True:
        its += step()
        n += 1
        if time.perf_counter() - t0 > budget_s / 2 or n >= 3:
            break
    dt = time.perf_counter() - t0
    return {"value": N * its / dt / 1e6, "unit": "MDoF*iter/s", "cores": blas_threads(), "kind": "oracle",
            "sample": "%d slab solve(s) of %s (setup excluded), %.2f s/slab, %d GMRES its" % (n, cfg["name"], dt / n, its)}


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    cfg = config(args.config)
    N, step = oracle_slab_solver(cfg)
    for _ in range(args.warmup):
        step()
    t0 = time.perf_counter()
    its = 0
    for _ in range(args.steps):
        its += step()
    dt = time.perf_counter() - t0
    val = N * its / dt / 1e6
    cores = blas_threads()
    sample = "%d slab solves of %s on host cores (oracle as it stands)" % (args.steps, cfg["name"])
    out = {"impl": "reference", "metric": "slab_solve_throughput", "value": val, "unit": "MDoF*iter/s",
           "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": cfg["name"], "dofs": N, "gmres_iterations": its},
           "cpu_baseline": {"value": val, "unit": "MDoF*iter/s", "cores": cores, "kind": "oracle", "sample": sample},
           "e2e": {"value": val, "unit": "MDoF*iter/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


# ---------------------------------------------------------------------------------------------- ours -------
def run_ours(args):
    import torch
    ws, rank, lrank = dist_env()
    if ws > 1:
        torch.cuda.set_device(lrank)
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", lrank))
    dev = torch.device("cuda", lrank if ws > 1 else 0)
    from paper_2303_06742_b200 import Solver
    from paper_2303_06742_b200.stgmg import nccl_unique_id, nccl_comm_create, nccl_comm_destroy, partition_plan
    from paper_2303_06742_b200.partition import window_index
    cfg = config(args.config)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    dd = ws > 1 and not args.replicas
    smoother = {"additive": 0, "colored": 1, "element": 2, "overwrite": 3}[args.smoother]
    comm = None
    t_setup = time.perf_counter()
    dd_error = None
    if dd:
        # the library's own NCCL communicator: rank 0 draws the id, torch.distributed broadcasts it (stgmg.h)
        try:
            uid = torch.tensor(list(nccl_unique_id()) if rank == 0 else [0] * 128, dtype=torch.uint8, device=dev)
            torch.distributed.broadcast(uid, 0)
            comm = nccl_comm_create(bytes(uid.cpu().tolist()), ws, rank)
            s = Solver(cfg, stream=stream, rank=rank, nranks=ws, comm=comm, smoother=smoother)
        except Exception as e:   # every rank fails the same way: report it and run replicas instead
            dd_error = "%s: %s" % (type(e).__name__, e)
            ok = torch.tensor([0.0], device=dev)
        else:
            ok = torch.tensor([1.0], device=dev)
        torch.distributed.all_reduce(ok, op=torch.distributed.ReduceOp.MIN)
        if ok.item() < 1.0:
            if dd_error is None:
                s.close()
                dd_error = "another rank failed to set up the decomposition"
            if comm is not None:
                nccl_comm_destroy(comm)
                comm = None
            dd = False
            print("bench: x-slab decomposition unavailable (%s); running %d replicas" % (dd_error, ws), file=sys.stderr)
            s = Solver(cfg, stream=stream, smoother=smoother)
    else:
        s = Solver(cfg, stream=stream, smoother=smoother)
    t_setup = time.perf_counter() - t_setup
    N = s.size()                       # this rank's (window) vector length
    Nglob = dof_count(cfg)             # DoFs of the global slab problem
    Lg = uniform_load(Nglob, cfg["seed"] or 1)
    if dd:
        idx, _own = window_index(cfg, cfg["levels"] - 1, partition_plan(cfg, cfg["levels"] - 1, rank, ws))
        Lg = Lg[idx]
    L = torch.as_tensor(Lg, device=dev)
    Xp = torch.zeros(N, dtype=torch.float64, device=dev)
    rhs = torch.zeros_like(Xp)
    x = torch.zeros_like(Xp)
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device=dev)   # > 126 MB L2
    rhs_launches = 1 << cfg["dim"]

    def step():
        s.slab_rhs(L, Xp, rhs)
        x.zero_()
        st = s.solve(rhs, x, tol=cfg["rtol"], restart=cfg["restart"])
        Xp.copy_(x)
        return st

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if ws > 1:
        torch.distributed.barrier()
    clocks = ClockSampler(dev.index)
    ev0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ev1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    its, launches, resid = 0, 0, []
    for i in range(args.steps):
        flush.fill_(float(i))                      # L2 flush between timed steps (untimed)
        ev0[i].record(stream)
        st = step()
        ev1[i].record(stream)
        its += st["iterations"]
        resid.append(st["rel_residual"])
        launches += s.launch_count() + rhs_launches
    torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in zip(ev0, ev1))
    # energy window: NVML's counter updates coarsely, so measure over >= 1.5 s of back-to-back slab solves
    # (same step, no flushes); the clock sampler keeps running through it
    e_start = nvml_energy_mj(dev.index)
    t_e0 = time.perf_counter()
    n_e = 0
    while True:
        step()
        n_e += 1
        if n_e >= args.steps and time.perf_counter() - t_e0 > 1.5:
            torch.cuda.synchronize()
            if time.perf_counter() - t_e0 > 1.5:
                break
    torch.cuda.synchronize()
    t_e = time.perf_counter() - t_e0
    e_end = nvml_energy_mj(dev.index)
    clk = clocks.stop()
    t_local = torch.tensor([ms], dtype=torch.float64, device=dev)
    its_t = torch.tensor([float(its)], dtype=torch.float64, device=dev)
    energy_j = (e_end - e_start) * 1e-3 if (e_start is not None and e_end is not None) else None
    if ws > 1:
        import torch.distributed as dist
        dist.all_reduce(t_local, op=dist.ReduceOp.MAX)
        if not dd:                     # replicas: every rank solved its own copy
            dist.all_reduce(its_t, op=dist.ReduceOp.SUM)
        if energy_j is not None:       # board energy of every participating GPU
            et = torch.tensor([energy_j], dtype=torch.float64, device=dev)
            dist.all_reduce(et, op=dist.ReduceOp.SUM)
            energy_j = float(et.item())
    t_max_s = float(t_local.item()) * 1e-3
    value = Nglob * float(its_t.item()) / t_max_s / 1e6    # DoF*iterations of the job / max-over-ranks time
    energy = {"joules_per_solve": energy_j / n_e if energy_j is not None else None,
              "avg_watts": energy_j / t_e if energy_j is not None else None, "solves": n_e, "window_s": t_e,
              "source": "NVML nvmlDeviceGetTotalEnergyConsumption (board), >= 1.5 s window of back-to-back solves"}

    # roofline of the dominant kernel: K2 patch GEMM on the fine level (FP64 DMMA), timed alone
    work = s.level_work()
    # whole-solve FP64 tensor work: 2 J_max patch-solve sweeps per smoothed level per V-cycle (one V-cycle per GMRES
    # iteration), the dominant flops of the solve (95-99 %)
    # levels at or below the folded sub-cycle run as one GEMV of 2 n_f^2 flops instead of their sweeps
    fold_lv = s.fold_level()
    vc_flops = sum(2 * 4 * s.level_work(l)["k2_flops"] for l in range(max(1, fold_lv + 1), cfg["levels"]))
    if fold_lv:
        vc_flops += 2.0 * float(s.size(fold_lv)) ** 2   # this rank's
    job_flops = torch.tensor([vc_flops * its], dtype=torch.float64, device=dev)
    if ws > 1:
        torch.distributed.all_reduce(job_flops, op=torch.distributed.ReduceOp.SUM)
    solve_tflops = float(job_flops.item()) / t_max_s / 1e12
    k2_ms = s.time_kernel(0, reps=50)
    k2_achieved = work["k2_flops"] / (k2_ms * 1e-3) / 1e12
    vc_ms = s.time_kernel(3, reps=20)
    k1_ms = s.time_kernel(1, reps=50)
    traffic = None
    tp = os.path.join(ROOT, "profiles", "k2_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(cfg["name"])
        except Exception:
            traffic = None

    # e2e: the same solve through the C ABI with host buffers (H2D rhs + x, D2H x inside the timed region)
    rhs_h = torch.empty(N, dtype=torch.float64).pin_memory()
    x_h = torch.zeros(N, dtype=torch.float64).pin_memory()
    rhs_h.copy_(L.cpu())
    e2e_its = 0
    for _ in range(1):
        x_h.zero_()
        s.solve_host(rhs_h, x_h)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        x_h.zero_()
        st = s.solve_host(rhs_h, x_h)
        e2e_its += st["iterations"]
    e2e_dt = time.perf_counter() - t0
    e2e_val = Nglob * e2e_its / e2e_dt / 1e6
    if ws > 1:
        tt = torch.tensor([e2e_dt], dtype=torch.float64, device=dev)
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
            "config": {"workload": cfg["name"], "dofs": Nglob, "levels": cfg["levels"], "r": cfg["r"], "k": cfg["k"],
                       "restart": cfg["restart"], "rtol": cfg["rtol"], "load": "uniform[-1,1) seed %s" % cfg["seed"],
                       "smoother": args.smoother,
                       "gmres_iterations_total": its, "final_rel_residual_max": max(resid),
                       "l2": "flushed between timed steps (256 MB write, untimed)",
                       "parallelism": ("x-slab decomposition over %d GPUs (NCCL halo exchange)" % ws) if dd else
                                      (("%d replicas" % ws + (" (decomposition unavailable: %s)" % dd_error
                                                              if dd_error else "")) if ws > 1 else "single GPU"),
                       "setup_s": t_setup,
                       "s_per_slab": t_max_s / args.steps,
                       "vcycle_ms": vc_ms, "k1_fine_apply_ms": k1_ms,
                       "coarse_fold": ({"level": fold_lv, "dofs": s.size(fold_lv),
                                        "note": "V-cycle of levels %d..0 (Alg. 1 sweeps, transfers, coarse solve) "
                                                "applied as its assembled matrix, built at setup from the same "
                                                "kernels; exact up to rounding (DESIGN.md 7.1)" % fold_lv}
                                       if fold_lv else None),
                       "k1_fine_hbm_gbs": work["k1_bytes"] / (k1_ms * 1e-3) / 1e9},
            "gpu_launches": launches,
            "energy": energy,
            "roofline": {"kernel": "K2 vanka_patch_gemm (fine level)", "bound": "tensor", "achieved": k2_achieved,
                         "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s", "frac": k2_achieved / FP64_PEAK_TFLOPS,
                         "traffic": traffic, "avg_launch_ms": k2_ms, "flops_per_launch": work["k2_flops"],
                         "algorithmic_bytes_per_launch": work["k2_bytes"],
                         "peak_source": "FP64 DMMA m8n8k4 microbenchmark on this pool (profiles/fp64_peak_r01.json); "
                                        "MEASURED_PEAKS.json has no fp64 entry",
                         "timing": "CUDA events on the bench stream around 50 graph-captured back-to-back launches of "
                                   "the fine-level K2 right after the timed region (inside the timed region it runs "
                                   "within the per-step graphs); its share of the step: profiles/launches_r01_cfg1.txt"},
            "solve_fp64": {"flops_per_vcycle": vc_flops, "achieved_tflops": solve_tflops,
                           "frac_of_dmma_peak": solve_tflops / (FP64_PEAK_TFLOPS * ws),
                           "note": "patch-solve (K2) flops of the whole slab solves / timed solve time; K1/K3/K5/K7 "
                                   "flops (<5 %) not counted"},
            "clocks": clk,
            "e2e": {"value": e2e_val, "unit": "MDoF*iter/s", "h2d_bytes_per_step": 16 * N * ws,
                    "d2h_bytes_per_step": 8 * N * ws},
            "cpu_baseline": cpu,
        }
        print(json.dumps(out), flush=True)
    s.close()
    if comm is not None:
        nccl_comm_destroy(comm)
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
