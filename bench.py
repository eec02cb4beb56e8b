"""Benchmark: implicit-Euler heat steps (RHS + Jacobi-PCG to tol 1e-10) of the
tensor B-spline heat problem at paper scale on B200.

Metric (BASELINE.json): CG iteration DoF/s (GDoF/s) -- sum over the timed
steps of (CG iterations x DoF) / device time, whole job.  One "step" is one
implicit-Euler time step: b = M u + dt F (fused mass kernel) and the full
Jacobi-PCG solve with x0 = u_prev.

Default workload (N=1): C3, 930^3 coefficients (928^3 = 0.80 B nodes), p=3,
lambda = dt/h^2 = 4, fp64, synthetic Gaussian IC/source.
N>1: the same global grid split in z-slabs, one rank per GPU (strong scaling).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--ncoef 930] [--impl reference]
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# pass A: read r, p_{k-1}; write Ap, p_k.  Pass B: read r, Ap; write r
# (24 B), and every P_RING-th iteration also read x and the last P_RING p's
# and write x (24 + 16 + 8 * P_RING B): x moves once per P_RING iterations
#
ALG_BYTES_PASS_A = 32
ALG_BYTES_PASS_B = 24 + (16 + 8 * 4) / 4  # 36: average over the ring period (P_RING = 4)
ALG_BYTES_ITER = ALG_BYTES_PASS_A + ALG_BYTES_PASS_B  # 68
SURVEY_BYTES_ITER = 80  # x, r, p, Ap streams of the textbook fused CG
# ncu-measured DRAM traffic per DoF for the kernels (profiles/, `--set full` at 512^3):
# filled from the committed profile summary when present
TRAFFIC = {}
_tp = os.path.join(ROOT, "profiles", "traffic.json")
if os.path.exists(_tp):
    with open(_tp) as _f:
        TRAFFIC = json.load(_f)


def measured_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() in ("active", "1", "yes"):
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": float(max(smax)) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU baseline / reference arm (oracle port -- the reference is pure Python and
# does not exist on the GPU box)


def cpu_port_rate(ncoef=64, iters=20, repeats=3, p=3):
    """Oracle port of the reference CG path (numpy/scipy Kronecker apply +
    the reference pcg recurrence) on the C1 heat problem: CG DoF-it/s.
    Single-threaded: scipy's sparse matvec holds the GIL (a thread pool over
    slabs measured 7.7x slower); the port is still ~6x faster than the
    reference's fastest strategy (sparse 1.78 MDoF-it/s)."""
    from oracle import bspde_oracle as O

    inp = O.heat_inputs(ncoef, p)
    N, h, dt = inp["N"], inp["h"], inp["dt"]
    A = O.KronOperator((N,) * 3, (h,) * 3, p, dt, 1.0)
    b = A.mass_apply(inp["u0"]) + dt * A.mass_apply(inp["q"])
    O.pcg(A.apply, A.jacobi_diagonal, b, tol=1e-30, max_iter=2, x0=inp["u0"])  # warm
    times = []
    for _ in range(repeats):
        t0 = time.perf_counter()
        _, rep = O.pcg(A.apply, A.jacobi_diagonal, b, tol=1e-30, max_iter=iters, x0=inp["u0"])
        times.append(time.perf_counter() - t0)
    dofs = int(np.prod(A.cext))
    t = float(np.median(times))
    return dofs * rep["iterations"] / t, dict(dofs=dofs, iterations=rep["iterations"], seconds=t)


def _ref_worker(p, iters, nstep, barrier, out):
    """One reference-arm worker process: builds its own C1 system, then times
    `nstep` PCG samples, each started at a barrier shared by all workers so the
    timed regions overlap (memory-bandwidth contention included)."""
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass
    from oracle import bspde_oracle as O

    inp = O.heat_inputs(64, p)
    N, h, dt = inp["N"], inp["h"], inp["dt"]
    A = O.KronOperator((N,) * 3, (h,) * 3, p, dt, 1.0)
    b = A.mass_apply(inp["u0"]) + dt * A.mass_apply(inp["q"])
    O.pcg(A.apply, A.jacobi_diagonal, b, tol=1e-30, max_iter=2, x0=inp["u0"])  # warm
    res = []
    for _ in range(nstep):
        barrier.wait()
        t0 = time.perf_counter()
        _, rep = O.pcg(A.apply, A.jacobi_diagonal, b, tol=1e-30, max_iter=iters, x0=inp["u0"])
        res.append((int(np.prod(A.cext)) * rep["iterations"], time.perf_counter() - t0,
                    rep["iterations"]))
    out.put(res)


def host_workers():
    try:
        n = len(os.sched_getaffinity(0))
    except AttributeError:
        n = os.cpu_count() or 1
    return max(1, min(n, int(os.environ.get("BSPDE_REF_WORKERS", n)), 256))


def run_reference(args, rank, world):
    """Reference arm: the oracle port of the reference CG path on every host
    core the process may use -- one single-threaded worker process per core
    (scipy's matvec holds the GIL, so threads do not scale), each solving its
    own C1 sample; a step's value is the summed DoF-iterations of all workers
    over the slowest worker's time."""
    if rank != 0:
        return
    import multiprocessing as mp

    steps, warm = max(args.steps, 1), max(args.warmup, 0)
    nw = host_workers()
    iters = 10
    ctx = mp.get_context("fork")
    barrier, out = ctx.Barrier(nw), ctx.Queue()
    procs = [ctx.Process(target=_ref_worker, args=(args.degree, iters, warm + steps, barrier, out))
             for _ in range(nw)]
    for pr in procs:
        pr.start()
    results = [out.get() for _ in procs]
    for pr in procs:
        pr.join()
    vals, times = [], []
    for i in range(warm, warm + steps):
        work = sum(r[i][0] for r in results)
        t = max(r[i][1] for r in results)
        vals.append(work / t)
        times.append(t)
    val = float(np.median(vals)) / 1e9
    its = results[0][0][2]
    sample = (f"C1 sample: 64^3 coefficients, p={args.degree}, lambda=4, {its} Jacobi-PCG "
              f"iterations per step in each of {nw} worker processes (one per host core, timed "
              f"between barriers; oracle port: scipy CSR 1-D factors, separable Kronecker "
              f"apply, reference pcg recurrence); full config {args.ncoef}^3 infeasible on CPU")
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "GDoF/s", "n_gpus": world,
        "steps": steps, "warmup": warm, "ms_per_step": float(np.median(times)) * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_of(args, world),
        "cpu_baseline": {"value": val, "unit": "GDoF/s", "cores": nw, "kind": "port",
                         "sample": sample},
        "e2e": {"value": val, "unit": "GDoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


METRIC = "CG iteration DoF/s (GDoF/s) and % HBM roofline at 0.8B nodes, 1/2/4/8 B200"


def config_of(args, world):
    from paper_1904_03057_b200.gram import basis_extension

    ncoef, p = args.ncoef, args.degree
    tag = "C3" if (ncoef, p) == (930, 3) else ("C4" if ncoef == 512 else "custom")
    nodes = ncoef - 2 * basis_extension(p)
    gb = ncoef ** 3 * 8 / 1e9
    return {"workload": f"{tag} heat: {ncoef}^3 coefficients ({nodes}^3 nodes), p={p}, "
                        f"implicit Euler lambda=4, Jacobi-PCG tol 1e-10, z-slabs x{world}",
            "ncoef": ncoef, "degree": p, "dofs": ncoef ** 3, "precision": "fp64",
            "parallelism": f"zslab{world}",
            "halo_overlap": (os.environ.get("BSPDE_HALO_OVERLAP", "pipeline") if world > 1
                             else "none (single slab)"),
            "l2": f"inputs ({gb:.1f} GB/vector) vs 126 MB L2"}


# ---------------------------------------------------------------------------


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_1904_03057_b200 import SolveConfig, make_operator
    from paper_1904_03057_b200.distributed import DistributedOperator
    from paper_1904_03057_b200.domain import Grid
    from paper_1904_03057_b200.heat import HeatSolver
    from paper_1904_03057_b200.synthetic import IC, SOURCE, gaussian_coeffs, heat_c_inputs
    from paper_1904_03057_b200.system import heat_system

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    p = args.degree
    N, h, dt = heat_c_inputs(args.ncoef, p)
    data = heat_system(Grid((N,) * 3, (h,) * 3), p, dt)
    dofs = int(np.prod(data.cext))
    cfg = SolveConfig(tol=1e-10, max_iter=5000, poll_every=args.poll)
    stream = torch.cuda.current_stream()

    if world == 1:
        op = make_operator(data, "b200", device=local_rank)
        lay = op.layout
        z_range = None
    else:
        op = DistributedOperator(data)
        lay = op.layout
        z_range = op.part.bounds()
    u = lay.alloc(dev)
    q = lay.alloc(dev)
    gaussian_coeffs(N, h, p, device=dev, out=u, layout=lay, z_range=z_range, **IC)
    gaussian_coeffs(N, h, p, device=dev, out=q, layout=lay, z_range=z_range, **SOURCE)
    F = lay.alloc(dev)
    op.mass_apply_device(q, F)
    del q
    u0 = u.clone()
    if world == 1:
        hs = HeatSolver.from_device(op, dt, u, F, cfg)
        step = hs.step
    else:
        b = lay.alloc(dev)

        def step():
            op.mass_apply_device(u, b, F, a=dt)
            return op.pcg_device(b, u, cfg, has_x0=True)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        step()
    barrier()
    plan = op.plan()
    launches0 = plan.launches
    clk = ClockSampler(local_rank)
    clk.start()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    barrier()
    ev0.record(stream)
    its = []
    for _ in range(args.steps):
        its.append(step().iterations)
    ev1.record(stream)
    barrier()
    clocks = clk.stop()
    ms = max_over_ranks(ev0.elapsed_time(ev1))
    launches = plan.launches - launches0
    total_its = int(sum(its))
    value = total_its * dofs / (ms * 1e-3) / 1e9

    # -- per-kernel durations (CUDA events on the launching stream) --
    kt = kernel_times(op, u, F, dt, stream, world)
    kt = {k: max_over_ranks(v) for k, v in kt.items()}
    peak, peak_kind = measured_peaks()
    local_dofs = int(np.prod(lay.owned_shape))
    a_gbs = ALG_BYTES_PASS_A * local_dofs / (kt["pass_a_ms"] * 1e-3) / 1e9
    b_gbs = ALG_BYTES_PASS_B * local_dofs / (kt["pass_b_ms"] * 1e-3) / 1e9
    dom = "pass_b" if kt["pass_b_ms"] >= kt["pass_a_ms"] else "pass_a"
    ach = b_gbs if dom == "pass_b" else a_gbs
    it_s = (kt["pass_a_ms"] + kt["pass_b_ms"]) * 1e-3
    it_gbs = ALG_BYTES_ITER * local_dofs / it_s / 1e9
    it_gbs80 = SURVEY_BYTES_ITER * local_dofs / it_s / 1e9  # DoF-it rate vs the 80 B roofline

    # -- end to end through the public API: u from/to pinned host memory each step --
    e2e = e2e_rate(step, u, u0, lay, dofs, min(args.steps, 3), stream, barrier, max_over_ranks)

    cpu = None
    if rank == 0 and not args.no_cpu_baseline:
        rate, info = cpu_port_rate(64, iters=20, repeats=3, p=args.degree)
        cpu = {"value": rate / 1e9, "unit": "GDoF/s", "cores": 1, "kind": "port",
               "sample": f"C1 64^3 p={args.degree} heat system, {info['iterations']} Jacobi-PCG iterations, "
                         "median of 3 (oracle port, scipy/numpy single thread)"}

    line = {
        "metric": METRIC, "value": value, "unit": "GDoF/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_of(args, world),
        "cg_iterations_per_step": its,
        "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                     "frac": ach / peak,
                     # ncu traffic is captured for the C3 workload (profiles/traffic.json)
                     "traffic": TRAFFIC.get(dom) if (args.ncoef, args.degree) == (930, 3) else None,
                     "kernel": dom,
                     "peak_source": peak_kind,
                     "alg_bytes_per_dof": ALG_BYTES_PASS_B if dom == "pass_b" else ALG_BYTES_PASS_A,
                     "pass_a_ms": kt["pass_a_ms"], "pass_b_ms": kt["pass_b_ms"],
                     "pass_a_gbs": a_gbs, "pass_b_gbs": b_gbs,
                     "cg_iteration_gbs": it_gbs, "cg_iteration_frac": it_gbs / peak,
                     "cg_iteration_frac_80B": it_gbs80 / peak},
        "clocks": clocks,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "cpu_baseline": cpu,
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def kernel_times(op, u, F, dt, stream, world, reps=9):
    """Average device duration of CG pass A and pass B (same stream, events),
    on a copy of the current state (the timed solve is already over)."""
    import torch

    plan = op.plan()
    lay = op.layout
    dev = u.device
    x = u.clone()
    b = lay.alloc(dev)
    r = lay.alloc(dev)
    pring = lay.alloc_ring(dev)
    ap = lay.alloc(dev)
    scratch = plan.scratch()
    op.mass_apply_device(x, b, F, a=dt)
    plan.cg_setup(scratch, None, 1e-300, 10 ** 6, False, True)
    plan.cg_residual(b, x, r, scratch, 1)
    ta, tb = [], []
    for k in range(reps):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(stream)
        R = pring.shape[0]
        plan.cg_pass_a(r, pring[(k - 1) % R], pring[k % R], ap, scratch, 1)
        e[1].record(stream)
        plan.cg_pass_b(x, r, pring, ap, scratch, 1)
        e[2].record(stream)
        torch.cuda.synchronize()
        ta.append(e[0].elapsed_time(e[1]))
        tb.append(e[1].elapsed_time(e[2]))
    del x, b, r, pring, ap
    torch.cuda.empty_cache()
    return {"pass_a_ms": float(np.mean(ta[1:])), "pass_b_ms": float(np.mean(tb[1:]))}


def e2e_rate(step, u, u0, lay, dofs, steps, stream, barrier, max_over_ranks):
    """Same metric through the public step API with the state copied from and
    back to pinned host memory every step (host<->device copies timed)."""
    from paper_1904_03057_b200.heat import run_steps_host

    import torch

    host = torch.empty(lay.owned_shape, dtype=torch.float64).pin_memory()
    own = lay.owned(u)
    # untimed warm-up of the same pipeline (first DMA through the freshly
    # pinned buffer and the side streams), then reset the input
    host.copy_(lay.owned(u0).cpu())
    run_steps_host(step, own, host, 1, chunks=16, stream=stream)
    torch.cuda.synchronize()
    host.copy_(lay.owned(u0).cpu())
    barrier()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    if os.environ.get("BSPDE_E2E_SEQ"):  # A/B: strictly sequential copies
        its = 0
        for _ in range(steps):
            own.copy_(host, non_blocking=True)
            its += step().iterations
            host.copy_(own, non_blocking=True)
    else:
        reps = run_steps_host(step, own, host, steps, chunks=16, stream=stream)
        its = sum(r.iterations for r in reps)
    ev1.record(stream)
    barrier()
    ms = max_over_ranks(ev0.elapsed_time(ev1))
    nbytes = int(np.prod(lay.owned_shape)) * 8
    return {"value": its * dofs / (ms * 1e-3) / 1e9, "unit": "GDoF/s",
            "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
            "steps": steps, "cg_iterations": int(its), "ms": ms,
            "api": "heat step (public API, heat.run_steps_host) with u copied from/to pinned host "
                   "memory every step; the result download of step k and the input upload of "
                   "step k+1 overlap chunk-wise (16 z-chunks, full-duplex PCIe)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--ncoef", type=int, default=930)
    ap.add_argument("--degree", type=int, default=3, help="B-spline degree (C4 sweep: 1..5)")
    ap.add_argument("--poll", type=int, default=16)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
