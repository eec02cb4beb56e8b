"""Benchmark: implicit-Euler heat steps (RHS + Jacobi-PCG to tol 1e-10) of the
tensor B-spline heat problem at paper scale on B200.

Metric (BASELINE.json): CG iteration DoF/s (GDoF/s) -- sum over the timed
steps of (CG iterations x DoF) / device time, whole job.  One "step" is one
implicit-Euler time step: b = M u + dt F (fused mass kernel) and the full
Jacobi-PCG solve with x0 = u_prev.

Default workload (N=1): C3, 930^3 coefficients (928^3 = 0.80 B nodes), p=3,
lambda = dt/h^2 = 4, fp64, synthetic Gaussian IC/source.
N>1: the same global grid split in z-slabs, one rank per GPU (strong scaling);
`--gpus N` without a launcher spawns the N ranks itself (torch.distributed.run).

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

# algorithmic bytes per DoF of the CG passes: alg_bytes() below
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
# CPU baseline / reference arm.  The reference (package `bspde`, pure Python)
# is installed into baseline/_ref; it runs on the host cores.
# When it cannot be imported, the oracle port (oracle/bspde_oracle.py) stands
# in and the line says kind "port".

REF_DIR = os.path.join(ROOT, "baseline", "_ref")
REF_SAMPLE_NCOEF = 64  # C1: the reference's own demo scale (BASELINE.json configs[0])


def _reference_modules():
    """The installed reference package, or None (then the oracle port is timed)."""
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        from bspde.assembly import basis_extension, build_system
        from bspde.domain import BoxDomain, Grid
        from bspde.operator import make_operator
        from bspde.solver import SolveConfig, pcg
    except Exception:
        return None
    return dict(basis_extension=basis_extension, build_system=build_system,
                BoxDomain=BoxDomain, Grid=Grid, make_operator=make_operator,
                SolveConfig=SolveConfig, pcg=pcg)


def _ref_system(R, p, ncoef=REF_SAMPLE_NCOEF):
    """The C1 heat system A = M + dt K through the reference's own API
     and a smooth right-hand side."""
    ext = R["basis_extension"](p)
    N = ncoef - 2 * ext
    h = 1.0 / (N - 1)
    dt = 4.0 * h * h
    g = R["Grid"]((N,) * 3, (h,) * 3)
    shp = tuple(n + 2 * ext for n in g.extents)
    data = R["build_system"](R["BoxDomain"](g), p, p, np.full(shp, dt), np.full(shp, 1.0), [])
    b = np.random.default_rng(0).normal(size=shp)
    return data, b


def _ref_sparse_worker(p, iters, nstep, barrier, out):
    """One reference-arm worker process: the reference's pcg over its fastest
    strategy (SparseMatrixOperator, scipy CSR) on its own C1 system; each step
    is `iters` CG iterations timed between barriers shared by all workers (so
    the timed regions overlap, memory-bandwidth contention included)."""
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass
    R = _reference_modules()
    data, b = _ref_system(R, p)
    A = R["make_operator"](data, "sparse")
    cfg = R["SolveConfig"](tol=1e-30, max_iter=iters)
    R["pcg"](A, b, R["SolveConfig"](tol=1e-30, max_iter=1))  # warm
    dofs = int(np.prod(b.shape))
    res = []
    for _ in range(nstep):
        barrier.wait()
        t0 = time.perf_counter()
        _, rep = R["pcg"](A, b, cfg)
        res.append((dofs * rep.iterations, time.perf_counter() - t0, rep.iterations))
    out.put(res)


def _ref_onthefly_rate(p, workers):
    """The reference's default / paper strategy: OnTheFlyOperator with
    `workers` threads, one CG iteration (one apply) on the C1 system."""
    R = _reference_modules()
    data, b = _ref_system(R, p)
    A = R["make_operator"](data, "onthefly", workers=workers)
    t0 = time.perf_counter()
    _, rep = R["pcg"](A, b, R["SolveConfig"](tol=1e-30, max_iter=1))
    t = time.perf_counter() - t0
    return int(np.prod(b.shape)) * rep.iterations / t, t


def _port_worker(p, iters, nstep, barrier, out):
    """Fallback worker: the oracle port (no reference package importable)."""
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(1)
    except Exception:
        pass
    from oracle import bspde_oracle as O

    inp = O.heat_inputs(REF_SAMPLE_NCOEF, p)
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


def host_workers(per_worker_bytes=0):
    try:
        n = len(os.sched_getaffinity(0))
    except AttributeError:
        n = os.cpu_count() or 1
    if per_worker_bytes:
        try:
            import psutil
            n = min(n, max(1, int(0.6 * psutil.virtual_memory().available // per_worker_bytes)))
        except Exception:
            pass
    return max(1, min(n, int(os.environ.get("BSPDE_REF_WORKERS", n)), 256))


def _run_workers(target, p, iters, steps, warm, nw):
    import multiprocessing as mp

    ctx = mp.get_context("fork")
    barrier, out = ctx.Barrier(nw), ctx.Queue()
    procs = [ctx.Process(target=target, args=(p, iters, warm + steps, barrier, out))
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
    return float(np.median(vals)), float(np.median(times)), results[0][0][2]


def cpu_reference_rate(p=3, iters=10, repeats=3):
    """Our arm's cpu_baseline: one reference process (sparse strategy, the
    reference's fastest) on the C1 system; oracle port if the reference is
    absent.  Returns (DoF-it/s, kind, sample)."""
    R = _reference_modules()
    if R is not None:
        data, b = _ref_system(R, p)
        A = R["make_operator"](data, "sparse")
        cfg = R["SolveConfig"](tol=1e-30, max_iter=iters)
        R["pcg"](A, b, R["SolveConfig"](tol=1e-30, max_iter=1))
        ts = []
        for _ in range(repeats):
            t0 = time.perf_counter()
            _, rep = R["pcg"](A, b, cfg)
            ts.append(time.perf_counter() - t0)
        rate = int(np.prod(b.shape)) * rep.iterations / float(np.median(ts))
        return rate, "reference", (f"C1 64^3 p={p}: the reference's pcg over SparseMatrixOperator "
                                   f"(baseline/_ref), {rep.iterations} iterations, median of "
                                   f"{repeats}, 1 process")
    from oracle import bspde_oracle as O

    inp = O.heat_inputs(REF_SAMPLE_NCOEF, p)
    N, h, dt = inp["N"], inp["h"], inp["dt"]
    A = O.KronOperator((N,) * 3, (h,) * 3, p, dt, 1.0)
    b = A.mass_apply(inp["u0"]) + dt * A.mass_apply(inp["q"])
    ts = []
    for _ in range(repeats):
        t0 = time.perf_counter()
        _, rep = O.pcg(A.apply, A.jacobi_diagonal, b, tol=1e-30, max_iter=iters, x0=inp["u0"])
        ts.append(time.perf_counter() - t0)
    rate = int(np.prod(A.cext)) * rep["iterations"] / float(np.median(ts))
    return rate, "port", (f"C1 64^3 p={p}: oracle port (reference package not importable), "
                          f"{rep['iterations']} iterations, median of {repeats}, 1 process")


def run_reference(args, rank, world):
    """Reference arm: the reference's own CPU path on every host core.  The
    reference parallelises nothing but its on-the-fly apply (threads over
    blocks), and its fastest strategy (sparse CSR SpMV) is single-threaded,
    so the arm runs one single-threaded sparse-strategy pcg process per core,
    each on its own C1 sample; a step's value is the summed DoF-iterations
    over the slowest worker's time.  The on-the-fly strategy with
    workers=cpu_count (the paper's algorithm) is timed beside it."""
    if rank != 0:
        return
    steps, warm = max(args.steps, 1), max(args.warmup, 0)
    R = _reference_modules()
    iters = 2
    if R is not None:
        nw = host_workers(per_worker_bytes=1.6e9)  # the C1 CSR matrix is ~1 GB per process
        val, t_med, its = _run_workers(_ref_sparse_worker, args.degree, iters, steps, warm, nw)
        kind = "reference"
        otf_rate, otf_t = _ref_onthefly_rate(args.degree, host_workers())
        extra = {"onthefly": {"value": otf_rate / 1e9, "unit": "GDoF/s", "workers": host_workers(),
                              "seconds_per_iteration": otf_t}}
        sample = (f"C1 sample: 64^3 coefficients, p={args.degree}, lambda=4 heat system; the "
                  f"reference's pcg over SparseMatrixOperator (baseline/_ref, scipy CSR, its "
                  f"fastest strategy), {its} CG iterations per step in each of {nw} "
                  f"single-threaded worker processes (one per host core) timed between barriers")
    else:
        nw = host_workers()
        val, t_med, its = _run_workers(_port_worker, args.degree, 10, steps, warm, nw)
        kind, extra = "port", {}
        sample = (f"C1 sample: 64^3 coefficients, p={args.degree}, lambda=4; oracle port "
                  f"(reference package not importable), {its} iterations per step in each of "
                  f"{nw} worker processes")
    val /= 1e9
    cfg = config_of(args, world)
    cfg.update(ncoef=REF_SAMPLE_NCOEF, dofs=REF_SAMPLE_NCOEF ** 3, parallelism="host cores",
               target_config=f"{args.ncoef}^3 p={args.degree} (our arm's workload)")
    cfg["workload"] = (f"C1 heat sample: {REF_SAMPLE_NCOEF}^3 coefficients, p={args.degree}, "
                       f"implicit Euler lambda=4 (the {args.ncoef}^3 config is infeasible for the "
                       f"reference on CPU: ~{args.ncoef ** 3 / 262144 * 0.17:.0f} s per sparse "
                       f"iteration and ~{args.ncoef ** 3 * 3.8e3 / 1e12:.1f} TB of CSR)")
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "GDoF/s", "n_gpus": world,
        "steps": steps, "warmup": warm, "ms_per_step": t_med * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": cfg,
        "cpu_baseline": {"value": val, "unit": "GDoF/s", "cores": nw, "kind": kind,
                         "sample": sample, **extra},
        "e2e": {"value": val, "unit": "GDoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


METRIC = "CG iteration DoF/s (GDoF/s) and % HBM roofline at 0.8B nodes, 1/2/4/8 B200"


def config_of(args, world, halo=None):
    from paper_1904_03057_b200.gram import basis_extension

    ncoef, p = args.ncoef, args.degree
    tag = {(930, 3): "C3", (256, 3): "C2"}.get((ncoef, p), "C4" if ncoef == 512 else (
        "C5" if ncoef in (1024, 1536) else "custom"))
    nodes = ncoef - 2 * basis_extension(p)
    gb = ncoef ** 3 * 8 / 1e9
    return {"workload": f"{tag} heat: {ncoef}^3 coefficients ({nodes}^3 nodes), p={p}, "
                        f"implicit Euler lambda=4, Jacobi-PCG tol 1e-10, z-slabs x{world}",
            "ncoef": ncoef, "degree": p, "dofs": ncoef ** 3, "precision": "fp64",
            "parallelism": f"zslab{world}",
            "halo_overlap": (halo or os.environ.get("BSPDE_HALO_OVERLAP", "peer or pipeline")
                             if world > 1 else "none (single slab)"),
            "l2": f"inputs ({gb:.1f} GB/vector) vs 126 MB L2"}


# ---------------------------------------------------------------------------


def alg_bytes():
    """Algorithmic bytes per DoF of pass A / pass B / a CG iteration: pass A
    reads r, p_{k-1}, x and writes Ap, p_k, x (48 B: it forms p_k, applies A
    and x += alpha_{k-1} p_{k-1}); pass B reads r, Ap and writes r (24 B)
    (DESIGN.md §5)."""
    return 48, 24, 72


def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist

    from paper_1904_03057_b200 import SolveConfig, make_operator
    from paper_1904_03057_b200.device import heat_memory_plan
    from paper_1904_03057_b200.distributed import DistributedOperator
    from paper_1904_03057_b200.domain import Grid
    from paper_1904_03057_b200.heat import HeatSolver
    from paper_1904_03057_b200.solver import _work
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
    mem = heat_memory_plan(data.cext, p, world)
    cfg = SolveConfig(tol=1e-10, max_iter=5000, poll_every=args.poll)
    stream = torch.cuda.current_stream()

    # resident fields: u, F and the CG work set (r, Ap = b, ring) -- nothing
    # else; q is staged in r, which the first solve overwrites
    if world == 1:
        op = make_operator(data, "b200", device=local_rank)
        lay = op.layout
        z_range = None
    else:
        op = DistributedOperator(data)
        lay = op.layout
        z_range = op.part.bounds()
    halo_mode = None
    u = lay.alloc(dev)
    F = lay.alloc(dev)
    gaussian_coeffs(N, h, p, device=dev, out=u, layout=lay, z_range=z_range, **IC)
    if world == 1:
        w = _work(op, cfg.max_iter)
        r_buf, ring = w.r, w.pring.shape[0]
    else:
        wb = op._work_buffers(cfg.max_iter)
        r_buf, ring = wb["r"], wb["pring"].shape[0]
        # peer: pass A / pass B store the halo planes into the neighbours'
        # fields (CUDA IPC over NVLink); else NCCL halo transfers
        halo_mode = os.environ.get("BSPDE_HALO_OVERLAP",
                                   "peer" if op._peers is not None else "pipeline")
    gaussian_coeffs(N, h, p, device=dev, out=r_buf, layout=lay, z_range=z_range, **SOURCE)
    op.mass_apply_device(r_buf, F)
    if world == 1:
        hs = HeatSolver.from_device(op, dt, u, F, cfg)
        step = hs.step
    else:
        def step():  # RHS fused into the first residual, as the single-GPU step
            return op.heat_step_device(u, F, dt, cfg)

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

    # -- end to end through the public API: u from/to pinned host memory each
    # step, restarted from the initial condition (regenerated in place) --
    gaussian_coeffs(N, h, p, device=dev, out=u, layout=lay, z_range=z_range, **IC)
    e2e = e2e_rate(step, u, lay, dofs, min(args.steps, 3), stream, barrier, max_over_ranks)

    # -- per-kernel durations (CUDA events on the launching stream), on the
    # solver's own work set (after the e2e run: these passes perturb u) --
    wset = _work(op, cfg.max_iter) if world == 1 else op._work_buffers(cfg.max_iter)
    kt = kernel_times(op, u, F, dt, stream, wset)
    kt = {k: max_over_ranks(v) for k, v in kt.items()}
    peak, peak_kind = measured_peaks()
    local_dofs = int(np.prod(lay.owned_shape))
    bytes_a, bytes_b, bytes_it = alg_bytes()
    a_gbs = bytes_a * local_dofs / (kt["pass_a_ms"] * 1e-3) / 1e9
    b_gbs = bytes_b * local_dofs / (kt["pass_b_ms"] * 1e-3) / 1e9
    dom = "pass_b" if kt["pass_b_ms"] >= kt["pass_a_ms"] else "pass_a"
    ach = b_gbs if dom == "pass_b" else a_gbs
    it_s = (kt["pass_a_ms"] + kt["pass_b_ms"]) * 1e-3
    it_gbs = bytes_it * local_dofs / it_s / 1e9
    it_gbs80 = SURVEY_BYTES_ITER * local_dofs / it_s / 1e9  # DoF-it rate vs the 80 B roofline

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        rate, kind, sample = cpu_reference_rate(p=args.degree)
        cpu = {"value": rate / 1e9, "unit": "GDoF/s", "cores": 1, "kind": kind, "sample": sample}

    line = {
        "metric": METRIC, "value": value, "unit": "GDoF/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": config_of(args, world, halo_mode),
        "cg_iterations_per_step": its,
        "memory": {"fields_per_rank": mem["fields"], "p_ring": int(ring),
                   "bytes_per_rank": mem["field_bytes"] * (4 + int(ring))},
        "roofline": {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                     "frac": ach / peak,
                     # ncu traffic is captured for the C3 workload (profiles/traffic.json)
                     "traffic": TRAFFIC.get(dom) if (args.ncoef, args.degree) == (930, 3) else None,
                     "kernel": dom,
                     "peak_source": peak_kind,
                     "alg_bytes_per_dof": bytes_b if dom == "pass_b" else bytes_a,
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


def kernel_times(op, u, F, dt, stream, wset, reps=9):
    """Average device duration of CG pass A and pass B (same stream, events)
    on the solver's own work set (r, ring, Ap = b, scratch) with x = u: no
    extra fields are allocated (the timed solve is already over)."""
    import torch

    plan = op.plan()
    if isinstance(wset, dict):
        r, pring, ap, scratch = wset["r"], wset["pring"], wset["ap"], wset["scratch"]
    else:
        r, pring, ap, scratch = wset.r, wset.pring, wset.ap, wset.scratch
    x = u
    op.mass_apply_device(x, ap, F, a=dt)  # b in Ap's storage
    R = pring.shape[0]
    plan.cg_setup(scratch, None, 1e-300, 10 ** 6, False, True, p_ring=R)
    plan.cg_residual(ap, x, r, scratch, 1)
    ta, tb = [], []
    for k in range(reps):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        e[0].record(stream)
        plan.cg_pass_a(x, r, pring[(k - 1) % R], pring[k % R], ap, scratch, 1)
        e[1].record(stream)
        plan.cg_pass_b(r, ap, scratch, 1)
        e[2].record(stream)
        torch.cuda.synchronize()
        ta.append(e[0].elapsed_time(e[1]))
        tb.append(e[1].elapsed_time(e[2]))
    plan.cg_flush_x(x, pring, scratch)
    torch.cuda.synchronize()
    return {"pass_a_ms": float(np.mean(ta[1:])), "pass_b_ms": float(np.mean(tb[1:]))}


def e2e_rate(step, u, lay, dofs, steps, stream, barrier, max_over_ranks):
    """Same metric through the public step API with the state copied from and
    back to pinned host memory every step (host<->device copies timed)."""
    from paper_1904_03057_b200.heat import run_steps_host

    import torch

    host = torch.empty(lay.owned_shape, dtype=torch.float64).pin_memory()
    own = lay.owned(u)
    # untimed warm-up of the same pipeline (first DMA through the freshly
    # pinned buffer and the side streams), then the timed steps start again
    # from the same input (the host copy of u on entry)
    u_in = own.cpu()
    host.copy_(u_in)
    run_steps_host(step, own, host, 1, chunks=16, stream=stream)
    torch.cuda.synchronize()
    host.copy_(u_in)
    del u_in
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


# ---------------------------------------------------------------------------
# launcher


def _free_port():
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def spawn(args_list, nproc):
    """`bench.py --gpus N` without a launcher: start N ranks (one per GPU)
    through torch.distributed.run on 127.0.0.1 and relay rank 0's line."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), os.path.abspath(__file__), *args_list]
    env = dict(os.environ)
    env.setdefault("OMP_NUM_THREADS", "1")
    return subprocess.call(cmd, env=env)


def run_dry(args, rank, world):
    """CPU dry run of the launch topology (gloo): partition, barrier and the
    max-over-ranks timing of a bench step without the GPU kernels.  Used by
    the CPU test of `bench.py --gpus N`; its line says "dry": true."""
    import torch
    import torch.distributed as dist

    from paper_1904_03057_b200.distributed import SlabPartition

    if world > 1:
        dist.init_process_group("gloo")
    part = SlabPartition(args.ncoef, world, rank)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        t = torch.ones(1, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(t)
    ms = (time.perf_counter() - t0) * 1e3
    tm = torch.tensor([ms], dtype=torch.float64)
    if world > 1:
        dist.all_reduce(tm, op=dist.ReduceOp.MAX)
        wsum = torch.tensor([float(part.nz)], dtype=torch.float64)
        dist.all_reduce(wsum)
        planes = int(wsum.item())
    else:
        planes = part.nz
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": None, "unit": "GDoF/s", "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "dry": True,
                          "ms_per_step": float(tm.item()) / max(args.steps, 1),
                          "planes_covered": planes, "config": config_of(args, world)}),
              flush=True)
    if world > 1:
        dist.destroy_process_group()


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
    ap.add_argument("--dry", action="store_true",
                    help="CPU/gloo dry run of the multi-rank launch (no kernels; tests)")
    args = ap.parse_args()
    env_world = os.environ.get("WORLD_SIZE")
    if env_world is None and args.gpus > 1:
        # no launcher: start one rank per GPU ourselves
        sys.exit(spawn(sys.argv[1:], args.gpus))
    world = int(env_world or "1")
    if args.gpus != world:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}; launch one rank per GPU "
                 f"(or drop the launcher and let bench.py spawn them)")
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.dry:
        run_dry(args, rank, world)
        return
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
