"""The reference's masked-domain run (acceptance criterion 9,
test_acceptance.py:351-383) on the B200: the 60x60x240 synthetic leg,
basis degree 1, D = 0.5, penalty 20 degC (eps 1e-3), source 1 on the
arteria, Jacobi-PCG to 1e-6 from x0 = 0 (no coarse initialisation).

    python tools/time_mask_leg.py            (GPU)
    python tools/time_mask_leg.py --reference  (this container: the reference, CPU)

Prints one JSON line: setup / solve seconds, iterations, residual and a
solution checksum (sum and 2-norm of the coefficients); then the full
criterion-9 pipeline (solve_problem with coarse_init_factor = 5)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

EXT = (60, 60, 240)


def ours():
    import torch
    from paper_1904_03057_b200 import (DirichletPenalty, Grid, MaskDomain, assembled_rhs,
                                       build_system, make_operator, pcg, realize_bc,
                                       transform_field)
    from paper_1904_03057_b200.solver import SolveConfig
    from paper_1904_03057_b200.synthetic import leg_mask

    mask, art = leg_mask(EXT)
    grid = Grid(EXT, (1.0, 1.0, 1.0))
    src = np.zeros(EXT)
    src[:-1, :-1, :-1][art] = 1.0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    dom = MaskDomain(grid, mask)
    specs = realize_bc(DirichletPenalty(20.0, 1e-3), grid, mask=True)
    data = build_system(dom, 1, 1, 0.5, 0.0, specs)
    op = make_operator(data, "b200")
    rhs = assembled_rhs(data, 1, transform_field(src, grid, 1))
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    x, rep = pcg(op, rhs, SolveConfig(tol=1e-6, max_iter=6000))
    t2 = time.perf_counter()
    # device-only solve (inputs resident): the PCG kernels alone
    b = torch.from_numpy(rhs).cuda()
    xd = torch.zeros_like(b)
    op.pcg_device(b, xd, SolveConfig(tol=1e-6, max_iter=6000), has_x0=False)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    xd.zero_()
    e0.record()
    rep2 = op.pcg_device(b, xd, SolveConfig(tol=1e-6, max_iter=6000), has_x0=False)
    e1.record()
    torch.cuda.synchronize()
    from paper_1904_03057_b200.problem import ProblemSpec, solve_problem
    spec = ProblemSpec(domain=dom, basis_degree=1, diffusion=0.5, absorption=0.0, source=src,
                       bc=DirichletPenalty(20.0, 1e-3))
    solve_problem(spec, SolveConfig(tol=1e-6, max_iter=6000, coarse_init_factor=5))  # warm
    torch.cuda.synchronize()
    runs = []
    for _ in range(5):  # host-side work dominates: median of 5 warm runs
        t3 = time.perf_counter()
        sol = solve_problem(spec, SolveConfig(tol=1e-6, max_iter=6000, coarse_init_factor=5))
        runs.append(time.perf_counter() - t3)
    return dict(impl="b200", pipeline_coarse5_s=round(float(np.median(runs)), 3),
                pipeline_coarse5_runs_s=[round(r, 3) for r in runs],
                pipeline_iterations=sol.report.iterations,
                pipeline_coarse_iterations=sol.coarse_info["coarse_iterations"],
                pipeline_checksum=[float(sol.samples.sum()), float(np.linalg.norm(sol.samples))],
                setup_s=round(t1 - t0, 3), solve_s=round(t2 - t1, 3),
                solve_device_ms=round(e0.elapsed_time(e1), 2), iterations=rep.iterations,
                iterations_device=rep2.iterations, residual=rep.relative_residual,
                unknowns=int(np.prod(data.cext)), active=int((data.mask.node_class != 0).sum()),
                boundary_rows=int(len(data.mask.brows)),
                checksum=[float(x.sum()), float(np.linalg.norm(x))])


def reference():
    sys.path.insert(0, "/root/reference/pkg/src")
    from bspde.domain import Grid, MaskDomain, make_leg_mask
    from bspde.problem import DirichletPenalty, ProblemSpec, assemble_system
    from bspde.solver import SolveConfig, pcg

    mask, art = make_leg_mask(EXT)
    grid = Grid(EXT, (1.0, 1.0, 1.0))
    src = np.zeros(EXT)
    src[:-1, :-1, :-1][art] = 1.0
    spec = ProblemSpec(domain=MaskDomain(grid, mask), basis_degree=1, diffusion=0.5,
                       absorption=0.0, source=src, bc=DirichletPenalty(20.0, 1e-3))
    t0 = time.perf_counter()
    sysm = assemble_system(spec, "sparse")
    t1 = time.perf_counter()
    x, rep = pcg(sysm.operator, sysm.rhs, SolveConfig(tol=1e-6, max_iter=6000))
    t2 = time.perf_counter()
    x = np.where(sysm.data.active, x, 0.0)
    from bspde.problem import solve_problem
    t3 = time.perf_counter()
    sol = solve_problem(spec, SolveConfig(tol=1e-6, max_iter=6000, coarse_init_factor=5),
                        strategy="blocktensor")
    t4 = time.perf_counter()
    return dict(impl="reference (sparse, 1 thread)", pipeline_coarse5_s=round(t4 - t3, 3),
                pipeline_strategy="blocktensor (as test_acceptance.py:351-383)",
                pipeline_iterations=sol.report.iterations,
                pipeline_coarse_iterations=sol.coarse_info["coarse_iterations"],
                pipeline_checksum=[float(sol.samples.sum()), float(np.linalg.norm(sol.samples))], setup_s=round(t1 - t0, 3),
                solve_s=round(t2 - t1, 3), iterations=rep.iterations,
                residual=rep.relative_residual, checksum=[float(x.sum()), float(np.linalg.norm(x))])


if __name__ == "__main__":
    print(json.dumps(reference() if "--reference" in sys.argv else ours()), flush=True)
