"""The paper's masked leg run at scale: p = 1, a synthetic
leg mask on a 600 x 600 x 2400 node grid (~0.86 B nodes, ~0.2 B active), D =
0.5, DirichletPenalty 20 degC on the exposed faces (eps 1e-3), unit source on
the arteria, Jacobi-PCG to 1e-6 from the coarse-grid initial guess
(coarse_init_factor 5: 120 x 120 x 480), through the public solve_problem
pipeline (transforms, assembly with compact active-row stencils, coarse
solve, prolongation, fine solve, node sampling -- every numeric stage on the
GPU).  The reference's acceptance test runs the same problem at 60 x 60 x 240
(test_acceptance.py:351-383; tools/time_mask_leg.py).

    python tools/leg_paper_scale.py [NX NY NZ]            (default 600 600 2400)

Prints one JSON line: stage times, unknowns / active / boundary rows,
coarse and fine iterations, fine-solve iterations per second and
active-DoF iterations per second, peak device memory.
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1904_03057_b200 import DirichletPenalty, Grid, MaskDomain  # noqa: E402
from paper_1904_03057_b200.problem import ProblemSpec, solve_problem  # noqa: E402
from paper_1904_03057_b200.solver import SolveConfig  # noqa: E402
from paper_1904_03057_b200.synthetic import leg_mask  # noqa: E402

ext = tuple(int(v) for v in sys.argv[1:4]) if len(sys.argv) >= 4 else (600, 600, 2400)
t0 = time.perf_counter()
mask, art = leg_mask(ext)
grid = Grid(ext, (1.0, 1.0, 1.0))
src = np.zeros(ext)
src[:-1, :-1, :-1][art] = 1.0
del art
spec = ProblemSpec(domain=MaskDomain(grid, mask), basis_degree=1, diffusion=0.5, absorption=0.0,
                   source=src, bc=DirichletPenalty(20.0, 1e-3))
t1 = time.perf_counter()
torch.cuda.reset_peak_memory_stats()
sol = solve_problem(spec, SolveConfig(tol=1e-6, max_iter=6000, coarse_init_factor=5))
torch.cuda.synchronize()
t2 = time.perf_counter()
rep = sol.report
info = sol.coarse_info or {}
n = int(np.prod(ext))
out = dict(extents=list(ext), nodes=n, setup_host_s=round(t1 - t0, 2),
           pipeline_s=round(t2 - t1, 2), coarse_extents=info.get("coarse_extents"),
           coarse_iterations=info.get("coarse_iterations"), iterations=rep.iterations,
           relative_residual=rep.relative_residual, converged=rep.converged,
           fine_solve_s=round(rep.wall_time, 3),
           iterations_per_s=round(rep.iterations / rep.wall_time, 1) if rep.wall_time else None,
           peak_device_GB=round(torch.cuda.max_memory_allocated() / 1e9, 2),
           sample_checksum=[float(sol.samples.sum()), float(np.linalg.norm(sol.samples))])
if hasattr(sol, "stats"):
    out.update(sol.stats)
print(json.dumps(out), flush=True)
