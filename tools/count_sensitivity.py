"""Rounding sensitivity of the reference's CG iteration counts (CPU, runs the
reference package from baseline/_ref).  Perturbs every dot product of the
reference's pcg (bspde.solver) by `eps` relative (one rounding unit ~1e-16)
with a seeded RNG and prints the counts, so a count difference between two
correct implementations can be told from a defect.

    python tools/count_sensitivity.py c2d [seeds] [eps]     # coarse c2d pipeline
    python tools/count_sensitivity.py c1 [seeds] [eps]      # C1 heat, 10 steps (slow: ~2 min/seed)

Measured (this container): c2d 94 unperturbed, 96 for 5 of 6 seeds at 1e-16;
C1 [45, 45, 47, 50, 63, 77, 91, 112, 120, 129] for every seed at 1e-16..1e-13
(oracle port).
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
sys.path.insert(0, "/root/reference/pkg/src")

import bspde.solver as BS  # noqa: E402


def perturb(seed, eps):
    rng = np.random.default_rng(seed)

    class NP:
        def __getattr__(self, k):
            return getattr(np, k)

        def vdot(self, a, b):
            v = np.vdot(a, b)
            return v * (1 + eps * rng.standard_normal()) if eps else v

    BS.np = NP()


def c2d():
    from bspde.domain import BoxDomain, Grid
    from bspde.problem import DirichletPenalty, ProblemSpec, solve_problem

    g3 = Grid((21, 17), (0.05, 0.06))
    yy2, xx2 = np.meshgrid(*[g3.node_coordinates(a) for a in range(2)], indexing="ij")
    spec = ProblemSpec(domain=BoxDomain(g3), basis_degree=2, diffusion=0.8, absorption=1.0,
                       source=np.cos(3 * xx2) + yy2, bc={"all": DirichletPenalty(1.0, 1e-3)})
    sol = solve_problem(spec, BS.SolveConfig(tol=1e-9, max_iter=4000, coarse_init_factor=3),
                        strategy="sparse")
    return sol.report.iterations


def c1():
    from bspde.assembly import basis_extension, build_system
    from bspde.bspline import BSplineBasis, direct_transform
    from bspde.domain import BoxDomain, Grid
    from bspde.operator import assembled_rhs, make_operator

    p, ncoef = 3, 64
    ext = basis_extension(p)
    N = ncoef - 2 * ext
    h = 1.0 / (N - 1)
    dt = 4 * h * h
    g = Grid((N,) * 3, (h,) * 3)
    shp = tuple(n + 2 * ext for n in g.extents)
    A = make_operator(build_system(BoxDomain(g), p, p, np.full(shp, dt), np.full(shp, 1.0), []),
                      "sparse")
    Md = build_system(BoxDomain(g), p, p, np.full(shp, 0.0), np.full(shp, 1.0), [])
    M = make_operator(Md, "sparse")
    X, Y, Z = np.meshgrid(*[g.node_coordinates(a) for a in range(3)], indexing="ij")

    def coef(s):
        return np.pad(direct_transform(s, BSplineBasis(p, g.step)), ext, mode="reflect")

    u = coef(np.exp(-40 * ((X - .5) ** 2 + (Y - .4) ** 2 + (Z - .6) ** 2)))
    F = assembled_rhs(Md, p, coef(10 * np.exp(-60 * ((X - .3) ** 2 + (Y - .6) ** 2 + (Z - .5) ** 2))))
    its = []
    for _ in range(10):
        u, rep = BS.pcg(A, M.apply(u) + dt * F, BS.SolveConfig(tol=1e-10, max_iter=5000), x0=u)
        its.append(rep.iterations)
    return its


if __name__ == "__main__":
    case = sys.argv[1] if len(sys.argv) > 1 else "c2d"
    seeds = int(sys.argv[2]) if len(sys.argv) > 2 else 6
    eps = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-16
    fn = {"c2d": c2d, "c1": c1}[case]
    perturb(0, 0.0)
    print(case, "unperturbed", fn(), flush=True)
    for seed in range(seeds):
        perturb(seed, eps)
        print(case, f"seed {seed} eps {eps:g}", fn(), flush=True)
