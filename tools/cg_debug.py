"""Full pcg vs oracle with small max_iter / poll variations (debug aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from oracle import bspde_oracle as O
from paper_1904_03057_b200 import BoxDomain, Grid, build_system, make_operator, pcg, SolveConfig
p, ext = 3, (12, 12, 12)
step = tuple(1.0 / (n - 1) for n in ext)
data = build_system(BoxDomain(Grid(ext, step)), p, p, 0.01, 1.0, [])
ora = O.KronOperator(ext, step, p, 0.01, 1.0)
b = np.random.default_rng(0).normal(size=data.cext)
op = make_operator(data, "b200")
for poll in (1, 2, 8):
    for mi in (1, 2, 3, 5):
        try:
            x, rep = pcg(op, b, SolveConfig(tol=1e-10, max_iter=mi, poll_every=poll))
        except Exception as e:
            print("poll", poll, "max_iter", mi, "EXC", str(e)[:80]); continue
        xo, ro = O.pcg(ora.apply, ora.jacobi_diagonal, b, tol=1e-10, max_iter=mi)
        print("poll", poll, "max_iter", mi, "its", rep.iterations, ro["iterations"], "relres", rep.relative_residual, ro["relative_residual"],
              "xerr", float(np.linalg.norm(x - xo) / np.linalg.norm(xo)), flush=True)
