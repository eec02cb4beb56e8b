"""Step-by-step GPU sanity check of each native entry point (debug aid)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import bspde_oracle as O
from paper_1904_03057_b200 import BoxDomain, Grid, build_system, make_operator, pcg, SolveConfig

def rel(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())

for p, ext in [(3, (12, 12, 12)), (3, (40, 37, 35)), (1, (9, 9, 9)), (5, (14, 13, 12))]:
    step = tuple(1.0 / (n - 1) for n in ext)
    data = build_system(BoxDomain(Grid(ext, step)), p, p, 0.01, 1.0, [])
    ora = O.KronOperator(ext, step, p, 0.01, 1.0)
    op = make_operator(data, "b200")
    c = np.random.default_rng(0).normal(size=data.cext)
    t = op.apply(c); torch.cuda.synchronize()
    print(p, ext, "apply rel", rel(t, ora.apply(c)), "diag rel", rel(op.jacobi_diagonal(), ora.jacobi_diagonal()), flush=True)
    for mi in (1, 5, 50):
        try:
            x, rep = pcg(op, c, SolveConfig(tol=1e-10, max_iter=mi))
            xo, ro = O.pcg(ora.apply, ora.jacobi_diagonal, c, tol=1e-10, max_iter=mi)
            print("   max_iter", mi, "its", rep.iterations, ro["iterations"], "relres", rep.relative_residual, ro["relative_residual"], flush=True)
        except Exception as e:
            print("   max_iter", mi, "EXC", type(e).__name__, str(e)[:90], flush=True)
